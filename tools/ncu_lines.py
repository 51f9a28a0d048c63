"""Summarise `ncu --page source --csv --print-source cuda,sass` output per CUDA line.
usage: python tools/ncu_lines.py REPORT KERNEL [TOP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None
hdr = None
agg = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    d = dict(zip(hdr, r))
    try:
        agg.append((int(d["Instructions Executed"]), int(d["Warp Stall Sampling (All Samples)"]), fname, r[0], r[1][:90]))
    except (ValueError, KeyError):
        pass
tot_i = sum(a[0] for a in agg) or 1
tot_s = sum(a[1] for a in agg) or 1
print(f"total warp-instr {tot_i:,}  stall samples {tot_s:,}")
print("--- by instructions")
for a in sorted(agg, reverse=True)[:top]:
    print(f"{100*a[0]/tot_i:5.1f}% i {100*a[1]/tot_s:5.1f}% s  {a[2]}:{a[3]}  {a[4]}")
print("--- by stall samples")
for a in sorted(agg, key=lambda x: -x[1])[:top]:
    print(f"{100*a[0]/tot_i:5.1f}% i {100*a[1]/tot_s:5.1f}% s  {a[2]}:{a[3]}  {a[4]}")
