"""Per-source-line instructions / stall samples of one kernel from an ncu report.
usage: python tools/ncu_lines2.py REPORT KERNEL_REGEX [FROM TO [MINPCT]]  (line range of dsmc_kernels.cu)"""
import csv, io, subprocess, sys
rep, kr = sys.argv[1], sys.argv[2]
lo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4]) if len(sys.argv) > 4 else 10**9
mp = float(sys.argv[5]) if len(sys.argv) > 5 else 0.3
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name-base", "demangled", "-k", "regex:" + kr,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
fname, agg = None, {}
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) < 8 or r[2] != "-" or not r[0].isdigit():
        continue
    try:
        w = int(r[4]); v = int(r[7])
    except ValueError:
        continue
    a = agg.setdefault((fname, int(r[0])), [0, 0, r[1]])
    a[0] += v; a[1] += w
ti = sum(a[0] for a in agg.values()) or 1; ts = sum(a[1] for a in agg.values()) or 1
print(f"total warp-instr {ti} stall samples {ts}")
for (f, l), (v, w, s) in sorted(agg.items()):
    if (f != "dsmc_kernels.cu" or lo <= l <= hi) and (100 * v / ti >= mp or 100 * w / ts >= mp):
        print(f"{f[:16]:16s} {l:5d} {100*v/ti:5.1f}% {100*w/ts:5.1f}%  {s.strip()[:90]}")
