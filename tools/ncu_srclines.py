"""Top source lines of one kernel by warp-instructions executed and stall samples, from the gzipped
source-page CSV that tools/ncu_export.sh writes.  usage: python tools/ncu_srclines.py SRC_CSV_GZ FUNC_SUBSTR [N]"""
import csv, gzip, io, sys
path, fsub = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(io.StringIO(gzip.open(path, "rt").read())))
fname = func = None
agg = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) == 2 and r[0] == "Function Name":
        func = r[1]; continue
    if not func or fsub not in func or len(r) < 8 or not r[0].isdigit():
        continue
    try:
        samp, ins = int(r[4]), int(r[7])
    except ValueError:
        continue
    a = agg.setdefault((fname, int(r[0])), [r[1].strip(), 0, 0])
    a[1] += ins; a[2] += samp
ti = sum(v[1] for v in agg.values()) or 1
ts = sum(v[2] for v in agg.values()) or 1
print(f"total warp-instructions {ti}, stall samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:N]:
    print(f"{k[0]}:{k[1]:5d}  instr {100*v[1]/ti:5.1f}%  stall {100*v[2]/ts:5.1f}%  {v[0][:90]}")
