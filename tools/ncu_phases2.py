"""Per-phase instruction / stall shares of a kernel from an ncu report with embedded source.
Lines are grouped by the last '// ---- X' marker (inside kernels) or by the enclosing
function (device helpers).  usage: python tools/ncu_phases2.py REPORT KERNEL_REGEX"""
import csv, io, re, subprocess, sys
rep, kr = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name-base", "demangled", "-k", "regex:" + kr,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
fname, lines = None, {}
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) < 8 or r[2] != "-" or not r[0].isdigit():
        continue
    try:
        w, v = int(r[4]), int(r[7])
    except ValueError:
        w, v = 0, 0
    lines[(fname, int(r[0]))] = (r[1], v, w)
srcfile = sys.argv[3] if len(sys.argv) > 3 else "paper_cs_9902024_b200/csrc/dsmc_kernels.cu"
text = open(srcfile).read().split("\n")   # must be the source the report was built from
group, agg = {}, {}
for f in sorted({f for f, _ in lines}):
    cur = f
    if f != "dsmc_kernels.cu":
        for k in lines:
            if k[0] == f: group[k] = f
        continue
    for l in range(1, len(text) + 1):
        src = text[l - 1]
        ff = f
        m = re.match(r"(?:__global__|__device__|__host__ __device__|    k_collide)[^(]*?(\w+)\s*\(", src)
        if m and m.group(1) == "__launch_bounds__":
            m = None
        if m:
            cur = m.group(1)
        m2 = re.match(r"\s*// ---- (\w+)", src)
        if m2:
            cur = cur.split(":")[0] + ":" + m2.group(1)
        group[(ff, l)] = cur
for k, (s, v, w) in lines.items():
    g = group.get(k, "?")
    a = agg.setdefault(g, [0, 0]); a[0] += v; a[1] += w
ti = sum(a[0] for a in agg.values()) or 1; ts = sum(a[1] for a in agg.values()) or 1
print(f"total warp-instr {ti}  stall samples {ts}")
for g, (v, w) in sorted(agg.items(), key=lambda x: -x[1][0]):
    if v / ti > 0.003 or w / ts > 0.003:
        print(f"{g:36s} {100*v/ti:5.1f}% instr {100*w/ts:5.1f}% stall")
