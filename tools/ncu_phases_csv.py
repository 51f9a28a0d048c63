"""Per-phase instruction / stall shares of one kernel from an exported source-page CSV (csv.gz of
tools/ncu_export.sh).  Lines of the body are grouped by the last '// ---- X' marker in the function
that contains them; helpers by their own signature line.  The source file must be the one the
report was built from.  usage: python tools/ncu_phases_csv.py SRC_CSV_GZ FUNC_SUBSTR SOURCE_FILE BODY_SIGNATURE"""
import csv, gzip, io, re, sys
path, fsub, srcf, sig = sys.argv[1:5]
rows = list(csv.reader(io.StringIO(gzip.open(path, "rt").read())))
src = open(srcf).read().split("\n")
start = next(i for i, l in enumerate(src) if sig in l)
end = next(i for i in range(start + 1, len(src)) if src[i].startswith("}"))
marker, cur = {}, "entry"
for i in range(start, end + 1):
    m = re.search(r"// ---- ([A-Z0-9]+)", src[i])
    if m:
        cur = m.group(1)
    marker[i + 1] = cur
fname = func = None
agg, tot = {}, 0
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) == 2 and r[0] == "Function Name":
        func = r[1]; continue
    if not func or fsub not in func or len(r) < 8 or not r[0].isdigit():
        continue
    try:
        ins, samp = int(r[7]), int(r[4])
    except ValueError:
        continue
    ln = int(r[0])
    if fname == src_name if (src_name := srcf.split("/")[-1]) else False:
        pass
    if fname == srcf.split("/")[-1] or fname == "dsmc_kernels.cu":
        if ln in marker:
            g = "phase " + marker[ln]
        else:
            j = ln - 1
            while j > 0 and not re.match(r"^(__device__|template|__global__|__host__)", src[j]):
                j -= 1
            g = "helper " + re.sub(r"\s+", " ", src[j + 1 if src[j].startswith("template") else j])[:70]
    else:
        g = fname
    a = agg.setdefault(g, [0, 0]); a[0] += ins; a[1] += samp; tot += ins
ts = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:24]:
    print(f"{100 * v[0] / tot:5.1f}% instr {100 * v[1] / ts:5.1f}% stall  {k}")
