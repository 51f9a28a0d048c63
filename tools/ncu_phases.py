"""Per-phase instruction / stall breakdown of k_collide from an ncu report.
usage: python tools/ncu_phases.py REPORT [N_CELLS_PER_LAUNCH] [N_LAUNCHES]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ncell = float(sys.argv[2]) if len(sys.argv) > 2 else 4.19e6
nl = float(sys.argv[3]) if len(sys.argv) > 3 else 2
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:k_collide", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None
hdr = None
agg, st = {}, {}
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
        v = int(d["Instructions Executed"])
        w = int(d["Warp Stall Sampling (All Samples)"])
    except (KeyError, ValueError):
        continue
    key = (fname, int(r[0]))
    agg[key] = agg.get(key, 0) + v
    st[key] = st.get(key, 0) + w
src = open("paper_cs_9902024_b200/csrc/dsmc_kernels.cu").read().split("\n")


def find(m):
    return next(i + 1 for i, l in enumerate(src) if m in l)


kstart = find("k_collide(Prm P, int mode, int slot_arg, int capw) {")
marks = [("A", kstart), ("B", find("    // ---- B")), ("C", find("    // ---- C")), ("D", find("    // ---- D")),
         ("E0", find("    // ---- E")), ("E1", find("      for (uint32_t base = 0; base < tot; base += CCW) {")),
         ("E2", find("        if (Mu) {")), ("Efin", find("      if (valid && M) {")),
         ("F", find("    // ---- F")), ("G", find("tile too large for the warp")),
         ("end", find("// per-run counters: aggregate") + 12)]
fns = [("marsaglia_pq", find("__device__ __forceinline__ void marsaglia_pq")),
       ("ntc_apply", find("// candidates k in [k_lo, k_hi)")), ("sort_net", find("template <int NN>")),
       ("sample_cell", find("__device__ __forceinline__ void sample_cell(")),
       ("sorts", find("__device__ __forceinline__ void insertion_sort")), ("x", kstart - 3)]
ph, phs = {}, {}
for (f, l), v in agg.items():
    w = st[(f, l)]
    if f == "dsmc_device.cuh":
        n = "philox/dev"
    elif f != "dsmc_kernels.cu":
        n = "intrinsics"
    else:
        n = None
        for (a, la), (b, lb) in zip(marks, marks[1:]):
            if la <= l < lb:
                n = a
        if n is None:
            for (a, la), (b, lb) in zip(fns, fns[1:]):
                if la <= l < lb:
                    n = a
        if n is None:
            n = "other"
    ph[n] = ph.get(n, 0) + v
    phs[n] = phs.get(n, 0) + w
tot, tots = sum(ph.values()), sum(phs.values())
for k, v in sorted(ph.items(), key=lambda x: -x[1]):
    print(f"{k:14s} {100 * v / tot:5.1f}% instr {100 * phs[k] / tots:5.1f}% stalls {v / nl / ncell:6.1f} warp-instr/cell")
