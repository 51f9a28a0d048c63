"""Write profiles/<tag>_*.md/json summaries from gpurun_out ncu artefacts.
usage: python tools/summarize_profiles.py TAG LAUNCH_CSV NCU_REP_OR_RAW_CSV_GZ CONFIG"""
import csv
import io
import json
import os
import subprocess
import sys

tag, launch_csv, rep, cfg = sys.argv[1:5]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_md = os.path.join(ROOT, "profiles", f"{tag}_{cfg}.md")
lines = []
# ---- launch list
rows = list(csv.reader(open(launch_csv)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
seq = [(r[ki].split("(")[0].replace("void ", "").split("<")[0], float(r[vi].replace(",", ""))) for r in rows[hi + 1:]
       if len(r) > vi and r[vi]]
agg = {}
for n, v in seq:
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += v
step_kernels = {"k_zero", "k_motion", "k_step_mid", "k_scan_reduce", "k_scan_partials", "k_scan_down", "k_scatter",
                "k_collide", "k_collide_list", "k_collide_triage", "k_step_end", "k_inflow_count", "k_inflow_emit"}
step_total = sum(v[1] for n, v in agg.items() if n in step_kernels)
lines.append(f"# {tag} profile summary — {cfg}\n")
lines.append(f"Launch list: `{os.path.basename(launch_csv)}` (ncu `--metrics gpu__time_duration.sum "
             f"--clock-control none`, cold-cache, serialised; compare shares, not absolutes).\n")
lines.append("| kernel | launches | mean µs | share of step-kernel time |")
lines.append("|---|---|---|---|")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    share = f"{100 * t / step_total:.1f}%" if n in step_kernels else "(setup)"
    lines.append(f"| {n} | {c} | {t / c / 1e3:.1f} | {share} |")
# ---- full metrics
if rep.endswith(".csv.gz"):       # exported on the GPU box by tools/ncu_export.sh
    import gzip
    out = gzip.open(rep, "rt").read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(out)))
h, u = rr[0], rr[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "lts__t_sector_op_write_hit_rate.pct"]
traffic, tcount = {}, {}
lines.append("\n## ncu --set full (one launch of each kernel per captured step; with K = 2 the two captured steps "
             "are a reorder and a non-reorder step, and `traffic` is their mean)\n")
lines.append("| kernel | " + " | ".join(w.replace(".sum", "").replace(".avg.pct_of_peak_sustained_elapsed", " %pk")
                                       .replace(".avg.pct_of_peak_sustained_active", " %") for w in want) + " |")
lines.append("|---|" + "---|" * len(want))
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
for r in rr[2:]:
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    vals = []
    for w in want:
        vals.append(f"{r[h.index(w)]} {u[h.index(w)]}" if w in h else "n/a")
    lines.append(f"| {name} | " + " | ".join(vals) + " |")
    b = 0.0
    for w in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        b += float(r[h.index(w)]) * scale.get(u[h.index(w)], 1.0)
    base = name.split("<")[0]
    traffic[base] = traffic.get(base, 0.0) + b
    tcount[base] = tcount.get(base, 0) + 1
stalls = []
for r in rr[2:]:
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    items = [(h[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), r[i])
             for i in range(len(h)) if "smsp__average_warps_issue_stalled" in h[i] and h[i].endswith("_per_issue_active.ratio")]
    items = sorted(items, key=lambda x: -float(x[1] or 0))[:5]
    stalls.append(f"- {name}: " + ", ".join(f"{a} {float(b):.2f}" for a, b in items))
lines.append("\nTop warp-stall reasons (cycles per issued instruction):\n")
lines += stalls
open(out_md, "w").write("\n".join(lines) + "\n")
traffic = {k: v / tcount[k] for k, v in traffic.items()}
lines.append("\nMean DRAM bytes per launch (`traffic` of the bench line): " +
             ", ".join(f"{k} {v / 1e9:.2f} GB" for k, v in traffic.items()))
json.dump(traffic, open(os.path.join(ROOT, "profiles", f"traffic_{cfg}.json"), "w"), indent=1)
print("\n".join(lines))
