"""Markdown table of the key metrics of every kernel in an exported ncu raw page (csv.gz from
tools/ncu_export.sh), with its top stall reasons.  usage: python tools/ncu_table.py RAW_CSV_GZ"""
import csv, gzip, io, sys
rr = list(csv.reader(io.StringIO(gzip.open(sys.argv[1], "rt").read())))
h, u = rr[0], rr[1]
want = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
        ("smsp__inst_executed.sum", "warp-instr"), ("smsp__issue_active.avg.per_cycle_active", "issue/cycle"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__registers_per_thread", "regs"), ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/instr")]
print("| kernel | " + " | ".join(n for _, n in want) + " | top stalls (cycles per issue) |")
print("|---|" + "---|" * (len(want) + 1))
for r in rr[2:]:
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    vals = []
    for w, _ in want:
        if w in h:
            v, un = r[h.index(w)], u[h.index(w)]
            try:
                v = f"{float(v.replace(',', '')):.4g}"
            except ValueError:
                pass
            vals.append(f"{v} {un}".strip().replace("register/thread", "").replace(" inst", ""))
        else:
            vals.append("n/a")
    st = sorted(((h[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(r[i] or 0))
                 for i in range(len(h)) if h[i].startswith("smsp__average_warps_issue_stalled_")
                 and h[i].endswith("_per_issue_active.ratio")), key=lambda x: -x[1])[:4]
    print(f"| {name} | " + " | ".join(vals) + " | " + ", ".join(f"{a} {b:.2f}" for a, b in st) + " |")
