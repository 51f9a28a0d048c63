"""c4 batching sweep (BASELINE configs[3]): particle-steps/s vs n on one GPU.
Writes gpurun_out/<tag>_c4_sweep.md (copied into profiles/).  usage: python tools/sweep_c4.py TAG"""
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = []
for n in (1, 4, 16, 64, 256):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--n-runs", str(n), "--steps", "20",
                          "--warmup", "3", "--no-cpu", "--no-e2e"], capture_output=True, text=True)
    line = [l for l in out.stdout.strip().split("\n") if l.startswith("{")]
    if not line:
        rows.append((n, None, out.stderr[-300:]))
        continue
    d = json.loads(line[-1])
    rows.append((n, d, None))
sys.path.insert(0, ROOT)
from workloads import configs  # noqa: E402
p = configs.get("c4")
fv, Nc = p["fnum_vc"], configs.n_cells(p)
# HS equilibrium: accepted pairs per run per step = 1/2 n_d^2 sigma <g> V dt / F_N (V_c = 1),
# n_d = 10 F_N/V_c, sigma = pi d^2, <g> = 4 sqrt(kT/(pi m)); E[N(N-1)] of a closed box: (1 - 1/N_tot)
expect_run = 0.5 * (10 * fv) ** 2 * math.pi * (4 / math.sqrt(math.pi)) * Nc * p["dt"] / fv * (1 - 1 / (10 * Nc))
lines = [f"# {tag}: c4 batching sweep (64^3 cells x 10 ppc per run, HS, K=2, 20 timed steps after 3)\n",
         "| n runs | particles | ms/step | particle-steps/s | collide share | collide GB/s (alg.) | accepted / (n x 1/2 n_d^2 sigma <g> V dt / F_N) |",
         "|---|---|---|---|---|---|---|"]
for n, d, err in rows:
    if d is None:
        lines.append(f"| {n} | error | | | | | {err} |")
        continue
    k = d["roofline"]["kernels"]["k_collide"]
    ratio = d["collisions"]["accepted_per_step"] / (n * expect_run)
    lines.append(f"| {n} | {n * 2621440:,} | {d['ms_per_step']:.3f} | {d['value']:.4g} | {k['share']:.2f} | {k['GB/s']} | "
                 f"{ratio:.4f} |")
txt = "\n".join(lines) + "\n"
print(txt)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
open(os.path.join(ROOT, "gpurun_out", f"{tag}_c4_sweep.md"), "w").write(txt)  # copied into profiles/ afterwards
