"""Bench line of every BASELINE config (c1..c5) at its own batch size: throughput
and the dominant kernel.  Writes gpurun_out/<tag>_configs.md.  usage: python tools/configs_bench.py TAG"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
lines = [f"# {tag}: bench line per config (20 timed steps after 3 warm-up steps, from the fill)\n",
         "| config | runs | particles/step | ms/step | particle-steps/s | dominant kernel | its share | GB/s (alg.) |",
         "|---|---|---|---|---|---|---|---|"]
for cfg in ("c1", "c2", "c3", "c4", "c5"):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "20",
                          "--warmup", "3", "--no-cpu", "--no-e2e"], capture_output=True, text=True)
    line = [l for l in out.stdout.strip().split("\n") if l.startswith("{")]
    if not line:
        lines.append(f"| {cfg} | error | | | | | | {out.stderr[-200:]!r} |")
        continue
    d = json.loads(line[-1])
    r = d["roofline"]
    lines.append(f"| {cfg} | {d['config']['n_runs_per_gpu']} | {d['config']['particles_per_step']:.4g} | "
                 f"{d['ms_per_step']:.3f} | {d['value']:.4g} | {r['kernel']} | {r['share_of_step']} | {r['achieved']} |")
txt = "\n".join(lines) + "\n"
print(txt)
open(os.path.join(ROOT, "gpurun_out", f"{tag}_configs.md"), "w").write(txt)
