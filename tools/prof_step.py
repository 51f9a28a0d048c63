"""Minimal driver for ncu: build a batch, warm up, then run a few graph steps.
usage: python tools/prof_step.py CONFIG N_RUNS WARMUP STEPS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_cs_9902024_b200 import dsmc  # noqa: E402
from workloads import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
n_runs = int(sys.argv[2]) if len(sys.argv) > 2 else 16
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 3
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
kw = dict(n_runs=n_runs)
if name == "c4":
    kw["n_steps"] = 100
p = configs.get(name, **kw)
sim = dsmc.Simulation(p)
sim.generate()
sim.step(warm)
torch.cuda.synchronize()
sim.step(steps)
torch.cuda.synchronize()
rc, st = sim.status()
print("ok", rc, st[0])
