"""NEXT-1: the TLPDPR-style heavy-tile queue (dynamic, two size tiers)
against a static block-per-heavy-tile mapping (one tier, tiles dealt round-robin) on c5
once the orifice jet has built dense cells.
usage: python tools/heavy_ab.py WARM STEPS   (set DSMC_STATIC_CELLS=1 for the static arm)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_cs_9902024_b200 import dsmc  # noqa: E402
from workloads import configs  # noqa: E402

warm, K = int(sys.argv[1]), int(sys.argv[2])
p = configs.get("c5", n_runs=2, n_steps=2000, cap_per_run=24 << 20)
sim = dsmc.Simulation(p)
sim.generate()
sim.step(warm)
torch.cuda.synchronize()
timed = sim.step_timed(K)
rc, st = sim.status()
col = {k: v[0] / v[1] for k, v in timed.items() if k.startswith("k_collide")}
print(json.dumps({"static": os.environ.get("DSMC_STATIC_CELLS", "0"), "warm": warm, "steps": K, "status": rc,
                  "live": sum(s["live"] for s in st), "ms_per_launch": col,
                  "interaction_ms": sum(col.values())}))
