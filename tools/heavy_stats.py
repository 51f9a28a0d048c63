"""Tile-size statistics of c5 after WARM steps: how many 32-cell tiles go to each
heavy tier and how large their cells are (input for tuning k_collide_heavy).
usage: python tools/heavy_stats.py WARM [N_RUNS]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_cs_9902024_b200 import dsmc  # noqa: E402
from workloads import configs  # noqa: E402

warm = int(sys.argv[1])
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p = configs.get("c5", n_runs=nr)
sim = dsmc.Simulation(p, debug=True)
sim.generate()
sim.step(warm)
torch.cuda.synchronize()
cnt = sim.get_index(0)["count"]
tiles = cnt.reshape(-1, 32)
ts = tiles.sum(1)
capw = int(os.environ.get("CAPW", "0")) or None
out = {"warm": warm, "live_run0": int(cnt.sum()), "cell_max": int(cnt.max()), "tile_max": int(ts.max())}
for lo, hi in [(0, 256), (256, 1024), (1024, 2048), (2048, 4096), (4096, 8192), (8192, 1 << 30)]:
    m = (ts > lo) & (ts <= hi)
    out[f"tiles_{lo}_{hi}"] = int(m.sum())
    if m.any():
        t = tiles[m]
        out[f"sumsq_over_sum_{lo}_{hi}"] = float((t.astype(np.float64) ** 2).sum() / t.sum())
        out[f"cellmax_mean_{lo}_{hi}"] = float(t.max(1).mean())
print(json.dumps(out))
