"""Per-tile work statistics of a configuration after WARM steps (debug build of the step, which
records candidates and accepted pairs per cell): particles, candidates and accepted pairs per
32-cell tile of run 0, idle tiles (no candidate), the largest candidate count per tile against the
mean (the lane-per-cell walk's length), and the tiles above the warp staging capacity.
usage: python tools/tile_stats.py CONFIG N_RUNS WARM [CAPW]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_cs_9902024_b200 import dsmc  # noqa: E402
from workloads import configs  # noqa: E402

name, nr, warm = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
capw = int(sys.argv[4]) if len(sys.argv) > 4 else 384
p = configs.get(name, n_runs=nr)
sim = dsmc.Simulation(p, debug=True)
sim.generate()
sim.step(warm)
torch.cuda.synchronize()
ix = sim.get_index(0)
cnt, cand, acc = ix["count"], ix["cand"], ix["acc"]
pad = (-len(cnt)) % 32
t_n = np.pad(cnt, (0, pad)).reshape(-1, 32)
t_m = np.pad(cand, (0, pad)).reshape(-1, 32)
t_a = np.pad(acc, (0, pad)).reshape(-1, 32)
tn, tm = t_n.sum(1), t_m.sum(1)
small = tn <= capw
out = {"config": name, "warm": warm, "cells": int(len(cnt)), "tiles": int(len(tn)), "live_run0": int(cnt.sum()),
       "ppc_mean": float(cnt.mean()), "cand_per_cell": float(cand.mean()), "acc_per_cell": float(acc.mean()),
       "tiles_empty": int((tn == 0).sum()), "tiles_no_cand": int((tm == 0).sum()),
       "tiles_over_capw": int((~small).sum()), "particles_in_heavy_tiles": int(tn[~small].sum()),
       "warp_tiles_with_cand": int(((tm > 0) & small).sum())}
w = (tm > 0) & small
if w.any():
    out["walk_passes_mean"] = float(t_m[w].max(1).mean())          # max M over the tile
    out["cand_per_lane_mean"] = float(t_m[w].mean())
    out["cand_per_tile_mean"] = float(tm[w].mean())
    out["particles_per_tile_mean"] = float(tn[w].mean())
    out["wN_mean"] = float(t_n[w].max(1).mean())                    # network width driver
    out["acc_per_tile_mean"] = float(t_a[w].sum(1).mean())
hist = np.bincount(np.minimum(tm[small], 64))
out["cand_per_tile_hist_0_64"] = hist.tolist()
print(json.dumps(out))
