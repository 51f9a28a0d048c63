import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_cs_9902024_b200 import dsmc
from oracle import oracle
from workloads import configs
warm, run = int(sys.argv[1]), int(sys.argv[2])
p = configs.get("c5", n_runs=2, n_steps=max(100, (warm // 50 + 1) * 50), cap_per_run=12 << 20)
p["dt_s"] = p["dt"] * 50
sim = dsmc.Simulation(p, debug=True)
sim.generate()
sim.step(warm)
st = sim.get_state(run)
ref = oracle.OracleRun(p, run)
ref.set_state(st, step=warm)
ref.set_gmax(sim.get_gmax(run))
sim.step(1)
ref.step(1)
gi, oi = sim.get_index(run), ref.get_index()
bad = np.nonzero(gi["lcr"] != oi["lcr"])[0]
print("lcr mismatches", len(bad), "of", len(gi["lcr"]))
cnt = gi["count"]
ends = np.cumsum(cnt)
cells = np.searchsorted(ends, bad, side="right")
tiles = cells // 32
tc = cnt[: len(cnt) // 32 * 32].reshape(-1, 32).sum(1)
ut = np.unique(tiles)
print("cells", np.unique(cells)[:20], "tiles", ut[:20], "tile counts", tc[ut][:20])
for c in np.unique(cells)[:3]:
    s0 = ends[c] - cnt[c]
    print("cell", c, "N", cnt[c], "gpu", gi["lcr"][s0:ends[c]][:40], "ora", oi["lcr"][s0:ends[c]][:40])
