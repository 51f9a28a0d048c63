import os, sys, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_cs_9902024_b200 import dsmc
from workloads import configs
steps = int(sys.argv[1]); debug = int(sys.argv[2]) if len(sys.argv) > 2 else 0
def run():
    p = configs.get("c5", n_runs=2, n_steps=max(100, (steps // 50 + 1) * 50), cap_per_run=12 << 20)
    p["dt_s"] = p["dt"] * 50
    sim = dsmc.Simulation(p, debug=bool(debug))
    sim.generate()
    out = []
    for s in range(0, steps, 50):
        sim.step(50)
        st = sim.get_state(1)
        out.append(hashlib.md5(b"".join(np.ascontiguousarray(st[k]).tobytes() for k in sorted(st))).hexdigest()[:8] + f":{len(st['x'])}")
    return out
for mode in (sys.argv[3] if len(sys.argv) > 3 else "1100"):
    os.environ["DSMC_COMPACT"] = mode
    print(mode, run())
