"""c5 with the jet developed: WARM graph steps, then K steps kernel by kernel with CUDA events
(dsmc_step_timed); per-kernel ms and algorithmic GB/s (bench.algorithmic_bytes), the phase
fractions of the north-star targets.  usage: python tools/c5_timed.py WARM K [N_RUNS]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_cs_9902024_b200 import dsmc  # noqa: E402
from workloads import configs  # noqa: E402

warm, K = int(sys.argv[1]), int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4
p = configs.get("c5", n_runs=n)
sim = dsmc.Simulation(p)
sim.generate()
sim.step(warm)
torch.cuda.synchronize()
_, s0 = sim.status()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(sim.stream)
sim.step(K)
e1.record(sim.stream)
torch.cuda.synchronize()
_, s1 = sim.status()
ms_graph = e0.elapsed_time(e1) / K
live = sum(b["particle_steps"] - a["particle_steps"] for a, b in zip(s0, s1)) / K
acc = sum(b["accepted"] - a["accepted"] for a, b in zip(s0, s1)) / K
timed = sim.step_timed(K)
cells = sim.R * sim.Nc
hbm, _ = bench.peaks()
out = {"config": f"c5 n={n} after {warm} steps", "live": live, "ms_per_step_graph": ms_graph,
       "particle_steps_per_s": live / (ms_graph / 1e3), "kernels": {}}
ph = {"motion+sort": [0.0, 0.0], "collide+sample": [0.0, 0.0]}
S, Kr = configs.sample_every(p), p["reorder_every"]
for name, (ms, cnt) in timed.items():
    m = ms / cnt
    b = bench.algorithmic_bytes(p, name, live, cells, acc, False, False)
    if name == "k_collide":   # reorder every Kr steps, sampling every S
        b = b + (bench.algorithmic_bytes(p, name, live, cells, acc, False, True) - b) / Kr \
            + (bench.algorithmic_bytes(p, name, live, cells, acc, True, False) - b) / S
    out["kernels"][name] = {"ms": round(m, 4), "GB/s": round(b / (m / 1e3) / 1e9, 1) if b else None}
    if name in ("k_zero", "k_motion", "k_scan_reduce", "k_scan_partials", "k_scan_down", "k_scatter"):
        ph["motion+sort"][0] += m; ph["motion+sort"][1] += b
    if name in ("k_collide_triage", "k_collide", "k_collide_heavy"):
        ph["collide+sample"][0] += m; ph["collide+sample"][1] += b
out["phases"] = {k: {"ms": round(v[0], 4), "frac_measured": round(v[1] / (v[0] / 1e3) / 1e9 / hbm, 4),
                     "frac_8TBs": round(v[1] / (v[0] / 1e3) / 1e9 / 8000, 4)} for k, v in ph.items()}
print(json.dumps(out))
