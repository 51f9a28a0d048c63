"""Golden fixtures (tests/golden/): the numbers PAPER.md prints for its efficiency
model and the worked toy examples SPEC.md states, each line with its citation,
checked against analysis/efficiency.py (NEXT-3) and the oracle (test
infrastructure).  The values are read from the fixture files, not retyped here."""
import os

import numpy as np
import pytest

from analysis import efficiency as ef
from workloads import configs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    out = {}
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        k, v = (s.strip() for s in line.split("=", 1))
        vals = [float(t) for t in v.split()]
        out[k] = vals[0] if len(vals) == 1 else vals
    return out


def test_paper_tlpdpr_printed_numbers():
    g = load("paper_efficiency.txt")
    beta, p2 = g["dpr.beta"], int(g["dpr.p2"])
    # Eq. 13 with p1 -> infinity and p2 (1 + PRI) -> infinity: 1 / beta, printed as 2.3
    assert round(ef.tlpdpr_speedup2(beta, 1e12, 0.0), 1) == g["dpr.max_speedup"]
    # TLP (PRI = 0) at p2 = 6: 80% of that maximum (Eq. 13 gives 0.82; the paper rounds to a tenth)
    assert round(ef.tlpdpr_speedup2(beta, p2, 0.0) * beta, 1) == g["dpr.tlp_fraction"]
    # TLPDPR at PRI* (Eq. 15) reaches at least the measured 93% (Eq. 13 assumes instant
    # reallocation, so it bounds the measurement from above)
    ps = ef.pri_star(beta, p2)
    assert ef.pri_condition_residual(int(g["dpr.p1"]) * p2, int(g["dpr.p1"]), p2, beta, ps) == pytest.approx(0, abs=1e-9)
    assert g["dpr.dpr_fraction"] <= ef.tlpdpr_speedup2(beta, p2, ps) * beta <= g["dpr.dpr_fraction"] + 0.03
    # "equivalent to TLP on a 120-processor computer (p1 = 6, p2 = 20)": TLP at p2 = 20 gives
    # the same fraction to within the paper's rounding
    assert g["dpr.equiv_p"] == g["dpr.p1"] * g["dpr.equiv_p2"]
    assert abs(ef.tlpdpr_speedup2(beta, int(g["dpr.equiv_p2"]), 0.0) * beta - g["dpr.dpr_fraction"]) < 0.015


def test_paper_tlp_comet_inputs():
    g = load("paper_efficiency.txt")
    p1, a1, a2 = int(g["tlp.p1"]), g["tlp.alpha1"], g["tlp.alpha2"]
    S = [ef.tlp_speedup(p1, a1, p2, a2) for p2 in range(1, int(g["tlp.p2_max"]) + 1)]
    # p2 = 1 is Amdahl's law on the first level alone; S grows with p2 and stays below p
    assert S[0] == pytest.approx(ef.amdahl_speedup(p1, a1), rel=1e-12)
    assert all(b > a for a, b in zip(S, S[1:]))
    assert all(s <= p1 * p2 for s, p2 in zip(S, range(1, 7)))
    # Eq. 10 is Eq. 9 over p = p1 p2
    assert ef.tlp_efficiency(p1, a1, 6, a2) == pytest.approx(S[-1] / 36, rel=1e-12)


def test_spec_index_toy(oracle_mod):
    g = load("spec_examples.txt")
    p = configs.get("c1")
    p["fnum_vc"] = 0.0
    p.update(nx=int(g["index.toy.cells"]), fill=[], cap_per_run=3)
    p["bc"] = [configs.SPECULAR] * 2 + [configs.PERIODIC] * 4
    x = np.array(g["index.toy.x"], np.float32)
    z = np.zeros(len(x), np.float32)
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(dict(x=x, y=z, z=z, vx=z, vy=z, vz=z, alive=np.ones(len(x), np.uint8)))
    o.step(1)
    ix = o.get_index()
    assert ix["count"].tolist() == [int(v) for v in g["index.toy.count"]]
    start = [int(v) for v in g["index.toy.start"]]
    assert ix["start"].tolist() == start[:-1] and len(ix["lcr"]) == start[-1]
    assert ix["lcr"].tolist() == [int(v) for v in g["index.toy.perm"]]


def test_spec_specular_toy(oracle_mod):
    g = load("spec_examples.txt")
    p = configs.get("c1")
    p["fnum_vc"] = 0.0
    L = np.float32(g["specular.toy.L"])
    assert float(L) == float(p["nx"])           # the wall is c1's x = L face
    v = np.array(g["specular.toy.v"], np.float32)
    st = dict(x=np.array([g["specular.toy.x"]], np.float32), y=np.zeros(1, np.float32),
              z=np.zeros(1, np.float32), vx=v[:1], vy=v[1:2], vz=v[2:], alive=np.ones(1, np.uint8))
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(st)
    o.step(1)
    out = o.get_state()
    free = np.float32(st["x"][0] + np.float32(st["vx"][0] * np.float32(p["dt"])))
    assert abs(float(out["x"][0]) - float(2 * L - free)) < 1e-4
    assert out["vx"][0] == -v[0] and out["vy"][0] == v[1] and out["vz"][0] == v[2]


def test_spec_sparse_cells_never_collide(oracle_mod):
    g = load("spec_examples.txt")
    p = configs.get("c4_small")
    p["fill"] = [dict(lo=[0, 0, 0], hi=[16, 16, 16], ppc=int(g["collide.sparse.ppc"]), T=1.0, u=[0.0, 0.0, 0.0])]
    p["reorder_every"] = 0
    o = oracle_mod.OracleRun(p, 0)
    o.fill()
    # positions on a grid (one particle per cell): no cell ever holds two
    st = o.get_state()
    n = len(st["x"])
    cells = np.arange(n)
    st["x"] = (cells % 16 + 0.5).astype(np.float32)
    st["y"] = (cells // 16 % 16 + 0.5).astype(np.float32)
    st["z"] = (cells // 256 + 0.5).astype(np.float32)
    for a in ("vx", "vy", "vz"):
        st[a] = np.zeros(n, np.float32)             # at rest: they stay in their cells
    o.set_state(st)
    o.step(1)
    assert o.counters()["candidates"] == 0 and o.counters()["accepted"] == 0
    out = o.get_state()
    assert (out["vx"] == 0).all() and (out["vy"] == 0).all() and (out["vz"] == 0).all()


def test_spec_vacuum_step(oracle_mod):
    g = load("spec_examples.txt")
    p = configs.get("c4_small")
    p["fill"] = []
    o = oracle_mod.OracleRun(p, 0)
    k = int(g["step.vacuum.steps"])
    o.step(k)
    assert o.n == 0 and o.step_index == k and o.status == 0
