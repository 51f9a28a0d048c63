"""NEXT-3: the paper's efficiency model (analysis/efficiency.py), pinned by the
numbers the paper prints and by its own identities."""
import math

import pytest

from analysis import efficiency as ef


def test_amdahl_forms_agree():
    # Eq. 4 and 5 follow from Eq. 3 with Eqs. 1-2, for any alpha, p
    for a in (0.0, 0.5, 0.97, 0.998, 1.0):
        for p in (1, 2, 6, 36, 1000):
            Tp = ef.time_parallel(1.0, p, a)
            assert math.isclose(ef.amdahl_speedup(p, a), ef.speedup(1.0, Tp), rel_tol=1e-12)
            assert math.isclose(ef.amdahl_efficiency(p, a), ef.efficiency(ef.speedup(1.0, Tp), p), rel_tol=1e-12)
            assert ef.amdahl_speedup(p, a) <= ef.amdahl_limit(a) + 1e-12       # Eq. 6
    assert ef.amdahl_speedup(6, 0.998) == pytest.approx(5.940594, abs=1e-6)


def test_tlp_comet_case():
    # p1 = 6, p2 = 1..6, alpha1 = 0.998, alpha2 = 0.97 (Fig. 10's curve)
    S = ef.tlp_speedup(6, 0.998, 6, 0.97)
    assert S == pytest.approx(ef.amdahl_speedup(6, 0.998) * 6 / (6 - 0.97 * 5), rel=1e-12)
    assert S == pytest.approx(30.9944, abs=1e-4)
    assert ef.tlp_efficiency(6, 0.998, 6, 0.97) == pytest.approx(S / 36, rel=1e-12)
    assert ef.tlp_speedup(6, 0.998, 1, 0.97) == pytest.approx(ef.amdahl_speedup(6, 0.998))


def test_tlpdpr_flow_past_body():
    beta, p1, p2, p = 0.437, 6, 6, 36
    # "The maximum speedup S_p2 ... comes to 2.3": Eq. 13 as p2 (1+PRI) -> infinity
    assert round(1.0 / beta, 1) == 2.3
    assert ef.tlpdpr_speedup2(beta, 1e12, 0.0) == pytest.approx(1.0 / beta, rel=1e-9)
    # "The TLP algorithm gives the speedup ... which is 80% of the maximum value"
    tlp = ef.tlpdpr_speedup2(beta, p2, 0.0)
    assert round(tlp * beta, 1) == 0.8
    # PRI* from Eq. 15 satisfies the condition Eq. 14 it was derived from (p = p1 p2)
    ps = ef.pri_star(beta, p2)
    assert ps == pytest.approx(3.880995, abs=1e-6)
    assert ef.pri_condition_residual(p, p1, p2, beta, ps) == pytest.approx(0.0, abs=1e-9)
    assert abs(ef.pri_condition_residual(p, p1, p2, beta, ps + 0.1)) > 0.1
    # the paper measured 93% at the optimum; Eq. 13 predicts more (it assumes instant reallocation)
    dpr = ef.tlpdpr_speedup2(beta, p2, ps) * beta
    assert 0.93 <= dpr <= 0.96
    # "equivalent to the usage of TLP algorithm on a 120-processor computer (p2 = 20)": 93% of the maximum
    assert round(ef.tlpdpr_speedup2(beta, 20, 0.0) * beta, 2) == 0.94
    assert ef.p2_actual(p2, ps) == pytest.approx(p2 * (1 + ps))                   # Eq. 12
    assert ef.beta_star(beta, p2) == pytest.approx(0.823234, abs=1e-6)            # Eq. 11


def test_fit_alpha_recovers_amdahl():
    ps = [1, 4, 16, 64, 256]
    for a in (0.3, 0.9, 0.99):
        S = [ef.amdahl_speedup(p, a) for p in ps]
        assert ef.fit_alpha(ps, S) == pytest.approx(a, abs=1e-6)


def test_batching_model_on_sweep():
    rows, alpha = ef.batching_model({1: 0.131, 4: 0.391, 16: 1.405, 64: 5.469, 256: 21.775})
    assert rows[0]["S"] == pytest.approx(1.0)
    assert all(r["E"] <= 1.0 for r in rows)
    assert 0.0 < alpha < 1.0
