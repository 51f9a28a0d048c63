"""Pins of oracle behaviours that the round-1 pin suite left open (VERDICT r01,
"What's weak" #1): each test below fails for the mutant named in its docstring.

  - the flight after a diffuse bounce uses the remaining time;
  - particles crossing the x=0 wall inside the orifice disk leave the domain
    (PAPER.md:124-127), those crossing outside it come back;
  - an effusive particle enters after a uniformly sampled fraction of dt;
  - the majorant (sigma g)_max is raised after the step to the largest sigma g seen
    (reading R13);
  - the jackknife SE has the leave-one-out scale (n-1)/n;
  - run-time faults latch by precedence, not by visiting order (reading R24).

Every expected value comes from a closed form, brute force or an exact identity
evaluated here, never from the CUDA path.
"""
import math
from fractions import Fraction

import numpy as np
from scipy import special, stats

from workloads import configs, inputs


def f32_round(q: Fraction) -> np.float32:
    f = np.float32(float(q))
    best = f
    for cand in (np.nextafter(f, np.float32(-np.inf)), np.nextafter(f, np.float32(np.inf))):
        d_c, d_b = abs(Fraction(float(cand)) - q), abs(Fraction(float(best)) - q)
        if d_c < d_b or (d_c == d_b and (cand.view(np.uint32) & 1) == 0):
            best = cand
    return best


def fmaf_exact(a, b, c):
    """Correctly rounded fp32 a*b + c (the reading's fmaf) by exact rationals."""
    return f32_round(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def div_f32(a, b):
    return f32_round(Fraction(float(a)) / Fraction(float(b)))


def no_collisions(p):
    q = dict(p)
    q["fnum_vc"] = 0.0
    return q


# ------------------------------------------------------------ diffuse bounce
def test_diffuse_bounce_flies_the_remaining_time(oracle_mod):
    """PAPER.md:98-100 (Motion with surface interaction, reading R10):
    a particle that hits the diffuse wall x=0 at t_h = (0 - x)/v_x is placed on
    the wall, re-emitted with v' and flies the REST of the step:
        x_end = 0 + v'_x (dt - t_h),  y_end = (y + v_y t_h) + v'_y (dt - t_h).
    Mutant killed: `tau = tau - t` -> `tau = tau` (the full dt flown again)."""
    p = no_collisions(configs.get("c2_small"))
    p["fill"] = []
    p["reorder_every"] = 0
    n = 40
    rng = np.random.Generator(np.random.PCG64(21))
    x0 = rng.uniform(0.01, 0.2, n).astype(np.float32)
    y0 = rng.uniform(20.0, 44.0, n).astype(np.float32)
    vx = rng.uniform(-4.0, -2.0, n).astype(np.float32)     # x0 + vx dt < 0 for every particle
    vy = rng.uniform(-1.0, 1.0, n).astype(np.float32)
    st = dict(x=x0, y=y0, z=np.zeros(n, np.float32), vx=vx, vy=vy,
              vz=rng.standard_normal(n).astype(np.float32), alive=np.ones(n, np.uint8))
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(st, step=0)
    o.step(1)
    out = o.get_state()
    dt = np.float32(p["dt"])
    assert (out["alive"] == 1).all()
    for i in range(n):
        assert fmaf_exact(vx[i], dt, x0[i]) < 0
        t_h = div_f32(np.float32(0.0) - x0[i], vx[i])
        y_h = fmaf_exact(vy[i], t_h, y0[i])
        vp = o.diffuse_velocity(0, 1, p["bc_T"][0], i, 0, 0)     # the bounce's draw (key: particle, step, bounce 0)
        assert vp[0] > 0
        rest = f32_round(Fraction(float(dt)) - Fraction(float(t_h)))
        assert out["x"][i] == fmaf_exact(vp[0], rest, np.float32(0.0)), i
        assert out["y"][i] == fmaf_exact(vp[1], rest, y_h), i
        assert (out["vx"][i], out["vy"][i], out["vz"][i]) == tuple(vp)


# --------------------------------------------------------------- orifice
def _orifice_problem(p):
    p = no_collisions(p)
    p.update(nx=8, ny=32, nz=32, orifice_cy=16.0, orifice_cz=16.0, orifice_r=4.0,
             inflow_kind=configs.INFLOW_NONE, inflow_count=0, reorder_every=0,
             fill=[dict(lo=[0, 8, 8], hi=[4, 24, 24], ppc=40, T=1.0, u=[0.0, 0.0, 0.0])])
    p["cap_per_run"] = 4 * 16 * 16 * 40
    return p


def test_orifice_removes_exactly_the_disk_crossings(oracle_mod):
    """PAPER.md:124-127 / reading R10 (c5): a particle whose straight flight crosses
    x=0 inside the staircase disk leaves the domain; outside the disk the diffuse
    wall returns it (v_x > 0).  Brute force over the pre-step state of 8 runs, and
    the removal count against the effusion closed form
        E[removed] = ppc * A_disk * dt * sqrt(T / 2 pi)      (within 3 sigma, Poisson).
    Mutant killed: the orifice-crossing removal deleted."""
    p = _orifice_problem(configs.get("c5_small"))
    jj, kk = np.meshgrid(np.arange(32), np.arange(32), indexing="ij")
    open_face = ((jj + 0.5 - 16) ** 2 + (kk + 0.5 - 16) ** 2) <= 16.0      # [j][k]
    A = int(open_face.sum())
    dt = np.float32(p["dt"])
    removed = 0
    for run in range(8):
        o = oracle_mod.OracleRun(p, run)
        o.fill()
        s0 = o.get_state()
        o.step(1)
        s1 = o.get_state()
        # sign of fmaf(v, dt, x) = sign of the exact v dt + x, which fp64 gets right
        x1 = s0["vx"].astype(np.float64) * float(dt) + s0["x"].astype(np.float64)
        hit = np.nonzero(x1 < 0)[0]
        expect_dead = set()
        for i in hit:
            t = div_f32(np.float32(0.0) - s0["x"][i], s0["vx"][i])
            yc = fmaf_exact(s0["vy"][i], t, s0["y"][i])
            zc = fmaf_exact(s0["vz"][i], t, s0["z"][i])
            if open_face[int(math.floor(yc)), int(math.floor(zc))]:
                expect_dead.add(int(i))
        dead = set(np.nonzero(s1["alive"] == 0)[0].tolist())
        assert dead == expect_dead, run
        back = [i for i in hit if int(i) not in expect_dead]
        assert len(back) > 100 and (s1["vx"][back] > 0).all()
        assert o.counters()["removed"] == len(dead)
        removed += len(dead)
    expect = 8 * 40 * A * float(dt) * math.sqrt(1.0 / (2 * math.pi))
    assert abs(removed - expect) < 3 * math.sqrt(expect), (removed, expect)


# ------------------------------------------------------------ effusive entry
def test_effusive_entry_fraction_is_uniform(oracle_mod):
    """SPEC.md:72 / reading R8: an effusive particle is placed on the face and
    advanced by a uniformly sampled fraction u of dt, so tau = x / v_x is U[0, dt)
    (KS).  Mutant killed: `u * dt` -> `dt`."""
    p = no_collisions(configs.get("c5"))
    p.update(nx=16, ny=128, nz=128, fill=[], cap_per_run=100_000, reorder_every=0)
    o = oracle_mod.OracleRun(p, 0)
    o.step(1)
    st = o.get_state()
    dt = float(np.float32(p["dt"]))
    tau = st["x"].astype(np.float64) / st["vx"].astype(np.float64)
    assert len(tau) == 208 * 100
    assert stats.kstest(tau / dt, "uniform").pvalue > 1e-3
    assert tau.mean() < 0.52 * dt


# ------------------------------------------------------- majorant update
def _sigma_c_vhs(omega):
    # sigma g = pi d^2 (2 k T_ref / (m_r g^2))^(omega - 1/2) g / Gamma(5/2 - omega), m_r = 1/2, d = T_ref = 1
    return math.pi * 4.0 ** (omega - 0.5) / special.gamma(2.5 - omega)


def test_majorant_raised_to_largest_sigma_g(oracle_mod):
    """Reading R13: (sigma g)_max is frozen during the step and afterwards becomes
    max((sigma g)_max, sigma g(max g^2)).  Two-particle cells with a majorant far
    below their sigma g and x = coef gmax ~ 1.5 (one or two candidates, every one
    accepted): with one candidate the new majorant is exactly fp32(sigma g(g^2))
    of the input pair; a majorant above every sigma g is left unchanged.
    Mutant killed: the post-step update deleted (or applied unconditionally)."""
    rng = np.random.Generator(np.random.PCG64(33))
    assert abs(_sigma_c_vhs(0.74) - 4.755628) < 1e-6          # SURVEY C-8's printed constant
    for model, omega, sc in ((configs.HS, 0.5, math.pi), (configs.VHS, 0.74, _sigma_c_vhs(0.74))):
        p = configs.get("c4_small")
        p.update(model=model, omega=omega)
        g_low = 1e-3
        p["fnum_vc"] = 1.5 / (g_low * p["dt"])
        o = oracle_mod.OracleRun(p, 0)
        n_one = 0
        for t in range(200):
            v = rng.standard_normal((3, 2)).astype(np.float32)
            d = (v[:, 0] - v[:, 1]).astype(np.float32)
            g2 = np.float32(np.float32(d[0] * d[0] + d[1] * d[1]) + np.float32(d[2] * d[2]))
            sg = sc * math.sqrt(float(g2)) if model == configs.HS else sc * float(g2) ** (1 - omega)
            r = o.interact_cell(t, 3, v[0], v[1], v[2], g_low)
            assert r["cand"] in (1, 2) and r["acc"] == r["cand"]
            if r["cand"] == 1:
                n_one += 1
                assert abs(r["gmax"] - np.float32(sg)) <= 1.2e-7 * sg, (model, t, r["gmax"], sg)
            else:   # the second candidate sees the post-collision pair: |g| preserved up to rounding
                assert abs(r["gmax"] / sg - 1) < 1e-5
            hi = np.float32(sg * 1.5)
            q = o.interact_cell(t, 4, v[0], v[1], v[2], hi)
            assert q["gmax"] == hi
        assert n_one > 50


# ------------------------------------------------------------- jackknife
def test_jackknife_scale_exact_for_density(oracle_mod):
    """SPEC.md:285, reading R18: the leave-one-run-out jackknife
    SE of a LINEAR statistic equals the textbook standard error of the mean,
        SE(rho) = sd(rho_r, ddof = 1) / sqrt(n),   rho_r = N_r F_N/V_c,
    exactly (up to rounding).  Mutant killed: factor (n-1)/n -> n/(n-1)."""
    rng = np.random.Generator(np.random.PCG64(5))
    for n in (2, 5, 16):
        Nc = 30
        sums = np.zeros((n, 5, Nc))
        sums[:, 0] = rng.integers(0, 40, (n, Nc))
        sums[:, 1:4] = rng.standard_normal((n, 3, Nc)) * 5
        sums[:, 4] = 60 + rng.uniform(0, 10, (n, Nc))
        fv = 0.0225
        e = oracle_mod.ensemble(sums, fv)
        rho_r = sums[:, 0] * fv
        se = rho_r.std(axis=0, ddof=1) / math.sqrt(n)
        assert np.allclose(e[:, 5], se, rtol=1e-10, atol=1e-14), n
        assert np.allclose(e[:, 0], rho_r.mean(axis=0), rtol=1e-12)


# ---------------------------------------------------------- fault latch
def test_fault_precedence_is_order_free(oracle_mod):
    """Reading R24: a NaN velocity makes both a non-finite velocity and (through the
    position) an indexing fault; the latch reports ENONFINITE (-6) whichever the
    particle order.  A particle far outside a periodic box alone gives EINDEX (-5)."""
    p = configs.get("c4_small", n_runs=1)
    for pos in (3, 4000):
        st = inputs.random_state(3, p, 4096)
        st["x"][7] = np.float32(3 * p["nx"] + 0.5)           # outside after the wrap: EINDEX
        st["vx"][7] = np.float32(0.0)
        st["vx"][pos] = np.float32("nan")                    # before or after it in store order
        o = oracle_mod.OracleRun(p, 0)
        o.set_state(st)
        o.step(1)
        assert o.status == -6, (pos, o.status)
    st = inputs.random_state(3, p, 4096)
    st["x"][7] = np.float32(3 * p["nx"] + 0.5)
    st["vx"][7] = np.float32(0.0)
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(st)
    o.step(1)
    assert o.status == -5


def test_periodic_exact_upper_face_wraps_to_lower(oracle_mod):
    """Reading R10 / SURVEY C-5 periodic rule 'x >= hi -> x - (hi - lo)': a flight that
    lands exactly on the upper face x = L comes back at 0 (the half-open cell [0, 1)),
    exactly.  Mutant killed: `x >= L` -> `x > L` (the particle kept on the face)."""
    p = no_collisions(configs.get("c4_small"))
    p["fill"] = []
    p["reorder_every"] = 0
    dt = np.float32(p["dt"])
    L = np.float32(p["nx"])
    xs, vs = [], []
    for v in np.linspace(0.5, 3.0, 40).astype(np.float32):
        x = np.float32(L - np.float32(v * dt))
        for _ in range(8):                         # nudge x until the fmaf lands on L exactly
            y = fmaf_exact(v, dt, x)
            if y == L:
                break
            x = np.nextafter(x, np.float32(-np.inf) if y > L else np.float32(np.inf))
        if fmaf_exact(v, dt, x) == L:
            xs.append(x)
            vs.append(v)
    n = len(xs)
    assert n >= 10
    st = dict(x=np.array(xs, np.float32), y=np.full(n, 5.5, np.float32), z=np.full(n, 7.5, np.float32),
              vx=np.array(vs, np.float32), vy=np.zeros(n, np.float32), vz=np.zeros(n, np.float32),
              alive=np.ones(n, np.uint8))
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(st)
    o.step(1)
    out = o.get_state()
    assert (out["x"] == 0.0).all(), out["x"]
    ix = o.get_index()
    assert ix["count"][0 + 16 * (5 + 16 * 7)] == n
