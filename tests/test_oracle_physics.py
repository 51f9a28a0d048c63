"""Pins of the oracle's DSMC step against closed forms, invariants and brute
force (SURVEY §8(c) "What pins each part"; SPEC S:75-131 examples).

Each test names the paper passage the oracle function follows and the
independent fact it is checked against.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
from scipy import integrate, special, stats

from workloads import configs, inputs


# ----------------------------------------------------------------- helpers
def f32_round(q: Fraction) -> np.float32:
    """Correctly rounded (ties-to-even) float32 of an exact rational."""
    f = np.float32(float(q))
    best = f
    for cand in (np.nextafter(f, np.float32(-np.inf)), np.nextafter(f, np.float32(np.inf))):
        d_c, d_b = abs(Fraction(float(cand)) - q), abs(Fraction(float(best)) - q)
        if d_c < d_b or (d_c == d_b and (cand.view(np.uint32) & 1) == 0):
            best = cand
    return best


def fmaf_exact(a, b, c):
    return f32_round(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def no_collisions(p):
    q = dict(p)
    q["fnum_vc"] = 0.0
    return q


def live_count(o):
    return int(o.get_state()["alive"].sum())


# ------------------------------------------------------------------ Motion
def test_free_flight_is_fmaf(oracle_mod):
    """PAPER.md:98-100 Motion: x <- x + v dt; with periodic faces far away the
    result must be the correctly rounded fma of the inputs (closed form)."""
    p = no_collisions(configs.get("c4_small"))
    p["reorder_every"] = 0
    st = inputs.random_state(1, p, 500, face_margin=0.05)
    st["x"] = (st["x"] * 0.5 + 3.0).astype(np.float32)   # stay inside [3, 11): no wrap
    st["y"] = (st["y"] * 0.5 + 3.0).astype(np.float32)
    st["z"] = (st["z"] * 0.5 + 3.0).astype(np.float32)
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(st, step=0)
    o.step(1)
    out = o.get_state()
    dt = np.float32(p["dt"])
    for i in range(0, 500, 5):
        for a, va in (("x", "vx"), ("y", "vy"), ("z", "vz")):
            assert out[a][i] == fmaf_exact(st[va][i], dt, st[a][i])
    assert (out["vx"] == st["vx"]).all()


def test_specular_mirror_example(oracle_mod):
    """specular wall at x=L, particle at L-eps moving +x: x -> 2L-(x+v dt),
    v_x -> -v_x."""
    p = no_collisions(configs.get("c1"))
    L = np.float32(100.0)
    st = dict(x=np.array([L - np.float32(0.01)], np.float32), y=np.zeros(1, np.float32),
              z=np.zeros(1, np.float32), vx=np.array([1.5], np.float32),
              vy=np.array([0.2], np.float32), vz=np.array([-0.3], np.float32),
              alive=np.ones(1, np.uint8))
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(st)
    o.step(1)
    out = o.get_state()
    x1 = fmaf_exact(st["vx"][0], np.float32(p["dt"]), st["x"][0])
    assert out["x"][0] == np.float32(2 * L) - x1
    assert out["vx"][0] == -st["vx"][0] and out["vy"][0] == st["vy"][0]
    # and the lower wall
    st["x"][0] = np.float32(0.05)
    st["vx"][0] = np.float32(-2.0)
    o.set_state(st)
    o.step(1)
    out = o.get_state()
    assert out["x"][0] == -fmaf_exact(st["vx"][0], np.float32(p["dt"]), st["x"][0])
    assert out["vx"][0] == np.float32(2.0)


def test_periodic_wrap_keeps_everything_inside(oracle_mod):
    p = no_collisions(configs.get("c4_small"))
    st = inputs.random_state(2, p, 20_000, T=25.0)   # fast particles cross faces
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(st)
    o.step(3)
    out = o.get_state()
    assert out["alive"].sum() == 20_000
    for a in "xyz":
        assert out[a].min() >= 0 and out[a].max() < 16


def test_diffuse_wall_conserves_count_and_reflects(oracle_mod):
    """c2's x=0 diffuse wall: particles hitting it come back with v_x>0; with
    all other faces outflow, count balance is exact."""
    p = no_collisions(configs.get("c2_small"))
    st = inputs.random_state(3, p, 5000)
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(st)
    before = live_count(o)
    o.step(5)
    c = o.counters()
    assert live_count(o) == before - c["removed"] + c["inserted"]
    assert c["removed"] > 0


def test_free_molecular_expansion(oracle_mod):
    """Collisionless release from a uniform square into vacuum with outflow on
    all sides (SURVEY C-pins 'free-molecular expansion'): the density is
    n0 * P_x * P_y with P = 1/2[erf((b-x)/(sqrt2 s)) - erf((a-x)/(sqrt2 s))],
    s = sqrt(T) t.  Cell averages by the antiderivative of erf; chi-square-
    like check against the Poisson/binomial count error over 8 runs."""
    p = no_collisions(configs.get("c2_small"))
    p["bc"] = [configs.OUTFLOW] * 4 + [configs.PERIODIC] * 2
    p["reorder_every"] = 0
    nsteps = 25
    x0, x1, y0, y1, ppc = 20, 32, 24, 40, 50
    p["fill"] = [dict(lo=[x0, y0, 0], hi=[x1, y1, 1], ppc=ppc, T=1.0, u=[0.0, 0.0, 0.0])]
    p["cap_per_run"] = (x1 - x0) * (y1 - y0) * ppc
    nx, ny = p["nx"], p["ny"]
    counts = np.zeros((ny, nx))
    R = 8
    for r in range(R):
        o = oracle_mod.OracleRun(p, r)
        o.fill()
        o.step(nsteps)
        st = o.get_state()
        al = st["alive"] == 1
        h, _, _ = np.histogram2d(st["y"][al], st["x"][al], bins=[ny, nx], range=[[0, ny], [0, nx]])
        counts += h
    t = nsteps * np.float32(p["dt"])
    s = math.sqrt(2.0) * t

    def G(z):  # antiderivative of erf
        return z * special.erf(z) + np.exp(-z * z) / math.sqrt(math.pi)

    def cell_frac(n, a, b):
        e = np.arange(n + 1, dtype=np.float64)
        # integral over [e_i, e_i+1] of 1/2[erf((b-x)/s) - erf((a-x)/s)] dx
        I = lambda x: 0.5 * s * (-G((b - x) / s) + G((a - x) / s))
        return np.diff(I(e))

    Px = cell_frac(nx, x0, x1)
    Py = cell_frac(ny, y0, y1)
    expect = R * ppc * np.outer(Py, Px)
    m = expect > 20
    z = (counts[m] - expect[m]) / np.sqrt(expect[m])
    assert abs(z.mean()) < 4 / math.sqrt(m.sum())
    assert (np.abs(z) < 5).all()
    assert 0.7 < (z * z).mean() < 1.3


# ------------------------------------------------------ Enumeration/Indexing
def test_index_toy_three_particles(oracle_mod):
    """3 particles in cell 0 of a 2-cell grid -> starts [0,3], perm [0,1,2]."""
    p = no_collisions(configs.get("c1"))
    p.update(nx=2, fill=[], cap_per_run=3)
    p["bc"] = [configs.SPECULAR] * 2 + [configs.PERIODIC] * 4
    st = dict(x=np.array([0.5, 0.25, 0.75], np.float32), y=np.zeros(3, np.float32),
              z=np.zeros(3, np.float32), vx=np.zeros(3, np.float32), vy=np.zeros(3, np.float32),
              vz=np.zeros(3, np.float32), alive=np.ones(3, np.uint8))
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(st)
    o.step(1)
    ix = o.get_index()
    assert ix["count"].tolist() == [3, 0]
    assert ix["start"].tolist() == [0, 3]
    assert ix["lcr"].tolist() == [0, 1, 2]


def test_index_empty_store(oracle_mod):
    """empty store -> all counts/starts zero."""
    p = no_collisions(configs.get("c4_small"))
    p["fill"] = []
    o = oracle_mod.OracleRun(p, 0)
    o.step(1)
    ix = o.get_index()
    assert (ix["count"] == 0).all() and (ix["start"] == 0).all() and len(ix["lcr"]) == 0


def test_index_brute_force(oracle_mod):
    """1e4 random particles; LCR segments equal a brute-force per-cell
    membership scan, in ascending store index (stable); dead excluded."""
    p = no_collisions(configs.get("c4_small"))
    p["reorder_every"] = 0
    st = inputs.random_state(5, p, 10_000, dead_frac=0.1)
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(st)
    o.step(1)
    out = o.get_state()
    ix = o.get_index()
    cell = (np.floor(out["x"]).astype(np.int64) + 16 * (np.floor(out["y"]).astype(np.int64)
            + 16 * np.floor(out["z"]).astype(np.int64)))
    alive = out["alive"] == 1
    for c in range(0, 16 ** 3, 7):
        members = np.nonzero(alive & (cell == c))[0]
        seg = ix["lcr"][ix["start"][c]: ix["start"][c] + ix["count"][c]]
        assert seg.tolist() == members.tolist()
    assert ix["count"].sum() == alive.sum()


# ------------------------------------------------------------- Interaction
def test_no_collisions_below_two(oracle_mod):
    p = configs.get("c4_small")
    o = oracle_mod.OracleRun(p, 0)
    for N in (0, 1):
        r = o.interact_cell(3, 0, np.ones(N), np.zeros(N), np.zeros(N), 50.0)
        assert r["acc"] == 0 and r["cand"] == 0


def test_pair_conservation(oracle_mod):
    """every accepted pair conserves momentum and energy (fp32: 1e-5 rel)."""
    p = configs.get("c4_small")
    o = oracle_mod.OracleRun(p, 0)
    rng = np.random.Generator(np.random.PCG64(7))
    n_acc = 0
    for c in range(300):
        N = 12
        vx, vy, vz = (rng.standard_normal(N).astype(np.float32) for _ in range(3))
        r = o.interact_cell(c, 1, vx, vy, vz, 40.0)
        n_acc += r["acc"]
        P0 = np.array([vx.sum(), vy.sum(), vz.sum()], np.float64)
        P1 = np.array([r["vx"].astype(np.float64).sum(), r["vy"].astype(np.float64).sum(),
                       r["vz"].astype(np.float64).sum()])
        E0 = (vx.astype(np.float64) ** 2 + vy.astype(np.float64) ** 2 + vz.astype(np.float64) ** 2).sum()
        E1 = (r["vx"].astype(np.float64) ** 2 + r["vy"].astype(np.float64) ** 2 + r["vz"].astype(np.float64) ** 2).sum()
        scale = math.sqrt(E0)
        assert np.abs(P1 - P0).max() <= 1e-5 * max(scale, np.abs(P0).max())
        assert abs(E1 - E0) <= 1e-5 * E0
    assert n_acc > 100


def test_ntc_all_pairs_identity(oracle_mod):
    """NTC pair law (SURVEY C-pins): with x = 1/2 N(N-1) coef gmax < 1 so M<=1,
    P(pair ab collides in a step) = coef * sigma(g_ab) g_ab exactly,
    independent of N and gmax.  Chi-square over keyed trials vs that law."""
    p = configs.get("c4_small")
    o = oracle_mod.OracleRun(p, 0)
    coef = p["fnum_vc"] * p["dt"]
    vx = np.array([0.0, 1.0, -0.5, 2.0], np.float32)
    vy = np.array([0.0, 0.5, 1.5, -1.0], np.float32)
    vz = np.array([0.0, -1.0, 0.25, 0.5], np.float32)
    N = 4
    sg = {}
    for i in range(N):
        for j in range(i + 1, N):
            g2 = float((np.float32(vx[i] - vx[j]) ** 2 + np.float32(vy[i] - vy[j]) ** 2)
                       + np.float32(vz[i] - vz[j]) ** 2)
            sg[(i, j)] = math.pi * math.sqrt(g2)
    gmax = np.float32(max(sg.values()) * 1.05)
    assert 0.5 * N * (N - 1) * coef * float(gmax) < 1
    trials = 100_000
    hits = {k: 0 for k in sg}
    for s in range(trials):
        r = o.interact_cell(11, s, vx, vy, vz, gmax, max_pairs=4)
        for i, j in r["pairs"]:
            hits[(min(i, j), max(i, j))] += 1
    obs = np.array([hits[k] for k in sg] + [trials - sum(hits.values())], np.float64)
    pk = np.array([coef * sg[k] for k in sg])
    exp = np.append(pk, 1 - pk.sum()) * trials
    assert stats.chisquare(obs, exp).pvalue > 1e-3


def test_ntc_selection_uniform_over_pairs(oracle_mod):
    """Each candidate picks an unordered pair with probability 2/(N(N-1)):
    tiny gmax makes every candidate accepted, so accepted pairs = candidates."""
    p = configs.get("c4_small")
    p["fnum_vc"] = 50.0
    o = oracle_mod.OracleRun(p, 0)
    rng = np.random.Generator(np.random.PCG64(8))
    N = 5
    cnt = np.zeros((N, N))
    for s in range(300):
        vx, vy, vz = (rng.standard_normal(N).astype(np.float32) * 3 for _ in range(3))
        r = o.interact_cell(2, s, vx, vy, vz, 1e-3, max_pairs=100000)
        assert r["acc"] == r["cand"]
        for i, j in r["pairs"]:
            cnt[min(i, j), max(i, j)] += 1
    obs = cnt[np.triu_indices(N, 1)]
    assert stats.chisquare(obs).pvalue > 1e-3


def _rate_box(oracle_mod, model, T, n_cells=14, steps=60, skip=10):
    p = configs.get("c4_small")
    p.update(nx=n_cells, ny=n_cells, nz=n_cells, model=model, omega=0.74 if model == configs.VHS else 0.5,
             cap_per_run=n_cells ** 3 * 10,
             fill=[dict(lo=[0, 0, 0], hi=[n_cells] * 3, ppc=10, T=T, u=[0.0, 0.0, 0.0])])
    o = oracle_mod.OracleRun(p, 0)
    o.fill()
    o.step(skip)
    a0 = o.counters()["accepted"]
    o.step(steps)
    acc = o.counters()["accepted"] - a0
    return p, acc


def test_hs_equilibrium_collision_rate(oracle_mod):
    """North star: HS equilibrium rate n^2 sigma <g> / 2 within 1%, with
    <g> = 4 sqrt(kT/(pi m)) (closed form)."""
    p, acc = _rate_box(oracle_mod, configs.HS, 1.0, n_cells=16, steps=100)
    Nc = 16 ** 3
    n_d = 10 * p["fnum_vc"]                      # real number density
    g_mean = 4.0 / math.sqrt(math.pi)
    expect = 0.5 * n_d * n_d * math.pi * g_mean * Nc * p["dt"] / p["fnum_vc"] * 100
    expect *= 1.0 - 1.0 / (Nc * 10)              # E[N(N-1)] for fixed total
    assert abs(acc / expect - 1.0) < 0.01, acc / expect
    assert abs(acc - expect) < 4 * math.sqrt(expect)


@pytest.mark.parametrize("T", [1.0, 2.0])
def test_vhs_equilibrium_collision_rate(oracle_mod, T):
    """VHS: <sigma g>(T) = pi d_ref^2 <g>_ref (T/T_ref)^(1-omega) (closed form of
    the VHS cross-section averaged over the Maxwellian relative speed)."""
    p, acc = _rate_box(oracle_mod, configs.VHS, T, n_cells=16, steps=100)
    Nc = 16 ** 3
    n_d = 10 * p["fnum_vc"]
    sg = math.pi * (4.0 / math.sqrt(math.pi)) * T ** (1 - 0.74)
    expect = 0.5 * n_d * n_d * sg * Nc * p["dt"] / p["fnum_vc"] * 100 * (1 - 1 / (Nc * 10))
    assert abs(acc / expect - 1.0) < 0.01, acc / expect


def test_maxwellian_preserved(oracle_mod):
    """Equilibrium box: per-component mean 0, variance T, kurtosis 3, KS normal."""
    p = configs.get("c4_small")
    o = oracle_mod.OracleRun(p, 0)
    o.fill()
    o.step(20)
    st = o.get_state()
    n = len(st["vx"])
    for k in ("vx", "vy", "vz"):
        v = st[k].astype(np.float64)
        assert abs(v.mean()) < 4 / math.sqrt(n)
        assert abs(v.var() - 1.0) < 4 * math.sqrt(2.0 / n)
        assert abs(stats.kurtosis(v, fisher=False) - 3.0) < 4 * math.sqrt(24.0 / n)
        assert stats.kstest(v, "norm").pvalue > 1e-3
    # total momentum / energy conserved by the collisions in a periodic box
    E = sum((st[k].astype(np.float64) ** 2).sum() for k in ("vx", "vy", "vz"))
    o2 = oracle_mod.OracleRun(p, 0)
    o2.fill()
    s0 = o2.get_state()
    E0 = sum((s0[k].astype(np.float64) ** 2).sum() for k in ("vx", "vy", "vz"))
    assert abs(E / E0 - 1) < 1e-5


def test_fill_exact_counts_and_maxwellian(oracle_mod):
    """Initial fill (C-3): exactly ppc per cell; velocities N(u, T)."""
    p = configs.get("c1")
    o = oracle_mod.OracleRun(p, 0)
    o.fill()
    st = o.get_state()
    cells = np.floor(st["x"]).astype(int)
    cnt = np.bincount(cells, minlength=100)
    assert (cnt[:50] == 40).all() and (cnt[50:] == 10).all()
    p3 = configs.get("c3_small")
    o3 = oracle_mod.OracleRun(p3, 0)
    o3.fill()
    s3 = o3.get_state()
    assert abs(s3["vx"].mean() - configs.MACH5_U) < 4 / math.sqrt(len(s3["vx"]))
    assert stats.kstest(s3["vy"], "norm").pvalue > 1e-3


# -------------------------------------------------------------- Generation
def _edge_loss(s):
    # expected fraction of an edge face cell's ghosts whose y leaves [0, ny)
    # during the entry flight: int_0^1 Phi(-y/s) dy
    return integrate.quad(lambda y: stats.norm.cdf(-y / s), 0, 1)[0]


def test_inflow_ghost_flux(oracle_mod):
    """mean inserted count = Phi A dt / F_N with the drifting-Maxwellian
    flux Phi = n (cbar/4)[exp(-s^2) + sqrt(pi) s (1 + erf s)]."""
    p = no_collisions(configs.get("c3_small"))
    p["fill"] = []
    p["plate_on"] = 0
    p["reorder_every"] = 1
    steps = 400
    o = oracle_mod.OracleRun(p, 0)
    ins = 0
    for _ in range(steps):
        o.step(1)
    ins = o.counters()["inserted"]
    T, U, n = p["inflow_T"], p["inflow_U"], p["inflow_n"]
    sr = U / math.sqrt(2 * T)
    cbar = math.sqrt(8 * T / math.pi)
    phi = n * cbar / 4 * (math.exp(-sr * sr) + math.sqrt(math.pi) * sr * (1 + math.erf(sr)))
    dt = float(np.float32(p["dt"]))
    per_face = phi * dt
    ny = p["ny"]
    expect = steps * per_face * (ny - 2 * _edge_loss(math.sqrt(T) * dt))
    # each face-step count is floor(x+u) (variance <= 1/4) thinned binomially
    sd = math.sqrt(steps * ny * (per_face + 0.25))
    assert abs(ins - expect) < 4 * sd, (ins, expect, sd)


def test_inflow_ghost_count_mean(oracle_mod):
    """E[floor(x + u)] = x for u ~ U[0,1) (C-4 count rule), over 1e4 steps."""
    p = configs.get("c3_small")
    o = oracle_mod.OracleRun(p, 0)
    w = (p["inflow_U"] + 6 * math.sqrt(p["inflow_T"])) * p["dt"]
    x = p["inflow_n"] * w
    c = np.array([o.inflow_count(f, s) for s in range(2000) for f in range(5)])
    assert set(np.unique(c)) <= {math.floor(x), math.floor(x) + 1}
    assert abs(c.mean() - x) < 4 * math.sqrt(0.25 / len(c))


def test_inflow_effusive(oracle_mod):
    """c5 orifice: the staircase disk of radius 8 has 208 face cells (brute
    force), exactly inflow_count per face cell per step, normal velocity
    Rayleigh(sqrt T) (flux-weighted half-Maxwellian)."""
    p = no_collisions(configs.get("c5"))
    jj, kk = np.meshgrid(np.arange(128), np.arange(128))
    assert int((((jj + 0.5 - 64) ** 2 + (kk + 0.5 - 64) ** 2) <= 64).sum()) == 208
    p.update(nx=16, ny=128, nz=128, fill=[], cap_per_run=100_000, reorder_every=0)
    o = oracle_mod.OracleRun(p, 0)
    assert o.n_face == 208
    o.step(1)
    c = o.counters()
    assert c["inserted"] == 208 * 100
    st = o.get_state()
    assert stats.kstest(st["vx"], stats.rayleigh().cdf).pvalue > 1e-3
    assert stats.kstest(st["vy"], "norm").pvalue > 1e-3
    tau = st["x"] / st["vx"]
    assert tau.min() >= 0 and tau.max() <= np.float32(p["dt"]) * (1 + 1e-6)


def test_open_system_count_balance(oracle_mod):
    """Delta count = inserts - removals, every config with open faces."""
    for name in ("c2_small", "c3_small", "c5_small"):
        p = configs.get(name, n_steps=20)
        o = oracle_mod.OracleRun(p, 0)
        o.fill()
        n0 = live_count(o)
        o.step(20)
        c = o.counters()
        assert live_count(o) == n0 + c["inserted"] - c["removed"], name
        assert o.status == 0, name


def test_closed_box_count_constant(oracle_mod):
    for name in ("c1", "c4_small"):
        p = configs.get(name)
        o = oracle_mod.OracleRun(p, 0)
        o.fill()
        n0 = o.n
        o.step(30)
        assert live_count(o) == n0 and o.status == 0


def test_plate_reflects(oracle_mod):
    """c3 plate: no particle crosses the zero-thickness plate in one step:
    start just below it moving up -> ends below it (diffuse, T_w = 2)."""
    p = no_collisions(configs.get("c3_small"))
    n = 2000
    rng = np.random.Generator(np.random.PCG64(4))
    st = dict(x=rng.uniform(20, 80, n).astype(np.float32),
              y=np.full(n, 11.95, np.float32), z=np.zeros(n, np.float32),
              vx=np.zeros(n, np.float32), vy=rng.uniform(1, 5, n).astype(np.float32),
              vz=np.zeros(n, np.float32), alive=np.ones(n, np.uint8))
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(st)
    o.step(1)
    out = o.get_state()
    assert (out["y"][:n] < 12.0).all()          # inflow appends after index n
    assert (out["vy"][:n] <= 0).all()


# ---------------------------------------------------------------- Sampling
def test_sampling_toys(oracle_mod):
    """empty cell -> zeros; one particle -> its own sums."""
    p = no_collisions(configs.get("c4_small"))
    p["dt_s"] = p["dt"]
    st = dict(x=np.array([0.5], np.float32), y=np.array([0.5], np.float32), z=np.array([0.5], np.float32),
              vx=np.array([0.1], np.float32), vy=np.array([0.0], np.float32), vz=np.array([0.0], np.float32),
              alive=np.ones(1, np.uint8))
    o = oracle_mod.OracleRun(p, 0)
    o.set_state(st)
    o.step(1)
    S = o.get_snap(0)
    c = 0
    assert S[0, c] == 1 and S[1, c] == np.float64(np.float32(0.1))
    assert S[4, c] == np.float64(np.float32(0.1)) ** 2
    assert S[:, 1:].sum() == 0


def test_ensemble_properties(oracle_mod):
    """single run -> SE 0; identical runs idempotent; SE ~ 1/sqrt(n)."""
    rng = np.random.Generator(np.random.PCG64(1))
    Nc = 50
    one = np.zeros((1, 5, Nc))
    one[0, 0] = 10
    one[0, 1:4] = rng.standard_normal((3, Nc)) * 3
    one[0, 4] = 30 + rng.uniform(0, 1, Nc)
    e1 = oracle_mod.ensemble(one, 0.02)
    assert (e1[:, 5:] == 0).all()
    e4 = oracle_mod.ensemble(np.repeat(one, 4, axis=0), 0.02)
    assert np.allclose(e4[:, :5], e1[:, :5], rtol=1e-12) and np.allclose(e4[:, 5:], 0, atol=1e-9)
    # equilibrium box: SE(n=4)/SE(n=16) ~ 2 within 30%
    p = configs.get("c4_small", n_runs=16, n_steps=5)
    sums = []
    for r in range(16):
        o = oracle_mod.OracleRun(p, r)
        o.fill()
        o.step(5)
        sums.append(o.get_snap(0))
    sums = np.array(sums)
    se4 = oracle_mod.ensemble(sums[:4], p["fnum_vc"])[:, 5:].mean(axis=0)
    se16 = oracle_mod.ensemble(sums, p["fnum_vc"])[:, 5:].mean(axis=0)
    ratio = se4 / se16
    assert ((ratio > 2 * 0.7) & (ratio < 2 * 1.3)).all(), ratio
    # equilibrium temperature within 3 SE of T=1 on the pooled cells
    e = oracle_mod.ensemble(sums, p["fnum_vc"])
    Tm = e[:, 4].mean()
    assert abs(Tm - 1.0) < 0.01


def test_run_deterministic(oracle_mod):
    """a run is a pure function of (problem, run id, seed)."""
    p = configs.get("c2_small", n_steps=20)
    a = oracle_mod.OracleRun(p, 3)
    a.fill()
    a.step(10)
    b = oracle_mod.OracleRun(p, 3)
    b.fill()
    b.step(10)
    sa, sb = a.get_state(), b.get_state()
    for k in sa:
        assert (sa[k] == sb[k]).all()


def test_time_average_accumulates_snapshots(oracle_mod):
    """Steady problems (NEXT-4): sample_add accumulates exactly the
    snapshot sums a separate run takes at the same moments, in order, and counts them."""
    p = configs.get("c4_small", n_steps=40)
    a = oracle_mod.OracleRun(p, 1)
    b = oracle_mod.OracleRun(p, 1)
    a.fill()
    b.fill()
    slot = configs.n_slots(p) - 1
    acc = np.zeros((5, a.Nc))
    for _ in range(6):
        a.step(3)
        b.step(3)
        a.sample_add(slot)
        b.sample(0)
        acc = acc + b.get_snap(0)
    assert a.snap_count(slot) == 6
    assert np.array_equal(a.get_snap(slot), acc)
    a.sample(slot)                       # a snapshot overwrites: count back to 1
    assert a.snap_count(slot) == 1


def test_time_average_estimators(oracle_mod):
    """Density of a time average of m samples = mean of the m snapshot densities
    (S_N F_N/V_c/(n m)); in a closed box its mean over cells is the exact particle
    count per cell; averaging shrinks the cell-to-cell density scatter."""
    p = configs.get("c4_small", n_steps=200)
    m, every = 25, 4
    runs = [oracle_mod.OracleRun(p, r) for r in range(2)]
    snaps = [[] for _ in runs]
    acc = []
    for o, sn in zip(runs, snaps):
        o.fill()
        for _ in range(m):
            o.step(every)
            o.sample(0)
            sn.append(o.get_snap(0))
        acc.append(np.sum(sn, axis=0))
    fv = p["fnum_vc"]
    avg = oracle_mod.ensemble(np.array(acc), fv, m)
    inst = [oracle_mod.ensemble(np.array([sn[k] for sn in snaps]), fv) for k in range(m)]
    assert np.allclose(avg[:, 0], np.mean([e[:, 0] for e in inst], axis=0), rtol=1e-12)
    Nc = configs.n_cells(p)
    n_tot = sum(o.n for o in runs)
    assert math.isclose(avg[:, 0].mean(), n_tot * fv / (2 * Nc), rel_tol=1e-12)
    sd_inst = np.mean([e[:, 0].std() for e in inst])
    assert avg[:, 0].std() < 0.5 * sd_inst, (avg[:, 0].std(), sd_inst)
    assert abs(np.nanmean(avg[:, 4]) - 1.0) < 0.01      # equilibrium temperature


def test_marsaglia_direction_isotropic(oracle_mod):
    """R14 pin: the post-collision direction is uniform on the sphere whichever
    try (the pair block's or a direction block's) produced it.  A two-particle
    cell with v = (+-1, 0, 0) keeps c_m = 0 and h = 1, so after the step v_0 is
    the last accepted candidate's unit vector e: its z must be uniform on
    [-1, 1] (Archimedes) and its azimuth uniform on (-pi, pi]."""
    p = configs.get("c4_small")
    gmax = 6.0                                   # < 2 pi: every candidate of g = 2 is accepted (HS)
    p["fnum_vc"] = 2.0 / (gmax * p["dt"])        # about two candidates per trial
    o = oracle_mod.OracleRun(p, 0)
    es = []
    for t in range(6000):
        r = o.interact_cell(t % 4096, t // 4096, np.array([1.0, -1.0]), np.zeros(2), np.zeros(2), gmax)
        if r["acc"]:
            assert r["acc"] == r["cand"]
            es.append((r["vx"][0], r["vy"][0], r["vz"][0]))
    e = np.array(es, np.float64)
    n = len(e)
    assert n > 4000
    assert np.allclose(np.linalg.norm(e, axis=1), 1.0, atol=1e-6)
    assert np.abs(e.mean(0)).max() < 4 / math.sqrt(3 * n)
    assert stats.kstest(e[:, 2], stats.uniform(loc=-1, scale=2).cdf).pvalue > 1e-3
    phi = np.arctan2(e[:, 1], e[:, 0])
    assert stats.kstest(phi, stats.uniform(loc=-math.pi, scale=2 * math.pi).cdf).pvalue > 1e-3
