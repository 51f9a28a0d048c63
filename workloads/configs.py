"""Workload definitions (inputs only) shared by the CUDA path and the oracle.

This module holds the *problem statements* of BASELINE.json's five configs as
plain dictionaries of numbers: grid, boundary kinds, clock (dt, dt_s, dt_L),
fill regions, inflow, seed, batch size.  It contains none of the method's
arithmetic (no motion, indexing, collision or sampling rule); both the CUDA
binding (`paper_cs_9902024_b200.dsmc`) and the oracle wrapper (`oracle.oracle`)
read these dicts and marshal them into their own, independently defined C
structs.

Units (reading R1): m = k = 1, unit cells, and the
cell width equals the mean free path of the config's reference state:
    n_d(lambda = 1) = 1/(sqrt(2) pi d^2),  F_N/V_c = n_d / N_ref,
    tau_ref = lambda / cbar = sqrt(pi/8),   dt = f * tau_ref.
PAPER.md:61-68 (Fig. 1 caption) names dt, dt_s, dt_L and n; the numbers are
BASELINE.json's configs[0..4].
"""
from __future__ import annotations

import copy
import math

# boundary kinds (same numeric codes are used by both C structs)
SPECULAR, PERIODIC, DIFFUSE, OUTFLOW, INFLOW = 0, 1, 2, 3, 4
HS, VHS = 0, 1
INFLOW_NONE, INFLOW_GHOST, INFLOW_EFFUSIVE = 0, 1, 2

# reference state: d = 1, T = 1, m = 1
N_D_LAMBDA1 = 1.0 / (math.sqrt(2.0) * math.pi)   # 0.2250790790392765
TAU_REF = math.sqrt(math.pi / 8.0)               # 0.6266570686577501
MACH5_U = 5.0 * math.sqrt(5.0 / 3.0)             # 6.454972243679028


def _base(**kw):
    p = dict(
        dim=3, nx=1, ny=1, nz=1,
        fnum_vc=1.0, model=HS, d_ref=1.0, omega=0.5, T_ref=1.0, mass=1.0,
        bc=[PERIODIC] * 6, bc_T=[1.0] * 6,
        plate_on=0, plate_axis=1, plate_span_axis=0, plate_pos=0.0,
        plate_lo=0.0, plate_hi=0.0, plate_T=1.0,
        orifice_on=0, orifice_cy=0.0, orifice_cz=0.0, orifice_r=0.0,
        inflow_kind=INFLOW_NONE, inflow_n=0.0, inflow_T=1.0, inflow_U=0.0,
        inflow_count=0,
        fill=[],            # list of dict(lo=[..3], hi=[..3], ppc=int, T=float, u=[..3])
        dt=0.1, dt_s=0.1, dt_L=0.1,
        seed=0, n_runs=1, run_id0=0, reorder_every=4, cap_per_run=0,
    )
    p.update(kw)
    return p


def _clock(f, n_steps, sample_every):
    dt = f * TAU_REF
    return dict(dt=dt, dt_s=dt * sample_every, dt_L=dt * n_steps)


def c1(n_runs=8):
    """configs[0]: 1D/3V shock tube, HS, 100 cells, specular ends, 40|10 ppc."""
    return _base(
        dim=1, nx=100, fnum_vc=N_D_LAMBDA1 / 40.0, model=HS,
        bc=[SPECULAR, SPECULAR, PERIODIC, PERIODIC, PERIODIC, PERIODIC],
        fill=[dict(lo=[0, 0, 0], hi=[50, 1, 1], ppc=40, T=1.0, u=[0.0, 0.0, 0.0]),
              dict(lo=[50, 0, 0], hi=[100, 1, 1], ppc=10, T=1.0, u=[0.0, 0.0, 0.0])],
        seed=1, n_runs=n_runs, reorder_every=4, cap_per_run=2500,
        **_clock(0.2, 200, 10))


def c2(n_runs=64, n_steps=400):
    """configs[1]: 2D/3V release into vacuum, HS, 256x256, source 32x32 at 50 ppc."""
    return _base(
        dim=2, nx=256, ny=256, fnum_vc=N_D_LAMBDA1 / 50.0, model=HS,
        bc=[DIFFUSE, OUTFLOW, OUTFLOW, OUTFLOW, PERIODIC, PERIODIC],
        fill=[dict(lo=[0, 112, 0], hi=[32, 144, 1], ppc=50, T=1.0, u=[0.0, 0.0, 0.0])],
        seed=2, n_runs=n_runs, reorder_every=4, cap_per_run=51200,
        **_clock(0.25, n_steps, 20))


def c3(n_runs=16, n_steps=1000, cap_per_run=4 << 20):
    """configs[2]: 2D/3V Mach-5 flow over a flat diffuse plate, VHS omega=0.74."""
    return _base(
        dim=2, nx=512, ny=256, fnum_vc=N_D_LAMBDA1 / 20.0, model=VHS, omega=0.74,
        bc=[INFLOW, OUTFLOW, OUTFLOW, OUTFLOW, PERIODIC, PERIODIC],
        plate_on=1, plate_axis=1, plate_span_axis=0, plate_pos=64.0,
        plate_lo=64.0, plate_hi=448.0, plate_T=2.0,
        inflow_kind=INFLOW_GHOST, inflow_n=20.0, inflow_T=1.0, inflow_U=MACH5_U,
        fill=[dict(lo=[0, 0, 0], hi=[512, 256, 1], ppc=20, T=1.0, u=[MACH5_U, 0.0, 0.0])],
        seed=3, n_runs=n_runs, reorder_every=4, cap_per_run=cap_per_run,
        **_clock(0.3, n_steps, 50))


def c4(n_runs=256, n_steps=100, sample_every=10):
    """configs[3]: 3D periodic equilibrium box 64^3, HS, 10 ppc (batching sweep).

    BASELINE gives no sampling interval for c4; reading R9 takes dt_s = 10 dt."""
    return _base(
        dim=3, nx=64, ny=64, nz=64, fnum_vc=N_D_LAMBDA1 / 10.0, model=HS,
        bc=[PERIODIC] * 6,
        fill=[dict(lo=[0, 0, 0], hi=[64, 64, 64], ppc=10, T=1.0, u=[0.0, 0.0, 0.0])],
        # physical reorder every 2 steps (measured on B200 at n = 256: 21.8 ms/step
        # against 22.4 for K = 4 and 22.0 for K = 3; K is a problem parameter)
        seed=4, n_runs=n_runs, reorder_every=2, cap_per_run=64 * 64 * 64 * 10,
        **_clock(0.2, n_steps, sample_every))


def c5(n_runs=4, n_steps=2000, cap_per_run=56 << 20):
    """configs[4]: 3D/3V jet from a radius-8 orifice in the x=0 wall, VHS."""
    return _base(
        dim=3, nx=256, ny=128, nz=128, fnum_vc=N_D_LAMBDA1 / 200.0, model=VHS, omega=0.74,
        bc=[DIFFUSE, OUTFLOW, OUTFLOW, OUTFLOW, OUTFLOW, OUTFLOW],
        orifice_on=1, orifice_cy=64.0, orifice_cz=64.0, orifice_r=8.0,
        inflow_kind=INFLOW_EFFUSIVE, inflow_T=1.0, inflow_count=100,
        fill=[dict(lo=[0, 0, 0], hi=[256, 128, 128], ppc=2, T=1.0, u=[0.0, 0.0, 0.0])],
        seed=5, n_runs=n_runs, reorder_every=4, cap_per_run=cap_per_run,
        **_clock(0.2, n_steps, 100))


# --- reduced variants: same physics and code paths, sizes the oracle finishes
# in seconds (parity tests).  Each keeps several collide tiles and a ragged tail.

def c2_small(n_runs=4, n_steps=60):
    p = c2(n_runs=n_runs, n_steps=n_steps)
    p.update(nx=64, ny=64, fill=[dict(lo=[0, 24, 0], hi=[12, 40, 1], ppc=50, T=1.0, u=[0.0, 0.0, 0.0])],
             cap_per_run=12 * 16 * 50)
    return p


def c3_small(n_runs=2, n_steps=80):
    p = c3(n_runs=n_runs, n_steps=n_steps, cap_per_run=200_000)
    p.update(nx=96, ny=48, plate_pos=12.0, plate_lo=12.0, plate_hi=84.0,
             fill=[dict(lo=[0, 0, 0], hi=[96, 48, 1], ppc=20, T=1.0, u=[MACH5_U, 0.0, 0.0])])
    p["dt_s"] = p["dt"] * 10
    return p


def c4_small(n_runs=2, n_steps=20, n=16):
    p = c4(n_runs=n_runs, n_steps=n_steps, sample_every=5)
    p.update(nx=n, ny=n, nz=n, fill=[dict(lo=[0, 0, 0], hi=[n, n, n], ppc=10, T=1.0, u=[0.0, 0.0, 0.0])],
             cap_per_run=n * n * n * 10)
    return p


def c5_small(n_runs=2, n_steps=60):
    p = c5(n_runs=n_runs, n_steps=n_steps, cap_per_run=400_000)
    p.update(nx=48, ny=32, nz=32, orifice_cy=16.0, orifice_cz=16.0, orifice_r=4.0,
             inflow_count=20,
             fill=[dict(lo=[0, 0, 0], hi=[48, 32, 32], ppc=2, T=1.0, u=[0.0, 0.0, 0.0])])
    p["dt_s"] = p["dt"] * 10
    return p


PRESETS = dict(c1=c1, c2=c2, c3=c3, c4=c4, c5=c5,
               c2_small=c2_small, c3_small=c3_small, c4_small=c4_small, c5_small=c5_small)


def get(name, **kw):
    return copy.deepcopy(PRESETS[name](**kw))


def n_cells(p):
    return p["nx"] * p["ny"] * p["nz"]


def n_steps(p):
    return int(round(p["dt_L"] / p["dt"]))


def sample_every(p):
    return int(round(p["dt_s"] / p["dt"]))


def n_slots(p):
    return n_steps(p) // sample_every(p)
