"""Seeded synthetic input generators shared by tests, bench and smoke.

Holds no arithmetic of the method: these produce arbitrary particle states
(positions uniform in the domain, normal velocities) and arbitrary per-cell
majorant tables with numpy's PCG64 so that the oracle and the CUDA path can be
started from the *same* state (SURVEY §8(d) parity protocol: "one step from
identical state").
"""
from __future__ import annotations

import numpy as np


def random_state(seed, p, n_particles, T=1.0, drift=(0.0, 0.0, 0.0), dead_frac=0.0,
                 face_margin=2e-5):
    """Return dict(x, y, z, vx, vy, vz, alive) as float32/uint8 numpy arrays.

    Positions are uniform over the domain of problem dict `p`, kept at least
    `face_margin` away from every cell face so the cell index is unambiguous
    (the 1e-5 band of north-star criterion (1) is then empty by construction).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    dims = [p["nx"], p["ny"], p["nz"]][: p["dim"]]
    out = {}
    for a, name in enumerate("xyz"):
        if a < p["dim"]:
            cell = rng.integers(0, dims[a], n_particles)
            frac = rng.uniform(face_margin, 1.0 - face_margin, n_particles)
            out[name] = (cell + frac).astype(np.float32)
        else:
            out[name] = np.zeros(n_particles, np.float32)
    sd = np.sqrt(T)
    for a, name in enumerate(("vx", "vy", "vz")):
        out[name] = (drift[a] + sd * rng.standard_normal(n_particles)).astype(np.float32)
    alive = np.ones(n_particles, np.uint8)
    if dead_frac > 0:
        alive[rng.uniform(size=n_particles) < dead_frac] = 0
    out["alive"] = alive
    return out


def clustered_state(seed, p, cells, ppc, T=1.0):
    """Particles concentrated in the listed flat cells (heavy-cell / skew tests)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    nx, ny = p["nx"], p["ny"]
    cells = np.repeat(np.asarray(cells, np.int64), ppc)
    n = cells.size
    ix = cells % nx
    iy = (cells // nx) % ny
    iz = cells // (nx * ny)
    out = {}
    for a, (name, ic) in enumerate(zip("xyz", (ix, iy, iz))):
        if a < p["dim"]:
            out[name] = (ic + rng.uniform(2e-5, 1 - 2e-5, n)).astype(np.float32)
        else:
            out[name] = np.zeros(n, np.float32)
    perm = rng.permutation(n)
    for k in out:
        out[k] = out[k][perm]
    for name in ("vx", "vy", "vz"):
        out[name] = (np.sqrt(T) * rng.standard_normal(n)).astype(np.float32)
    out["alive"] = np.ones(n, np.uint8)
    return out


def random_gmax(seed, n_cells, lo, hi):
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(lo, hi, n_cells).astype(np.float32)
