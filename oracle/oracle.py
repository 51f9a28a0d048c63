"""ctypes wrapper of the C oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this module.  It imports nothing from the
product package `paper_cs_9902024_b200` (and the product never imports it).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
# mutation testing (tools/mutate_oracle.py) points this at a mutant build
LIB_OVERRIDE = os.environ.get("DSMC_ORACLE_LIB")
SRC = os.path.join(HERE, "dsmc_oracle.c")
CFLAGS = ["-O2", "-std=gnu11", "-Wall", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force=False):
    """Compile the oracle (plain gcc, no FMA contraction)."""
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "dsmc_oracle.h"))):
        return LIB_PATH
    subprocess.check_call(["gcc", *CFLAGS, "-o", LIB_PATH, SRC, "-lm"])
    return LIB_PATH


class Fill(C.Structure):
    _fields_ = [("lo", C.c_int32 * 3), ("hi", C.c_int32 * 3), ("ppc", C.c_int32),
                ("T", C.c_double), ("u", C.c_double * 3)]


class Problem(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
        ("fnum_vc", C.c_double),
        ("model", C.c_int32), ("d_ref", C.c_double), ("omega", C.c_double),
        ("T_ref", C.c_double), ("mass", C.c_double),
        ("bc", C.c_int32 * 6), ("bc_T", C.c_double * 6),
        ("plate_on", C.c_int32), ("plate_axis", C.c_int32), ("plate_span_axis", C.c_int32),
        ("plate_pos", C.c_double), ("plate_lo", C.c_double), ("plate_hi", C.c_double),
        ("plate_T", C.c_double),
        ("orifice_on", C.c_int32), ("orifice_cy", C.c_double), ("orifice_cz", C.c_double),
        ("orifice_r", C.c_double),
        ("inflow_kind", C.c_int32), ("inflow_n", C.c_double), ("inflow_T", C.c_double),
        ("inflow_U", C.c_double), ("inflow_count", C.c_int32),
        ("n_fill", C.c_int32), ("fill", Fill * 4),
        ("dt", C.c_double), ("dt_s", C.c_double), ("dt_L", C.c_double),
        ("seed", C.c_uint32), ("n_runs", C.c_int32), ("run_id0", C.c_int32),
        ("reorder_every", C.c_int32), ("cap_per_run", C.c_int64),
    ]


def make_problem(p):
    s = Problem()
    for name, _ in Problem._fields_:
        if name in ("bc", "bc_T", "fill", "n_fill"):
            continue
        setattr(s, name, p[name])
    for f in range(6):
        s.bc[f] = p["bc"][f]
        s.bc_T[f] = p["bc_T"][f]
    s.n_fill = len(p["fill"])
    for k, F in enumerate(p["fill"]):
        for a in range(3):
            s.fill[k].lo[a] = F["lo"][a]
            s.fill[k].hi[a] = F["hi"][a]
            s.fill[k].u[a] = F["u"][a]
        s.fill[k].ppc = F["ppc"]
        s.fill[k].T = F["T"]
    return s


_lib = None


def lib():
    global _lib
    if _lib is None:
        if LIB_OVERRIDE:
            L = C.CDLL(LIB_OVERRIDE)
        else:
            build()
            L = C.CDLL(LIB_PATH)
        P = C.POINTER
        vp = C.c_void_p
        L.orc_create.restype = vp
        L.orc_create.argtypes = [P(Problem), C.c_int32, P(C.c_int32)]
        L.orc_destroy.argtypes = [vp]
        for fn in ("orc_fill_initial", "orc_step", "orc_status", "orc_step_index", "orc_n_face"):
            getattr(L, fn).restype = C.c_int32
            getattr(L, fn).argtypes = [vp]
        L.orc_steps.restype = C.c_int32
        L.orc_steps.argtypes = [vp, C.c_int32]
        L.orc_sample.restype = C.c_int32
        L.orc_sample.argtypes = [vp, C.c_int32]
        L.orc_sample_add.restype = C.c_int32
        L.orc_sample_add.argtypes = [vp, C.c_int32]
        L.orc_snap_count.restype = C.c_int32
        L.orc_snap_count.argtypes = [vp, C.c_int32]
        L.orc_n_store.restype = C.c_int64
        L.orc_n_store.argtypes = [vp]
        L.orc_counters.argtypes = [vp, vp]
        L.orc_get_state.argtypes = [vp] + [vp] * 7
        L.orc_set_state.restype = C.c_int32
        L.orc_set_state.argtypes = [vp, C.c_int64] + [vp] * 7 + [C.c_int32]
        L.orc_get_gmax.argtypes = [vp, vp]
        L.orc_set_gmax.argtypes = [vp, vp]
        L.orc_get_index.restype = C.c_int64
        L.orc_get_index.argtypes = [vp, vp, vp, vp, vp]
        L.orc_get_cell_stats.argtypes = [vp, vp, vp]
        L.orc_get_snap.restype = C.c_int32
        L.orc_get_snap.argtypes = [vp, C.c_int32, vp]
        L.orc_interact_cell.restype = C.c_int64
        L.orc_interact_cell.argtypes = [vp, C.c_int64, C.c_int32, C.c_int32, vp, vp, vp, vp, vp,
                                        C.c_int64, vp]
        L.orc_diffuse_velocity.argtypes = [vp, C.c_int32, C.c_int32, C.c_double, C.c_uint32,
                                           C.c_uint32, C.c_uint32, vp]
        L.orc_inflow_count.restype = C.c_int64
        L.orc_inflow_count.argtypes = [vp, C.c_int32, C.c_int32]
        L.orc_ensemble.argtypes = [C.c_int32, C.c_int64, vp, C.c_double, vp]
        L.orc_ensemble_m.argtypes = [C.c_int32, C.c_int64, vp, C.c_double, C.c_int32, vp]
        L.orc_philox4x32_10.argtypes = [vp, vp, vp]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def philox(ctr, key):
    c = np.asarray(ctr, np.uint32)
    k = np.asarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def ensemble(sums, fnum_vc, m=1):
    """sums: float64 [n_runs][5][Nc], each run's holding m samples -> [Nc][10]."""
    sums = np.ascontiguousarray(sums, np.float64)
    n_runs, five, Nc = sums.shape
    out = np.zeros((Nc, 10), np.float64)
    lib().orc_ensemble_m(n_runs, Nc, _ptr(sums), fnum_vc, int(m), _ptr(out))
    return out


class OracleRun:
    """One statistically independent run of the oracle."""

    def __init__(self, p, run_id):
        self.p = p
        self.Nc = p["nx"] * p["ny"] * p["nz"]
        self._prob = make_problem(p)
        err = C.c_int32(0)
        h = lib().orc_create(C.byref(self._prob), run_id, C.byref(err))
        if not h:
            raise ValueError(f"oracle rejected problem: code {err.value}")
        self.h = C.c_void_p(h)
        self.run_id = run_id

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def fill(self):
        return lib().orc_fill_initial(self.h)

    def step(self, k=1):
        return lib().orc_steps(self.h, k)

    def sample(self, slot):
        return lib().orc_sample(self.h, slot)

    def sample_add(self, slot):
        """Time averaging (steady problems): add the current state's sums to the slot."""
        return lib().orc_sample_add(self.h, slot)

    def snap_count(self, slot):
        return lib().orc_snap_count(self.h, slot)

    @property
    def n(self):
        return lib().orc_n_store(self.h)

    @property
    def step_index(self):
        return lib().orc_step_index(self.h)

    @property
    def status(self):
        return lib().orc_status(self.h)

    def counters(self):
        out = np.zeros(4, np.int64)
        lib().orc_counters(self.h, _ptr(out))
        return dict(inserted=int(out[0]), removed=int(out[1]), candidates=int(out[2]), accepted=int(out[3]))

    def get_state(self):
        n = self.n
        arrs = {k: np.zeros(n, np.float32) for k in ("x", "y", "z", "vx", "vy", "vz")}
        arrs["alive"] = np.zeros(n, np.uint8)
        lib().orc_get_state(self.h, *[_ptr(arrs[k]) for k in ("x", "y", "z", "vx", "vy", "vz", "alive")])
        return arrs

    def set_state(self, st, step=0):
        n = len(st["x"])
        a = {k: np.ascontiguousarray(st[k], np.float32) for k in ("x", "y", "z", "vx", "vy", "vz")}
        a["alive"] = np.ascontiguousarray(st["alive"], np.uint8)
        rc = lib().orc_set_state(self.h, n, *[_ptr(a[k]) for k in ("x", "y", "z", "vx", "vy", "vz", "alive")], step)
        if rc:
            raise ValueError(f"set_state failed {rc}")

    def get_gmax(self):
        out = np.zeros(self.Nc, np.float32)
        lib().orc_get_gmax(self.h, _ptr(out))
        return out

    def set_gmax(self, g):
        g = np.ascontiguousarray(g, np.float32)
        lib().orc_set_gmax(self.h, _ptr(g))

    def get_index(self):
        n = self.n
        cell = np.zeros(max(n, 1), np.int32)
        count = np.zeros(self.Nc, np.int64)
        start = np.zeros(self.Nc, np.int64)
        lcr = np.zeros(max(n, 1), np.int64)
        live = lib().orc_get_index(self.h, _ptr(cell), _ptr(count), _ptr(start), _ptr(lcr))
        return dict(cell=cell[:n], count=count, start=start, lcr=lcr[:live])

    def get_cell_stats(self):
        cand = np.zeros(self.Nc, np.int64)
        acc = np.zeros(self.Nc, np.int32)
        lib().orc_get_cell_stats(self.h, _ptr(cand), _ptr(acc))
        return cand, acc

    def get_snap(self, slot):
        out = np.zeros((5, self.Nc), np.float64)
        rc = lib().orc_get_snap(self.h, slot, _ptr(out))
        if rc:
            raise ValueError(f"slot {slot} not written ({rc})")
        return out

    def interact_cell(self, cell, step, vx, vy, vz, gmax, max_pairs=4096):
        vx = np.ascontiguousarray(vx, np.float32).copy()
        vy = np.ascontiguousarray(vy, np.float32).copy()
        vz = np.ascontiguousarray(vz, np.float32).copy()
        g = np.array([gmax], np.float32)
        pairs = np.zeros(2 * max_pairs, np.int32)
        ncand = C.c_int64(0)
        acc = lib().orc_interact_cell(self.h, cell, step, len(vx), _ptr(vx), _ptr(vy), _ptr(vz), _ptr(g),
                                      _ptr(pairs), max_pairs, C.byref(ncand))
        return dict(acc=int(acc), cand=int(ncand.value), vx=vx, vy=vy, vz=vz, gmax=float(g[0]),
                    pairs=pairs[: 2 * min(acc, max_pairs)].reshape(-1, 2))

    def diffuse_velocity(self, axis, sign, Tw, idx, step, bounce):
        v = np.zeros(3, np.float32)
        lib().orc_diffuse_velocity(self.h, axis, sign, Tw, idx, step, bounce, _ptr(v))
        return v

    def inflow_count(self, face, step):
        return lib().orc_inflow_count(self.h, face, step)

    @property
    def n_face(self):
        return lib().orc_n_face(self.h)


def run_ensemble(p, run_ids=None, steps=None):
    """Run the oracle for the given run ids (default: all n_runs) and return
    (runs, per-slot sums [n_slots][n_runs][5][Nc])."""
    from workloads import configs  # input module only
    run_ids = list(range(p["run_id0"], p["run_id0"] + p["n_runs"])) if run_ids is None else run_ids
    steps = configs.n_steps(p) if steps is None else steps
    runs = []
    for r in run_ids:
        o = OracleRun(p, r)
        o.fill()
        o.step(steps)
        runs.append(o)
    return runs
