"""Thin ctypes binding of libdsmc.so (include/dsmc.h): argument marshalling only.

Every step of the DSMC path runs in the CUDA kernels of libdsmc.so; torch is
used for device memory (caller-owned buffers) and the CUDA stream.  There is
no CPU fallback: if the library is missing or no GPU is visible, calls raise.
Function names mirror the C ABI (dsmc_create, dsmc_generate, dsmc_step,
dsmc_sample, dsmc_read_macros, ...); `Simulation` bundles them.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdsmc.so")

DSMC_ERRORS = {0: "OK", -1: "EINVAL", -2: "ECLOCK", -3: "EPARAM", -4: "ECAP", -5: "EINDEX",
               -6: "ENONFINITE", -7: "ECUDA", -8: "ESCHED", -9: "EBOUNCE", -10: "ECELL"}
MAX_KERNELS = 16
STATUS_COLS = 9          # DSMC_STATUS_COLS of include/dsmc.h


class DsmcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{DSMC_ERRORS.get(code, code)} ({code}): {msg}")
        self.code = code


class FillRegion(C.Structure):
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
        ("n_fill", C.c_int32), ("fill", FillRegion * 4),
        ("dt", C.c_double), ("dt_s", C.c_double), ("dt_L", C.c_double),
        ("seed", C.c_uint32), ("n_runs", C.c_int32), ("run_id0", C.c_int32),
        ("reorder_every", C.c_int32), ("cap_per_run", C.c_int64),
    ]


class Sizes(C.Structure):
    _fields_ = [("P", C.c_size_t), ("key", C.c_size_t), ("lcr", C.c_size_t), ("cell", C.c_size_t),
                ("gmax", C.c_size_t), ("C", C.c_size_t), ("ctl", C.c_size_t), ("scratch", C.c_size_t),
                ("stride", C.c_int64), ("n_cells", C.c_int64),
                ("n_steps", C.c_int32), ("sample_every", C.c_int32), ("n_slots", C.c_int32)]


BUFFER_NAMES = ("P", "key", "lcr", "cell", "gmax", "C", "ctl", "scratch")


class Buffers(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in BUFFER_NAMES]


def make_problem(p) -> Problem:
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

# (name, restype, argtypes) of every symbol include/dsmc.h declares
_VP = C.c_void_p
SIGNATURES = [
    ("dsmc_query_sizes", C.c_int, [C.POINTER(Problem), C.c_int32, C.POINTER(Sizes)]),
    ("dsmc_create", C.c_int, [C.POINTER(Problem), C.POINTER(Buffers), C.c_int32, _VP, C.POINTER(_VP)]),
    ("dsmc_generate", C.c_int, [_VP]),
    ("dsmc_step", C.c_int, [_VP, C.c_int32]),
    ("dsmc_sample", C.c_int, [_VP, C.c_int32]),
    ("dsmc_sample_add", C.c_int, [_VP, C.c_int32]),
    ("dsmc_slot_samples", C.c_int, [_VP, C.c_int32, _VP]),
    ("dsmc_read_macros", C.c_int, [_VP, C.c_int32, _VP]),
    ("dsmc_read_sums", C.c_int, [_VP, C.c_int32, _VP]),
    ("dsmc_slot_sums_ptr", C.c_int, [_VP, C.c_int32, C.POINTER(_VP)]),
    ("dsmc_read_macros_gathered", C.c_int, [_VP, C.c_int32, _VP, C.c_int32, _VP]),
    ("dsmc_status", C.c_int, [_VP, _VP]),
    ("dsmc_get_state", C.c_int, [_VP, C.c_int32, C.POINTER(C.c_int64)] + [_VP] * 7),
    ("dsmc_set_state", C.c_int, [_VP, C.c_int32, C.c_int64] + [_VP] * 7 + [C.c_int32]),
    ("dsmc_get_gmax", C.c_int, [_VP, C.c_int32, _VP]),
    ("dsmc_set_gmax", C.c_int, [_VP, C.c_int32, _VP]),
    ("dsmc_get_index", C.c_int, [_VP, C.c_int32, C.POINTER(C.c_int64), _VP, _VP, _VP, _VP, _VP]),
    ("dsmc_selftest_philox", C.c_int, [C.c_int64, _VP, C.c_uint32, C.c_uint32, _VP, _VP]),
    ("dsmc_kernels_per_step", C.c_int, [_VP, C.POINTER(C.c_int32)]),
    ("dsmc_step_timed", C.c_int, [_VP, C.c_int32, _VP, _VP]),
    ("dsmc_kernel_name", C.c_char_p, [C.c_int32]),
    ("dsmc_destroy", C.c_int, [_VP]),
    ("dsmc_last_error", C.c_char_p, []),
]


def load_library(path=None):
    """Load libdsmc.so (or $DSMC_LIB, for A/B builds); raises, never falls back."""
    global _lib
    path = path or os.environ.get("DSMC_LIB") or LIB_PATH
    if _lib is None:
        if not os.path.exists(path):
            raise DsmcError(-7, f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(path)
        ab = "DSMC_LIB" in os.environ     # A/B builds of older commits may lack newer entry points
        for name, res, args in SIGNATURES:
            if ab and not hasattr(L, name):
                continue
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise DsmcError(rc, load_library().dsmc_last_error().decode())
    return rc


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def dsmc_query_sizes(p, debug=False):
    s = Sizes()
    prob = make_problem(p)
    _check(load_library().dsmc_query_sizes(C.byref(prob), int(debug), C.byref(s)))
    return s


def dsmc_selftest_philox(ctr, k0, k1, with_ref=True):
    ctr = np.ascontiguousarray(ctr, np.uint32).reshape(-1, 4)
    n = ctr.shape[0]
    out = np.zeros((n, 4), np.uint32)
    ref = np.zeros((n, 4), np.uint32) if with_ref else None
    _check(load_library().dsmc_selftest_philox(n, _ptr(ctr), k0, k1, _ptr(out),
                                                _ptr(ref) if with_ref else None))
    return out, ref


def dsmc_kernel_name(k):
    return load_library().dsmc_kernel_name(k).decode()


class Simulation:
    """One dsmc_ctx over torch-owned device buffers (n runs batched)."""

    def __init__(self, p, debug=False, device="cuda:0", stream=None):
        import torch
        if not torch.cuda.is_available():
            raise DsmcError(-7, "no CUDA device: the DSMC path has no CPU fallback")
        L = load_library()
        self.p = p
        self.debug = bool(debug)
        self.device = torch.device(device)
        self.prob = make_problem(p)
        self.sizes = dsmc_query_sizes(p, debug)
        self.Nc = int(self.sizes.n_cells)
        self.R = int(p["n_runs"])
        self.cap = int(p["cap_per_run"])
        self.n_slots = int(self.sizes.n_slots)
        self.n_steps = int(self.sizes.n_steps)
        self.bufs = {}
        cbuf = Buffers()
        for name in BUFFER_NAMES:
            nbytes = max(int(getattr(self.sizes, name)), 16)
            t = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self.bufs[name] = t
            setattr(cbuf, name, t.data_ptr())
        self._cbuf = cbuf
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        _check(L.dsmc_create(C.byref(self.prob), C.byref(cbuf), int(debug),
                             C.c_void_p(self.stream.cuda_stream), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            load_library().dsmc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- the five calls of the boundary
    def generate(self):
        _check(load_library().dsmc_generate(self.h))

    def step(self, n=1):
        _check(load_library().dsmc_step(self.h, int(n)))

    def sample(self, slot):
        _check(load_library().dsmc_sample(self.h, int(slot)))

    def sample_add(self, slot):
        """Time averaging (steady problems): add the current state to the slot."""
        _check(load_library().dsmc_sample_add(self.h, int(slot)))

    def slot_samples(self, slot):
        n = C.c_int32(0)
        _check(load_library().dsmc_slot_samples(self.h, int(slot), C.byref(n)))
        return n.value

    def time_average(self, slot, n_samples, every):
        """Steady flow: n_samples samples of the current run state, `every` steps apart,
        accumulated in `slot` (the unsteady schedule keeps writing its own slots)."""
        for _ in range(int(n_samples)):
            self.step(every)
            self.sample_add(slot)

    def read_macros(self, slot):
        out = np.zeros((self.Nc, 10), np.float64)
        _check(load_library().dsmc_read_macros(self.h, int(slot), _ptr(out)))
        return out

    def read_sums(self, slot):
        out = np.zeros((5, self.R, self.Nc), np.float64)
        _check(load_library().dsmc_read_sums(self.h, int(slot), _ptr(out)))
        return out

    def slot_sums_device(self, slot):
        """The slot's sums [5][R*Nc] fp64 as a torch view of the caller-owned C buffer
        (no copy): the send buffer of the one exchange (runs.gather_slot_sums)."""
        import torch
        ptr = C.c_void_p()
        _check(load_library().dsmc_slot_sums_ptr(self.h, int(slot), C.byref(ptr)))
        n = 5 * self.R * self.Nc
        base = self.bufs["C"]
        off = ptr.value - base.data_ptr()
        assert off % 8 == 0 and off + 8 * n <= base.numel()
        return base[off: off + 8 * n].view(torch.float64)

    def read_macros_gathered(self, slot, sums_dev, n_blocks):
        """Ensemble over n_blocks * R runs from device sums [n_blocks][5][R*Nc] (blocks in
        ascending run id; e.g. an all-gather of every rank's slot_sums_device)."""
        out = np.zeros((self.Nc, 10), np.float64)
        assert sums_dev.is_cuda and sums_dev.dtype.itemsize == 8 and sums_dev.is_contiguous()
        assert sums_dev.numel() == int(n_blocks) * 5 * self.R * self.Nc
        _check(load_library().dsmc_read_macros_gathered(self.h, int(slot), C.c_void_p(sums_dev.data_ptr()),
                                                        int(n_blocks), _ptr(out)))
        return out

    # --- status, checkpoint and test hooks
    def status(self, raise_on_fault=True):
        out = np.zeros((self.R, STATUS_COLS), np.int64)
        rc = load_library().dsmc_status(self.h, _ptr(out))
        if raise_on_fault:
            _check(rc)
        keys = ("inserted", "removed", "candidates", "accepted", "n_store", "step", "live", "particle_steps",
                "max_ppc")
        return rc, [dict(zip(keys, map(int, row))) for row in out]

    def get_state(self, run):
        st = {k: np.zeros(self.cap, np.float32) for k in ("x", "y", "z", "vx", "vy", "vz")}
        st["alive"] = np.zeros(self.cap, np.uint8)
        n = C.c_int64(0)
        _check(load_library().dsmc_get_state(self.h, int(run), C.byref(n),
                                             *[_ptr(st[k]) for k in ("x", "y", "z", "vx", "vy", "vz", "alive")]))
        return {k: v[: n.value].copy() for k, v in st.items()}

    def set_state(self, run, st, step=0):
        n = len(st["x"])
        a = {k: np.ascontiguousarray(st[k], np.float32) for k in ("x", "y", "z", "vx", "vy", "vz")}
        alive = st.get("alive")
        alive_p = None if alive is None else _ptr(np.ascontiguousarray(alive, np.uint8))
        _check(load_library().dsmc_set_state(self.h, int(run), n,
                                             *[_ptr(a[k]) for k in ("x", "y", "z", "vx", "vy", "vz")],
                                             alive_p, int(step)))

    def get_gmax(self, run):
        out = np.zeros(self.Nc, np.float32)
        _check(load_library().dsmc_get_gmax(self.h, int(run), _ptr(out)))
        return out

    def set_gmax(self, run, g):
        g = np.ascontiguousarray(g, np.float32)
        _check(load_library().dsmc_set_gmax(self.h, int(run), _ptr(g)))

    def get_index(self, run):
        live = C.c_int64(0)
        count = np.zeros(self.Nc, np.int64)
        start = np.zeros(self.Nc, np.int64)
        lcr = np.zeros(self.cap + 1, np.int64)
        cand = np.zeros(self.Nc, np.int64)
        acc = np.zeros(self.Nc, np.int32)
        _check(load_library().dsmc_get_index(self.h, int(run), C.byref(live), _ptr(count), _ptr(start),
                                             _ptr(lcr), _ptr(cand), _ptr(acc)))
        return dict(count=count, start=start, lcr=lcr[: live.value], cand=cand, acc=acc)

    def kernels_per_step(self):
        n = C.c_int32(0)
        _check(load_library().dsmc_kernels_per_step(self.h, C.byref(n)))
        return n.value

    def step_timed(self, n):
        ms = np.zeros(MAX_KERNELS, np.float64)
        cnt = np.zeros(MAX_KERNELS, np.int64)
        _check(load_library().dsmc_step_timed(self.h, int(n), _ptr(ms), _ptr(cnt)))
        return {dsmc_kernel_name(k): (float(ms[k]), int(cnt[k])) for k in range(MAX_KERNELS) if cnt[k]}
