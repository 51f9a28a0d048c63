"""Host-side checks of the C ABI (no GPU needed): the library loads, exports
every function include/dsmc.h declares, and validates problems (error codes
of include/dsmc.h) without touching a device."""
import ctypes as C
import os
import re

import pytest

from workloads import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dsmc_mod():
    from paper_cs_9902024_b200 import build, dsmc
    build.build()
    dsmc.load_library()
    return dsmc


def header_functions():
    src = open(os.path.join(ROOT, "include", "dsmc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(dsmc_\w+)\s*\(", src, flags=re.M)))


def test_exports_every_declared_symbol(dsmc_mod):
    names = header_functions()
    assert len(names) >= 18
    lib = C.CDLL(dsmc_mod.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    bound = {s[0] for s in dsmc_mod.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_no_oracle_in_product():
    """The product path never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_cs_9902024_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower().replace("oracle/ is test-only", ""), f


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5", "c2_small", "c3_small", "c4_small", "c5_small"])
def test_query_sizes_presets(dsmc_mod, name):
    p = configs.get(name)
    s = dsmc_mod.dsmc_query_sizes(p)
    assert s.n_cells == configs.n_cells(p)
    assert s.n_steps == configs.n_steps(p)
    assert s.n_slots == configs.n_slots(p)
    assert s.stride % 32 == 0 and s.stride >= p["cap_per_run"]
    assert s.P == 2 * 6 * 4 * s.stride * p["n_runs"]
    assert s.cell >= 4 * s.n_cells * p["n_runs"]


def test_c4_n256_fits_one_b200(dsmc_mod):
    s = dsmc_mod.dsmc_query_sizes(configs.get("c4", n_runs=256))
    total = sum(getattr(s, k) for k in ("P", "key", "lcr", "cell", "gmax", "C", "ctl", "scratch"))
    assert total < 120e9, total


@pytest.mark.parametrize("mut,code", [
    (dict(dt_s=0.15), -2),                 # dt_s not a multiple of dt
    (dict(dt=-1.0), -2),
    (dict(model=1, omega=0.3), -3),        # omega outside [0.5, 1]
    (dict(dim=4), -1),
    (dict(n_runs=0), -1),
    (dict(bc=[1, 0, 1, 1, 1, 1]), -3),     # periodic on one face only
])
def test_validation_codes(dsmc_mod, mut, code):
    p = configs.get("c4_small")
    p["dt"] = 0.1
    p["dt_s"] = 0.5
    p["dt_L"] = 1.0
    p.update(mut)
    with pytest.raises(dsmc_mod.DsmcError) as e:
        dsmc_mod.dsmc_query_sizes(p)
    assert e.value.code == code


def test_simulation_refuses_without_gpu(dsmc_mod):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(dsmc_mod.DsmcError):
        dsmc_mod.Simulation(configs.get("c4_small"))


def test_too_many_runs_rejected(dsmc_mod):
    """n_runs is the grid y dimension of the generation kernels (<= 65535): a larger
    batch is rejected at validation with EINVAL, not by a failing launch later."""
    p = configs.get("c1", n_runs=65536)
    with pytest.raises(dsmc_mod.DsmcError) as e:
        dsmc_mod.dsmc_query_sizes(p)
    assert e.value.code == -1
    p = configs.get("c1", n_runs=65535)
    assert dsmc_mod.dsmc_query_sizes(p).n_cells == 100


def test_32bit_key_overflow_rejected(dsmc_mod):
    """Keys and LCR entries are 32-bit (run * Nc + cell, run * stride + i): a batch whose
    slots reach 2^32 is rejected at validation (EINVAL), never wrapped silently."""
    p = configs.get("c4", n_runs=1700)               # 1700 * 2,621,440 slots > 2^32
    with pytest.raises(dsmc_mod.DsmcError) as e:
        dsmc_mod.dsmc_query_sizes(p)
    assert e.value.code == -1
    p = configs.get("c4", n_runs=1600)               # 4.19e9 < 2^32 - 1: accepted
    assert dsmc_mod.dsmc_query_sizes(p).n_cells == 64 ** 3
