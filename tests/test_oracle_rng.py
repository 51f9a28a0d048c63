"""Pins of the oracle's RNG layer (PAPER.md:113-115 'shift
random number generator'; SPEC S:179-199 rng examples).

* Philox4x32-10 block function vs ATen's independent implementation
  (at::Philox4_32, torch/include/ATen/core/PhiloxRNGEngine.h) on many
  (counter, key) pairs -- a library routine, not the oracle itself.
* statistical pins of the variates built on it (chi-square, KS, correlation).
"""
import os
import subprocess

import numpy as np
import pytest
from scipy import stats

HERE = os.path.dirname(os.path.abspath(__file__))

ATEN_SRC = r"""
#include <ATen/core/PhiloxRNGEngine.h>
#include <cstdio>
#include <cstdlib>
// reads lines "seed subsequence offset", prints the 4 words of one block
int main() {
  unsigned long long seed, sub, off;
  while (scanf("%llu %llu %llu", &seed, &sub, &off) == 3) {
    at::Philox4_32 e(seed, sub, off);
    unsigned a = e(), b = e(), c = e(), d = e();
    printf("%u %u %u %u\n", a, b, c, d);
  }
}
"""


@pytest.fixture(scope="module")
def aten_philox(tmp_path_factory):
    import torch
    inc = os.path.join(os.path.dirname(torch.__file__), "include")
    d = tmp_path_factory.mktemp("aten")
    src = d / "p.cpp"
    src.write_text(ATEN_SRC)
    exe = d / "p"
    subprocess.check_call(["g++", "-std=c++17", "-O1", f"-I{inc}", str(src), "-o", str(exe)])
    return str(exe)


def test_philox_matches_aten(oracle_mod, aten_philox):
    rng = np.random.Generator(np.random.PCG64(11))
    ctrs = rng.integers(0, 2**32, size=(400, 4), dtype=np.uint64)
    keys = rng.integers(0, 2**32, size=(400, 2), dtype=np.uint64)
    # edge counters/keys
    ctrs[0] = 0
    keys[0] = 0
    ctrs[1] = 2**32 - 1
    keys[1] = 2**32 - 1
    # ATen layout: key = seed (lo, hi), counter = (offset lo, offset hi, subseq lo, subseq hi)
    lines = []
    for c, k in zip(ctrs, keys):
        seed = int(k[0]) | (int(k[1]) << 32)
        off = int(c[0]) | (int(c[1]) << 32)
        sub = int(c[2]) | (int(c[3]) << 32)
        lines.append(f"{seed} {sub} {off}")
    out = subprocess.run([aten_philox], input="\n".join(lines) + "\n", capture_output=True,
                         text=True, check=True).stdout.split("\n")
    for c, k, line in zip(ctrs, keys, out):
        want = [int(w) for w in line.split()]
        got = oracle_mod.philox(c.astype(np.uint32), k.astype(np.uint32))
        assert list(map(int, got)) == want, (c, k)


def _stream(oracle_mod, key, n_blocks, c1=0):
    return np.concatenate([oracle_mod.philox([i, c1, 0, 0], key) for i in range(n_blocks)])


def test_uniform_chi_square(oracle_mod):
    w = _stream(oracle_mod, [4, 0], 25_000)          # 1e5 words
    u = (w >> 8).astype(np.float64) * 2.0**-24        # u_co
    assert u.min() >= 0.0 and u.max() < 1.0
    hist, _ = np.histogram(u, bins=100, range=(0, 1))
    p = stats.chisquare(hist).pvalue
    assert p > 1e-3, p


def test_runs_uncorrelated(oracle_mod):
    a = (_stream(oracle_mod, [4, 0], 5000) >> 8) * 2.0**-24
    b = (_stream(oracle_mod, [4, 1], 5000) >> 8) * 2.0**-24
    assert abs(np.corrcoef(a, b)[0, 1]) < 0.01 * 3   # 2e4 samples: SE 0.007
    # disjoint streams: no identical blocks
    assert len(set(a.tolist()) & set(b.tolist())) < 50


def test_replay_deterministic(oracle_mod):
    a = _stream(oracle_mod, [9, 3], 100)
    b = _stream(oracle_mod, [9, 3], 100)
    assert (a == b).all()


def test_lemire_index_unbiased(oracle_mod):
    # i = (w * N) >> 32 hits every index in [0, N) with equal probability
    w = _stream(oracle_mod, [5, 5], 20_000).astype(np.uint64)
    N = 7
    idx = (w * N) >> 32
    assert idx.max() < N
    p = stats.chisquare(np.bincount(idx.astype(np.int64), minlength=N)).pvalue
    assert p > 1e-3


def test_diffuse_velocity_distribution(oracle_mod):
    """diffuse re-emission = flux-weighted half-Maxwellian.  Normal
    component ~ Rayleigh(sqrt(Tw)), tangential ~ N(0, Tw) (KS, 1e5 draws is
    too slow through ctypes; 2e4 draws keeps the test under seconds)."""
    from workloads import configs
    p = configs.get("c2_small")
    o = oracle_mod.OracleRun(p, 0)
    Tw = 2.0
    v = np.array([o.diffuse_velocity(0, 1, Tw, i, 3, 0) for i in range(20_000)])
    assert (v[:, 0] >= 0).all()
    assert stats.kstest(v[:, 0], stats.rayleigh(scale=np.sqrt(Tw)).cdf).pvalue > 1e-3
    assert stats.kstest(v[:, 1], stats.norm(scale=np.sqrt(Tw)).cdf).pvalue > 1e-3
    assert stats.kstest(v[:, 2], stats.norm(scale=np.sqrt(Tw)).cdf).pvalue > 1e-3
    # the upper face emits with negative normal velocity, on axis 1
    w = np.array([o.diffuse_velocity(1, -1, Tw, i, 3, 1) for i in range(2000)])
    assert (w[:, 1] <= 0).all()
