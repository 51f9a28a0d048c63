"""The canonical-order sorting networks of k_collide (phase C), checked on the host.

The CUDA source's `sort_oem<NN, NE>` (Batcher odd-even merge, comparators past NE
dropped) is compiled with g++ and run on every 0/1 input for NE <= 24 (0-1
principle: a comparator network sorts every input iff it sorts all 0/1 inputs)
and on random inputs for NE = 32.  Reading R11 (canonical LCR order) depends on it.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_cs_9902024_b200", "csrc", "dsmc_kernels.cu")

DRIVER = r"""
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#define __host__
#define __device__
#define __forceinline__ inline
%s
template <int NN, int NE> long check(bool exhaustive) {
  long bad = 0; std::mt19937 g(7);
  const long n = exhaustive ? (1L << NE) : 300000;
  for (long m = 0; m < n; m++) {
    uint32_t a[NN], b[NN];
    for (int i = 0; i < NN; i++)
      a[i] = i < NE ? (exhaustive ? (uint32_t)((m >> i) & 1) : (uint32_t)(g() %% 40)) : 0xFFFFFFFFu;
    std::copy(a, a + NN, b); std::sort(b, b + NN);
    sort_oem<NN, NE>(a);
    if (!std::equal(a, a + NN, b)) bad++;
  }
  return bad;
}
int main() {
  long bad = check<4, 4>(true) + check<8, 8>(true) + check<16, 12>(true) + check<16, 16>(true) +
             check<32, 20>(true) + check<32, 24>(true) + check<32, 32>(false);
  printf("%%ld\n", bad);
  return bad != 0;
}
"""


def test_sorting_networks_sort(tmp_path):
    src = open(SRC).read()
    m = re.search(r"template <int NN, int NE>\n__host__ __device__ __forceinline__ void sort_oem.*?\n}\n", src, re.S)
    assert m, "sort_oem not found in dsmc_kernels.cu"
    cpp = tmp_path / "net.cpp"
    cpp.write_text(DRIVER % m.group(0))
    exe = tmp_path / "net"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-o", str(exe), str(cpp)])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == "0", out.stdout + out.stderr
