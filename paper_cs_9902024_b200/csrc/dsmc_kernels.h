// dsmc_kernels.h -- host-side launchers of the kernels in dsmc_kernels.cu
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "dsmc_device.cuh"

namespace dsmc {

enum KernelSlot {
  KSLOT_ZERO = 0,
  KSLOT_INFLOW_COUNT,
  KSLOT_INFLOW_EMIT,
  KSLOT_MOTION,
  KSLOT_STEP_MID,
  KSLOT_SCAN_REDUCE,
  KSLOT_SCAN_PARTIALS,
  KSLOT_SCAN_DOWN,
  KSLOT_SCATTER,
  KSLOT_COLLIDE,
  KSLOT_STEP_END,
  KSLOT_COLLIDE_HEAVY,
  KSLOT_COLLIDE_TRIAGE,
  KSLOT_COUNT
};

// optional per-launch callbacks (event timing); empty by default
struct LaunchHook {
  void (*fn)(void* user, int slot, int after) = nullptr;
  void* user = nullptr;
  void before(int slot) const { if (fn) fn(user, slot, 0); }
  void after(int slot) const { if (fn) fn(user, slot, 1); }
};

int64_t scan_tiles(int64_t L);
void launch_zero(uint32_t* a, int64_t n, cudaStream_t st);
void launch_fill_f32(float* a, int64_t n, float v, cudaStream_t st);
void launch_scan(uint32_t* a, int64_t L, uint32_t* part, cudaStream_t st, const LaunchHook& hook);
void launch_fill(const Prm& P, cudaStream_t st);
void launch_macros(const Prm& P, const double* sums, int n_blocks, int m, double fnum_vc, cudaStream_t st);
void launch_selftest_philox(int64_t n, const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out,
                            uint32_t* out_ref, cudaStream_t st);
// an optional second branch for graph capture: the heavy tiles of a triaged (sparse)
// step run on `st` forked from and joined back into the main stream by the two events
struct Branch {
  cudaStream_t st = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
void issue_step(const Prm& P, cudaStream_t st, const LaunchHook& hook, const Branch& br = Branch{});
void issue_sample(const Prm& P, int slot, int add, cudaStream_t st);
const char* kernel_slot_name(int k);

}  // namespace dsmc
