// dsmc_kernels.cu -- sm_100a kernels of the batched unsteady-DSMC step.
//
// Step = inner loop (1) of PAPER.md Fig. 1 (lines 95-110), batched over the
// n independent runs of the outer loop (2) (lines 112-115):
//
//   k_zero          counts <- 0                                   (LCR prep)
//   k_inflow_count  per (run, face cell): kept inflow particles   Generation
//   k_inflow_emit   append them at each run's tail, key, count    Generation
//   k_motion        free flight + surfaces, cell key, count       Motion, Enumeration
//   k_step_mid      store lengths, reorder flags                  (control)
//   k_scan_*        exclusive scan of counts -> starts            Indexing
//   k_scatter       LCR[start + rank] = particle                  Indexing
//   k_collide       per cell: canonical order, NTC, Sampling,     Interaction, Sampling
//                   (sigma g)_max, physical reorder
//   k_step_end      parity/length after reorder, step++           (control)
//
// The paper's "Indexing ... can not be parallelized, so it is performed by one
// processor" is replaced by a parallel counting sort; the
// within-cell order (ascending store index, reading R11) is restored inside
// k_collide, which stages each tile of cells in shared memory.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <curand_kernel.h>

#include "dsmc_device.cuh"
#include "dsmc_kernels.h"

namespace dsmc {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int DSMC_MODEL_HS = 0, DSMC_MODEL_VHS = 1;   // Prm::model

// ------------------------------------------------------------- async copies
// Bulk (TMA 1D) copy global -> shared completing on an mbarrier (sm_90+; SASS
// UBLKCP / SYNCS), and 4-byte cp.async (LDGSTS) gathers that land in shared
// memory without holding registers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ====================================================================== util
__global__ void k_zero(uint32_t* __restrict__ a, int64_t n) {
  const int64_t n4 = n >> 2;
  uint4* a4 = reinterpret_cast<uint4*>(a);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride)
    a4[i] = make_uint4(0, 0, 0, 0);
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) a[n4 * 4 + threadIdx.x] = 0;
}

__global__ void k_fill_f32(float* __restrict__ a, int64_t n, float v) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = v;
}

// ==================================================================== scan
// three-phase exclusive scan of uint32 counts (tile = 2048 elements / block)
constexpr int SCAN_T = 256, SCAN_PER = 8, SCAN_TILE = SCAN_T * SCAN_PER;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t t = lane < nw ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(FULL, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) s_warp[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  total = s_warp[nw - 1];
  const uint32_t wpre = wid ? s_warp[wid - 1] : 0;
  __syncthreads();
  return wpre + x - v;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_reduce(const uint32_t* __restrict__ a, int64_t L,
                                                        uint32_t* __restrict__ part) {
  __shared__ uint32_t s_warp[32];
  const int64_t b = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_PER;
  uint32_t s = 0;
  if (b + SCAN_PER <= L) {
    const uint4 v0 = __ldg(reinterpret_cast<const uint4*>(a + b));
    const uint4 v1 = __ldg(reinterpret_cast<const uint4*>(a + b + 4));
    s = v0.x + v0.y + v0.z + v0.w + v1.x + v1.y + v1.z + v1.w;
  } else {
    for (int i = 0; i < SCAN_PER; i++) if (b + i < L) s += a[b + i];
  }
  uint32_t total;
  block_excl_scan(s, s_warp, total);
  if (threadIdx.x == 0) part[blockIdx.x] = total;
}

// one block: each warp scans a contiguous segment of the tile sums 32 at a time
// (coalesced loads, all issued up front), then the warp totals are scanned
__global__ void __launch_bounds__(1024) k_scan_partials(uint32_t* __restrict__ part, int64_t nb) {
  __shared__ uint32_t s_warp[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t seg = (nb + 1023) / 1024 * 32;     // elements per warp, a multiple of 32
  const int64_t b = (int64_t)wid * seg;
  uint32_t tot = 0;
  for (int64_t c0 = 0; c0 < seg; c0 += 32 * 16) {
    uint32_t v[16];
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const int64_t i = b + c0 + u * 32 + lane;
      v[u] = c0 + u * 32 < seg && i < nb ? part[i] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 16; u++) tot += __reduce_add_sync(FULL, v[u]);
  }
  if (lane == 0) s_warp[wid] = tot;
  __syncthreads();
  if (wid == 0) {
    const uint32_t x = s_warp[lane];
    uint32_t y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const uint32_t z = __shfl_up_sync(FULL, y, o); if (lane >= o) y += z; }
    s_warp[lane] = y - x;                          // exclusive warp offsets
    if (lane == 31) part[nb] = y;
  }
  __syncthreads();
  uint32_t run = s_warp[wid];
  for (int64_t c0 = 0; c0 < seg; c0 += 32 * 16) {
    uint32_t v[16];
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const int64_t i = b + c0 + u * 32 + lane;
      v[u] = c0 + u * 32 < seg && i < nb ? part[i] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 16; u++) {
      uint32_t y = v[u];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) { const uint32_t z = __shfl_up_sync(FULL, y, o); if (lane >= o) y += z; }
      const int64_t i = b + c0 + u * 32 + lane;
      if (c0 + u * 32 < seg && i < nb) part[i] = run + y - v[u];
      run += __shfl_sync(FULL, y, 31);
    }
  }
}

__global__ void __launch_bounds__(SCAN_T) k_scan_down(uint32_t* __restrict__ a, int64_t L,
                                                      const uint32_t* __restrict__ part) {
  __shared__ uint32_t s_warp[32];
  const int64_t b = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_PER;
  uint32_t v[SCAN_PER];
  const bool full = b + SCAN_PER <= L;
  if (full) {
    const uint4 v0 = *reinterpret_cast<const uint4*>(a + b);
    const uint4 v1 = *reinterpret_cast<const uint4*>(a + b + 4);
    v[0] = v0.x; v[1] = v0.y; v[2] = v0.z; v[3] = v0.w; v[4] = v1.x; v[5] = v1.y; v[6] = v1.z; v[7] = v1.w;
  } else {
    for (int i = 0; i < SCAN_PER; i++) v[i] = b + i < L ? a[b + i] : 0;
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_PER; i++) s += v[i];
  uint32_t total;
  uint32_t run = block_excl_scan(s, s_warp, total) + part[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SCAN_PER; i++) { const uint32_t t = v[i]; v[i] = run; run += t; }
  if (full) {
    *reinterpret_cast<uint4*>(a + b) = make_uint4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<uint4*>(a + b + 4) = make_uint4(v[4], v[5], v[6], v[7]);
  } else {
    for (int i = 0; i < SCAN_PER; i++) if (b + i < L) a[b + i] = v[i];
  }
}

// ==================================================================== fill
__device__ __forceinline__ int fill_region(const Prm& P, int64_t c, int32_t ic[3]) {
  ic[0] = (int32_t)(c % P.nx);
  ic[1] = (int32_t)((c / P.nx) % P.ny);
  ic[2] = (int32_t)(c / ((int64_t)P.nx * P.ny));
  for (int k = 0; k < P.n_fill; k++) {
    bool in = true;
    for (int a = 0; a < 3; a++) in = in && ic[a] >= P.fill_lo[k][a] && ic[a] < P.fill_hi[k][a];
    if (in) return k;
  }
  return -1;
}

__global__ void k_fill_count(Prm P) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P.Nc) return;
  int32_t ic[3];
  const int k = fill_region(P, c, ic);
  P.cell[c] = k < 0 ? 0u : (uint32_t)P.fill_ppc[k];
}

// warp per (cell, run); store order (cell, k) (reading R7)
__global__ void k_fill_emit(Prm P) {
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int r = blockIdx.y, lane = threadIdx.x & 31;
  if (c >= P.Nc) return;
  int32_t ic[3];
  const int k = fill_region(P, c, ic);
  if (k < 0) return;
  const uint32_t off = P.cell[c];
  const int ppc = P.fill_ppc[k];
  const uint2 key = run_key(P, r);
  const int64_t base = (int64_t)r * P.stride;
  const double sq = P.fill_sqrtT[k];
  for (int q = lane; q < ppc; q += 32) {
    const int64_t i = (int64_t)off + q;
    if (i >= P.cap) { latch(P, ST_CAP); continue; }
    const uint4 w = draw(key, (uint32_t)c, FILL_STEP, TAG_FILL, (uint32_t)q, 0);
    const uint4 u = draw(key, (uint32_t)c, FILL_STEP, TAG_FILL, (uint32_t)q, 1);
    const uint32_t ww[3] = {w.x, w.y, w.z};
    for (int a = 0; a < 3; a++) parr(P, 0, a)[base + i] = a < P.dim ? place(ic[a], ww[a]) : 0.0f;
    double n1, n2, n3, n4;
    box_muller(u.x, u.y, n1, n2);
    box_muller(u.z, u.w, n3, n4);
    parr(P, 0, 3)[base + i] = (float)(P.fill_u[k][0] + sq * n1);
    parr(P, 0, 4)[base + i] = (float)(P.fill_u[k][1] + sq * n2);
    parr(P, 0, 5)[base + i] = (float)(P.fill_u[k][2] + sq * n3);
  }
}

// per run: lengths and control reset after a fill
__global__ void k_fill_finish(Prm P) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r == 0) { *P.ctl.step = 0; }
  if (r < P.n_slots) P.ctl.slot_done[r] = 0;
  if (r >= P.R) return;
  int32_t ic[3];
  const int k = fill_region(P, P.Nc - 1, ic);
  int64_t total = (int64_t)P.cell[P.Nc - 1] + (k < 0 ? 0 : P.fill_ppc[k]);
  if (total > P.cap) total = P.cap;
  P.ctl.n_store[r] = total;
  P.ctl.live[r] = total;
  P.ctl.psteps[r] = 0;
  P.ctl.parity[r] = 0;
  P.ctl.reorder[r] = 0;
  P.ctl.inserted[r] = 0;
  for (int q = 0; q < 4; q++) P.ctl.counters[r * 4 + q] = 0;
}

// ============================================================== Generation
// one inflow particle (reading R8): ghost buffer (drifting Maxwellian, flies
// dt from behind the face) or effusion (Rayleigh normal speed, flies u dt)
__device__ __forceinline__ bool gen_particle(const Prm& P, uint2 key, int f, uint32_t s, uint32_t k, float pos[3],
                                             float vel[3]) {
  const uint4 a = draw(key, (uint32_t)f, s, TAG_INFLOW_PARTICLE, k, 0);
  const uint4 b = draw(key, (uint32_t)f, s, TAG_INFLOW_PARTICLE, k, 1);
  double n1, n2, n3, n4;
  box_muller(b.x, b.y, n1, n2);
  box_muller(b.z, b.w, n3, n4);
  const double sq = P.sqrt_inflowT;
  float x0[3], tau;
  x0[1] = place(P.face_j[f], a.y);
  x0[2] = place(P.face_k[f], a.z);
  if (P.inflow_kind == 1) {
    x0[0] = -(P.ghost_w_f * (float)u_oc_d(a.x));
    vel[0] = (float)(P.inflow_U + sq * n1);
    vel[1] = (float)(0.0 + sq * n2);
    vel[2] = (float)(0.0 + sq * n3);
    tau = P.dt_f;
  } else {
    x0[0] = 0.0f;
    vel[0] = (float)(sq * sqrt(-2.0 * log(u_oc_d(a.w))));
    vel[1] = (float)(0.0 + sq * n1);
    vel[2] = (float)(0.0 + sq * n2);
    tau = u_co(a.x) * P.dt_f;
  }
  bool kept = true;
#pragma unroll
  for (int d = 0; d < 3; d++) {
    pos[d] = d < P.dim ? fmaf(vel[d], tau, x0[d]) : 0.0f;
    if (d < P.dim && !(pos[d] >= 0.0f && pos[d] <= (float)axis_n(P, d))) kept = false;
  }
  return kept;
}

__device__ __forceinline__ int64_t inflow_n(const Prm& P, uint2 key, int f, uint32_t s) {
  if (P.inflow_kind == 2) return P.inflow_count;
  const uint4 w = draw(key, (uint32_t)f, s, TAG_INFLOW_COUNT, 0, 0);
  return (int64_t)floor(P.ghost_x + u_co_d(w.x));
}

// warp per (run, face cell): number of kept particles
__global__ void k_inflow_count(Prm P) {
  const int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int r = blockIdx.y, lane = threadIdx.x & 31;
  if (f >= P.n_face) return;
  const uint2 key = run_key(P, r);
  const uint32_t s = *P.ctl.step;
  const int64_t cnt = inflow_n(P, key, f, s);
  int kept = 0;
  for (int64_t k0 = 0; k0 < cnt; k0 += 32) {
    bool kp = false;
    if (k0 + lane < cnt) {
      float pos[3], vel[3];
      kp = gen_particle(P, key, f, s, (uint32_t)(k0 + lane), pos, vel);
    }
    kept += __popc(__ballot_sync(FULL, kp));
  }
  if (lane == 0) P.face_kept[(int64_t)r * P.n_face + f] = kept;
}

// warp per (run, face cell): append in (face, k) order at the run's tail
__global__ void k_inflow_emit(Prm P) {
  const int f = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int r = blockIdx.y, lane = threadIdx.x & 31;
  if (f >= P.n_face) return;
  const int32_t* kept_r = P.face_kept + (int64_t)r * P.n_face;
  uint32_t pre = 0;
  for (int q = lane; q < f; q += 32) pre += kept_r[q];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(FULL, pre, o);
  const uint2 key = run_key(P, r);
  const uint32_t s = *P.ctl.step;
  const int64_t n0 = P.ctl.n_store[r];
  const int h = P.ctl.parity[r];
  const int64_t base = (int64_t)r * P.stride;
  const int64_t cnt = inflow_n(P, key, f, s);
  int64_t pos_out = n0 + pre;
  for (int64_t k0 = 0; k0 < cnt; k0 += 32) {
    float pos[3], vel[3];
    bool kp = false;
    if (k0 + lane < cnt) kp = gen_particle(P, key, f, s, (uint32_t)(k0 + lane), pos, vel);
    const unsigned bal = __ballot_sync(FULL, kp);
    if (kp) {
      const int64_t i = pos_out + __popc(bal & ((1u << lane) - 1u));
      if (i < P.cap) {
        for (int a = 0; a < 3; a++) {
          parr(P, h, a)[base + i] = pos[a];
          parr(P, h, 3 + a)[base + i] = vel[a];
        }
        int32_t ic[3] = {0, 0, 0};
        for (int a = 0; a < P.dim; a++) {
          int32_t c = (int32_t)floorf(pos[a]);
          const int32_t L = axis_n(P, a);
          ic[a] = c > L - 1 ? L - 1 : c;
        }
        const uint32_t kk = (uint32_t)r * (uint32_t)P.Nc + (uint32_t)(ic[0] + P.nx * (ic[1] + P.ny * ic[2]));
        P.key[base + i] = kk;
        atomicAdd(&P.cell[kk], 1u);
      } else {
        latch(P, ST_CAP);
      }
    }
    pos_out += __popc(bal);
  }
  if (f == P.n_face - 1 && lane == 0) {
    int64_t total = pos_out - n0;
    if (n0 + total > P.cap) total = P.cap - n0;
    P.ctl.inserted[r] = (int32_t)total;
    P.ctl.counters[r * 4 + 0] += (unsigned long long)total;
  }
}

// ================================================================= Motion
// Full-accommodation diffuse re-emission (reading R10): Rayleigh normal speed
// into the domain, N(0, T) tangential components, in fp64 then rounded.
#ifndef DSMC_DIFFUSE_NOINLINE
#define DSMC_DIFFUSE_NOINLINE 0
#endif
#ifndef DSMC_MOTION_EV_MINB
// __launch_bounds__ min blocks/SM of k_motion: 4 caps it at 64 registers (without the cap the
// event-surface variants took 116; a min of 1 gave the plain c4 variant 80 registers, 4.40 -> 5.02 ms)
// (c5 after 300 steps: motion 0.75 -> 0.56 ms; c3: 2.01 -> 1.86 ms/step; 3 blocks: 0.62 ms)
#define DSMC_MOTION_EV_MINB 4
#endif
#if DSMC_DIFFUSE_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
void diffuse(uint2 key, uint32_t idx, uint32_t s, uint32_t b, int a, int sign, double sq,
                                        float v[3]) {
  const uint4 w = draw(key, idx, s, TAG_WALL, b, 0);
  const double vn = sq * sqrt(-2.0 * log(u_oc_d(w.x)));
  double t1, t2;
  box_muller(w.y, w.z, t1, t2);
  // normal component on axis a, the tangential ones in axis order (selects: a runtime
  // index into v[] would put the particle's registers in local memory)
  const float fn = (float)(sign > 0 ? vn : -vn), f1 = (float)(0.0 + sq * t1), f2 = (float)(0.0 + sq * t2);
  v[0] = a == 0 ? fn : f1;
  v[1] = a == 1 ? fn : (a == 0 ? f1 : f2);
  v[2] = a == 2 ? fn : f2;
}

// component a (runtime) of a 3-vector, and its assignment, without dynamic indexing
__device__ __forceinline__ float comp(const float x[3], int a) { return a == 0 ? x[0] : (a == 1 ? x[1] : x[2]); }
__device__ __forceinline__ void set_comp(float x[3], int a, float val) {
  x[0] = a == 0 ? val : x[0];
  x[1] = a == 1 ? val : x[1];
  x[2] = a == 2 ? val : x[2];
}

// Motion with surface interaction (reading R10).  Returns
// true if the particle left the domain.  EV = the problem has event surfaces
// (diffuse / outflow / inflow faces or the plate).
template <int D, bool EV>
__device__ __forceinline__ bool move_one(const Prm& P, uint2 key, uint32_t idx, uint32_t s, float x[3], float v[3],
                                         bool& vchg, bool& inside) {
  float tau = P.dt_f;
  {
    // the straight flight ends in [0, L) on every axis (in 2D also on its side of the
    // plate), velocity finite: no event, no wrap and no index fault -- the position the
    // event loop and the wrap below would compute, decided in ~4 instructions per axis
    // (c5: most particles; the full path's surface and boundary tests were ~40% of
    // k_motion's instructions)
    float x1[3] = {x[0], x[1], x[2]};
    bool in = true;
#pragma unroll
    for (int a = 0; a < D; a++) {
      x1[a] = fmaf(v[a], tau, x[a]);
      in = in && x1[a] >= 0.0f && x1[a] < (float)axis_n(P, a);
    }
#pragma unroll
    for (int a = D; a < 3; a++) in = in && isfinite(v[a]);
    if (EV && D == 2 && P.plate_on)
      in = in && ((comp(x, P.plate_axis) >= P.plate_pos) == (comp(x1, P.plate_axis) >= P.plate_pos));
    if (in) {
#pragma unroll
      for (int a = 0; a < D; a++) x[a] = x1[a];
      inside = true;
      return false;
    }
  }
  if (EV) {
    for (int b = 0;; b++) {
      float x1[3] = {x[0], x[1], x[2]};
#pragma unroll
      for (int a = 0; a < D; a++) x1[a] = fmaf(v[a], tau, x[a]);
      int ev = -1;
      float tbest = __int_as_float(0x7f800000);
#pragma unroll
      for (int a = 0; a < D; a++) {
#pragma unroll
        for (int f = 0; f < 2; f++) {
          const int bc = P.bc[2 * a + f];
          if (bc == BC_SPECULAR || bc == BC_PERIODIC) continue;
          const float L = f ? (float)axis_n(P, a) : 0.0f;
          const bool crossed = f ? (x1[a] > L) : (x1[a] < L);
          if (crossed) {
            const float t = (L - x[a]) / v[a];
            if (t < tbest) { tbest = t; ev = 2 * a + f; }
          }
        }
      }
      bool s0 = false;
      if (D == 2 && P.plate_on) {
        const int pa = P.plate_axis, qa = P.plate_span_axis;
        const float pc = P.plate_pos;
        s0 = comp(x, pa) >= pc;
        const bool s1 = comp(x1, pa) >= pc;
        if (s0 != s1) {
          const float t = (pc - comp(x, pa)) / comp(v, pa);
          const float xq = fmaf(comp(v, qa), t, comp(x, qa));
          if (xq >= P.plate_lo && xq <= P.plate_hi && t < tbest) { tbest = t; ev = 6; }
        }
      }
      if (ev < 0) {
#pragma unroll
        for (int a = 0; a < D; a++) x[a] = x1[a];
        break;
      }
      const float t = tbest < tau ? tbest : tau;
      if (ev < 6) {
        const int a = ev >> 1, f = ev & 1, bc = P.bc[ev];
        if (bc == BC_OUTFLOW || bc == BC_INFLOW) return true;
#pragma unroll
        for (int c = 0; c < D; c++) if (c != a) x[c] = fmaf(v[c], t, x[c]);
        set_comp(x, a, f ? (float)axis_n(P, a) : 0.0f);
        if (D == 3 && P.orifice_on && a == 0 && f == 0) {
          int32_t j = (int32_t)floorf(x[1]), k = (int32_t)floorf(x[2]);
          j = j < 0 ? 0 : (j > P.ny - 1 ? P.ny - 1 : j);
          k = k < 0 ? 0 : (k > P.nz - 1 ? P.nz - 1 : k);
          if (P.open_face[(int64_t)k * P.ny + j]) return true;
        }
        if (b == MAX_BOUNCE) { latch(P, ST_BOUNCE); break; }
        diffuse(key, idx, s, (uint32_t)b, a, f ? -1 : 1, P.sqrt_bcT[ev], v);
      } else {
        const int pa = P.plate_axis;
        const float pc = P.plate_pos;
#pragma unroll
        for (int c = 0; c < D; c++) if (c != pa) x[c] = fmaf(v[c], t, x[c]);
        set_comp(x, pa, s0 ? pc : nextafterf(pc, -__int_as_float(0x7f800000)));
        if (b == MAX_BOUNCE) { latch(P, ST_BOUNCE); break; }
        diffuse(key, idx, s, (uint32_t)b, pa, s0 ? 1 : -1, P.sqrt_plateT, v);
      }
      vchg = true;
      tau = tau - t;
    }
  } else {
#pragma unroll
    for (int a = 0; a < D; a++) x[a] = fmaf(v[a], tau, x[a]);
  }
#pragma unroll
  for (int a = 0; a < D; a++) {
    const float L = (float)axis_n(P, a);
    if (P.bc[2 * a] == BC_PERIODIC) {
      if (x[a] >= L) x[a] = x[a] - L;
      else if (x[a] < 0.0f) { x[a] = x[a] + L; if (x[a] >= L) x[a] = 0.0f; }
    } else {
      if (x[a] < 0.0f && P.bc[2 * a] == BC_SPECULAR) { x[a] = -x[a]; v[a] = -v[a]; vchg = true; }
      else if (x[a] > L && P.bc[2 * a + 1] == BC_SPECULAR) { x[a] = 2.0f * L - x[a]; v[a] = -v[a]; vchg = true; }
    }
  }
  return false;
}

// Dynamic work queue for the persistent particle kernels: blocks take items
// (ITEM_M / ITEM_S consecutive particles of one run, run-major) from a global cursor, so
// the items in flight stay within a window of ~one run and the cell counters
// / LCR segments they hit stay resident in L2.  The last block to finish
// resets the cursor for the next launch.
constexpr int ITEM_M = 8192;   // Motion's work item (measured at c4: 4096 / 8192 / 16384: 4.50 / 4.38 / 4.40 ms)
constexpr int ITEM_S = 4096;   // the scatter's (2048 / 4096 / 8192: 2.42 / 2.32 / 2.40 ms)
__device__ __forceinline__ int64_t queue_next(unsigned long long* q, int64_t* s_item) {
  __syncthreads();
  if (threadIdx.x == 0) *s_item = (int64_t)atomicAdd(q, 1ull);
  __syncthreads();
  return *s_item;
}
__device__ __forceinline__ void queue_done(unsigned long long* q) {
  if (threadIdx.x == 0 && atomicAdd(q + 1, 1ull) == gridDim.x - 1) { q[0] = 0; q[1] = 0; }
}

// work items of the persistent particle kernels: items[r] = sum over runs r' < r
// of ceil(n_store[r'] / ITEM), items[R] = total -- only the occupied part of each
// run's window is walked (open systems sized for growth leave most of it empty)
template <int ITEM>
__global__ void __launch_bounds__(1024) k_items(Prm P) {
  __shared__ uint32_t s_warp[32];
  __shared__ int64_t s_carry;
  __shared__ int s_uniform;
  if (threadIdx.x == 0) { s_carry = 0; s_uniform = 1; }
  __syncthreads();
  const uint32_t v0 = (uint32_t)((P.ctl.n_store[0] + ITEM - 1) / ITEM);
  for (int r0 = 0; r0 < P.R; r0 += 1024) {
    const int r = r0 + (int)threadIdx.x;
    const uint32_t v = r < P.R ? (uint32_t)((P.ctl.n_store[r] + ITEM - 1) / ITEM) : 0u;
    if (r < P.R && v != v0) s_uniform = 0;
    uint32_t total;
    const uint32_t pre = block_excl_scan(v, s_warp, total);
    if (r < P.R) P.ctl.items[r] = s_carry + (int64_t)pre;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += (int64_t)total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    P.ctl.items[P.R] = s_carry;
    P.ctl.items[P.R + 1] = s_uniform ? (int64_t)v0 : 0;   // items per run when all runs hold as many
  }
}

// run of work item `item`: the last r with items[r] <= item (empty runs share
// their successor's start, so the last one is the occupied run)
__device__ __forceinline__ int item_run(const Prm& P, int64_t item) {
  const int64_t per = P.ctl.items[P.R + 1];
  if (per > 0) return (int)(item / per);                         // every run holds as many items (closed box)
  int lo = 0, hi = P.R;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (P.ctl.items[mid] <= item) lo = mid; else hi = mid;
  }
  return lo;
}

// Enumeration (reading R11): floor per axis, clamped.
template <int D>
__device__ __forceinline__ uint32_t enumerate(const Prm& P, const float x[3], const float v[3], uint32_t kbase) {
  int32_t ic[3] = {0, 0, 0};
  // a non-finite velocity is reported as such (it also makes the position non-finite)
  if (!(isfinite(v[0]) && isfinite(v[1]) && isfinite(v[2]))) latch(P, ST_NONFINITE);
#pragma unroll
  for (int a = 0; a < D; a++) {
    const int32_t L = axis_n(P, a);
    if (!(x[a] >= 0.0f && x[a] <= (float)L)) latch(P, ST_INDEX);
    int32_t c = x[a] >= 0.0f ? (int32_t)floorf(x[a]) : 0;
    ic[a] = c > L - 1 ? L - 1 : c;
  }
  return kbase + (uint32_t)(ic[0] + P.nx * (ic[1] + P.ny * ic[2]));
}

// the same for a position move_one found in [0, L) on every axis with a finite
// velocity: nothing to report, floor = truncation, no clamp needed
template <int D>
__device__ __forceinline__ uint32_t enumerate_in(const Prm& P, const float x[3], uint32_t kbase) {
  int32_t ic[3] = {0, 0, 0};
#pragma unroll
  for (int a = 0; a < D; a++) ic[a] = (int32_t)x[a];
  return kbase + (uint32_t)(ic[0] + P.nx * (ic[1] + P.ny * ic[2]));
}

// persistent over (run = blockIdx.y, warp chunks of 128 particles; lane owns
// particles chunk + 32 j + lane, j < 4, so that the 32 keys of one warp
// instruction are consecutive store slots -- after a reorder they share few
// cells and the warp-aggregated histogram needs few atomics).
// mode 0: move + enumerate, mode 1: enumerate only (explicit Sampling)
template <int D, bool EV>
__global__ void __launch_bounds__(256, EV ? DSMC_MOTION_EV_MINB : 0) k_motion(Prm P, int mode) {
  const int lane = threadIdx.x & 31;
  const uint32_t s = (uint32_t)*P.ctl.step;
  const int64_t n_items = P.ctl.items[P.R];
  __shared__ int64_t s_item;
  for (int64_t item = queue_next(P.ctl.queue, &s_item); item < n_items; item = queue_next(P.ctl.queue, &s_item)) {
  const int r = item_run(P, item);
  const int64_t n = P.ctl.n_store[r];
  const int64_t ibase = (item - P.ctl.items[r]) * ITEM_M;
  const int h = P.ctl.parity[r];
  const int64_t base = (int64_t)r * P.stride;
  float* X[3];
  float* V[3];
#pragma unroll
  for (int a = 0; a < 3; a++) { X[a] = parr(P, h, a) + base; V[a] = parr(P, h, 3 + a) + base; }
  uint32_t* K = P.key + base;
  const uint2 key = run_key(P, r);
  const uint32_t kbase = (uint32_t)r * (uint32_t)P.Nc;
  uint32_t removed = 0;
  for (int64_t i0w = ibase + (threadIdx.x >> 5) * 128; i0w < ibase + ITEM_M && i0w < n; i0w += 1024) {
    float x[4][3], v[4][3];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int64_t i = i0w + j * 32 + lane;
      const bool in = i < n;
#pragma unroll
      for (int a = 0; a < D; a++) x[j][a] = in ? X[a][i] : DEAD_X;
#pragma unroll
      for (int a = D; a < 3; a++) x[j][a] = 0.0f;
#pragma unroll
      for (int a = 0; a < 3; a++) v[j][a] = in ? V[a][i] : 0.0f;
    }
    uint32_t kk[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int64_t i = i0w + j * 32 + lane;
      bool vchg = false, inside = false;
      if (x[j][0] < -1.0e29f) {
        kk[j] = DEAD_KEY;
      } else {
        bool dead = false;
        if (mode == 0) {
          dead = move_one<D, EV>(P, key, (uint32_t)i, s, x[j], v[j], vchg, inside);
          if (dead) { x[j][0] = DEAD_X; removed++; }
        }
        kk[j] = dead ? DEAD_KEY : (inside ? enumerate_in<D>(P, x[j], kbase) : enumerate<D>(P, x[j], v[j], kbase));
        if (mode == 0) {
          X[0][i] = x[j][0];
          if (!dead) {
#pragma unroll
            for (int a = 1; a < D; a++) X[a][i] = x[j][a];
            if (vchg) {
#pragma unroll
              for (int a = 0; a < 3; a++) V[a][i] = v[j][a];
            }
          }
        }
      }
      if (i < n) K[i] = kk[j];
    }
    // warp-aggregated histogram of cell keys
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const unsigned m = __match_any_sync(FULL, kk[j]);
      if (kk[j] != DEAD_KEY && lane == __ffs(m) - 1) atomicAdd(&P.cell[kk[j]], (uint32_t)__popc(m));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) removed += __shfl_xor_sync(FULL, removed, o);
  if (lane == 0 && removed) atomicAdd(&P.ctl.counters[r * 4 + 1], (unsigned long long)removed);
  }
  queue_done(P.ctl.queue);
}

// ================================================================ control
__global__ void k_step_mid(Prm P) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= P.R) return;
  const int32_t s = *P.ctl.step;
  const int64_t n = P.ctl.n_store[r] + P.ctl.inserted[r];
  P.ctl.n_store[r] = n;
  P.ctl.psteps[r] += (unsigned long long)(P.ctl.live[r] + P.ctl.inserted[r]);
  P.ctl.inserted[r] = 0;
  P.ctl.maxn[r] = 0u;          // k_collide takes the maximum over the step's cells
  const int K = P.reorder_every;
  P.ctl.reorder[r] = ((K > 0 && (s + 1) % K == 0) || (P.cap - n < P.insert_bound)) ? 1 : 0;
  if (r == 0)   // Sampling of this step (R2: after step s when (s+1) is a multiple of the interval), or -1
    *P.ctl.step_slot = ((s + 1) % P.sample_every == 0 && (s + 1) / P.sample_every - 1 < P.n_slots)
                           ? (s + 1) / P.sample_every - 1 : -1;
}

__device__ __forceinline__ uint32_t run_lcr_base(const Prm& P, int r) {
  return r == 0 ? 0u : P.cell[(int64_t)r * P.Nc - 1];
}

__global__ void k_step_end(Prm P, int mode, int slot) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < 2 * HEAVY_TIERS) P.ctl.heavy[r] = 0;   // heavy-tile queues of k_collide
  if (r == 0) P.ctl.tiles[0] = 0;                // k_collide_triage's tile list
  if (mode != 0) {  // explicit sample (1: snapshot, 2: added to the slot's time average)
    if (r == 0) P.ctl.slot_done[slot] = mode == 1 ? 1 : P.ctl.slot_done[slot] + 1;
    return;
  }
  const int32_t s = *P.ctl.step;
  if (r < P.R) {
    const uint32_t b = run_lcr_base(P, r);
    const uint32_t e = P.cell[(int64_t)(r + 1) * P.Nc - 1];
    P.ctl.live[r] = (int64_t)(e - b);
    if (P.ctl.reorder[r]) {
      P.ctl.n_store[r] = (int64_t)(e - b);
      P.ctl.parity[r] ^= 1;
    }
  }
  if (r == 0) {
    if ((s + 1) % P.sample_every == 0) {
      const int sl = (s + 1) / P.sample_every - 1;
      if (sl < P.n_slots) P.ctl.slot_done[sl] = 1;
    }
    *P.ctl.step = s + 1;
  }
}

// ================================================================ Indexing
// LCR[start[key] + rank] = global store index; warp-aggregated cursors over
// lane-contiguous particles (same chunking as k_motion); the four atomics of
// a chunk are issued before any result is consumed.
#ifdef DSMC_SCATTER_LDCS          // A/B: the keys (read once) by streaming loads
#define DSMC_LDK(p) __ldcs(p)
#else
#define DSMC_LDK(p) (*(p))
#endif
__global__ void __launch_bounds__(256) k_scatter(Prm P) {
  const int lane = threadIdx.x & 31;
  constexpr int SL = 2;      // 32-particle slices per warp iteration (returning atomics in flight)
  const unsigned lt = (1u << lane) - 1u;
  const int64_t n_items = P.ctl.items[P.R];
  __shared__ int64_t s_item;
  for (int64_t item = queue_next(P.ctl.queue + 2, &s_item); item < n_items;
       item = queue_next(P.ctl.queue + 2, &s_item)) {
    const int r = item_run(P, item);
    const int64_t n = P.ctl.n_store[r];
    const int64_t ibase = (item - P.ctl.items[r]) * ITEM_S;
    const int64_t base = (int64_t)r * P.stride;
    const uint32_t* K = P.key + base;
    // the next slice's keys are loaded before this slice's returning atomics, so
    // the HBM latency of one overlaps the L2 atomic latency of the other
    const int64_t iend = ibase + ITEM_S < n ? ibase + ITEM_S : n;
    uint32_t kn[SL];
    int64_t i0w = ibase + (threadIdx.x >> 5) * (32 * SL);
#pragma unroll
    for (int j = 0; j < SL; j++) {
      const int64_t i = i0w + j * 32 + lane;
      kn[j] = i < iend ? DSMC_LDK(K + i) : DEAD_KEY;
    }
    for (; i0w < iend; i0w += 256 * SL) {
    uint32_t kk[SL], m[SL], p0[SL];
#pragma unroll
    for (int j = 0; j < SL; j++) kk[j] = kn[j];
    if (i0w + 256 * SL < iend) {
#pragma unroll
      for (int j = 0; j < SL; j++) {
        const int64_t i = i0w + 256 * SL + j * 32 + lane;
        kn[j] = i < iend ? DSMC_LDK(K + i) : DEAD_KEY;
      }
    }
#pragma unroll
    for (int j = 0; j < SL; j++) m[j] = __match_any_sync(FULL, kk[j]);
#pragma unroll
    for (int j = 0; j < SL; j++) {
      p0[j] = 0;
      if (kk[j] != DEAD_KEY && lane == __ffs(m[j]) - 1) p0[j] = atomicAdd(&P.cell[kk[j]], (uint32_t)__popc(m[j]));
    }
#pragma unroll
    for (int j = 0; j < SL; j++) {
      const uint32_t b = __shfl_sync(FULL, p0[j], __ffs(m[j]) - 1);
      if (kk[j] != DEAD_KEY) P.lcr[b + __popc(m[j] & lt)] = (uint32_t)(base + i0w + j * 32 + lane);
    }
    }
  }
  queue_done(P.ctl.queue + 2);
}

// ============================================================= Interaction
// Isotropic direction, Marsaglia (reading R14): the first try from words z, w
// of the candidate's pair block, further tries two per COLL_DIR block
__device__ __forceinline__ void marsaglia(uint2 key, uint32_t c, uint32_t s, uint32_t k, uint4 wpair, float e[3]) {
  uint4 w = wpair;
  int h0 = 1;
#pragma unroll 1
  for (int32_t blk = -1; blk < 64; blk++) {
    if (blk >= 0) { w = draw(key, c, s, TAG_COLL_DIR, k, (uint32_t)blk); h0 = 0; }
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
    for (int h = h0; h < 2; h++) {
      const float pp = 2.0f * u_co(ww[2 * h]) - 1.0f;
      const float qq = 2.0f * u_co(ww[2 * h + 1]) - 1.0f;
      const float rho = pp * pp + qq * qq;
      if (rho < 1.0f) {
        const float sr = sqrtf(1.0f - rho);
        e[0] = 2.0f * pp * sr;
        e[1] = 2.0f * qq * sr;
        e[2] = 1.0f - 2.0f * rho;
        return;
      }
    }
  }
  e[0] = 0.0f; e[1] = 0.0f; e[2] = 1.0f;
}

// the candidate pair of R13 from the first word of its pair block:
// m = w N, i = m >> 32, j = lemire(m mod 2^32, N - 1), j += (j >= i)
__device__ __forceinline__ void pair_of(uint32_t w, uint32_t N, uint32_t& i, uint32_t& j) {
  const uint64_t m = (uint64_t)w * N;
  i = (uint32_t)(m >> 32);
  j = lemire((uint32_t)m, N - 1);
  if (j >= i) j++;
}

// velocity accessors: shared-memory tile, or global memory through LCR
// build-time A/B switches (tools/build_variant.sh passes -D): all give bit-identical results
// k_collide's F writes every velocity of the tile back (no collided flags to set,
// clear and scan).  About 20% of the particles collide per step at c4, so ~83% of
// the 32-byte sectors of the velocity arrays are written either way: the full
// write-back adds ~20% DRAM writes and saves the flag work (c4 n=256: k_collide
// 12.35 -> 12.15 ms).
#ifndef DSMC_COLLIDE_MINB
// __launch_bounds__ min blocks per SM of k_collide (1 warp per block): 16 caps it at
// 128 registers, the most that keeps 16 warps per SM (130 registers: 15 warps, +3%)
#define DSMC_COLLIDE_MINB 16
#endif
#ifndef DSMC_NET_MAX
#define DSMC_NET_MAX 32      // widest register network chosen by the warp's largest segment
#endif
#ifndef DSMC_CCW
#define DSMC_CCW 128        // pre-drawn candidates per pass of k_collide's E1
#endif
#ifndef DSMC_LANE_UNROLL_N
#define DSMC_LANE_UNROLL_N 1   // unroll of k_collide's lane-strided gather / write-back loops (A/B; see below)
#endif
#define DSMC_PRAGMA(x) _Pragma(#x)
#define DSMC_PRAGMA_UNROLL(n) DSMC_PRAGMA(unroll n)
#ifdef DSMC_LANE_UNROLL_NONE
#define DSMC_LANE_UNROLL
#else
#define DSMC_LANE_UNROLL DSMC_PRAGMA_UNROLL(DSMC_LANE_UNROLL_N)
#endif
// Loop unrolling in k_collide, measured at c4 n = 256 (k_collide ms): the compiler's own
// unrolling of the lane-strided gather / write-back loops 11.46, kept rolled 10.10 (2x:
// 10.35, 4x: 10.62) -- the unrolled copies cost more in code size and registers than the
// loop overhead they save; the candidate walk rolled as well 10.02 (compiler: 10.10, 4x:
// 10.73); the other runtime-trip loops (E1 passes, Sampling, rank sort) rolled: 10.06-10.07,
// left to the compiler: 10.02.
#ifdef DSMC_LOOP_UNROLL_ONE         // A/B: the other runtime-trip loops rolled
#define DSMC_LOOP_UNROLL DSMC_PRAGMA_UNROLL(1)
#else
#define DSMC_LOOP_UNROLL
#endif
#ifndef DSMC_OWNMAP
#define DSMC_OWNMAP 1          // E1 finds a candidate's cell in a byte map instead of a search (A/B)
#endif
#ifndef DSMC_WALK_UNROLL_N
#define DSMC_WALK_UNROLL_N 1   // 0: the compiler's choice
#endif
#ifndef DSMC_CCARITH
#define DSMC_CCARITH 1         // E1 takes a one-run tile's owner cell as c(lane 0) + owner, not by a shuffle
#endif                         // (c4 k_collide 9.82 -> 9.78-9.79 ms; 0: the shuffle, A/B)
// k_collide's staged cell: velocities as 3 floats per particle (12-byte stride: lane-strided
// LDS.32 are conflict-free).  float4 (one LDS.128 per particle) costs 4 more bytes per staged
// particle, and the kernel's speed follows the L1 its shared memory leaves: at c4 the 16 one-warp
// blocks of an SM then need 190 KB (196 KB carveout, 60 KB of L1) against 160 KB (164 KB carveout,
// 92 KB of L1): k_collide 9.80 -> 8.93 ms at n = 256 (float3 under a forced 196 KB carveout: 9.62)
constexpr int VS = 3;       // floats per staged velocity
// k_collide reads its cell data (ends, majorant) once and writes velocities and positions it
// never reads again: streaming loads / stores (evict-first) keep them from displacing the
// sectors the gathers share in L1 and L2 (c4 n = 256: k_collide 8.94 -> 8.79 ms; loads alone
// 8.93, stores alone 8.82)
#define DSMC_LD1(p) __ldcs(p)
#define DSMC_ST1(p, v) __stcs(p, v)
struct SmemCellV {
  float* v;
  __device__ void ld(uint32_t i, float a[3]) const { a[0] = v[3 * i]; a[1] = v[3 * i + 1]; a[2] = v[3 * i + 2]; }
  __device__ void st(uint32_t i, const float a[3]) const { v[3 * i] = a[0]; v[3 * i + 1] = a[1]; v[3 * i + 2] = a[2]; }
};
struct SmemCell {
  float* vx; float* vy; float* vz; uint8_t* mod;
  __device__ void ld(uint32_t i, float a[3]) const { a[0] = vx[i]; a[1] = vy[i]; a[2] = vz[i]; }
  __device__ void st(uint32_t i, const float a[3]) const { vx[i] = a[0]; vy[i] = a[1]; vz[i] = a[2]; mod[i] = 1; }
};
struct GlobCell {
  const uint32_t* idx; float* vx; float* vy; float* vz;
  __device__ void ld(uint32_t i, float a[3]) const { const uint32_t g = idx[i]; a[0] = vx[g]; a[1] = vy[g]; a[2] = vz[g]; }
  __device__ void st(uint32_t i, const float a[3]) const { const uint32_t g = idx[i]; vx[g] = a[0]; vy[g] = a[1]; vz[g] = a[2]; }
};

// VHS acceptance of R13, u (sigma g)_max < sigma_c (g^2)^(1-omega), decided
// exactly but mostly without the fp64 pow: the two sides are first compared
// as fp32 base-2 logarithms (MUFU.LG2, absolute error < 2^-21 over the range
// used, plus the float roundings of both arguments, all far below 2^-10), and
// only a decision within 2^-10 of the threshold -- about one candidate in a
// thousand -- evaluates the fp64 expression itself.
__device__ __forceinline__ bool vhs_accept(const Prm& P, uint32_t uword, double gm, float g2) {
  const double lhs = u_co_d(uword) * gm;
  const float l_lhs = __log2f((float)lhs);
  const float l_rhs = __log2f((float)P.sigma_c) + (float)P.omega1 * __log2f(g2);
  if (l_lhs < l_rhs - 0.0009765625f) return true;      // lhs < rhs by more than a factor 2^(1/1024)
  if (l_lhs > l_rhs + 0.0009765625f) return false;
  return lhs < P.sigma_c * pow((double)g2, P.omega1);   // near the threshold (and 0, inf cases): exact
}

// NTC in one cell (readings R12-R15): M = floor(1/2 N(N-1) coef gmax + u);
// candidate k: i = lemire(a, N), j = lemire(b, N-1) (+1 if >= i); accept iff
// u (sigma g)_max < sigma g in fp64; g_max frozen during the step.
template <class A>
__device__ __forceinline__ void collide_cell(const Prm& P, uint2 key, uint32_t c, uint32_t s, uint32_t N, const A& acc,
                                             float& gmax, uint32_t& ncand, uint32_t& nacc) {
  ncand = 0;
  nacc = 0;
  if (N < 2) return;
  const double gm = (double)gmax;
  const double ghat = gm / P.sigma_c;
  const double x = ((double)((int64_t)N * (int64_t)(N - 1)) * 0.5) * P.coef * gm;
  uint4 w = draw(key, c, s, TAG_COLL_COUNT, 0, 0);
  int64_t M = (int64_t)floor(x + u_co_d(w.x));
  if (M > 0xFFFFFF) { latch(P, ST_CELL); M = 0xFFFFFF; }
  float maxg2 = 0.0f;
  for (uint32_t k = 0; k < (uint32_t)M; k++) {
    w = draw(key, c, s, TAG_COLL_PAIR, k, 0);
    uint32_t i, j;
    pair_of(w.x, N, i, j);
    float a[3], b[3];
    acc.ld(i, a);
    acc.ld(j, b);
    const float dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
    const float g2 = (dx * dx + dy * dy) + dz * dz;
    if (g2 > maxg2) maxg2 = g2;
    bool accept;
    if (P.model == 0) {
      const double lhs = u_co_d(w.y) * ghat;
      accept = lhs * lhs < (double)g2;
    } else {
      accept = vhs_accept(P, w.y, gm, g2);
    }
    if (accept) {
      float e[3];
      marsaglia(key, c, s, k, w, e);
      const float cmx = (a[0] + b[0]) * 0.5f, cmy = (a[1] + b[1]) * 0.5f, cmz = (a[2] + b[2]) * 0.5f;
      const float hh = 0.5f * sqrtf(g2);
      const float pa[3] = {cmx + hh * e[0], cmy + hh * e[1], cmz + hh * e[2]};
      const float pb[3] = {cmx - hh * e[0], cmy - hh * e[1], cmz - hh * e[2]};
      acc.st(i, pa);
      acc.st(j, pb);
      nacc++;
    }
  }
  ncand = (uint32_t)M;
  if (M > 0) {
    const double sgm = P.model == 0 ? P.sigma_c * sqrt((double)maxg2) : P.sigma_c * pow((double)maxg2, P.omega1);
    if (sgm > gm) gmax = (float)sgm;
  }
}

// NTC, split for lane efficiency inside k_collide's shared-memory path:
// ntc_count() draws M for a cell; the pair draws of all candidates of the tile
// are then computed lane-parallel (E1) and ntc_apply_pre() walks one cell's
// candidates in increasing k (E2), exactly the order of collide_cell().
__device__ __forceinline__ uint32_t ntc_count(const Prm& P, uint2 key, uint32_t c, uint32_t s, uint32_t N, float gmax) {
  if (N < 2) return 0;
  const double x = ((double)((int64_t)N * (int64_t)(N - 1)) * 0.5) * P.coef * (double)gmax;
  const uint4 w = draw(key, c, s, TAG_COLL_COUNT, 0, 0);
  int64_t M = (int64_t)floor(x + u_co_d(w.x));
  if (M > 0xFFFFFF) { latch(P, ST_CELL); M = 0xFFFFFF; }
  return (uint32_t)M;
}

// Marsaglia pair from direction block b0 on (the first try, from the pair block, is made inline)
__device__ __noinline__ void marsaglia_pq_from(uint2 key, uint32_t c, uint32_t s, uint32_t k, uint32_t b0,
                                               float& pp_out, float& qq_out) {
#pragma unroll 1   // cold (both tries of block 0 rejected): keep the code small
  for (uint32_t blk = b0; blk < 64; blk++) {
    const uint4 w = draw(key, c, s, TAG_COLL_DIR, k, blk);
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const float pp = 2.0f * u_co(ww[2 * h]) - 1.0f;
      const float qq = 2.0f * u_co(ww[2 * h + 1]) - 1.0f;
      const float rho = pp * pp + qq * qq;
      if (rho < 1.0f) { pp_out = pp; qq_out = qq; return; }
    }
  }
  pp_out = 0.0f;   // never reached in practice; gives e = (0, 0, 1) like marsaglia()
  qq_out = 0.0f;
}

// candidates of one cell in increasing k with everything velocity-independent
// drawn ahead (k_collide): ij = i | j << 16; thr = HS threshold F (accept iff
// g2 > F) or the raw VHS acceptance word; (ex, ey, ez) the unit vector (R14)
// rec[k] = (ex, ey, ez, threshold bits): one LDS.128 per candidate
template <int MODEL, class A>
__device__ __forceinline__ void ntc_apply_pre(const Prm& P, const A& acc, double gm, const uint32_t* ij,
                                              const float4* rec, uint32_t n, float& maxg2, uint32_t& nacc) {
#if DSMC_WALK_UNROLL_N > 0
  DSMC_PRAGMA_UNROLL(DSMC_WALK_UNROLL_N)
#endif
  for (uint32_t k = 0; k < n; k++) {
    const uint32_t pr = ij[k];
    const uint32_t i = pr & 0xFFFFu, j = pr >> 16;
    float a[3], b[3];
    acc.ld(i, a);
    acc.ld(j, b);
    const float4 rc = rec[k];
    const float dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
    const float g2 = (dx * dx + dy * dy) + dz * dz;
    maxg2 = g2 > maxg2 ? g2 : maxg2;
    const bool accept = MODEL == DSMC_MODEL_HS ? g2 > rc.w
                                     : vhs_accept(P, __float_as_uint(rc.w), gm, g2);
    if (accept) {
      const float e[3] = {rc.x, rc.y, rc.z};
      const float cmx = (a[0] + b[0]) * 0.5f, cmy = (a[1] + b[1]) * 0.5f, cmz = (a[2] + b[2]) * 0.5f;
      const float hh = 0.5f * sqrtf(g2);
      const float pa[3] = {cmx + hh * e[0], cmy + hh * e[1], cmz + hh * e[2]};
      const float pb[3] = {cmx - hh * e[0], cmy - hh * e[1], cmz - hh * e[2]};
      acc.st(i, pa);
      acc.st(j, pb);
      nacc++;
    }
  }
}

// odd-even merge sorting network (Batcher) over the first NE <= NN entries,
// ascending; NN a power of two.  Comparators reaching past NE are dropped:
// with the tail padded by +inf they never swap (0-1 principle; exhaustively
// checked by tests/test_sortnet.py).
template <int NN, int NE>
__host__ __device__ __forceinline__ void sort_oem(uint32_t (&a)[NN]) {
  // stage (p, k) compares x with x + k for every x with (x - k%p) mod 2k < k
  // inside one 2p-block; every loop bound is a constant, so the network
  // unrolls completely and a[] stays in registers
#pragma unroll
  for (int p = 1; p < NN; p <<= 1) {
#pragma unroll
    for (int k = p; k >= 1; k >>= 1) {
#pragma unroll
      for (int x = 0; x < NN; x++) {
        const int j0 = k % p;
        if (x >= j0 && (x - j0) % (2 * k) < k && x + k < NE && x / (2 * p) == (x + k) / (2 * p)) {
          const uint32_t u = a[x], v = a[x + k];
          a[x] = u < v ? u : v;
          a[x + k] = u < v ? v : u;
        }
      }
    }
  }
}

// sort a segment of N <= NE from src into dst (shared memory), in registers
template <int NN, int NE>
__device__ __forceinline__ void sort_segment(const uint32_t* src, uint32_t* dst, uint32_t N) {
  uint32_t v[NN];
#pragma unroll
  for (int i = 0; i < NN; i++) v[i] = (i < NE && (uint32_t)i < N) ? src[i] : 0xFFFFFFFFu;
  sort_oem<NN, NE>(v);
#pragma unroll
  for (int i = 0; i < NE; i++) if ((uint32_t)i < N) dst[i] = v[i];
}

// Sampling of one cell into slot `slot` of array C (R17); add: accumulate
// (time averaging for steady problems) instead of overwrite
template <class A>
__device__ __forceinline__ void sample_cell(const Prm& P, int slot, int64_t k, uint32_t N, const A& acc,
                                            bool add = false) {
  double sx = 0.0, sy = 0.0, sz = 0.0, se = 0.0;
  DSMC_LOOP_UNROLL
  for (uint32_t i = 0; i < N; i++) {
    float a[3];
    acc.ld(i, a);
    const double vx = (double)a[0], vy = (double)a[1], vz = (double)a[2];
    sx += vx; sy += vy; sz += vz;
    se += (vx * vx + vy * vy) + vz * vz;
  }
  const int64_t RN = (int64_t)P.R * P.Nc;
  double* C = P.C + (int64_t)slot * 5 * RN + k;
  if (add) {
    C[0] += (double)N; C[RN] += sx; C[2 * RN] += sy; C[3 * RN] += sz; C[4 * RN] += se;
  } else {
    C[0] = (double)N; C[RN] = sx; C[2 * RN] = sy; C[3 * RN] = sz; C[4 * RN] = se;
  }
}

__device__ __forceinline__ void insertion_sort(uint32_t* a, uint32_t n) {
  for (uint32_t i = 1; i < n; i++) {
    const uint32_t t = a[i];
    uint32_t j = i;
    while (j > 0 && a[j - 1] > t) { a[j] = a[j - 1]; j--; }
    a[j] = t;
  }
}

__device__ void heap_sort(uint32_t* a, uint32_t n) {
  auto sift = [&](uint32_t root, uint32_t end) {
    while (2 * root + 1 < end) {
      uint32_t ch = 2 * root + 1;
      if (ch + 1 < end && a[ch] < a[ch + 1]) ch++;
      if (a[root] < a[ch]) { const uint32_t t = a[root]; a[root] = a[ch]; a[ch] = t; root = ch; }
      else return;
    }
  };
  for (uint32_t st = n / 2; st-- > 0;) sift(st, n);
  for (uint32_t end = n; end-- > 1;) {
    const uint32_t t = a[0]; a[0] = a[end]; a[end] = t;
    sift(0, end);
  }
}

// ---------------------------------------------------------------------------
// k_collide: Interaction + Sampling (+ physical reorder) for tiles of 32
// consecutive (run, cell) keys.  Each WARP owns one tile independently (lane
// = cell): per-cell scalars stay in registers and are exchanged by shuffles,
// the tile's particles are staged in the warp's slice of shared memory, and
// phases are separated by __syncwarp only, so the warps of an SM overlap
// their memory and compute phases freely.
//   A  segment bounds from the LCR ends, run metadata
//   B  stage the tile's LCR slice; tag each position with its cell (lane)
//   C  canonical order (R11): lanes sort segments of <= NET in registers
//      (bitonic network); bigger segments rank every element
//   D  gather velocities in canonical order; on reorder steps copy positions
//      to their canonical rank in the other half of P
//   E  NTC: M per cell, warp prefix, cells reassigned to lanes in order of M
//      (bitonic over the warp); rounds of pre-drawn candidates (pair,
//      acceptance word, Marsaglia pair), then each lane walks one cell's
//      candidates in increasing k -- the method's sequential order
//   F  write modified velocities back (or the whole tile to its new rank)
// mode 0: full step; mode 1: sample only into `slot_arg` (dsmc_sample);
// mode 2: sample added to `slot_arg` (dsmc_sample_add, time averaging).
#ifndef DSMC_WPB
#define DSMC_WPB 1
#endif
constexpr int WPB = DSMC_WPB;   // warps per block (1: the tile index, hence run and key, is uniform)
constexpr int CCW = DSMC_CCW;   // pre-drawn candidates per round per warp

struct WarpSmem {           // carve-out of one warp's slice of dynamic smem
  uint32_t* sorted;         // [capw] canonical (sorted) store indices of the tile
  uint32_t* a;              // [capw + APAD] the staged LCR slice (aliases vf: dead after phase C)
  float* vf;                // [capw][VS] velocities (x, y, z) in canonical order
  float4* rec;              // [CCW] pre-drawn candidate: unit vector (R14) and acceptance threshold / word
  uint32_t* cij;            // [CCW] candidate pair i | j << 16
  uint8_t* cell; uint8_t* fl;
  uint8_t* own;             // [CCW] owning cell (lane) of each candidate of the E1 pass (DSMC_OWNMAP)
};

// the staged LCR slice `a` (the bulk copy's 16-byte aligned window around [S, E): up
// to 3 words of slack on either side) aliases the 12 capw bytes of vf
// `one`: every tile of the kernel lies in one run (ONE): the tags are then used by the rank
// sort of C only and can share the records' bytes (capw <= 16 CCW is checked by the host)
__host__ __device__ inline bool cell_aliased(int capw, bool one) { return one && capw <= 16 * CCW; }
__host__ __device__ inline size_t warp_smem_bytes(int capw, bool one) {   // capw a multiple of 32
  return (size_t)capw * (4 + 4 * VS + (cell_aliased(capw, one) ? 0 : 1)) +
         (size_t)CCW * (16 + 4 + 1 + (DSMC_OWNMAP ? 1 : 0)) + 16;
}

__device__ __forceinline__ WarpSmem warp_smem(uint8_t* base, int capw, bool one) {
  WarpSmem w;
  w.sorted = reinterpret_cast<uint32_t*>(base);
  w.vf = reinterpret_cast<float*>(w.sorted + capw);          // 16-byte aligned (capw % 4 == 0)
  w.a = reinterpret_cast<uint32_t*>(w.vf);                   // capw + APAD words fit in 3 capw words
  w.rec = reinterpret_cast<float4*>(w.vf + (size_t)VS * capw);
  w.cij = reinterpret_cast<uint32_t*>(w.rec + CCW);
  w.fl = reinterpret_cast<uint8_t*>(w.cij + CCW);      // candidates whose first Marsaglia try was rejected
  w.own = w.fl + CCW;
  w.cell = cell_aliased(capw, one) ? reinterpret_cast<uint8_t*>(w.rec) : w.own + CCW;
  return w;
}

// E1 of k_collide: candidates [base, base + lim) of the tile drawn lane-parallel
// (two per lane per pass: four independent Philox chains in flight); owner
// cell of a candidate = last lane with prefix mst <= index.  UK: the tile
// lies in one run, whose key key_u is then warp-uniform.
template <bool UK, int MODEL>
__device__ __forceinline__ void ntc_predraw(const Prm& P, const WarpSmem& W, int lane, uint32_t base, uint32_t lim,
                                            uint32_t mst, uint32_t M, uint32_t N, double ghatu, int r, uint32_t c,
                                            uint32_t s, uint2 key_u) {
    const unsigned lt = (1u << lane) - 1u;
    uint32_t nfail = 0;        // candidates whose first Marsaglia try (pair block) was rejected
    const uint32_t c0 = (UK && DSMC_CCARITH) ? __shfl_sync(FULL, c, 0) : 0u;   // one run: c(lane) = c0 + lane
#if DSMC_OWNMAP
    // owner of each candidate of the pass: every lane marks its cell's range (at most
    // the cell's M entries) -- one byte load per candidate instead of a 5-step search
    {
      const uint32_t a0 = mst > base ? mst : base;
      const uint32_t a1 = mst + M < base + lim ? mst + M : base + lim;
      DSMC_LOOP_UNROLL
      for (uint32_t k = a0; k < a1; k++) W.own[k - base] = (uint8_t)lane;
      __syncwarp();
    }
#endif
    DSMC_LOOP_UNROLL
    for (uint32_t q0 = 0; q0 < lim; q0 += 64) {
      uint32_t qq[2], kq[2], nc[2];
      double gq_hat[2];
      int rc[2];
      uint32_t cc[2];
#pragma unroll
      for (int hh = 0; hh < 2; hh++) {
        qq[hh] = q0 + 32 * hh + lane;
        const uint32_t gq = base + qq[hh];
        // owning cell of candidate gq: last lane with mst <= gq
#if DSMC_OWNMAP
        const int lo = qq[hh] < lim ? (int)W.own[qq[hh]] : 0;
#else
        int lo = 0;     // (binary search over lanes)
#pragma unroll
        for (int stp = 16; stp > 0; stp >>= 1) {
          const uint32_t m = __shfl_sync(FULL, mst, lo + stp);
          if (m <= gq && lo + stp < 32) lo += stp;
        }
#endif
        nc[hh] = __shfl_sync(FULL, N, lo);
        gq_hat[hh] = __shfl_sync(FULL, ghatu, lo);
        kq[hh] = gq - __shfl_sync(FULL, mst, lo);
        rc[hh] = __shfl_sync(FULL, r, lo);
        cc[hh] = (UK && DSMC_CCARITH) ? c0 + (uint32_t)lo : __shfl_sync(FULL, c, lo);
      }
      uint4 wp[2];
#pragma unroll
      for (int hh = 0; hh < 2; hh++) {
        const uint2 keyc = UK ? key_u : run_key(P, rc[hh]);
        wp[hh] = draw(keyc, cc[hh], s, TAG_COLL_PAIR, kq[hh], 0);
      }
#pragma unroll
      for (int hh = 0; hh < 2; hh++) {
        const uint32_t q = qq[hh];
        const float pp = 2.0f * u_co(wp[hh].z) - 1.0f, qv = 2.0f * u_co(wp[hh].w) - 1.0f;
        const float rho = pp * pp + qv * qv;
        const bool fail = q < lim && !(rho < 1.0f);
        const unsigned fm = __ballot_sync(FULL, fail);
        if (fail) W.fl[nfail + __popc(fm & lt)] = (uint8_t)q;
        nfail += __popc(fm);
        if (q < lim) {
          uint32_t i, j;
          pair_of(wp[hh].x, nc[hh], i, j);
          W.cij[q] = i | (j << 16);
          uint32_t thr;
          if (MODEL == DSMC_MODEL_HS) {
            // HS: accept iff (double)g2 > (u ghat)^2 (R13)  <=>  g2 > F, F the largest
            // float <= (u ghat)^2 -- the same decision as one fp32 compare in the walk
            const double lhs = u_co_d(wp[hh].y) * gq_hat[hh];
            thr = __float_as_uint(__double2float_rd(lhs * lhs));
          } else {
            thr = wp[hh].y;
          }
          if (!fail) {   // unit vector of R14 from the pair block's try
            const float sr = sqrtf(1.0f - rho);
            W.rec[q] = make_float4(2.0f * pp * sr, 2.0f * qv * sr, 1.0f - 2.0f * rho, __uint_as_float(thr));
          } else {
            reinterpret_cast<float*>(W.rec + q)[3] = __uint_as_float(thr);
          }
        }
      }
    }
    // rejected first tries (about one candidate in five), compacted: direction blocks
    __syncwarp();
    DSMC_LOOP_UNROLL
    for (uint32_t f0 = 0; f0 < nfail; f0 += 32) {
      const bool act = f0 + lane < nfail;
      const uint32_t q = act ? W.fl[f0 + lane] : 0u;
      const uint32_t gq = base + q;
#if DSMC_OWNMAP
      const int lo = act ? (int)W.own[q] : 0;
#else
      int lo = 0;
#pragma unroll
      for (int stp = 16; stp > 0; stp >>= 1) {
        const uint32_t m = __shfl_sync(FULL, mst, lo + stp);
        if (m <= gq && lo + stp < 32) lo += stp;
      }
#endif
      const uint32_t kq = gq - __shfl_sync(FULL, mst, lo);
      const uint32_t cc = (UK && DSMC_CCARITH) ? c0 + (uint32_t)lo : __shfl_sync(FULL, c, lo);
      const int rc = __shfl_sync(FULL, r, lo);
      if (act) {
        const uint2 keyc = UK ? key_u : run_key(P, rc);
        const uint4 wd = draw(keyc, cc, s, TAG_COLL_DIR, kq, 0);
        float pp = 2.0f * u_co(wd.x) - 1.0f, qv = 2.0f * u_co(wd.y) - 1.0f;
        if (!(pp * pp + qv * qv < 1.0f)) {
          pp = 2.0f * u_co(wd.z) - 1.0f;
          qv = 2.0f * u_co(wd.w) - 1.0f;
          if (!(pp * pp + qv * qv < 1.0f)) marsaglia_pq_from(keyc, cc, s, kq, 1, pp, qv);
        }
        const float rho = pp * pp + qv * qv;
        const float sr = sqrtf(1.0f - rho);
        float* rq = reinterpret_cast<float*>(W.rec + q);
        rq[0] = 2.0f * pp * sr;
        rq[1] = 2.0f * qv * sr;
        rq[2] = 1.0f - 2.0f * rho;
      }
    }
}

// sample slot of this launch: the schedule's (R2: after step s when (s+1) is a
// multiple of the sampling interval) in mode 0, the caller's otherwise
__device__ __forceinline__ int sched_slot(const Prm& P, int mode, int32_t s, int slot_arg) {
  (void)s;
  return mode != 0 ? slot_arg : *P.ctl.step_slot;   // k_step_mid decided it for this step
}

// MODEL: the collision model is a template parameter so that the hard-sphere
// kernel carries no VHS code (its presence cost 2.4% at c4)
// ONE: every 32-cell tile lies in one run (Nc % 32 == 0 or a single run): the
// multi-run paths are compiled out (c4: 6336 -> 5328 SASS instructions, k_collide
// 12.15 -> 11.59 ms at n = 256, fewer instruction-cache misses)
// LIST: the tile comes from k_collide_triage's list (k_collide_list: persistent
// blocks; the mbarrier is initialised once per block and completes one phase per
// staged tile; the triage already took the run's largest cell count and queued
// the heavy tiles)
template <int D, int NET, int MODEL, bool STEP, bool ONE, bool LIST>
__device__ __forceinline__ void collide_tile(const Prm& P, const int mode_arg, const int slot_arg, const int capw,
                                             const WarpSmem& W, uint64_t* bar, uint32_t& bar_phase,
                                             const int64_t k0) {
  const int mode = STEP ? 0 : mode_arg;      // STEP: the kernel of dsmc_step (mode 0) only
  const int lane = threadIdx.x & 31;
  const int64_t RN = (int64_t)P.R * P.Nc;
  const int64_t RS = (int64_t)P.R * P.stride;
  float* const P0 = P.P;
  float* const P1 = P.P + P.half;
  if (k0 >= RN) return;                          // whole warp leaves together
  const int64_t k = k0 + lane;
  const bool valid = k < RN;
  const int64_t klast = k0 + 31 < RN ? k0 + 31 : RN - 1;
  const int last_lane = (int)(klast - k0);
  const uint32_t Nc32 = (uint32_t)P.Nc;          // R*Nc < 2^31 (checked in dsmc_create)
  const int r_first = (int)run_of(P, (uint32_t)k0);
  const int r_last = (int)run_of(P, (uint32_t)klast);
  const bool one_run = ONE || r_first == r_last;
  // ---- A
  uint32_t st = 0, en = 0;
  if (valid) {
    st = k == 0 ? 0u : DSMC_LD1(P.cell + k - 1);
    en = DSMC_LD1(P.cell + k);
  }
  const int r = ONE ? r_first : (valid ? (int)run_of(P, (uint32_t)k) : r_last);
  const uint32_t c = valid ? (uint32_t)k - (uint32_t)r * Nc32 : 0u;
  const uint32_t N = en - st;
  const uint32_t S = __shfl_sync(FULL, st, 0);
  const uint32_t E = __shfl_sync(FULL, en, last_lane);
  const uint32_t cnt = E - S;
  const uint32_t off = st - S;
  const int h = P.ctl.parity[r];
  const int reo = mode == 0 ? P.ctl.reorder[r] : 0;
  const uint32_t rbase = run_lcr_base(P, r);
  // the step index (device memory: the graph replays) is first needed by the
  // draws of E; the schedule decision below uses it only at Sampling, so its
  // load latency hides behind B-D
  const int32_t s = *P.ctl.step;
  const uint2 key = run_key(P, r);
  uint32_t ncand = 0, nacc = 0;
  // cell-occupancy skew: the step's largest particle count per cell, per run
  if (LIST) {
  } else if (one_run) {
    const uint32_t wmax = __reduce_max_sync(FULL, valid ? N : 0u);
    if (lane == 0 && wmax) atomicMax(P.ctl.maxn + r_first, wmax);
  } else if (valid && N) {
    atomicMax(P.ctl.maxn + r, N);
  }
  if (!LIST && cnt > (uint32_t)capw) {
    // tile too large for the warp's shared memory: hand it to k_collide_heavy
    // (a whole block with a large staging area -- the "heap" of TLPDPR)
    // (tiered by size: the smaller the staging area, the more blocks per SM;
    // the static NEXT-1 arm puts every such tile in the large tier)
    if (lane == 0) {
      const int q = (P.heavy_static || cnt + HEAVY_SLACK > (uint32_t)P.caph_tier[0]) ? 1 : 0;   // HEAVY_TIERS == 2
      P.heavy_list[(int64_t)q * P.heavy_stride + atomicAdd(P.ctl.heavy + 2 * q, 1u)] = (uint32_t)(k0 / 32);
    }
    return;
  }
  float gm = valid ? DSMC_LD1(P.gmax + k) : 0.0f;
  const float gm0 = gm;
  {
    // ---- B: the tile's LCR slice [S, E) is contiguous: one lane moves its 16-byte
    // aligned window into shared memory with a bulk (TMA) copy completing on an
    // mbarrier, and the candidate counts of E0 (which need only N and the majorant)
    // are drawn while it is in flight.  (The lcr buffer is a whole number of
    // 32-slot run windows, so the window rounded up to 4 words stays inside it.)
    uint32_t* const wa = W.a + (S & 3u);
    if (cnt > 0) {
      if (lane == 0) {
        const uint32_t s0 = S & ~3u, e0 = (E + 3u) & ~3u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes before the async copy
        if (!LIST) mbar_init(bar, 1u);
        mbar_arrive_expect_tx(bar, (e0 - s0) * 4u);
        bulk_g2s(W.a, P.lcr + s0, (e0 - s0) * 4u, bar);
      }
      __syncwarp();
    }
    // ---- E0: candidate count M per cell (R12) and its exclusive warp prefix mst
    uint32_t M = 0, mst = 0, tot = 0;
    if (mode == 0) {
      M = valid ? ntc_count(P, one_run ? run_key(P, r_first) : key, c, (uint32_t)s, N, gm) : 0u;
      tot = __reduce_add_sync(FULL, M);
      if (tot) {                                 // (an idle tile needs no prefix)
        mst = M;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(FULL, mst, o); if (lane >= o) mst += y; }
        mst -= M;
      }
    }
    const int slot = sched_slot(P, mode, s, slot_arg);
    // a tile with no candidate, no Sampling and no reorder this step changes nothing
    // (most of c5's sparse background): only the bulk copy is drained before the warp leaves
    const bool idle = mode == 0 && tot == 0 && slot < 0 && !P.debug && __all_sync(FULL, reo == 0);
    if (idle) {
      if (cnt > 0) { mbar_wait(bar, bar_phase); bar_phase ^= 1u; }
    } else {
    // largest segment of the warp (network width); element -> cell tags only
    // where the rank sort or the multi-run paths need them
    const uint32_t wN = __reduce_max_sync(FULL, valid ? N : 0u);
    if (valid && (wN > DSMC_NET_MAX || !one_run)) for (uint32_t i = 0; i < N; i++) W.cell[off + i] = (uint8_t)lane;
    if (cnt > 0) { mbar_wait(bar, bar_phase); bar_phase ^= 1u; }
    __syncwarp();
    // ---- C: network width by the warp's largest segment (warp-uniform)
    if (wN <= DSMC_NET_MAX) {
      if (valid && N > 0) {
        const uint32_t* src = wa + off;
        uint32_t* dst = W.sorted + off;
#ifndef DSMC_NETS
#define DSMC_NETS 5    // network widths: 8, 16, 20, 24, 32 (7 adds 4 and 12: c4 11.61 against 11.48-11.53 ms; c5 0.959 against 0.947)
#endif
        if (DSMC_NETS >= 7 && wN <= 4) sort_segment<4, 4>(src, dst, N);
        else if (wN <= 8) sort_segment<8, 8>(src, dst, N);
        else if (DSMC_NETS >= 6 && wN <= 12) sort_segment<16, 12>(src, dst, N);
        else if (wN <= 16) sort_segment<16, 16>(src, dst, N);
        else if (wN <= 20 || DSMC_NET_MAX <= 20) sort_segment<32, 20>(src, dst, N);
        else if (DSMC_NETS >= 5 && wN <= 24) sort_segment<32, 24>(src, dst, N);
        else sort_segment<32, 32>(src, dst, N);
      }
    } else {
      if (valid && N <= (uint32_t)NET) sort_segment<NET, NET>(wa + off, W.sorted + off, N);
      DSMC_LOOP_UNROLL
      for (uint32_t q0 = 0; q0 < cnt; q0 += 32) {
        const uint32_t q = q0 + lane;
        const int cq = q < cnt ? W.cell[q] : 0;
        const uint32_t n = __shfl_sync(FULL, N, cq), b = __shfl_sync(FULL, off, cq);
        if (q < cnt && n > (uint32_t)NET) {
          const uint32_t v = wa[q];
          uint32_t rank = 0;
          DSMC_LOOP_UNROLL
          for (uint32_t p = 0; p < n; p++) rank += wa[b + p] < v ? 1u : 0u;
          W.sorted[b + rank] = v;
        }
      }
    }
    __syncwarp();
    // ---- D
    float* const vf = W.vf;
    if (one_run) {
      // per-array base pointers indexed by 32-bit offsets (one IMAD.WIDE per access)
      const float* __restrict__ sx = (h ? P1 : P0) + 3 * RS;
      const float* __restrict__ sy = sx + RS;
      const float* __restrict__ sz = sy + RS;
      // velocities in canonical order: 4-byte cp.async gathers straight into shared
      // memory (no registers held while they are in flight); they complete while
      // E1 draws the candidates, and the walk E2 waits for them
      DSMC_LANE_UNROLL
      for (uint32_t q = lane; q < cnt; q += 32) {
        const uint32_t g = W.sorted[q];
        float* d = vf + VS * q;
        cp_async4(d, sx + g);
        cp_async4(d + 1, sy + g);
        cp_async4(d + 2, sz + g);
      }
      cp_async_commit();
      // (on reorder steps the positions move in F, once the staging arrays are free)
    } else {
      DSMC_LOOP_UNROLL
      for (uint32_t q0 = 0; q0 < cnt; q0 += 32) {
        const uint32_t q = q0 + lane;
        const int cq = q < cnt ? W.cell[q] : 0;
        const int hq = __shfl_sync(FULL, h, cq), rq = __shfl_sync(FULL, reo, cq);
        const int runq = __shfl_sync(FULL, r, cq);
        const uint32_t bq = __shfl_sync(FULL, rbase, cq);
        if (q < cnt) {
          const uint32_t g = W.sorted[q];
          const float* src = (hq ? P1 : P0) + g;
          if (rq) {
            float* d = (hq ? P0 : P1) + (int64_t)runq * P.stride + (int64_t)(S + q - bq);
#pragma unroll
            for (int a = 0; a < D; a++) d[a * RS] = src[a * RS];
          }
          vf[VS * q] = src[3 * RS];
          vf[VS * q + 1] = src[4 * RS];
          vf[VS * q + 2] = src[5 * RS];
        }
      }
    }
    __syncwarp();
    // ---- E
    if (mode == 0) {
      ncand = M;
      const uint32_t Mu = M, mstu = mst;
      const double gmu = (double)gm, ghatu = gmu / P.sigma_c;
      SmemCellV Au{vf + VS * off};
      float maxg2 = 0.0f;
      uint32_t naccu = 0;
      DSMC_LOOP_UNROLL
      for (uint32_t base = 0; base < tot; base += CCW) {
        const uint32_t lim = tot - base < (uint32_t)CCW ? tot - base : (uint32_t)CCW;
        // two candidates per lane per pass: four independent Philox chains in flight
        if (one_run)
          ntc_predraw<true, MODEL>(P, W, lane, base, lim, mst, M, N, ghatu, r, c, (uint32_t)s, run_key(P, r_first));
        else
          ntc_predraw<false, MODEL>(P, W, lane, base, lim, mst, M, N, ghatu, r, c, (uint32_t)s, run_key(P, r_first));
        cp_async_wait_all();                      // the velocity gathers of D (pending in the first pass only)
        __syncwarp();
        if (Mu) {
          const uint32_t a0 = mstu > base ? mstu : base;
          const uint32_t a1 = mstu + Mu < base + lim ? mstu + Mu : base + lim;
          if (a0 < a1)
            ntc_apply_pre<MODEL>(P, Au, gmu, W.cij + (a0 - base), W.rec + (a0 - base), a1 - a0, maxg2, naccu);
        }
        __syncwarp();
      }
      if (valid && M) {
        nacc = naccu;
        const double sgm = MODEL == DSMC_MODEL_HS ? P.sigma_c * sqrt((double)maxg2)
                                                  : P.sigma_c * pow((double)maxg2, P.omega1);
        if (sgm > (double)gm) gm = (float)sgm;
      }
    }
    cp_async_wait_all();                          // no candidates (or no Interaction): gathers of D
    __syncwarp();
    if (valid && slot >= 0) sample_cell(P, slot, k, N, SmemCellV{vf + VS * off}, mode == 2);
    // a tile without an accepted collision changed no velocity: nothing to write back
    // on a non-reorder step (sparse tiles, e.g. c5's background)
    const bool any_acc = __any_sync(FULL, nacc != 0);
    __syncwarp();
    // ---- F
    if (one_run) {
      if (reo) {
        // the tile to its canonical rank in the other half: velocities from the
        // staging arrays, then the positions gathered into them by cp.async (every
        // load of the tile in flight at once) and written out the same way
        float* __restrict__ dx = (h ? P0 : P1) + (int64_t)r * P.stride + (S - rbase);
        float* __restrict__ dy = dx + RS;
        float* __restrict__ dz = dy + RS;
        DSMC_LANE_UNROLL
        for (uint32_t q = lane; q < cnt; q += 32) {
          float v[3];
          SmemCellV{vf}.ld(q, v);
          DSMC_ST1(dx + 3 * RS + q, v[0]);
          DSMC_ST1(dy + 3 * RS + q, v[1]);
          DSMC_ST1(dz + 3 * RS + q, v[2]);
        }
        __syncwarp();
        const float* __restrict__ px = (h ? P1 : P0);
        const float* __restrict__ py = px + RS;
        const float* __restrict__ pz = py + RS;
        DSMC_LANE_UNROLL
        for (uint32_t q = lane; q < cnt; q += 32) {
          const uint32_t g = W.sorted[q];
          float* d = vf + VS * q;
          cp_async4(d, px + g);
          if (D > 1) cp_async4(d + 1, py + g);
          if (D > 2) cp_async4(d + 2, pz + g);
        }
        cp_async_commit();
        cp_async_wait_all();
        __syncwarp();
        DSMC_LANE_UNROLL
        for (uint32_t q = lane; q < cnt; q += 32) {
          float v[3];
          SmemCellV{vf}.ld(q, v);
          DSMC_ST1(dx + q, v[0]);
          if (D > 1) DSMC_ST1(dy + q, v[1]);
          if (D > 2) DSMC_ST1(dz + q, v[2]);
        }
      } else if (any_acc) {
        float* __restrict__ vxp = (h ? P1 : P0) + 3 * RS;
        float* __restrict__ vyp = vxp + RS;
        float* __restrict__ vzp = vyp + RS;
        DSMC_LANE_UNROLL
        for (uint32_t q = lane; q < cnt; q += 32) {
          const uint32_t g = W.sorted[q];
          float v[3];
          SmemCellV{vf}.ld(q, v);
          DSMC_ST1(vxp + g, v[0]);
          DSMC_ST1(vyp + g, v[1]);
          DSMC_ST1(vzp + g, v[2]);
        }
      }
    } else {
      DSMC_LOOP_UNROLL
      for (uint32_t q0 = 0; q0 < cnt; q0 += 32) {
        const uint32_t q = q0 + lane;
        const int cq = q < cnt ? W.cell[q] : 0;
        const int hq = __shfl_sync(FULL, h, cq), rq = __shfl_sync(FULL, reo, cq);
        const int runq = __shfl_sync(FULL, r, cq);
        const uint32_t bq = __shfl_sync(FULL, rbase, cq);
        if (q < cnt) {
          if (rq) {
            float* d = (hq ? P0 : P1) + (int64_t)runq * P.stride + (int64_t)(S + q - bq);
            float v[3];
            SmemCellV{vf}.ld(q, v);
            d[3 * RS] = v[0];
            d[4 * RS] = v[1];
            d[5 * RS] = v[2];
          } else {                               // full write-back (no collided flags)
            float* d = (hq ? P1 : P0) + W.sorted[q];
            float v[3];
            SmemCellV{vf}.ld(q, v);
            d[3 * RS] = v[0];
            d[4 * RS] = v[1];
            d[5 * RS] = v[2];
          }
        }
      }
    }
    if (P.debug)
      for (uint32_t q = lane; q < cnt; q += 32) P.lcr[S + q] = W.sorted[q];
    }   // !idle
  }
  if (valid && gm != gm0) P.gmax[k] = gm;
  if (valid && P.debug && mode == 0) { P.dbg_cand[k] = ncand; P.dbg_acc[k] = (int32_t)nacc; }
  // per-run counters: aggregate lanes of the same run
  if (ONE) {
    if (mode == 0) {
      const uint32_t sc = __reduce_add_sync(FULL, ncand);
      if (sc) {
        const uint32_t sa = __reduce_add_sync(FULL, nacc);
        if (lane == 0) {
          atomicAdd(&P.ctl.counters[r_first * 4 + 2], (unsigned long long)sc);
          atomicAdd(&P.ctl.counters[r_first * 4 + 3], (unsigned long long)sa);
        }
      }
    }
  } else if (mode == 0) {
    const uint32_t rk = valid ? (uint32_t)r : 0xFFFFFFFFu;
    const unsigned m = __match_any_sync(FULL, rk);
    const uint32_t sc = __reduce_add_sync(m, ncand), sa = __reduce_add_sync(m, nacc);
    if (valid && lane == __ffs(m) - 1 && sc) {
      atomicAdd(&P.ctl.counters[r * 4 + 2], (unsigned long long)sc);
      atomicAdd(&P.ctl.counters[r * 4 + 3], (unsigned long long)sa);
    }
  }
}

template <int D, int NET, int MODEL, bool STEP, bool ONE>
__global__ void __launch_bounds__(WPB * 32, DSMC_COLLIDE_MINB / WPB) k_collide(Prm P, int mode_arg, int slot_arg, int capw) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ __align__(8) uint64_t s_bars[WPB];  // completion of each warp's bulk copy of its LCR slice
  uint64_t& s_bar = s_bars[threadIdx.x >> 5];
  const int wid = threadIdx.x >> 5;
  const WarpSmem W = warp_smem(dsm + (size_t)wid * warp_smem_bytes(capw, ONE), capw, ONE);
  uint32_t ph = 0;
  collide_tile<D, NET, MODEL, STEP, ONE, false>(P, mode_arg, slot_arg, capw, W, &s_bar, ph,
                                                ((int64_t)blockIdx.x * WPB + wid) * 32);
}

// Sparse problems (mean fill below DSMC_COMPACT_PPC particles per cell: c5's background,
// c2): most tiles draw no candidate, and on a step without Sampling or reorder such a
// tile changes nothing, but a one-warp block per tile still pays its launch and two
// dependent global round trips (524288 blocks of c5 launch in 0.27 ms on their own).
// k_collide_triage draws the candidate counts of R12 with one thread per cell -- the
// same draws E0 repeats -- at full occupancy, queues the heavy tiles as k_collide would,
// and lists the tiles with work; persistent k_collide_list blocks then take the list.
constexpr int TRIAGE_T = 1024;
constexpr int TRIAGE_TPW = 4;    // tiles per warp: 128 tiles per block, one list atomic per block
template <bool ONE>
__global__ void __launch_bounds__(TRIAGE_T) k_collide_triage(Prm P, int capw) {
  __shared__ uint32_t s_cls[TRIAGE_T / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t RN = (int64_t)P.R * P.Nc;
  const int32_t s = *P.ctl.step;
  const bool all = *P.ctl.step_slot >= 0 || P.debug;     // Sampling (or debug): every tile has work
  uint32_t cls = 0;                // 2 bits per tile of this warp: 0 idle, 1 warp list, 2 / 3 heavy tier 0 / 1
#pragma unroll
  for (int t = 0; t < TRIAGE_TPW; t++) {
    const int64_t k0 = (((int64_t)blockIdx.x * (TRIAGE_T / 32) + wid) * TRIAGE_TPW + t) * 32;
    if (k0 >= RN) break;
    const int64_t k = k0 + lane;
    const bool valid = k < RN;
    const int64_t klast = k0 + 31 < RN ? k0 + 31 : RN - 1;
    const int last_lane = (int)(klast - k0);
    const int r_first = (int)run_of(P, (uint32_t)k0);
    const int r_last = (int)run_of(P, (uint32_t)klast);
    const bool one_run = ONE || r_first == r_last;
    const uint32_t en = valid ? P.cell[k] : 0u;
    uint32_t st = __shfl_up_sync(FULL, en, 1);
    if (lane == 0) st = k == 0 ? 0u : P.cell[k - 1];
    const int r = ONE ? r_first : (valid ? (int)run_of(P, (uint32_t)k) : r_last);
    const uint32_t c = valid ? (uint32_t)k - (uint32_t)r * (uint32_t)P.Nc : 0u;
    const uint32_t N = valid ? en - st : 0u;
    const uint32_t S = __shfl_sync(FULL, st, 0);
    const uint32_t E = __shfl_sync(FULL, en, last_lane);
    // (read first: the run's maximum settles within a few tiles, and thousands of
    // atomics per microsecond on one address would serialise)
    if (one_run) {
      const uint32_t wmax = __reduce_max_sync(FULL, N);
      if (lane == 0 && wmax > P.ctl.maxn[r_first]) atomicMax(P.ctl.maxn + r_first, wmax);
    } else if (N > P.ctl.maxn[r]) {
      atomicMax(P.ctl.maxn + r, N);
    }
    uint32_t ct;
    if (E - S > (uint32_t)capw) {
      ct = (P.heavy_static || E - S + HEAVY_SLACK > (uint32_t)P.caph_tier[0]) ? 3u : 2u;   // HEAVY_TIERS == 2
    } else {
      const float gm = valid ? P.gmax[k] : 0.0f;
      const uint32_t M = valid ? ntc_count(P, run_key(P, r), c, (uint32_t)s, N, gm) : 0u;
      ct = (all || __any_sync(FULL, M != 0u || P.ctl.reorder[r] != 0)) ? 1u : 0u;
    }
    cls |= ct << (2 * t);
  }
  if (lane == 0) s_cls[wid] = cls;
  __syncthreads();
  if (wid == 0) {
    // the block's 128 tiles in order (warp w holds 4w .. 4w+3): one atomic per list
    const uint32_t a = s_cls[lane];
    const uint32_t t0 = (blockIdx.x * (TRIAGE_T / 32) + lane) * TRIAGE_TPW;
#pragma unroll
    for (uint32_t q = 1; q <= 3; q++) {
      uint32_t mine = 0;
#pragma unroll
      for (int t = 0; t < TRIAGE_TPW; t++) mine |= ((a >> (2 * t)) & 3u) == q ? 1u << t : 0u;
      const uint32_t n = __popc(mine);
      uint32_t pre = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(FULL, pre, o); if (lane >= o) pre += y; }
      const uint32_t tot = __shfl_sync(FULL, pre, 31);
      if (tot == 0) continue;
      pre -= n;
      uint32_t* const cnt = q == 1 ? P.ctl.tiles : P.ctl.heavy + 2 * (q - 2);
      uint32_t* const lst = q == 1 ? P.tile_list : P.heavy_list + (int64_t)(q - 2) * P.heavy_stride;
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(cnt, tot);
      base = __shfl_sync(FULL, base, 0) + pre;
#pragma unroll
      for (int t = 0; t < TRIAGE_TPW; t++)
        if (mine & (1u << t)) lst[base + __popc(mine & ((1u << t) - 1u))] = t0 + t;
    }
  }
}

template <int D, int NET, int MODEL, bool ONE>
__global__ void __launch_bounds__(32, DSMC_COLLIDE_MINB) k_collide_list(Prm P, int capw) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ __align__(8) uint64_t s_bar;
  const WarpSmem W = warp_smem(dsm, capw, ONE);
  if (threadIdx.x == 0) mbar_init(&s_bar, 1u);
  __syncwarp();
  uint32_t ph = 0;
  const uint32_t n = *P.ctl.tiles;
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
    collide_tile<D, NET, MODEL, true, ONE, true>(P, 0, -1, capw, W, &s_bar, ph, (int64_t)P.tile_list[i] * 32);
    // every lane's generic shared-memory accesses of this tile are ordered before the
    // next tile's bulk copy (async proxy) overwrites the staging area
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// k_collide_heavy: the warp tiles k_collide could not stage (dense cells, e.g.
// c5's orifice jet).  The GPU analog of TLPDPR's processor heap (PAPER.md
// 501-515, Eq. 12): a persistent block "borrows" 256 threads and a large
// shared-memory staging area for one such tile at a time, taken from the
// queue k_collide filled.  Same phases and arithmetic as k_collide:
// block-parallel staging, rank sort, gather and candidate pre-draws; the
// per-cell candidate walk stays sequential (thread per cell).
constexpr int CCH = 1024;   // pre-drawn candidates per round

__host__ __device__ inline size_t heavy_smem_bytes(int caph) { return (size_t)caph * 22 + (size_t)CCH * 17 + 32; }

template <int D, int HT>   // HT threads per block: 256 (small tier, two blocks per SM) or 512
__global__ void __launch_bounds__(HT) k_collide_heavy(Prm P, int mode, int slot_arg, int caph, int queue) {
  extern __shared__ __align__(16) uint8_t dsm[];
  uint32_t* s_sorted = reinterpret_cast<uint32_t*>(dsm);
  uint32_t* s_a = s_sorted + caph;
  float* s_vx = reinterpret_cast<float*>(s_a);
  float* s_vy = reinterpret_cast<float*>(s_a + caph);
  float* s_vz = s_vy + caph;
  uint32_t* s_cij = reinterpret_cast<uint32_t*>(s_vz + caph);
  uint32_t* s_cur = s_cij + CCH;
  float* s_cp = reinterpret_cast<float*>(s_cur + CCH);
  float* s_cq = s_cp + CCH;
  uint32_t* s_min = reinterpret_cast<uint32_t*>(s_cq + CCH);   // earliest undone candidate on a particle
  uint8_t* s_clo = reinterpret_cast<uint8_t*>(s_min + caph);     // owner cell (lane) of a candidate
  uint8_t* s_cell = s_clo + CCH;
  uint8_t* s_mod = s_cell + caph;
  __shared__ uint32_t c_st[33], c_N[32], c_M[32], c_mst[33], c_c[32], c_base[32], c_nacc[32];
  __shared__ float c_mg2[32];
  __shared__ int c_r[32], c_h[32], c_reo[32];
  __shared__ float c_gm[32];
  __shared__ double c_gh[32];
  __shared__ uint32_t s_tile, c_k[33], s_nmax;
  __shared__ __align__(8) uint64_t s_hbar;       // completion of the tile's LCR bulk copy
  const int t = threadIdx.x;
  const int64_t RN = (int64_t)P.R * P.Nc;
  const int64_t RS = (int64_t)P.R * P.stride;
  const uint32_t Nc32 = (uint32_t)P.Nc;
  const int32_t s = *P.ctl.step;
  int slot = -1;
  if (mode == 0) {
    if ((s + 1) % P.sample_every == 0 && (s + 1) / P.sample_every - 1 < P.n_slots) slot = (s + 1) / P.sample_every - 1;
  } else {
    slot = slot_arg;
  }
  const uint32_t* const hlist = P.heavy_list + (int64_t)queue * P.heavy_stride;
  uint32_t* const hctr = P.ctl.heavy + 2 * queue;
  const uint32_t n_heavy = hctr[0];
  if (t == 0) mbar_init(&s_hbar, 1u);            // initialised once; each staged tile completes one phase
  uint32_t hphase = 0;
  for (uint32_t it = 0;; it++) {
    __syncthreads();
    // dynamic: the next tile from the queue; static (NEXT-1 A/B arm): block b takes
    // tiles b, b + G, b + 2G, ... whatever their sizes
    if (t == 0) s_tile = P.heavy_static ? blockIdx.x + it * gridDim.x : atomicAdd(hctr + 1, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= n_heavy) break;
    const int64_t k0 = (int64_t)hlist[tile] * 32;
    // ---- A (thread per cell)
    const bool valid = t < 32 && k0 + t < RN;
    uint32_t N = 0, c = 0;
    int r = 0, h = 0, reo = 0;
    float gm = 0.0f;
    if (t < 32) {
      const int64_t k = k0 + t;
      uint32_t st = 0, en = 0;
      if (valid) {
        st = k == 0 ? 0u : P.cell[k - 1];
        en = P.cell[k];
        r = (int)((uint32_t)k / Nc32);
        c = (uint32_t)k - (uint32_t)r * Nc32;
        h = P.ctl.parity[r];
        reo = mode == 0 ? P.ctl.reorder[r] : 0;
        gm = P.gmax[k];
        c_base[t] = run_lcr_base(P, r);
      } else {
        st = en = 0xFFFFFFFFu;
      }
      N = en - st;
      c_st[t] = st;
      c_N[t] = valid ? N : 0u;
      c_c[t] = c;
      c_r[t] = r;
      c_h[t] = h;
      c_reo[t] = reo;
      c_gm[t] = gm;
      c_gh[t] = (double)gm / P.sigma_c;
      // 64-element sort chunks per cell (prefix) and the largest cell, for phase C
      const uint32_t nch = valid ? (N + 63u) >> 6 : 0u;
      uint32_t xk = nch;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(FULL, xk, o); if (t >= o) xk += y; }
      c_k[t] = xk - nch;
      if (t == 31) c_k[32] = xk;
      const uint32_t nm = __reduce_max_sync(FULL, valid ? N : 0u);
      if (t == 0) s_nmax = nm;
    }
    __syncthreads();
    int last = 31;
    while (c_st[last] == 0xFFFFFFFFu) last--;
    const uint32_t S = c_st[0], E = c_st[last] + c_N[last], cnt = E - S;
    if (t == 32) c_st[32] = E;
    // every thread's generic accesses of the previous tile's staging ordered before
    // this tile's bulk copy (async proxy) overwrites it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const float gm0 = gm;
    uint32_t ncand = 0, nacc = 0;
    // the bulk copy's 16-byte aligned window puts the slice at offset S & 3 (<= 3 words)
    // of the staging buffer: the slice itself must fit, or its last words would land
    // in the buffer C's chunk sort writes while other warps still read them
    if (cnt + HEAVY_SLACK <= (uint32_t)caph) {
      // ---- B: the tile's LCR slice is contiguous: one thread moves its 16-byte aligned
      // window into shared memory with a bulk copy on an mbarrier while the block tags
      // every element with its cell.  It lands in the buffer the chunk sort of C does
      // not write (C reads it at offset S & 3); the window's up-to-3-word overhang
      // past cnt spills into the next buffer, which C or D overwrites afterwards.
      int nlev = 0;
      for (uint32_t L = 64; L < s_nmax; L <<= 1) nlev++;
      uint32_t* const stage = (nlev & 1) ? s_sorted : s_a;   // C's chunk sort writes the other one
      if (t == 0 && cnt > 0) {
        const uint32_t s0 = S & ~3u, e0 = (E + 3u) & ~3u;
        // the previous tile's generic-proxy writes to this shared memory (ordered by the
        // block barriers since) must be ordered before the bulk copy's async-proxy writes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(&s_hbar, (e0 - s0) * 4u);
        bulk_g2s(stage, P.lcr + s0, (e0 - s0) * 4u, &s_hbar);
      }
      for (uint32_t q = t; q < cnt; q += HT) {
        int lo = 0;
#pragma unroll
        for (int stp = 16; stp > 0; stp >>= 1)
          if (lo + stp <= last && c_st[lo + stp] <= S + q) lo += stp;
        s_cell[q] = (uint8_t)lo;
      }
      __syncthreads();
      if (cnt > 0) { mbar_wait(&s_hbar, hphase); hphase ^= 1u; }   // one phase per staged tile
      const uint32_t* const s_in = stage + (S & 3u);
      // ---- C: sort every cell's segment: a warp bitonic sort of each 64-element
      // chunk, then merge rounds in which every element finds its place by a
      // binary search of the partner run (keys are distinct store slots).  An
      // O(n^2) rank count was 62% of this kernel's instructions at c5; a block
      // bitonic sort of the whole tile (91 barriers per 8192 elements) was 35%
      // slower than that.
      {
        const uint32_t nmax = s_nmax;
        uint32_t* from = (nlev & 1) ? s_a : s_sorted;   // the last round lands in s_sorted
        const int ln = t & 31;
        const uint32_t nchk = c_k[32];
        for (uint32_t ch = (uint32_t)(t >> 5); ch < nchk; ch += HT / 32) {
          int lo = 0;
#pragma unroll
          for (int stp = 16; stp > 0; stp >>= 1)
            if (lo + stp < 32 && c_k[lo + stp] <= ch) lo += stp;
          const uint32_t b = c_st[lo] - S + ((ch - c_k[lo]) << 6), n = c_st[lo] - S + c_N[lo];
          const bool in0 = b + ln < n, in1 = b + 32 + ln < n;
          uint32_t x0 = in0 ? s_in[b + ln] : 0xFFFFFFFFu, x1 = in1 ? s_in[b + 32 + ln] : 0xFFFFFFFFu;
          // 64-element bitonic sort, element e = lane + 32 h in x_h
#pragma unroll
          for (int k = 2; k <= 64; k <<= 1)
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
              if (j == 32) {                       // partners in one lane (k == 64: ascending)
                const uint32_t lo_ = min(x0, x1), hi_ = max(x0, x1);
                x0 = lo_;
                x1 = hi_;
              } else {
                const uint32_t y0 = __shfl_xor_sync(FULL, x0, j), y1 = __shfl_xor_sync(FULL, x1, j);
                const bool lower = (ln & j) == 0;
                x0 = (lower == ((ln & k) == 0)) ? min(x0, y0) : max(x0, y0);
                x1 = (lower == (((ln + 32) & k) == 0)) ? min(x1, y1) : max(x1, y1);
              }
            }
          if (in0) from[b + ln] = x0;
          if (in1) from[b + 32 + ln] = x1;
        }
        __syncthreads();
        uint32_t* to = from == s_a ? s_sorted : s_a;
        int lg = 6;
        for (uint32_t L = 64; L < nmax; L <<= 1, lg++) {
          // merge path: each thread writes MV consecutive outputs; it locates the
          // split of its first output in the run pair by a binary search along the
          // diagonal, then merges sequentially (again where a pair or segment ends)
          constexpr uint32_t MV = 8;
          for (uint32_t g0 = t * MV; g0 < cnt; g0 += HT * MV) {
            uint32_t cur = 0xFFFFFFFFu, la = 0, lb = 0, ai = 0, bi = 0, va = 0, vb = 0;
            const uint32_t* A = from;
            const uint32_t* B = from;
#pragma unroll
            for (uint32_t u = 0; u < MV; u++) {
              const uint32_t q = g0 + u;
              if (q >= cnt) break;
              const int cq = s_cell[q];
              const uint32_t b = c_st[cq] - S, n = c_N[cq];
              const uint32_t off = ((q - b) >> (lg + 1)) << (lg + 1);   // pair start in the segment
              if (b + off != cur) {
                cur = b + off;
                la = min(n - off, L);
                lb = n - off > L ? min(n - off - L, L) : 0u;
                A = from + cur;
                B = A + L;
                const uint32_t diag = q - cur;
                uint32_t lo = diag > lb ? diag - lb : 0u, hi = min(diag, la);
                while (lo < hi) {
                  const uint32_t mid = (lo + hi) >> 1;
                  if (A[mid] < B[diag - 1 - mid]) lo = mid + 1; else hi = mid;
                }
                ai = lo;
                bi = diag - lo;
                va = ai < la ? A[ai] : 0xFFFFFFFFu;
                vb = bi < lb ? B[bi] : 0xFFFFFFFFu;
              }
              if (va < vb) {
                to[q] = va;
                ai++;
                va = ai < la ? A[ai] : 0xFFFFFFFFu;
              } else {
                to[q] = vb;
                bi++;
                vb = bi < lb ? B[bi] : 0xFFFFFFFFu;
              }
            }
          }
          __syncthreads();
          uint32_t* tmp = from; from = to; to = tmp;
        }
      }
      // ---- D: gather velocities by cp.async (they land while E0/E1 draw; the claim
      // rounds wait for them), move positions on reorder steps
      for (uint32_t q = t; q < cnt; q += HT) {
        const int cq = s_cell[q];
        const float* src = P.P + (int64_t)c_h[cq] * P.half + s_sorted[q];
        cp_async4(s_vx + q, src + 3 * RS);
        cp_async4(s_vy + q, src + 4 * RS);
        cp_async4(s_vz + q, src + 5 * RS);
        s_mod[q] = 0;
        s_min[q] = 0xFFFFFFFFu;
      }
      cp_async_commit();
      if (mode == 0) {
        for (uint32_t q0 = t; q0 < cnt; q0 += 4 * HT) {
          float xs[4][D];
          int cqs[4];
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const uint32_t q = q0 + u * HT;
            cqs[u] = q < cnt ? s_cell[q] : 0;
            if (q < cnt && c_reo[cqs[u]]) {
              const float* src = P.P + (int64_t)c_h[cqs[u]] * P.half + s_sorted[q];
#pragma unroll
              for (int a = 0; a < D; a++) xs[u][a] = src[a * RS];
            }
          }
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const uint32_t q = q0 + u * HT;
            if (q < cnt && c_reo[cqs[u]]) {
              const int cq = cqs[u], hq = c_h[cq];
              float* d = P.P + (int64_t)(hq ^ 1) * P.half + (int64_t)c_r[cq] * P.stride + (int64_t)(S + q - c_base[cq]);
#pragma unroll
              for (int a = 0; a < D; a++) d[a * RS] = xs[u][a];
            }
          }
        }
      }
      __syncthreads();
      // ---- E: NTC
      if (mode == 0) {
        uint32_t M = 0;
        if (valid) M = ntc_count(P, run_key(P, r), c, (uint32_t)s, N, gm);
        ncand = M;
        if (t < 32) {
          uint32_t x = M;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(FULL, x, o); if (t >= o) x += y; }
          c_mst[t] = x - M;
          c_M[t] = M;
          if (t == 31) c_mst[32] = x;
        }
        __syncthreads();
        const uint32_t tot = c_mst[32];
        const double gmd = (double)gm;
        if (t < 32) { c_mg2[t] = 0.0f; c_nacc[t] = 0; }
        uint32_t rnd = 0;                          // claim rounds so far in this tile
        for (uint32_t base = 0; base < tot; base += CCH) {
          const uint32_t lim = tot - base < (uint32_t)CCH ? tot - base : (uint32_t)CCH;
          // candidates drawn flattened: owner cell, tile-local particle slots, HS
          // threshold (as in k_collide's E1) and Marsaglia pair
          for (uint32_t q = t; q < lim; q += HT) {
            const uint32_t gq = base + q;
            int lo = 0;
#pragma unroll
            for (int stp = 16; stp > 0; stp >>= 1)
              if (lo + stp < 32 && c_mst[lo + stp] <= gq) lo += stp;
            const uint32_t nc = c_N[lo], kq = gq - c_mst[lo], o = c_st[lo] - S;
            const uint2 keyc = run_key(P, c_r[lo]);
            const uint4 w = draw(keyc, c_c[lo], (uint32_t)s, TAG_COLL_PAIR, kq, 0);
            uint32_t i, j;
            pair_of(w.x, nc, i, j);
            s_cij[q] = (o + i) | ((o + j) << 16);
            s_clo[q] = (uint8_t)lo;
            if (P.model == 0) {
              const double lhs = u_co_d(w.y) * c_gh[lo];
              s_cur[q] = __float_as_uint(__double2float_rd(lhs * lhs));
            } else {
              s_cur[q] = w.y;
            }
            float pp = 2.0f * u_co(w.z) - 1.0f, qv = 2.0f * u_co(w.w) - 1.0f;
            if (!(pp * pp + qv * qv < 1.0f)) marsaglia_pq_from(keyc, c_c[lo], (uint32_t)s, kq, 0, pp, qv);
            s_cp[q] = pp;
            s_cq[q] = qv;
          }
          if (base == 0) cp_async_wait_all();       // the velocity gathers of D
          __syncthreads();
          // dependency rounds: an undone candidate claims both its particles
          // (atomicMin of its index) and runs once it is the earliest undone
          // candidate on both.  Candidates that run together touch disjoint
          // particles, and every candidate runs after all earlier ones of its cell
          // that share a particle: the result is that of walking each cell's
          // candidates in increasing k.  (Replaces dependency waves assigned by a
          // thread per cell, whose serial loop the whole block waited for.)
          // A claim is (0xFFFF - round) << 16 | q: a later round's claims beat any
          // left from earlier rounds, so claims need no release pass.
          // each thread owns candidates t + u HT; which are undone is a register mask
          constexpr int OWN = CCH / HT;
          uint32_t undone = 0;
#pragma unroll
          for (int u = 0; u < OWN; u++) if (t + u * HT < lim) undone |= 1u << u;
          for (;;) {
            const uint32_t rtag = (0xFFFFu - rnd) << 16;
            rnd++;
#pragma unroll
            for (int u = 0; u < OWN; u++)
              if (undone >> u & 1u) {
                const uint32_t q = t + u * HT, pr = s_cij[q];
                atomicMin(&s_min[pr & 0xFFFFu], rtag | q);
                atomicMin(&s_min[pr >> 16], rtag | q);
              }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < OWN; u++) {
              if (!(undone >> u & 1u)) continue;
              const uint32_t q = t + u * HT, pr = s_cij[q];
              const uint32_t i = pr & 0xFFFFu, j = pr >> 16;
              if (s_min[i] != (rtag | q) || s_min[j] != (rtag | q)) continue;
              undone &= ~(1u << u);
              const int lo = s_clo[q];
              const float ax = s_vx[i], ay = s_vy[i], az = s_vz[i];
              const float bx = s_vx[j], by = s_vy[j], bz = s_vz[j];
              const float dx = ax - bx, dy = ay - by, dz = az - bz;
              const float g2 = (dx * dx + dy * dy) + dz * dz;
              atomicMax(reinterpret_cast<uint32_t*>(&c_mg2[lo]), __float_as_uint(g2));  // g^2 >= 0: int order
              const bool accept = P.model == 0 ? g2 > __uint_as_float(s_cur[q])
                                               : vhs_accept(P, s_cur[q], (double)c_gm[lo], g2);
              if (accept) {
                const float pp = s_cp[q], qq = s_cq[q];
                const float rho = pp * pp + qq * qq;
                const float sr = sqrtf(1.0f - rho);
                const float ex = 2.0f * pp * sr, ey = 2.0f * qq * sr, ez = 1.0f - 2.0f * rho;
                const float cmx = (ax + bx) * 0.5f, cmy = (ay + by) * 0.5f, cmz = (az + bz) * 0.5f;
                const float hh = 0.5f * sqrtf(g2);
                s_vx[i] = cmx + hh * ex; s_vy[i] = cmy + hh * ey; s_vz[i] = cmz + hh * ez;
                s_vx[j] = cmx - hh * ex; s_vy[j] = cmy - hh * ey; s_vz[j] = cmz - hh * ez;
                s_mod[i] = 1;
                s_mod[j] = 1;
                atomicAdd(&c_nacc[lo], 1u);
              }
            }
            int more = undone != 0u;
            more = __syncthreads_or(more);
            if (rnd > 0xFFF0u) {                       // round tags nearly exhausted: reset the claims
              for (uint32_t q = t; q < cnt; q += HT) s_min[q] = 0xFFFFFFFFu;
              rnd = 0;
              __syncthreads();
            }
            if (!more) break;
          }
        }
        if (valid && M) {
          nacc = c_nacc[t];
          const float maxg2 = c_mg2[t];
          const double sgm = P.model == 0 ? P.sigma_c * sqrt((double)maxg2) : P.sigma_c * pow((double)maxg2, P.omega1);
          if (sgm > gmd) gm = (float)sgm;
        }
      }
      cp_async_wait_all();                          // no candidates (or no Interaction): gathers of D
      __syncthreads();
      if (valid && slot >= 0) {
        const uint32_t off = c_st[t] - S;
        sample_cell(P, slot, k0 + t, N, SmemCell{s_vx + off, s_vy + off, s_vz + off, s_mod + off}, mode == 2);
      }
      __syncthreads();
      // ---- F: write back
      for (uint32_t q = t; q < cnt; q += HT) {
        const int cq = s_cell[q];
        const int hq = c_h[cq];
        if (c_reo[cq]) {
          float* d = P.P + (int64_t)(hq ^ 1) * P.half + (int64_t)c_r[cq] * P.stride + (int64_t)(S + q - c_base[cq]);
          d[3 * RS] = s_vx[q];
          d[4 * RS] = s_vy[q];
          d[5 * RS] = s_vz[q];
        } else if (s_mod[q]) {
          float* d = P.P + (int64_t)hq * P.half + s_sorted[q];
          d[3 * RS] = s_vx[q];
          d[4 * RS] = s_vy[q];
          d[5 * RS] = s_vz[q];
        }
        if (P.debug) P.lcr[S + q] = s_sorted[q];
      }
    } else if (valid) {
      // beyond even the heavy staging area: thread per cell in global memory
      const uint32_t st = c_st[t];
      uint32_t* seg = P.lcr + st;
      if (N <= 32) insertion_sort(seg, N);
      else heap_sort(seg, N);
      GlobCell A{seg, parr(P, h, 3), parr(P, h, 4), parr(P, h, 5)};
      if (mode == 0) collide_cell(P, run_key(P, r), c, (uint32_t)s, N, A, gm, ncand, nacc);
      if (slot >= 0) sample_cell(P, slot, k0 + t, N, A, mode == 2);
      if (reo) {
        const uint32_t rb = c_base[t];
        for (uint32_t i = 0; i < N; i++) {
          const uint32_t g = seg[i];
          const int64_t dst = (int64_t)r * P.stride + (int64_t)(st + i - rb);
#pragma unroll
          for (int a = 0; a < D; a++) parr(P, h ^ 1, a)[dst] = parr(P, h, a)[g];
#pragma unroll
          for (int a = 3; a < 6; a++) parr(P, h ^ 1, a)[dst] = parr(P, h, a)[g];
        }
      }
    }
    if (valid) {
      const int64_t k = k0 + t;
      if (gm != gm0) P.gmax[k] = gm;
      if (P.debug && mode == 0) { P.dbg_cand[k] = ncand; P.dbg_acc[k] = (int32_t)nacc; }
      if (mode == 0 && ncand) {
        atomicAdd(&P.ctl.counters[r * 4 + 2], (unsigned long long)ncand);
        atomicAdd(&P.ctl.counters[r * 4 + 3], (unsigned long long)nacc);
      }
    }
  }
}

// ============================================================== Ensemble
// pooled ratio estimates over runs, ascending run id, + jackknife (R18)
__device__ __forceinline__ void moments(double sn, double sx, double sy, double sz, double se, double fnum_vc,
                                        double nr, double o[5]) {
  o[0] = sn * fnum_vc / nr;
  if (sn > 0) {
    const double ux = sx / sn, uy = sy / sn, uz = sz / sn;
    o[1] = ux; o[2] = uy; o[3] = uz;
    o[4] = (se / sn - (ux * ux + uy * uy + uz * uz)) / 3.0;
  } else {
    o[1] = o[2] = o[3] = o[4] = __longlong_as_double(0x7ff8000000000000ll);
  }
}

// S: n_blocks blocks of [5][R*Nc] (block b = the slot sums of the context holding
// runs b*R .. b*R + R - 1 of the job, e.g. gathered from every rank); the fold over
// runs is in ascending global run id, so one block is the single-context case
__global__ void k_macros(Prm P, const double* __restrict__ S, int n_blocks, int m_i, double fnum_vc) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P.Nc) return;
  const int64_t RN = (int64_t)P.R * P.Nc;
  const int nr = n_blocks * P.R;
  auto at = [&](int q, int r) {   // sums of quantity q, global run r
    const int b = r / P.R, rl = r - b * P.R;
    return S[((int64_t)b * 5 + q) * RN + (int64_t)rl * P.Nc + c];
  };
  double tot[5] = {0, 0, 0, 0, 0};
  for (int r = 0; r < nr; r++)
    for (int q = 0; q < 5; q++) tot[q] += at(q, r);
  // samples per run in the slot: 1 for a snapshot, m for a time average
  const double m = m_i > 0 ? (double)m_i : 1.0;
  double full[5];
  moments(tot[0], tot[1], tot[2], tot[3], tot[4], fnum_vc, (double)nr * m, full);
  double* o = P.macros + c * 10;
  for (int q = 0; q < 5; q++) o[q] = full[q];
  if (nr < 2) { for (int q = 0; q < 5; q++) o[5 + q] = 0.0; return; }
  // two passes over runs: mean of leave-one-out estimates, then spread
  double mean[5] = {0, 0, 0, 0, 0};
  for (int r = 0; r < nr; r++) {
    double part[5], loo[5];
    for (int q = 0; q < 5; q++) part[q] = tot[q] - at(q, r);
    moments(part[0], part[1], part[2], part[3], part[4], fnum_vc, (double)(nr - 1) * m, loo);
    for (int q = 0; q < 5; q++) mean[q] += loo[q];
  }
  for (int q = 0; q < 5; q++) mean[q] /= (double)nr;
  double ss[5] = {0, 0, 0, 0, 0};
  for (int r = 0; r < nr; r++) {
    double part[5], loo[5];
    for (int q = 0; q < 5; q++) part[q] = tot[q] - at(q, r);
    moments(part[0], part[1], part[2], part[3], part[4], fnum_vc, (double)(nr - 1) * m, loo);
    for (int q = 0; q < 5; q++) { const double d = loo[q] - mean[q]; ss[q] += d * d; }
  }
  for (int q = 0; q < 5; q++) o[5 + q] = sqrt((double)(nr - 1) / (double)nr * ss[q]);
}

__global__ void k_selftest_philox(int64_t n, const uint32_t* ctr, uint2 key, uint32_t* out, uint32_t* out_ref) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4 c = make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]);
  const uint4 o = philox(c, key);
  out[4 * i] = o.x; out[4 * i + 1] = o.y; out[4 * i + 2] = o.z; out[4 * i + 3] = o.w;
  if (out_ref) {
    const uint4 q = curand_Philox4x32_10(c, key);
    out_ref[4 * i] = q.x; out_ref[4 * i + 1] = q.y; out_ref[4 * i + 2] = q.z; out_ref[4 * i + 3] = q.w;
  }
}

// ============================================================ host launchers
// per-device launch caches (function attributes and occupancy are per device):
// indexed by the current device ordinal
constexpr int MAX_DEV = 64;
static int cur_dev() {
  int d = 0;
  cudaGetDevice(&d);
  return d >= 0 && d < MAX_DEV ? d : 0;
}
static int g_num_sms[MAX_DEV] = {0};
static int num_sms() {
  const int dev = cur_dev();
  if (!g_num_sms[dev]) {
    cudaDeviceGetAttribute(&g_num_sms[dev], cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms[dev] <= 0) g_num_sms[dev] = 148;
  }
  return g_num_sms[dev];
}

static unsigned grid_cap(int64_t work, int threads, int64_t max_blocks) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (unsigned)b;
}

void launch_zero(uint32_t* a, int64_t n, cudaStream_t st) {
  k_zero<<<grid_cap(n / 4 + 1, 256, (int64_t)num_sms() * 8), 256, 0, st>>>(a, n);
}

void launch_fill_f32(float* a, int64_t n, float v, cudaStream_t st) {
  k_fill_f32<<<grid_cap(n, 256, (int64_t)num_sms() * 8), 256, 0, st>>>(a, n, v);
}

int64_t scan_tiles(int64_t L) { return (L + SCAN_TILE - 1) / SCAN_TILE; }

void launch_scan(uint32_t* a, int64_t L, uint32_t* part, cudaStream_t st, const LaunchHook& hook) {
  const int64_t nb = scan_tiles(L);
  hook.before(KSLOT_SCAN_REDUCE);
  k_scan_reduce<<<(unsigned)nb, SCAN_T, 0, st>>>(a, L, part);
  hook.after(KSLOT_SCAN_REDUCE);
  hook.before(KSLOT_SCAN_PARTIALS);
  k_scan_partials<<<1, 1024, 0, st>>>(part, nb);
  hook.after(KSLOT_SCAN_PARTIALS);
  hook.before(KSLOT_SCAN_DOWN);
  k_scan_down<<<(unsigned)nb, SCAN_T, 0, st>>>(a, L, part);
  hook.after(KSLOT_SCAN_DOWN);
}

void launch_fill(const Prm& P, cudaStream_t st) {
  k_fill_count<<<grid_cap(P.Nc, 256, 1 << 30), 256, 0, st>>>(P);
  launch_scan(P.cell, P.Nc, P.scan_part, st, LaunchHook{});
  dim3 g((unsigned)((P.Nc + 7) / 8), (unsigned)P.R);
  k_fill_emit<<<g, 256, 0, st>>>(P);
  k_fill_finish<<<grid_cap((P.R > P.n_slots ? P.R : P.n_slots), 128, 1 << 20), 128, 0, st>>>(P);
  launch_fill_f32(P.gmax, (int64_t)P.R * P.Nc, P.gmax0, st);
}

template <int D, bool EV>
static void motion_t(const Prm& P, int mode, cudaStream_t st) {
  static int occ_dev[MAX_DEV] = {0};
  int& occ = occ_dev[cur_dev()];
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_motion<D, EV>, 256, 0);
    if (occ < 1) occ = 1;
  }
  // persistent: one wave of resident blocks walks the (run-major) items, so
  // the cell counters being hit at any moment belong to one or two runs
  const int64_t items = (P.cap + ITEM_M - 1) / ITEM_M * P.R;
  int64_t g = (int64_t)num_sms() * occ;
  if (g > items) g = items;
  k_motion<D, EV><<<(unsigned)g, 256, 0, st>>>(P, mode);
}

void launch_motion(const Prm& P, int mode, cudaStream_t st) {
  const bool ev = P.has_events != 0;
  switch (P.dim * 2 + (ev ? 1 : 0)) {
    case 2: motion_t<1, false>(P, mode, st); break;
    case 3: motion_t<1, true>(P, mode, st); break;
    case 4: motion_t<2, false>(P, mode, st); break;
    case 5: motion_t<2, true>(P, mode, st); break;
    case 6: motion_t<3, false>(P, mode, st); break;
    default: motion_t<3, true>(P, mode, st); break;
  }
}

void launch_items(const Prm& P, cudaStream_t st, bool motion) {
  if (motion) k_items<ITEM_M><<<1, 1024, 0, st>>>(P);
  else k_items<ITEM_S><<<1, 1024, 0, st>>>(P);
}

void launch_scatter(const Prm& P, cudaStream_t st) {
  static int occ_dev[MAX_DEV] = {0};
  int& occ = occ_dev[cur_dev()];
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scatter, 256, 0);
    if (occ < 1) occ = 1;
  }
  const int64_t items = (P.cap + ITEM_S - 1) / ITEM_S * P.R;
  int64_t g = (int64_t)num_sms() * occ;
  if (g > items) g = items;
  k_scatter<<<(unsigned)g, 256, 0, st>>>(P);
}

void launch_inflow(const Prm& P, cudaStream_t st, const LaunchHook& hook) {
  if (P.inflow_kind == 0 || P.n_face == 0) return;
  dim3 g((unsigned)((P.n_face + 3) / 4), (unsigned)P.R);
  hook.before(KSLOT_INFLOW_COUNT);
  k_inflow_count<<<g, 128, 0, st>>>(P);
  hook.after(KSLOT_INFLOW_COUNT);
  hook.before(KSLOT_INFLOW_EMIT);
  k_inflow_emit<<<g, 128, 0, st>>>(P);
  hook.after(KSLOT_INFLOW_EMIT);
}

void launch_step_mid(const Prm& P, cudaStream_t st) {
  k_step_mid<<<(P.R + 127) / 128, 128, 0, st>>>(P);
}

template <int D, int NET, int MODEL, bool STEP, bool ONE>
static void collide_t(const Prm& P, int mode, int slot, int capw, cudaStream_t st) {
  const int64_t RN = (int64_t)P.R * P.Nc;
  const int64_t warps = (RN + 31) / 32;
  const unsigned g = (unsigned)((warps + WPB - 1) / WPB);
  const size_t smem = WPB * warp_smem_bytes(capw, ONE);
  static size_t configured_dev[MAX_DEV] = {0};
  size_t& configured = configured_dev[cur_dev()];
  if (smem > configured) {
    cudaFuncSetAttribute(k_collide<D, NET, MODEL, STEP, ONE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (const char* e = getenv("DSMC_CARVEOUT"))   // A/B experiments: shared-memory carveout (percent)
      cudaFuncSetAttribute(k_collide<D, NET, MODEL, STEP, ONE>, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(e));
    configured = smem;
  }
  k_collide<D, NET, MODEL, STEP, ONE><<<g, WPB * 32, smem, st>>>(P, mode, slot, capw);
}

template <int D, int NET, int MODEL, bool ONE>
static void collide_list_t(const Prm& P, int capw, cudaStream_t st) {
  const size_t smem = warp_smem_bytes(capw, ONE);
  static size_t configured_dev[MAX_DEV] = {0};
  static int occ_dev[MAX_DEV] = {0};
  const int dev = cur_dev();
  if (smem > configured_dev[dev]) {
    cudaFuncSetAttribute(k_collide_list<D, NET, MODEL, ONE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured_dev[dev] = smem;
    occ_dev[dev] = 0;
  }
  int& occ = occ_dev[dev];
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_collide_list<D, NET, MODEL, ONE>, 32, smem);
    if (occ < 1) occ = 1;
  }
  const int64_t tiles = ((int64_t)P.R * P.Nc + 31) / 32;
  int64_t g = (int64_t)num_sms() * occ;
  if (g > tiles) g = tiles;
  k_collide_list<D, NET, MODEL, ONE><<<(unsigned)g, 32, smem, st>>>(P, capw);
}

template <int D, int NET>
static void collide_list_m(const Prm& P, cudaStream_t st) {
  const bool one = P.Nc % 32 == 0 || P.R == 1;
  if (P.model == DSMC_MODEL_HS) {
    if (one) collide_list_t<D, NET, DSMC_MODEL_HS, true>(P, P.capw, st);
    else collide_list_t<D, NET, DSMC_MODEL_HS, false>(P, P.capw, st);
  } else {
    if (one) collide_list_t<D, NET, DSMC_MODEL_VHS, true>(P, P.capw, st);
    else collide_list_t<D, NET, DSMC_MODEL_VHS, false>(P, P.capw, st);
  }
}

// sparse problems: the tiles with work listed by k_collide_triage, then collided
// by persistent k_collide_list blocks (mode 0 only)
void launch_collide_heavy(const Prm& P, int mode, int slot, cudaStream_t st);

static void launch_collide_compact(const Prm& P, cudaStream_t st, const LaunchHook& hook, const Branch& br) {
  const int64_t tiles = ((int64_t)P.R * P.Nc + 31) / 32;
  const bool one = P.Nc % 32 == 0 || P.R == 1;
  const int64_t per_block = TRIAGE_T / 32 * TRIAGE_TPW;
  const unsigned g = (unsigned)((tiles + per_block - 1) / per_block);
  hook.before(KSLOT_COLLIDE_TRIAGE);
  if (one) k_collide_triage<true><<<g, TRIAGE_T, 0, st>>>(P, P.capw);
  else k_collide_triage<false><<<g, TRIAGE_T, 0, st>>>(P, P.capw);
  hook.after(KSLOT_COLLIDE_TRIAGE);
  // the triage queued the heavy tiles: with a second branch they run beside the
  // warp-tile list (the tiers' persistent blocks fill SMs the list's tail leaves idle)
  if (br.st) {
    cudaEventRecord(br.fork, st);
    cudaStreamWaitEvent(br.st, br.fork, 0);
    launch_collide_heavy(P, 0, -1, br.st);
    cudaEventRecord(br.join, br.st);
  }
  hook.before(KSLOT_COLLIDE);
  const bool wide = P.net_wide != 0;
  if (P.dim == 1) {
    if (wide) collide_list_m<1, 32>(P, st); else collide_list_m<1, 16>(P, st);
  } else if (P.dim == 2) {
    if (wide) collide_list_m<2, 32>(P, st); else collide_list_m<2, 16>(P, st);
  } else {
    if (wide) collide_list_m<3, 32>(P, st); else collide_list_m<3, 16>(P, st);
  }
  hook.after(KSLOT_COLLIDE);
}

template <int D, int NET>
static void collide_m(const Prm& P, int mode, int slot, int capw, cudaStream_t st) {
  if (mode == 0) {
    const bool one = P.Nc % 32 == 0 || P.R == 1;    // no tile spans two runs
    if (P.model == DSMC_MODEL_HS) {
      if (one) collide_t<D, NET, DSMC_MODEL_HS, true, true>(P, mode, slot, capw, st);
      else collide_t<D, NET, DSMC_MODEL_HS, true, false>(P, mode, slot, capw, st);
    } else {
      if (one) collide_t<D, NET, DSMC_MODEL_VHS, true, true>(P, mode, slot, capw, st);
      else collide_t<D, NET, DSMC_MODEL_VHS, true, false>(P, mode, slot, capw, st);
    }
  } else {   // explicit Sampling: no Interaction, so the model is irrelevant
    collide_t<D, NET, DSMC_MODEL_HS, false, false>(P, mode, slot, capw, st);
  }
}

void launch_collide(const Prm& P, int mode, int slot, cudaStream_t st) {
  // register sorting network width for segments beyond 32: 16 (sparse) or 32 (dense fills)
  const bool wide = P.net_wide != 0;
  const int capw = P.capw;
  if (P.dim == 1) {
    if (wide) collide_m<1, 32>(P, mode, slot, capw, st); else collide_m<1, 16>(P, mode, slot, capw, st);
  } else if (P.dim == 2) {
    if (wide) collide_m<2, 32>(P, mode, slot, capw, st); else collide_m<2, 16>(P, mode, slot, capw, st);
  } else {
    if (wide) collide_m<3, 32>(P, mode, slot, capw, st); else collide_m<3, 16>(P, mode, slot, capw, st);
  }
}

template <int D, int HT>
static void heavy_t(const Prm& P, int mode, int slot, int caph, int queue, cudaStream_t st) {
  const size_t smem = heavy_smem_bytes(caph);
  static bool configured_dev[MAX_DEV] = {false};
  static int occ_dev[MAX_DEV] = {0};
  const int dev = cur_dev();
  bool& configured = configured_dev[dev];
  int& occ = occ_dev[dev];
  if (!configured) {
    cudaFuncSetAttribute(k_collide_heavy<D, HT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)heavy_smem_bytes(8192));
    configured = true;
  }
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_collide_heavy<D, HT>, HT, smem);
    if (occ < 1) occ = 1;
  }
  k_collide_heavy<D, HT><<<num_sms() * occ, HT, smem, st>>>(P, mode, slot, caph, queue);
}

template <int D>
static void heavy_q(const Prm& P, int mode, int slot, int q, cudaStream_t st) {
  // the large tier has one block per SM (shared memory): 512 threads hide more latency
  if (q == 0) heavy_t<D, 256>(P, mode, slot, P.caph_tier[q], q, st);
  else heavy_t<D, 512>(P, mode, slot, P.caph_tier[q], q, st);
}

// the heap of TLPDPR in HEAVY_TIERS sizes: each tier's persistent blocks stage
// up to caph_tier[q] particles, so the tiers of small heavy tiles run several
// blocks per SM; tiles beyond the last tier take its global-memory path
void launch_collide_heavy(const Prm& P, int mode, int slot, cudaStream_t st) {
  if (!P.heavy_list) return;
  // the large tier first: beside the warp-tile list (second graph branch) its one block per
  // SM leaves the list room, and the small tier's finer blocks make the shorter tail
  // (c5 after 500 steps: 1.858 -> 1.822 ms per step; c2 0.307 -> 0.311); a graph branch per
  // tier changed nothing (c5 1.857 -> 1.865): the tiers' 96-193 KB blocks cannot share an SM
  for (int q = HEAVY_TIERS - 1; q >= 0; q--) {
    if (P.dim == 1) heavy_q<1>(P, mode, slot, q, st);
    else if (P.dim == 2) heavy_q<2>(P, mode, slot, q, st);
    else heavy_q<3>(P, mode, slot, q, st);
  }
}

void launch_step_end(const Prm& P, int mode, int slot, cudaStream_t st) {
  k_step_end<<<(P.R + 127) / 128, 128, 0, st>>>(P, mode, slot);
}

void launch_macros(const Prm& P, const double* sums, int n_blocks, int m, double fnum_vc, cudaStream_t st) {
  k_macros<<<(unsigned)((P.Nc + 127) / 128), 128, 0, st>>>(P, sums, n_blocks, m, fnum_vc);
}

void launch_selftest_philox(int64_t n, const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out,
                            uint32_t* out_ref, cudaStream_t st) {
  k_selftest_philox<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(n, ctr, make_uint2(k0, k1), out, out_ref);
}

// one full step: kernel order of PAPER.md Fig. 1
void issue_step(const Prm& P, cudaStream_t st, const LaunchHook& hook, const Branch& br_in) {
  const Branch br = (P.compact && !hook.fn && !std::getenv("DSMC_NO_BRANCH")) ? br_in : Branch{};
  hook.before(KSLOT_ZERO);
  launch_zero(P.cell, (int64_t)P.R * P.Nc, st);
  hook.after(KSLOT_ZERO);
  launch_inflow(P, st, hook);
  launch_items(P, st, true);
  hook.before(KSLOT_MOTION);
  launch_motion(P, 0, st);
  hook.after(KSLOT_MOTION);
  hook.before(KSLOT_STEP_MID);
  launch_step_mid(P, st);
  hook.after(KSLOT_STEP_MID);
  launch_scan(P.cell, (int64_t)P.R * P.Nc, P.scan_part, st, hook);
  launch_items(P, st, false);
  hook.before(KSLOT_SCATTER);
  launch_scatter(P, st);
  hook.after(KSLOT_SCATTER);
  if (P.compact) {
    launch_collide_compact(P, st, hook, br);
  } else {
    hook.before(KSLOT_COLLIDE);
    launch_collide(P, 0, -1, st);
    hook.after(KSLOT_COLLIDE);
  }
  if (br.st) {
    cudaStreamWaitEvent(st, br.join, 0);
  } else {
    hook.before(KSLOT_COLLIDE_HEAVY);
    launch_collide_heavy(P, 0, -1, st);
    hook.after(KSLOT_COLLIDE_HEAVY);
  }
  hook.before(KSLOT_STEP_END);
  launch_step_end(P, 0, 0, st);
  hook.after(KSLOT_STEP_END);
}

void issue_sample(const Prm& P, int slot, int add, cudaStream_t st) {
  launch_zero(P.cell, (int64_t)P.R * P.Nc, st);
  launch_zero(P.ctl.maxn, P.R, st);             // max_ppc of this Indexing
  launch_items(P, st, true);
  launch_motion(P, 1, st);
  launch_scan(P.cell, (int64_t)P.R * P.Nc, P.scan_part, st, LaunchHook{});
  launch_items(P, st, false);
  launch_scatter(P, st);
  launch_collide(P, add ? 2 : 1, slot, st);
  launch_collide_heavy(P, add ? 2 : 1, slot, st);
  launch_step_end(P, add ? 2 : 1, slot, st);
}

const char* kernel_slot_name(int k) {
  switch (k) {
    case KSLOT_ZERO: return "k_zero";
    case KSLOT_INFLOW_COUNT: return "k_inflow_count";
    case KSLOT_INFLOW_EMIT: return "k_inflow_emit";
    case KSLOT_MOTION: return "k_motion";
    case KSLOT_STEP_MID: return "k_step_mid";
    case KSLOT_SCAN_REDUCE: return "k_scan_reduce";
    case KSLOT_SCAN_PARTIALS: return "k_scan_partials";
    case KSLOT_SCAN_DOWN: return "k_scan_down";
    case KSLOT_SCATTER: return "k_scatter";
    case KSLOT_COLLIDE: return "k_collide";
    case KSLOT_COLLIDE_HEAVY: return "k_collide_heavy";
    case KSLOT_COLLIDE_TRIAGE: return "k_collide_triage";
    case KSLOT_STEP_END: return "k_step_end";
    default: return "";
  }
}

}  // namespace dsmc
