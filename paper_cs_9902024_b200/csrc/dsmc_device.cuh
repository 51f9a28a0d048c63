// dsmc_device.cuh -- device-side parameter block and arithmetic primitives of
// the B200 DSMC path.  Independent of the oracle (oracle/ is test-only and is
// neither included nor linked here).
//
// Every rounding-sensitive expression is written in the order DESIGN.md
// readings R1-R18 fix; the library is compiled with -fmad=false so that no
// a*b+c is contracted behind our back, and fmaf() appears only where the
// reading says "fma".
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dsmc {

constexpr uint32_t TAG_FILL = 1, TAG_INFLOW_COUNT = 2, TAG_INFLOW_PARTICLE = 3, TAG_WALL = 4,
                   TAG_COLL_COUNT = 5, TAG_COLL_PAIR = 6, TAG_COLL_DIR = 7;
constexpr uint32_t FILL_STEP = 0xFFFFFFFFu;
constexpr uint32_t DEAD_KEY = 0xFFFFFFFFu;
constexpr float DEAD_X = -1.0e30f;           // x of a removed, not yet compacted slot
constexpr int MAX_BOUNCE = 8;
constexpr int HEAVY_TIERS = 2;               // heavy-tile queues by size (k_collide_heavy; k_collide picks 0/1)
constexpr uint32_t HEAVY_SLACK = 3;          // words before the LCR slice in k_collide_heavy's staging (bulk-copy alignment)
constexpr double TWO_PI = 6.283185307179586;

enum { BC_SPECULAR = 0, BC_PERIODIC = 1, BC_DIFFUSE = 2, BC_OUTFLOW = 3, BC_INFLOW = 4 };
enum { ST_OK = 0, ST_CAP = -4, ST_INDEX = -5, ST_NONFINITE = -6, ST_BOUNCE = -9, ST_CELL = -10 };

// control block (device memory, in the caller-owned ctl buffer)
struct Ctl {
  int32_t* step;             // [1] current step index s
  int32_t* status;           // [1] first latched fault
  int64_t* n_store;          // [R] store length (live + removed-not-compacted)
  int32_t* parity;           // [R] which half of P holds run r
  int32_t* reorder;          // [R] reorder run r at the end of this step
  int32_t* inserted;         // [R] particles generated this step
  unsigned long long* counters;  // [R][4] inserted, removed, candidates, accepted
  int64_t* live;             // [R] live particles (after the last Indexing)
  unsigned long long* psteps;    // [R] sum over steps of live particles after Generation
  int32_t* slot_done;        // [n_slots]
  int32_t* step_slot;        // [1] sample slot of the current step (R2), or -1 -- set by k_step_mid
  uint32_t* maxn;            // [R] largest particle count of one cell at the step's Indexing
  unsigned long long* queue; // [4][2] work-queue cursors (item, blocks done) per persistent kernel
  int64_t* items;            // [R+2] work items of the particle kernels: prefix over runs, total, items per
                             //       run if all runs hold as many (else 0) -- k_items
  uint32_t* heavy;           // [2*HEAVY_TIERS] heavy-tile queues: count, next per size tier
  uint32_t* tiles;           // [2] k_collide_triage's list of tiles with work: count, (spare)
};

struct Prm {
  // grid / batch
  int32_t dim, nx, ny, nz;
  int64_t Nc;                // cells per run
  uint32_t nc_mul;           // key / Nc = __umulhi(key, nc_mul) >> nc_shift for keys < 2^31 (nc_mul = 0: Nc = 1)
  int32_t nc_shift;
  int32_t R;                 // runs in the batch
  int64_t stride;            // slots per run window
  int64_t cap;               // capacity per run
  int64_t half;              // floats per half of P (6 * R * stride)
  uint32_t seed, run_id0;
  // clock
  float dt_f;
  int32_t sample_every, n_slots, reorder_every;
  int64_t insert_bound;
  // collisions
  int32_t model;
  double coef;               // F_N/V_c * dt
  double sigma_c;            // sigma g = sigma_c (g^2)^(1-omega)
  double omega1;             // 1 - omega
  float gmax0;               // initial (sigma g)_max
  // boundaries
  int32_t bc[6];
  double sqrt_bcT[6];
  int32_t has_events;        // any DIFFUSE/OUTFLOW/INFLOW face or plate
  int32_t plate_on, plate_axis, plate_span_axis;
  float plate_pos, plate_lo, plate_hi;
  double sqrt_plateT;
  int32_t orifice_on;
  const uint8_t* open_face;  // [ny*nz]
  // inflow
  int32_t inflow_kind, n_face, inflow_count;
  const int32_t* face_j;
  const int32_t* face_k;
  double ghost_x;            // n * w
  float ghost_w_f;
  double inflow_U, sqrt_inflowT;
  int32_t* face_kept;        // [R][n_face]
  // fill
  int32_t n_fill;
  int32_t fill_lo[4][3], fill_hi[4][3], fill_ppc[4];
  double fill_sqrtT[4], fill_u[4][3];
  // buffers
  float* P;                  // [2][6][R*stride]
  uint32_t* key;             // [R*stride]
  uint32_t* lcr;             // [R*stride]
  uint32_t* cell;            // [R*Nc]
  float* gmax;               // [R*Nc]
  double* C;                 // [n_slots][5][R*Nc]
  uint32_t* scan_part;       // scan tile partials
  double* macros;            // [Nc][10] staging
  int32_t debug;
  int32_t net_wide;          // k_collide sorts segments of <= 32 (else 16) in registers
  int32_t capw;              // particles a warp tile (32 cells) stages in shared memory
  int32_t caph;              // particles k_collide_heavy stages per tile
  uint32_t* heavy_list;      // [HEAVY_TIERS][heavy_stride] tiles k_collide handed to k_collide_heavy, by size tier
  int32_t heavy_static;      // NEXT-1 A/B arm: one tier, tiles dealt to blocks round-robin (no queue)
  int64_t heavy_stride;      // entries per tier list (R*Nc/32 + 1)
  int32_t caph_tier[HEAVY_TIERS];   // staging capacity of each tier (the last one is caph)
  int32_t compact;           // sparse problem: k_collide_triage lists the tiles with work for k_collide_list
  uint32_t* tile_list;       // [R*Nc/32 + 1] that list
  int64_t* dbg_cand;         // [R*Nc]
  int32_t* dbg_acc;          // [R*Nc]
  Ctl ctl;
};

// ------------------------------------------------------------------ Philox
// Philox4x32-10 (Salmon et al., SC'11): 10 rounds, multipliers 0xD2511F53 /
// 0xCD9E8D57, Weyl increments 0x9E3779B9 / 0xBB67AE85.
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ uint4 draw(uint2 key, uint32_t unit, uint32_t step, uint32_t tag, uint32_t sub,
                                      uint32_t block) {
  return philox(make_uint4(unit, step, (tag << 24) | (sub & 0xFFFFFFu), block), key);
}

// run of a (run, cell) key k < 2^31 (R*Nc < 2^31 is checked at create): k / Nc by a
// multiply-shift (host-computed magic, exact for 31-bit dividends)
__device__ __forceinline__ uint32_t run_of(const Prm& P, uint32_t k) {
  return P.nc_mul ? __umulhi(k, P.nc_mul) >> P.nc_shift : k;
}

__device__ __forceinline__ uint2 run_key(const Prm& P, int r) { return make_uint2(P.seed, P.run_id0 + (uint32_t)r); }

__device__ __forceinline__ float u_co(uint32_t w) { return (float)(w >> 8) * (1.0f / 16777216.0f); }
__device__ __forceinline__ double u_co_d(uint32_t w) { return (double)(w >> 8) * (1.0 / 16777216.0); }
__device__ __forceinline__ double u_oc_d(uint32_t w) { return (double)((w >> 8) + 1u) * (1.0 / 16777216.0); }
__device__ __forceinline__ uint32_t lemire(uint32_t w, uint32_t N) {
  return (uint32_t)(((uint64_t)w * (uint64_t)N) >> 32);
}

// Box-Muller in fp64: radius from w0 (u in (0,1]), angle from w1 (u in [0,1))
__device__ __forceinline__ void box_muller(uint32_t w0, uint32_t w1, double& n1, double& n2) {
  const double r = sqrt(-2.0 * log(u_oc_d(w0)));
  const double th = TWO_PI * u_co_d(w1);
  double s, c;
  sincos(th, &s, &c);
  n1 = r * c;
  n2 = r * s;
}

// uniform coordinate inside cell i (reading R7: pulled below the upper face)
__device__ __forceinline__ float place(int32_t i, uint32_t w) {
  float x = (float)i + u_co(w);
  const float top = (float)(i + 1);
  if (x >= top) x = nextafterf(top, 0.0f);
  return x;
}

__device__ __forceinline__ int32_t axis_n(const Prm& P, int a) { return a == 0 ? P.nx : (a == 1 ? P.ny : P.nz); }

// Fault latch (reading R24): the control word keeps the most severe fault seen,
// ENONFINITE > EINDEX > ECELL > EBOUNCE > ECAP, whatever the order in which
// threads report them -- atomicMax over rank << 8 | -code; the host decodes it
// with status_code().
__host__ __device__ __forceinline__ uint32_t fault_word(int32_t code) {
  const uint32_t rank = code == ST_NONFINITE ? 5u : code == ST_INDEX ? 4u : code == ST_CELL ? 3u
                      : code == ST_BOUNCE ? 2u : code == ST_CAP ? 1u : 0u;
  return rank ? (rank << 8) | (uint32_t)(-code) : 0u;
}
__host__ __device__ __forceinline__ int32_t status_code(uint32_t word) { return -(int32_t)(word & 0xFFu); }
__device__ __forceinline__ void latch(const Prm& P, int32_t code) {
  atomicMax(reinterpret_cast<unsigned int*>(P.ctl.status), fault_word(code));
}

// P array a (0..5 = x,y,z,vx,vy,vz) of half h
__device__ __forceinline__ float* parr(const Prm& P, int h, int a) {
  return P.P + (int64_t)h * P.half + (int64_t)a * P.R * P.stride;
}

}  // namespace dsmc
