// dsmc_api.cu -- the extern "C" boundary of libdsmc.so (declared in
// include/dsmc.h).  Host logic only: validation, buffer layout, the step
// graph, host<->device marshalling.  Every step of the method runs in the
// kernels of dsmc_kernels.cu; there is no CPU fallback.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "dsmc.h"

// mean fill density (particles per cell) below which the step lists the collide tiles
// with work first (k_collide_triage); DSMC_COMPACT=0/1 overrides it
#ifndef DSMC_COMPACT_PPC
#define DSMC_COMPACT_PPC 4.0
#endif
#include "dsmc_device.cuh"
#include "dsmc_kernels.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return DSMC_ECUDA;
}

#define CK(call)                                         \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// NVTX range over one ABI call (host timeline of nsys / ncu --nvtx; no-ops without a tool)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

struct Layout {
  dsmc_sizes sz;
  int64_t Nc, stride, RN;
  int32_t n_face;
  // ctl offsets
  size_t c_maxn, c_stepslot, c_step, c_status, c_nstore, c_parity, c_reorder, c_inserted, c_counters, c_live, c_psteps, c_slot, c_queue, c_heavy,
      c_items, c_tiles;
  // scratch offsets
  size_t s_face_j, s_face_k, s_open, s_kept, s_part, s_macros, s_heavy, s_tiles, s_cand, s_acc;
};

// face-cell lists of the x- face (reading R8)
void face_lists(const dsmc_problem* p, std::vector<int32_t>& fj, std::vector<int32_t>& fk,
                std::vector<uint8_t>& open) {
  open.assign((size_t)p->ny * p->nz, 0);
  fj.clear();
  fk.clear();
  for (int32_t k = 0; k < p->nz; k++)
    for (int32_t j = 0; j < p->ny; j++) {
      bool is_open = false;
      if (p->orifice_on) {
        const double dy = j + 0.5 - p->orifice_cy, dz = k + 0.5 - p->orifice_cz;
        is_open = dy * dy + dz * dz <= p->orifice_r * p->orifice_r;
        open[(size_t)k * p->ny + j] = is_open ? 1 : 0;
      }
      const bool face = p->inflow_kind == DSMC_INFLOW_GHOST || (p->inflow_kind == DSMC_INFLOW_EFFUSIVE && is_open);
      if (face) { fj.push_back(j); fk.push_back(k); }
    }
}

int validate(const dsmc_problem* p) {
  if (!p) return fail(DSMC_EINVAL, "null problem");
  if (p->dim < 1 || p->dim > 3 || p->nx < 1 || p->ny < 1 || p->nz < 1) return fail(DSMC_EINVAL, "bad grid");
  if ((p->dim < 2 && p->ny != 1) || (p->dim < 3 && p->nz != 1)) return fail(DSMC_EINVAL, "unused axes must have 1 cell");
  if (p->n_runs < 1 || p->cap_per_run < 1 || p->n_fill < 0 || p->n_fill > 4) return fail(DSMC_EINVAL, "bad batch/fill");
  // the run index is gridDim.y of the fill and inflow kernels
  if (p->n_runs > 65535) return fail(DSMC_EINVAL, "n_runs > 65535 (grid y limit of the generation kernels)");
  if (!(p->dt > 0) || !(p->dt_s >= p->dt) || !(p->dt_L >= p->dt_s)) return fail(DSMC_ECLOCK, "need 0 < dt <= dt_s <= dt_L");
  const double ks = p->dt_s / p->dt, kl = p->dt_L / p->dt_s;
  if (std::fabs(ks - std::floor(ks + 0.5)) > 1e-9 * ks || std::fabs(kl - std::floor(kl + 0.5)) > 1e-9 * kl)
    return fail(DSMC_ECLOCK, "dt_s must be a multiple of dt and dt_L of dt_s");
  if (p->model != DSMC_HS && p->model != DSMC_VHS) return fail(DSMC_EPARAM, "unknown model");
  if (p->model == DSMC_VHS && !(p->omega >= 0.5 && p->omega <= 1.0)) return fail(DSMC_EPARAM, "omega outside [0.5,1]");
  if (!(p->d_ref > 0) || !(p->mass > 0) || !(p->T_ref > 0) || !(p->fnum_vc >= 0)) return fail(DSMC_EPARAM, "bad gas");
  bool has_diffuse = p->plate_on != 0;
  for (int f = 0; f < 2 * p->dim; f++) {
    if (p->bc[f] < 0 || p->bc[f] > 4) return fail(DSMC_EPARAM, "unknown boundary kind");
    if (p->bc[f] == DSMC_DIFFUSE) {
      has_diffuse = true;
      if (!(p->bc_T[f] > 0)) return fail(DSMC_EPARAM, "wall temperature <= 0");
    }
  }
  for (int a = 0; a < p->dim; a++) {
    const int lo = p->bc[2 * a], hi = p->bc[2 * a + 1];
    if ((lo == DSMC_PERIODIC) != (hi == DSMC_PERIODIC)) return fail(DSMC_EPARAM, "periodic needs both faces");
    if ((lo == DSMC_INFLOW && a != 0) || hi == DSMC_INFLOW) return fail(DSMC_EPARAM, "inflow only on x-");
    if ((lo == DSMC_SPECULAR || hi == DSMC_SPECULAR) && has_diffuse)
      return fail(DSMC_EPARAM, "specular faces cannot be combined with diffuse surfaces");
  }
  if (p->plate_on && (p->dim != 2 || !(p->plate_T > 0) || p->plate_axis == p->plate_span_axis ||
                      p->plate_axis < 0 || p->plate_axis > 1 || p->plate_span_axis < 0 || p->plate_span_axis > 1))
    return fail(DSMC_EPARAM, "bad plate");
  if (p->orifice_on && (p->dim != 3 || p->bc[0] != DSMC_DIFFUSE)) return fail(DSMC_EPARAM, "orifice needs a 3D diffuse x- wall");
  if (p->inflow_kind == DSMC_INFLOW_GHOST && (p->bc[0] != DSMC_INFLOW || !(p->inflow_T > 0)))
    return fail(DSMC_EPARAM, "ghost inflow needs an INFLOW x- face");
  if (p->inflow_kind == DSMC_INFLOW_EFFUSIVE && (!p->orifice_on || !(p->inflow_T > 0) || p->inflow_count < 0))
    return fail(DSMC_EPARAM, "effusive inflow needs the orifice");
  if (p->inflow_kind < 0 || p->inflow_kind > 2) return fail(DSMC_EPARAM, "unknown inflow");
  for (int k = 0; k < p->n_fill; k++)
    if (!(p->fill[k].T > 0) || p->fill[k].ppc < 0) return fail(DSMC_EPARAM, "bad fill region");
  return DSMC_OK;
}

int make_layout(const dsmc_problem* p, int debug, Layout& L) {
  int rc = validate(p);
  if (rc) return rc;
  std::memset(&L, 0, sizeof(L));
  L.Nc = (int64_t)p->nx * p->ny * p->nz;
  L.stride = (int64_t)align_up((size_t)p->cap_per_run, 32);
  L.RN = (int64_t)p->n_runs * L.Nc;
  if ((int64_t)p->n_runs * L.stride >= (int64_t)0xFFFFFFFFll || L.RN >= (int64_t)0x7FFFFFFFll)
    return fail(DSMC_EINVAL, "batch too large for 32-bit particle/cell keys");
  std::vector<int32_t> fj, fk;
  std::vector<uint8_t> open;
  face_lists(p, fj, fk, open);
  L.n_face = (int32_t)fj.size();
  dsmc_sizes& s = L.sz;
  s.stride = L.stride;
  s.n_cells = L.Nc;
  s.n_steps = (int32_t)std::floor(p->dt_L / p->dt + 0.5);
  s.sample_every = (int32_t)std::floor(p->dt_s / p->dt + 0.5);
  s.n_slots = s.n_steps / s.sample_every;
  const size_t slots = (size_t)p->n_runs * L.stride;
  s.P = 2 * 6 * slots * sizeof(float);
  s.key = slots * sizeof(uint32_t);
  s.lcr = slots * sizeof(uint32_t);
  s.cell = align_up((size_t)L.RN * sizeof(uint32_t), 16);
  s.gmax = (size_t)L.RN * sizeof(float);
  s.C = (size_t)s.n_slots * 5 * (size_t)L.RN * sizeof(double);
  if (s.C == 0) s.C = 8;
  const size_t R = (size_t)p->n_runs;
  size_t o = 0;
  L.c_step = o; o += 4;
  L.c_status = o; o += 4;
  o = align_up(o, 16);
  L.c_nstore = o; o = align_up(o + 8 * R, 16);
  L.c_parity = o; o = align_up(o + 4 * R, 16);
  L.c_reorder = o; o = align_up(o + 4 * R, 16);
  L.c_inserted = o; o = align_up(o + 4 * R, 16);
  L.c_counters = o; o = align_up(o + 8 * 4 * R, 16);
  L.c_live = o; o = align_up(o + 8 * R, 16);
  L.c_psteps = o; o = align_up(o + 8 * R, 16);
  L.c_slot = o; o = align_up(o + 4 * (size_t)(s.n_slots > 0 ? s.n_slots : 1), 16);
  L.c_stepslot = o; o = align_up(o + 4, 16);
  L.c_maxn = o; o = align_up(o + 4 * R, 16);
  L.c_queue = o; o = align_up(o + 8 * 8, 16);
  L.c_items = o; o = align_up(o + 8 * ((size_t)R + 2), 16);
  L.c_heavy = o; o = align_up(o + 4 * 2 * dsmc::HEAVY_TIERS, 16);
  L.c_tiles = o; o = align_up(o + 4 * 2, 16);
  s.ctl = o;
  const size_t F = (size_t)p->ny * p->nz;
  o = 0;
  L.s_face_j = o; o = align_up(o + 4 * F, 256);
  L.s_face_k = o; o = align_up(o + 4 * F, 256);
  L.s_open = o; o = align_up(o + F, 256);
  L.s_kept = o; o = align_up(o + 4 * R * (size_t)(L.n_face > 0 ? L.n_face : 1), 256);
  const int64_t Lscan = L.RN > L.Nc ? L.RN : L.Nc;
  L.s_part = o; o = align_up(o + 4 * ((size_t)dsmc::scan_tiles(Lscan) + 1), 256);
  L.s_macros = o; o = align_up(o + 8 * 10 * (size_t)L.Nc, 256);
  L.s_heavy = o; o = align_up(o + 4 * dsmc::HEAVY_TIERS * ((size_t)(L.RN + 31) / 32 + 1), 256);
  L.s_tiles = o; o = align_up(o + 4 * ((size_t)(L.RN + 31) / 32 + 1), 256);
  if (debug) {
    L.s_cand = o; o = align_up(o + 8 * (size_t)L.RN, 256);
    L.s_acc = o; o = align_up(o + 4 * (size_t)L.RN, 256);
  }
  s.scratch = o;
  return DSMC_OK;
}

// (sigma g) of the model at relative speed g (reading R13/R15); HS: pi d^2 g
void gas_constants(const dsmc_problem* p, double& sigma_c, double& omega1, double& gmax0) {
  if (p->model == DSMC_HS) {
    sigma_c = M_PI * p->d_ref * p->d_ref;
    omega1 = 0.5;
  } else {
    const double m_r = 0.5 * p->mass;
    sigma_c = M_PI * p->d_ref * p->d_ref * std::pow(2.0 * p->T_ref / m_r, p->omega - 0.5) / std::tgamma(2.5 - p->omega);
    omega1 = 1.0 - p->omega;
  }
  // g0 = |U|max + 5 sqrt(2 T_max / m) over every state in the problem
  double Tmax = 0.0, Umax = 0.0;
  for (int k = 0; k < p->n_fill; k++) {
    Tmax = std::fmax(Tmax, p->fill[k].T);
    const double u = std::sqrt(p->fill[k].u[0] * p->fill[k].u[0] + p->fill[k].u[1] * p->fill[k].u[1] +
                               p->fill[k].u[2] * p->fill[k].u[2]);
    Umax = std::fmax(Umax, u);
  }
  if (p->inflow_kind != DSMC_INFLOW_NONE) {
    Tmax = std::fmax(Tmax, p->inflow_T);
    Umax = std::fmax(Umax, std::fabs(p->inflow_U));
  }
  for (int f = 0; f < 6; f++) if (p->bc[f] == DSMC_DIFFUSE) Tmax = std::fmax(Tmax, p->bc_T[f]);
  if (p->plate_on) Tmax = std::fmax(Tmax, p->plate_T);
  if (Tmax <= 0) Tmax = p->T_ref;
  const double g0 = Umax + 5.0 * std::sqrt(2.0 * Tmax / p->mass);
  gmax0 = p->model == DSMC_HS ? sigma_c * g0 : sigma_c * std::pow(g0 * g0, 1.0 - p->omega);
}

}  // namespace

struct dsmc_ctx {
  dsmc_problem prob;
  Layout L;
  dsmc::Prm P;
  dsmc_buffers buf;
  int debug;
  cudaStream_t stream;
  cudaStream_t cap_stream;
  cudaStream_t aux_stream;   // the graph's second branch (heavy tiles beside the warp-tile list)
  cudaEvent_t fork, join;
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  int kernels_per_step;
};

extern "C" {

const char* dsmc_last_error(void) { return g_err.c_str(); }

int dsmc_query_sizes(const dsmc_problem* prob, int32_t debug, dsmc_sizes* out) {
  if (!out) return fail(DSMC_EINVAL, "null out");
  Layout L;
  const int rc = make_layout(prob, debug, L);
  if (rc) return rc;
  *out = L.sz;
  return DSMC_OK;
}

int dsmc_create(const dsmc_problem* prob, const dsmc_buffers* buf, int32_t debug, void* stream, dsmc_ctx** out) {
  if (!buf || !out) return fail(DSMC_EINVAL, "null argument");
  Layout L;
  int rc = make_layout(prob, debug, L);
  if (rc) return rc;
  const void* ptrs[8] = {buf->P, buf->key, buf->lcr, buf->cell, buf->gmax, buf->C, buf->ctl, buf->scratch};
  for (const void* q : ptrs) if (!q) return fail(DSMC_EINVAL, "null device buffer");
  dsmc_ctx* c = new dsmc_ctx();
  c->prob = *prob;
  c->L = L;
  c->buf = *buf;
  c->debug = debug;
  c->stream = (cudaStream_t)stream;
  dsmc::Prm& P = c->P;
  std::memset(&P, 0, sizeof(P));
  const dsmc_problem* p = prob;
  P.dim = p->dim; P.nx = p->nx; P.ny = p->ny; P.nz = p->nz;
  P.Nc = L.Nc; P.R = p->n_runs; P.stride = L.stride; P.cap = p->cap_per_run;
  // magic divisor for run = key / Nc (keys < 2^31): l = ceil(log2 Nc), m = ceil(2^(31+l) / Nc) < 2^32,
  // q = umulhi(k, m) >> (l - 1); exact since k * (m Nc - 2^(31+l)) < 2^31 Nc <= 2^(31+l)
  if (L.Nc > 1) {
    int l = 0;
    while ((1ll << l) < L.Nc) l++;
    const uint64_t m = ((1ull << (31 + l)) + (uint64_t)L.Nc - 1) / (uint64_t)L.Nc;
    P.nc_mul = (uint32_t)m;
    P.nc_shift = l - 1;
    for (uint64_t kk : {(uint64_t)0, (uint64_t)L.Nc - 1, (uint64_t)L.Nc, (uint64_t)L.RN - 1, (uint64_t)0x7FFFFFFE}) {
      const uint32_t q = (uint32_t)(((kk * m) >> 32) >> (l - 1));
      if (kk < 0x80000000ull && q != kk / (uint64_t)L.Nc) { delete c; return fail(DSMC_EINVAL, "run divisor"); }
    }
  }
  P.half = 6 * (int64_t)p->n_runs * L.stride;
  P.seed = p->seed; P.run_id0 = (uint32_t)p->run_id0;
  P.dt_f = (float)p->dt;
  P.sample_every = L.sz.sample_every; P.n_slots = L.sz.n_slots; P.reorder_every = p->reorder_every;
  P.model = p->model;
  P.coef = p->fnum_vc * p->dt;
  double gm0;
  gas_constants(p, P.sigma_c, P.omega1, gm0);
  P.gmax0 = (float)gm0;
  P.has_events = p->plate_on ? 1 : 0;
  for (int f = 0; f < 6; f++) {
    P.bc[f] = p->bc[f];
    P.sqrt_bcT[f] = std::sqrt(p->bc_T[f] > 0 ? p->bc_T[f] : 1.0);
    if (f < 2 * p->dim && (p->bc[f] == DSMC_DIFFUSE || p->bc[f] == DSMC_OUTFLOW || p->bc[f] == DSMC_INFLOW))
      P.has_events = 1;
  }
  P.plate_on = p->plate_on; P.plate_axis = p->plate_axis; P.plate_span_axis = p->plate_span_axis;
  P.plate_pos = (float)p->plate_pos; P.plate_lo = (float)p->plate_lo; P.plate_hi = (float)p->plate_hi;
  P.sqrt_plateT = std::sqrt(p->plate_T > 0 ? p->plate_T : 1.0);
  P.orifice_on = p->orifice_on;
  P.inflow_kind = p->inflow_kind; P.n_face = L.n_face; P.inflow_count = p->inflow_count;
  const double w = (p->inflow_U + 6.0 * std::sqrt(p->inflow_T)) * p->dt;
  P.ghost_x = p->inflow_n * w;
  P.ghost_w_f = (float)w;
  P.inflow_U = p->inflow_U;
  P.sqrt_inflowT = std::sqrt(p->inflow_T > 0 ? p->inflow_T : 1.0);
  if (p->inflow_kind == DSMC_INFLOW_GHOST) P.insert_bound = (int64_t)L.n_face * (int64_t)std::ceil(P.ghost_x);
  else if (p->inflow_kind == DSMC_INFLOW_EFFUSIVE) P.insert_bound = (int64_t)L.n_face * p->inflow_count;
  {  // mean initial particles per cell decides the register sorting-network width
    double filled = 0.0;
    for (int k = 0; k < p->n_fill; k++) {
      double vol = 1.0;
      for (int a = 0; a < 3; a++) vol *= (double)(p->fill[k].hi[a] - p->fill[k].lo[a]);
      filled += vol * p->fill[k].ppc;
    }
    const double ppc = filled / (double)L.Nc;
    P.net_wide = (ppc > 12.0 || p->inflow_kind == DSMC_INFLOW_EFFUSIVE) ? 1 : 0;
    // sparse fills: most tiles draw no candidate; list the ones with work (k_collide_triage)
    P.compact = ppc < DSMC_COMPACT_PPC ? 1 : 0;
    if (const char* e = std::getenv("DSMC_COMPACT")) P.compact = std::atoi(e) ? 1 : 0;   // A/B experiments
    // warp-tile staging capacity: the densest fill region's 32 cells with a
    // wide margin (tiles beyond it take the per-lane global-memory path)
    int32_t ppc_max = 0;
    for (int k = 0; k < p->n_fill; k++) ppc_max = p->fill[k].ppc > ppc_max ? p->fill[k].ppc : ppc_max;
    if (p->inflow_kind == DSMC_INFLOW_GHOST) ppc_max = std::max(ppc_max, (int32_t)std::ceil(p->inflow_n));
    // (3.5 sigma of the Poisson tile count: 16 one-warp blocks then stay under the
    // 196 KB shared-memory carveout, which leaves the L1 the gathers need; the
    // ~2e-4 of c4's tiles beyond it take the heavy blocks)
    int32_t capw = 32 * ppc_max + (int32_t)std::ceil(3.5 * std::sqrt(32.0 * ppc_max));
    capw = std::max(256, std::min(capw, 4096));
    // an effusive source builds a dense plume the fills do not predict: tiles of a
    // few hundred particles are then common, and they are cheaper in the warp path
    // than in the heavy queue (c5 after 500 steps, capw 256 / 512 / 768 / 1024:
    // 3.92 / 3.65 / 3.66 / 3.90 ms per step)
    if (p->inflow_kind == DSMC_INFLOW_EFFUSIVE) capw = std::max(capw, 512);
    // dense fills (cells beyond the 32-wide register sort, ~100 candidates per cell):
    // one lane walking a cell's candidates is the bottleneck, and the heavy blocks'
    // claim rounds walk them in parallel (c2 from the fill, capw 512 / 1024 / 1832:
    // 0.451 / 0.512 / 0.628 ms per step; c3 at 20 per cell stays faster in the warp path)
    if (ppc_max > 32) capw = 512;
    if (const char* e = std::getenv("DSMC_CAPW")) capw = std::max(256, std::min(std::atoi(e), 4096));   // A/B experiments
    P.capw = (capw + 31) / 32 * 32;
  }
  P.n_fill = p->n_fill;
  for (int k = 0; k < p->n_fill; k++) {
    for (int a = 0; a < 3; a++) {
      P.fill_lo[k][a] = p->fill[k].lo[a];
      P.fill_hi[k][a] = p->fill[k].hi[a];
      P.fill_u[k][a] = p->fill[k].u[a];
    }
    P.fill_ppc[k] = p->fill[k].ppc;
    P.fill_sqrtT[k] = std::sqrt(p->fill[k].T);
  }
  char* sc = (char*)buf->scratch;
  char* ct = (char*)buf->ctl;
  P.P = (float*)buf->P;
  P.key = (uint32_t*)buf->key;
  P.lcr = (uint32_t*)buf->lcr;
  P.cell = (uint32_t*)buf->cell;
  P.gmax = (float*)buf->gmax;
  P.C = (double*)buf->C;
  P.face_j = (const int32_t*)(sc + L.s_face_j);
  P.face_k = (const int32_t*)(sc + L.s_face_k);
  P.open_face = (const uint8_t*)(sc + L.s_open);
  P.face_kept = (int32_t*)(sc + L.s_kept);
  P.scan_part = (uint32_t*)(sc + L.s_part);
  P.macros = (double*)(sc + L.s_macros);
  P.debug = debug;
  if (debug) {
    P.dbg_cand = (int64_t*)(sc + L.s_cand);
    P.dbg_acc = (int32_t*)(sc + L.s_acc);
  }
  P.ctl.step = (int32_t*)(ct + L.c_step);
  P.ctl.status = (int32_t*)(ct + L.c_status);
  P.ctl.n_store = (int64_t*)(ct + L.c_nstore);
  P.ctl.parity = (int32_t*)(ct + L.c_parity);
  P.ctl.reorder = (int32_t*)(ct + L.c_reorder);
  P.ctl.inserted = (int32_t*)(ct + L.c_inserted);
  P.ctl.counters = (unsigned long long*)(ct + L.c_counters);
  P.ctl.live = (int64_t*)(ct + L.c_live);
  P.ctl.psteps = (unsigned long long*)(ct + L.c_psteps);
  P.ctl.slot_done = (int32_t*)(ct + L.c_slot);
  P.ctl.step_slot = (int32_t*)(ct + L.c_stepslot);
  P.ctl.maxn = (uint32_t*)(ct + L.c_maxn);
  P.ctl.queue = (unsigned long long*)(ct + L.c_queue);
  P.ctl.items = (int64_t*)(ct + L.c_items);
  P.ctl.heavy = (uint32_t*)(ct + L.c_heavy);
  P.ctl.tiles = (uint32_t*)(ct + L.c_tiles);
  P.tile_list = (uint32_t*)(sc + L.s_tiles);
  P.heavy_list = (uint32_t*)(sc + L.s_heavy);
  P.heavy_stride = (L.RN + 31) / 32 + 1;
  // NEXT-1 A/B: DSMC_STATIC_CELLS=1 replaces the dynamic, size-tiered
  // heavy-tile queue by a static block-per-tile mapping: every tile beyond the warp
  // staging area goes to the large tier, dealt to its blocks round-robin -- the
  // static mapping against which the TLPDPR-style reallocation is measured
  if (const char* e = std::getenv("DSMC_STATIC_CELLS")) if (std::atoi(e)) P.heavy_static = 1;
  P.caph = 8192;
  P.caph_tier[0] = 3584;      // 2 blocks per SM within the 196 KB carveout (4096: 215 KB, L1 down to 28 KB, 2-3% slower; a third tier of 1024, register-limited to 2 blocks too, measured slower)
  P.caph_tier[1] = P.caph;    // 1 block per SM

  auto bail = [&](int code) {   // release whatever was created before the failure
    if (c->exec) cudaGraphExecDestroy(c->exec);
    if (c->graph) cudaGraphDestroy(c->graph);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
    if (c->fork) cudaEventDestroy(c->fork);
    if (c->join) cudaEventDestroy(c->join);
    delete c;
    return code;
  };
  std::vector<int32_t> fj, fk;
  std::vector<uint8_t> open;
  face_lists(p, fj, fk, open);
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming)) != cudaSuccess)
    return bail(cuda_fail(e, "cudaStreamCreate"));
  if (!fj.empty()) {
    cudaMemcpyAsync((void*)P.face_j, fj.data(), 4 * fj.size(), cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync((void*)P.face_k, fk.data(), 4 * fk.size(), cudaMemcpyHostToDevice, c->stream);
  }
  cudaMemcpyAsync((void*)P.open_face, open.data(), open.size(), cudaMemcpyHostToDevice, c->stream);
  cudaMemsetAsync(buf->ctl, 0, L.sz.ctl, c->stream);
  cudaMemsetAsync(buf->cell, 0, L.sz.cell, c->stream);
  if (debug) {
    cudaMemsetAsync(P.dbg_cand, 0, 8 * (size_t)L.RN, c->stream);
    cudaMemsetAsync(P.dbg_acc, 0, 4 * (size_t)L.RN, c->stream);
  }
  dsmc::launch_fill_f32(P.gmax, L.RN, P.gmax0, c->stream);
  if ((e = cudaStreamSynchronize(c->stream)) != cudaSuccess) return bail(cuda_fail(e, "create init"));
  // capture one step as a graph (device-side schedule: one graph for all steps)
  if ((e = cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
    return bail(cuda_fail(e, "cudaStreamBeginCapture"));
  dsmc::issue_step(P, c->cap_stream, dsmc::LaunchHook{}, dsmc::Branch{c->aux_stream, c->fork, c->join});
  if ((e = cudaStreamEndCapture(c->cap_stream, &c->graph)) != cudaSuccess) {
    c->graph = nullptr;
    return bail(cuda_fail(e, "cudaStreamEndCapture"));
  }
  if ((e = cudaGraphInstantiate(&c->exec, c->graph, 0)) != cudaSuccess) {
    c->exec = nullptr;
    return bail(cuda_fail(e, "cudaGraphInstantiate"));
  }
  size_t nn = 0;
  cudaGraphGetNodes(c->graph, nullptr, &nn);
  std::vector<cudaGraphNode_t> nodes(nn);
  cudaGraphGetNodes(c->graph, nodes.data(), &nn);
  c->kernels_per_step = 0;
  for (auto& nd : nodes) {
    cudaGraphNodeType t;
    cudaGraphNodeGetType(nd, &t);
    if (t == cudaGraphNodeTypeKernel) c->kernels_per_step++;
  }
  *out = c;
  return DSMC_OK;
}

int dsmc_destroy(dsmc_ctx* c) {
  if (!c) return DSMC_OK;
  if (c->exec) cudaGraphExecDestroy(c->exec);
  if (c->graph) cudaGraphDestroy(c->graph);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
  if (c->fork) cudaEventDestroy(c->fork);
  if (c->join) cudaEventDestroy(c->join);
  delete c;
  return DSMC_OK;
}

int dsmc_generate(dsmc_ctx* c) {
  if (!c) return fail(DSMC_EINVAL, "null ctx");
  Nvtx nv("dsmc_generate");
  dsmc::launch_fill(c->P, c->stream);
  CK(cudaGetLastError());
  return DSMC_OK;
}

int dsmc_step(dsmc_ctx* c, int32_t nsteps) {
  if (!c || nsteps < 0) return fail(DSMC_EINVAL, "bad argument");
  Nvtx nv("dsmc_step");
  for (int32_t i = 0; i < nsteps; i++) CK(cudaGraphLaunch(c->exec, c->stream));
  return DSMC_OK;
}

namespace {
struct TimedHook {
  cudaEvent_t ev[dsmc::KSLOT_COUNT][2];
  bool used[dsmc::KSLOT_COUNT];
  cudaStream_t st;
  static void cb(void* u, int slot, int after) {
    TimedHook* h = (TimedHook*)u;
    if (!after) nvtxRangePushA(dsmc::kernel_slot_name(slot));   // one NVTX range per kernel launch
    cudaEventRecord(h->ev[slot][after], h->st);
    if (after) { h->used[slot] = true; nvtxRangePop(); }
  }
};
}  // namespace

int dsmc_step_timed(dsmc_ctx* c, int32_t nsteps, double* ms_accum, int64_t* launches) {
  if (!c || !ms_accum) return fail(DSMC_EINVAL, "bad argument");
  TimedHook h;
  h.st = c->stream;
  std::memset(h.ev, 0, sizeof(h.ev));
  auto destroy_events = [&]() {
    for (int k = 0; k < dsmc::KSLOT_COUNT; k++)
      for (int a = 0; a < 2; a++) if (h.ev[k][a]) cudaEventDestroy(h.ev[k][a]);
  };
  for (int k = 0; k < dsmc::KSLOT_COUNT; k++)
    for (int a = 0; a < 2; a++) {
      const cudaError_t e = cudaEventCreate(&h.ev[k][a]);
      if (e != cudaSuccess) {
        h.ev[k][a] = nullptr;
        destroy_events();
        return cuda_fail(e, "cudaEventCreate");
      }
    }
  dsmc::LaunchHook hook;
  hook.fn = &TimedHook::cb;
  hook.user = &h;
  int rc = DSMC_OK;
  for (int32_t i = 0; i < nsteps && rc == DSMC_OK; i++) {
    std::memset(h.used, 0, sizeof(h.used));
    dsmc::issue_step(c->P, c->stream, hook);
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) { rc = cuda_fail(e, "step_timed"); break; }
    for (int k = 0; k < dsmc::KSLOT_COUNT; k++) {
      if (!h.used[k]) continue;
      float ms = 0;
      cudaEventElapsedTime(&ms, h.ev[k][0], h.ev[k][1]);
      ms_accum[k] += ms;
      if (launches) launches[k] += 1;
    }
  }
  destroy_events();
  return rc;
}

const char* dsmc_kernel_name(int32_t k) { return dsmc::kernel_slot_name(k); }

int dsmc_kernels_per_step(dsmc_ctx* c, int32_t* out) {
  if (!c || !out) return fail(DSMC_EINVAL, "bad argument");
  *out = c->kernels_per_step;
  return DSMC_OK;
}

static int slot_written(dsmc_ctx* c, int32_t slot, bool* ok);

int dsmc_sample(dsmc_ctx* c, int32_t slot) {
  if (!c) return fail(DSMC_EINVAL, "null ctx");
  Nvtx nv("dsmc_sample");
  if (slot < 0 || slot >= c->L.sz.n_slots) return fail(DSMC_ESCHED, "slot out of range");
  dsmc::issue_sample(c->P, slot, 0, c->stream);
  CK(cudaGetLastError());
  return DSMC_OK;
}

int dsmc_sample_add(dsmc_ctx* c, int32_t slot) {
  if (!c) return fail(DSMC_EINVAL, "null ctx");
  Nvtx nv("dsmc_sample_add");
  if (slot < 0 || slot >= c->L.sz.n_slots) return fail(DSMC_ESCHED, "slot out of range");
  bool written = false;
  const int rc = slot_written(c, slot, &written);
  if (rc) return rc;
  if (!written) CK(cudaMemsetAsync(c->P.C + (size_t)slot * 5 * (size_t)c->L.RN, 0, 8 * 5 * (size_t)c->L.RN, c->stream));
  dsmc::issue_sample(c->P, slot, 1, c->stream);
  CK(cudaGetLastError());
  return DSMC_OK;
}

int dsmc_slot_samples(dsmc_ctx* c, int32_t slot, int32_t* out) {
  if (!c || !out) return fail(DSMC_EINVAL, "bad argument");
  if (slot < 0 || slot >= c->L.sz.n_slots) return fail(DSMC_ESCHED, "slot out of range");
  CK(cudaMemcpyAsync(out, c->P.ctl.slot_done + slot, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return DSMC_OK;
}

static int latched(dsmc_ctx* c, int32_t* st) {
  uint32_t w = 0;
  CK(cudaMemcpyAsync(&w, c->P.ctl.status, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *st = dsmc::status_code(w);
  return DSMC_OK;
}

static int slot_written(dsmc_ctx* c, int32_t slot, bool* ok) {
  int32_t v = 0;
  CK(cudaMemcpyAsync(&v, c->P.ctl.slot_done + slot, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *ok = v != 0;
  return DSMC_OK;
}

// ensemble of n_blocks blocks of slot sums (block 0 may be this context's own slot) -> host out
static int macros_from(dsmc_ctx* c, int32_t slot, const double* sums, int32_t n_blocks, double* out) {
  Nvtx nv("dsmc_read_macros");
  int32_t m = 0;
  CK(cudaMemcpyAsync(&m, c->P.ctl.slot_done + slot, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  dsmc::launch_macros(c->P, sums, n_blocks, m, c->prob.fnum_vc, c->stream);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, c->P.macros, 8 * 10 * (size_t)c->L.Nc, cudaMemcpyDeviceToHost, c->stream));
  int32_t st = 0;
  const int rc = latched(c, &st);
  if (rc) return rc;
  if (st) return fail(st, "latched device fault");
  return DSMC_OK;
}

int dsmc_read_macros(dsmc_ctx* c, int32_t slot, double* out) {
  if (!c || !out) return fail(DSMC_EINVAL, "bad argument");
  if (slot < 0 || slot >= c->L.sz.n_slots) return fail(DSMC_ESCHED, "slot out of range");
  bool ok = false;
  int rc = slot_written(c, slot, &ok);
  if (rc) return rc;
  if (!ok) return fail(DSMC_ESCHED, "slot not written yet");
  return macros_from(c, slot, c->P.C + (size_t)slot * 5 * (size_t)c->L.RN, 1, out);
}

int dsmc_read_macros_gathered(dsmc_ctx* c, int32_t slot, const double* sums_dev, int32_t n_blocks, double* out) {
  if (!c || !out || !sums_dev || n_blocks < 1) return fail(DSMC_EINVAL, "bad argument");
  if (slot < 0 || slot >= c->L.sz.n_slots) return fail(DSMC_ESCHED, "slot out of range");
  if ((int64_t)n_blocks * c->prob.n_runs > 0x7FFFFFFF) return fail(DSMC_EINVAL, "too many runs");
  bool ok = false;
  int rc = slot_written(c, slot, &ok);
  if (rc) return rc;
  if (!ok) return fail(DSMC_ESCHED, "slot not written yet");
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, sums_dev) != cudaSuccess || pa.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return fail(DSMC_EINVAL, "sums_dev is not device memory");
  }
  return macros_from(c, slot, sums_dev, n_blocks, out);
}

int dsmc_slot_sums_ptr(dsmc_ctx* c, int32_t slot, const double** out) {
  if (!c || !out) return fail(DSMC_EINVAL, "bad argument");
  if (slot < 0 || slot >= c->L.sz.n_slots) return fail(DSMC_ESCHED, "slot out of range");
  *out = c->P.C + (size_t)slot * 5 * (size_t)c->L.RN;
  return DSMC_OK;
}

int dsmc_read_sums(dsmc_ctx* c, int32_t slot, double* out) {
  if (!c || !out) return fail(DSMC_EINVAL, "bad argument");
  if (slot < 0 || slot >= c->L.sz.n_slots) return fail(DSMC_ESCHED, "slot out of range");
  bool ok = false;
  int rc = slot_written(c, slot, &ok);
  if (rc) return rc;
  if (!ok) return fail(DSMC_ESCHED, "slot not written yet");
  const size_t n = 5 * (size_t)c->L.RN;
  CK(cudaMemcpyAsync(out, c->P.C + (size_t)slot * n, 8 * n, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return DSMC_OK;
}

int dsmc_status(dsmc_ctx* c, int64_t* counters_out) {
  if (!c) return fail(DSMC_EINVAL, "null ctx");
  const int R = c->prob.n_runs;
  std::vector<unsigned long long> cnt(4 * (size_t)R);
  std::vector<int64_t> ns((size_t)R), live((size_t)R);
  std::vector<unsigned long long> ps((size_t)R);
  std::vector<uint32_t> mx((size_t)R);
  int32_t step = 0;
  uint32_t stw = 0;
  CK(cudaMemcpyAsync(cnt.data(), c->P.ctl.counters, 8 * 4 * (size_t)R, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(ns.data(), c->P.ctl.n_store, 8 * (size_t)R, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(live.data(), c->P.ctl.live, 8 * (size_t)R, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(ps.data(), c->P.ctl.psteps, 8 * (size_t)R, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(mx.data(), c->P.ctl.maxn, 4 * (size_t)R, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&step, c->P.ctl.step, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&stw, c->P.ctl.status, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const int32_t st = dsmc::status_code(stw);
  if (counters_out)
    for (int r = 0; r < R; r++) {
      int64_t* o = counters_out + (size_t)r * DSMC_STATUS_COLS;
      for (int q = 0; q < 4; q++) o[q] = (int64_t)cnt[r * 4 + q];
      o[4] = ns[r];
      o[5] = step;
      o[6] = live[r];
      o[7] = (int64_t)ps[r];
      o[8] = (int64_t)mx[r];
    }
  if (st) return fail(st, "latched device fault");
  return DSMC_OK;
}

static int run_window(dsmc_ctx* c, int32_t run, int64_t* n, int32_t* parity) {
  if (run < 0 || run >= c->prob.n_runs) return fail(DSMC_EINVAL, "run out of range");
  CK(cudaMemcpyAsync(n, c->P.ctl.n_store + run, 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(parity, c->P.ctl.parity + run, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return DSMC_OK;
}

static float* arr(dsmc_ctx* c, int h, int a, int32_t run) {
  return c->P.P + (int64_t)h * c->P.half + (int64_t)a * c->P.R * c->P.stride + (int64_t)run * c->P.stride;
}

int dsmc_get_state(dsmc_ctx* c, int32_t run, int64_t* n_out, float* x, float* y, float* z, float* vx, float* vy,
                   float* vz, uint8_t* alive) {
  if (!c || !n_out) return fail(DSMC_EINVAL, "bad argument");
  int64_t n = 0;
  int32_t h = 0;
  int rc = run_window(c, run, &n, &h);
  if (rc) return rc;
  *n_out = n;
  float* dst[6] = {x, y, z, vx, vy, vz};
  for (int a = 0; a < 6; a++) {
    if (!dst[a] || !n) continue;
    if (a < 3 && a >= c->prob.dim) std::memset(dst[a], 0, 4 * (size_t)n);  // axes >= dim are 0
    else CK(cudaMemcpyAsync(dst[a], arr(c, h, a, run), 4 * (size_t)n, cudaMemcpyDeviceToHost, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  if (alive) {
    std::vector<float> tmp;
    const float* xs = x;
    if (!xs) {
      tmp.resize((size_t)n);
      CK(cudaMemcpy(tmp.data(), arr(c, h, 0, run), 4 * (size_t)n, cudaMemcpyDeviceToHost));
      xs = tmp.data();
    }
    for (int64_t i = 0; i < n; i++) alive[i] = xs[i] < -1.0e29f ? 0 : 1;
  }
  return DSMC_OK;
}

int dsmc_set_state(dsmc_ctx* c, int32_t run, int64_t n, const float* x, const float* y, const float* z,
                   const float* vx, const float* vy, const float* vz, const uint8_t* alive, int32_t step) {
  if (!c || !x || !vx || !vy || !vz) return fail(DSMC_EINVAL, "bad argument");
  if (n < 0 || n > c->prob.cap_per_run) return fail(DSMC_ECAP, "n exceeds capacity");
  int64_t n0 = 0;
  int32_t h = 0;
  int rc = run_window(c, run, &n0, &h);
  if (rc) return rc;
  std::vector<float> xs;
  int64_t live = n;
  if (alive) {
    xs.assign(x, x + n);
    for (int64_t i = 0; i < n; i++) if (!alive[i]) { xs[i] = dsmc::DEAD_X; live--; }
  }
  std::vector<float> zero;
  const float* src[6] = {alive ? xs.data() : x, y, z, vx, vy, vz};
  for (int a = 0; a < 6; a++) {
    const float* s = src[a];
    if (!s) { zero.assign((size_t)n, 0.0f); s = zero.data(); }
    if (n) CK(cudaMemcpyAsync(arr(c, h, a, run), s, 4 * (size_t)n, cudaMemcpyHostToDevice, c->stream));
    if (s == zero.data()) CK(cudaStreamSynchronize(c->stream));
  }
  CK(cudaMemcpyAsync(c->P.ctl.n_store + run, &n, 8, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->P.ctl.live + run, &live, 8, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->P.ctl.step, &step, 4, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return DSMC_OK;
}

int dsmc_get_gmax(dsmc_ctx* c, int32_t run, float* out) {
  if (!c || !out || run < 0 || run >= c->prob.n_runs) return fail(DSMC_EINVAL, "bad argument");
  CK(cudaMemcpyAsync(out, c->P.gmax + (int64_t)run * c->L.Nc, 4 * (size_t)c->L.Nc, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return DSMC_OK;
}

int dsmc_set_gmax(dsmc_ctx* c, int32_t run, const float* in) {
  if (!c || !in || run < 0 || run >= c->prob.n_runs) return fail(DSMC_EINVAL, "bad argument");
  CK(cudaMemcpyAsync(c->P.gmax + (int64_t)run * c->L.Nc, in, 4 * (size_t)c->L.Nc, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return DSMC_OK;
}

int dsmc_get_index(dsmc_ctx* c, int32_t run, int64_t* live_out, int64_t* count, int64_t* start, int64_t* lcr,
                   int64_t* cand, int32_t* acc) {
  if (!c || !live_out || run < 0 || run >= c->prob.n_runs) return fail(DSMC_EINVAL, "bad argument");
  if (!c->debug) return fail(DSMC_EINVAL, "get_index needs a debug context");
  const int64_t Nc = c->L.Nc;
  std::vector<uint32_t> ends((size_t)Nc + 1);
  const int64_t k0 = (int64_t)run * Nc;
  if (run == 0) {
    ends[0] = 0;
    CK(cudaMemcpyAsync(ends.data() + 1, c->P.cell, 4 * (size_t)Nc, cudaMemcpyDeviceToHost, c->stream));
  } else {
    CK(cudaMemcpyAsync(ends.data(), c->P.cell + k0 - 1, 4 * ((size_t)Nc + 1), cudaMemcpyDeviceToHost, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  const uint32_t base = ends[0];
  const int64_t live = (int64_t)(ends[Nc] - base);
  *live_out = live;
  for (int64_t q = 0; q < Nc; q++) {
    if (count) count[q] = (int64_t)(ends[q + 1] - ends[q]);
    if (start) start[q] = (int64_t)(ends[q] - base);
  }
  if (lcr && live) {
    std::vector<uint32_t> g((size_t)live);
    CK(cudaMemcpyAsync(g.data(), c->P.lcr + base, 4 * (size_t)live, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int64_t q = 0; q < live; q++) lcr[q] = (int64_t)g[q] - (int64_t)run * c->L.stride;
  }
  if (cand) CK(cudaMemcpyAsync(cand, c->P.dbg_cand + k0, 8 * (size_t)Nc, cudaMemcpyDeviceToHost, c->stream));
  if (acc) CK(cudaMemcpyAsync(acc, c->P.dbg_acc + k0, 4 * (size_t)Nc, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return DSMC_OK;
}

int dsmc_selftest_philox(int64_t n, const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out, uint32_t* out_ref) {
  if (n <= 0 || !ctr || !out) return fail(DSMC_EINVAL, "bad argument");
  uint32_t *d_ctr = nullptr, *d_out = nullptr, *d_ref = nullptr;
  const size_t b = 16 * (size_t)n;
  int rc = DSMC_OK;
  cudaError_t e = cudaSuccess;
  // test hook: the only entry point that allocates device memory (freed on every exit path)
  if ((e = cudaMalloc(&d_ctr, b)) != cudaSuccess || (e = cudaMalloc(&d_out, b)) != cudaSuccess ||
      (out_ref && (e = cudaMalloc(&d_ref, b)) != cudaSuccess) ||
      (e = cudaMemcpy(d_ctr, ctr, b, cudaMemcpyHostToDevice)) != cudaSuccess) {
    rc = cuda_fail(e, "selftest setup");
  } else {
    dsmc::launch_selftest_philox(n, d_ctr, k0, k1, d_out, d_ref, 0);
    if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaMemcpy(out, d_out, b, cudaMemcpyDeviceToHost)) != cudaSuccess ||
        (out_ref && (e = cudaMemcpy(out_ref, d_ref, b, cudaMemcpyDeviceToHost)) != cudaSuccess))
      rc = cuda_fail(e, "selftest");
  }
  if (d_ctr) cudaFree(d_ctr);
  if (d_out) cudaFree(d_out);
  if (d_ref) cudaFree(d_ref);
  return rc;
}

}  // extern "C"
