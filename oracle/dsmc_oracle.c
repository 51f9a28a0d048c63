/*
 * dsmc_oracle.c -- TEST INFRASTRUCTURE ONLY (see dsmc_oracle.h).
 *
 * Plain sequential C; one run at a time; fp32 particle state, fp64 per-cell
 * scalars; compiled with -ffp-contract=off so every rounding is the one the
 * expression spells out (fmaf only where written).  The step follows
 * PAPER.md Fig. 1 / §1.1 (lines 95-110) literally:
 *
 *     Generation -> Motion (each of N_p particles) -> Enumeration, Indexing
 *     (readdressing array LCR) -> Interaction (each of N_c cells) ->
 *     Sampling (at sample moments) [-> reorder of P by LCR]
 *
 * Every free choice the paper leaves open is the DESIGN.md reading cited at
 * the function (R-numbers), taken from SURVEY.md §8(c) C-0..C-11.
 */
#include "dsmc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define TAG_FILL 1u
#define TAG_INFLOW_COUNT 2u
#define TAG_INFLOW_PARTICLE 3u
#define TAG_WALL 4u
#define TAG_COLL_COUNT 5u
#define TAG_COLL_PAIR 6u
#define TAG_COLL_DIR 7u
#define FILL_STEP 0xFFFFFFFFu
#define MAX_BOUNCE 8
#define TWO_PI 6.283185307179586

struct orc_run {
  orc_problem p;
  int32_t run_id;
  uint32_t key[2];
  int64_t Nc, cap, n;
  int32_t n_steps, sample_every, n_slots, step, status;
  float dt_f;
  double coef;      /* F_N/V_c * dt */
  double sigma_c;   /* sigma*g = sigma_c * (g^2)^(1-omega)  (HS: sigma_c*sqrt(g^2)) */
  double ghost_w, ghost_x;
  int64_t insert_bound;
  int32_t n_face;
  int32_t* face_j;
  int32_t* face_k;
  uint8_t* open_face;  /* [ny*nz] orifice map on x- face */
  float* x[3];
  float* v[3];
  uint8_t* alive;
  int32_t* cell;
  int64_t* count;
  int64_t* start;
  int64_t* lcr;
  int64_t* cand;
  int32_t* acc;
  float* gmax;
  double* snap;
  int32_t* snap_done;        /* samples accumulated in the slot (0 = never written) */
  int64_t inserted, removed, candidates, accepted;
};

/* ---------------------------------------------------------------- RNG -- */
/* Philox4x32-10: 10 rounds of the S-box on (c0,c1,c2,c3) with multipliers
 * 0xD2511F53, 0xCD9E8D57 and Weyl key bumps 0x9E3779B9, 0xBB67AE85
 * (Salmon, Moraes, Dror, Shaw, SC'11).  PAPER.md:113-115 "shift random number
 * generator": the key is (seed, run id) (reading R5, SURVEY C-2). */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; round++) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    if (round < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void draw(const orc_run* R, uint32_t unit, uint32_t step, uint32_t tag, uint32_t sub,
                 uint32_t block, uint32_t out[4]) {
  uint32_t ctr[4] = {unit, step, (tag << 24) | (sub & 0xFFFFFFu), block};
  orc_philox4x32_10(ctr, R->key, out);
}

/* u in [0,1): top 24 bits * 2^-24 ; u in (0,1]: (top 24 bits + 1) * 2^-24 */
static float u_co(uint32_t w) { return (float)(w >> 8) * (1.0f / 16777216.0f); }
static double u_co_d(uint32_t w) { return (double)(w >> 8) * (1.0 / 16777216.0); }
static double u_oc_d(uint32_t w) { return (double)((w >> 8) + 1u) * (1.0 / 16777216.0); }
/* index in [0,N): Lemire's multiply-shift */
static int64_t lemire(uint32_t w, int64_t N) { return (int64_t)(((uint64_t)w * (uint64_t)N) >> 32); }

/* Box-Muller pair in fp64 from (w0 -> radius, w1 -> angle) */
static void box_muller(uint32_t w0, uint32_t w1, double* n1, double* n2) {
  double r = sqrt(-2.0 * log(u_oc_d(w0)));
  double th = TWO_PI * u_co_d(w1);
  *n1 = r * cos(th);
  *n2 = r * sin(th);
}

/* uniform position inside cell i of an axis; a sum that rounds up to the
 * next face is pulled back below it (reading R7: exactly N per cell). */
static float place(int32_t i, uint32_t w) {
  float x = (float)i + u_co(w);
  float top = (float)(i + 1);
  if (x >= top) x = nextafterf(top, 0.0f);
  return x;
}

/* ----------------------------------------------------------- problem -- */
static int32_t axis_n(const orc_problem* p, int a) { return a == 0 ? p->nx : (a == 1 ? p->ny : p->nz); }

static double sigma_g(const orc_run* R, float g2) {
  if (R->p.model == ORC_HS) return R->sigma_c * sqrt((double)g2);
  return R->sigma_c * pow((double)g2, 1.0 - R->p.omega);
}

static int32_t validate(const orc_problem* p) {
  if (p->dim < 1 || p->dim > 3 || p->nx < 1 || p->ny < 1 || p->nz < 1) return ORC_EINVAL;
  if (p->dim < 2 && p->ny != 1) return ORC_EINVAL;
  if (p->dim < 3 && p->nz != 1) return ORC_EINVAL;
  if (p->n_runs < 1 || p->cap_per_run < 1 || p->n_fill < 0 || p->n_fill > 4) return ORC_EINVAL;
  if (!(p->dt > 0) || !(p->dt_s >= p->dt) || !(p->dt_L >= p->dt_s)) return ORC_ECLOCK;
  double ks = p->dt_s / p->dt, kl = p->dt_L / p->dt_s;
  if (fabs(ks - floor(ks + 0.5)) > 1e-9 * ks || fabs(kl - floor(kl + 0.5)) > 1e-9 * kl) return ORC_ECLOCK;
  if (p->model == ORC_VHS && !(p->omega >= 0.5 && p->omega <= 1.0)) return ORC_EPARAM;
  if (!(p->d_ref > 0) || !(p->mass > 0) || !(p->T_ref > 0) || !(p->fnum_vc >= 0)) return ORC_EPARAM;
  int has_diffuse = p->plate_on;
  for (int f = 0; f < 6; f++) {
    if (p->bc[f] < 0 || p->bc[f] > 4) return ORC_EPARAM;
    if (p->bc[f] == ORC_DIFFUSE) { has_diffuse = 1; if (!(p->bc_T[f] > 0)) return ORC_EPARAM; }
  }
  for (int a = 0; a < p->dim; a++) {
    int lo = p->bc[2 * a], hi = p->bc[2 * a + 1];
    if ((lo == ORC_PERIODIC) != (hi == ORC_PERIODIC)) return ORC_EPARAM;
    if (lo == ORC_INFLOW && a != 0) return ORC_EPARAM;
    if (hi == ORC_INFLOW) return ORC_EPARAM;
  }
  for (int a = 0; a < p->dim; a++)
    if ((p->bc[2 * a] == ORC_SPECULAR || p->bc[2 * a + 1] == ORC_SPECULAR) && has_diffuse) return ORC_EPARAM;
  if (p->plate_on && (p->dim != 2 || !(p->plate_T > 0) || p->plate_axis == p->plate_span_axis)) return ORC_EPARAM;
  if (p->orifice_on && (p->dim != 3 || p->bc[0] != ORC_DIFFUSE)) return ORC_EPARAM;
  if (p->inflow_kind == ORC_INFLOW_GHOST && (p->bc[0] != ORC_INFLOW || !(p->inflow_T > 0))) return ORC_EPARAM;
  if (p->inflow_kind == ORC_INFLOW_EFFUSIVE && (!p->orifice_on || !(p->inflow_T > 0) || p->inflow_count < 0)) return ORC_EPARAM;
  for (int k = 0; k < p->n_fill; k++) if (!(p->fill[k].T > 0) || p->fill[k].ppc < 0) return ORC_EPARAM;
  return ORC_OK;
}

orc_run* orc_create(const orc_problem* p, int32_t run_id, int32_t* err) {
  int32_t e = validate(p);
  if (err) *err = e;
  if (e) return NULL;
  orc_run* R = (orc_run*)calloc(1, sizeof(orc_run));
  R->p = *p;
  R->run_id = run_id;
  R->key[0] = p->seed;
  R->key[1] = (uint32_t)run_id;
  R->Nc = (int64_t)p->nx * p->ny * p->nz;
  R->cap = p->cap_per_run;
  R->sample_every = (int32_t)floor(p->dt_s / p->dt + 0.5);
  R->n_steps = (int32_t)floor(p->dt_L / p->dt + 0.5);
  R->n_slots = R->n_steps / R->sample_every;
  R->dt_f = (float)p->dt;
  R->coef = p->fnum_vc * p->dt;
  double omega = p->model == ORC_HS ? 0.5 : p->omega;
  if (p->model == ORC_HS) {
    R->sigma_c = M_PI * p->d_ref * p->d_ref;
  } else { /* VHS (Bird 1994 eq. 4.63): sigma = pi d^2 (2kT_ref/(m_r g^2))^(omega-1/2) / Gamma(5/2-omega) */
    double m_r = 0.5 * p->mass;
    R->sigma_c = M_PI * p->d_ref * p->d_ref * pow(2.0 * p->T_ref / m_r, omega - 0.5) / tgamma(2.5 - omega);
  }
  /* C-0: (sigma g)_max initial = sigma(g0) g0, g0 = |U|max + 5 sqrt(2 T_max / m) */
  double Tmax = 0.0, Umax = 0.0;
  for (int k = 0; k < p->n_fill; k++) {
    if (p->fill[k].T > Tmax) Tmax = p->fill[k].T;
    double u = sqrt(p->fill[k].u[0] * p->fill[k].u[0] + p->fill[k].u[1] * p->fill[k].u[1] +
                    p->fill[k].u[2] * p->fill[k].u[2]);
    if (u > Umax) Umax = u;
  }
  if (p->inflow_kind != ORC_INFLOW_NONE) {
    if (p->inflow_T > Tmax) Tmax = p->inflow_T;
    if (fabs(p->inflow_U) > Umax) Umax = fabs(p->inflow_U);
  }
  for (int f = 0; f < 6; f++) if (p->bc[f] == ORC_DIFFUSE && p->bc_T[f] > Tmax) Tmax = p->bc_T[f];
  if (p->plate_on && p->plate_T > Tmax) Tmax = p->plate_T;
  if (Tmax <= 0) Tmax = p->T_ref;
  double g0 = Umax + 5.0 * sqrt(2.0 * Tmax / p->mass);
  double sg0 = p->model == ORC_HS ? R->sigma_c * g0 : R->sigma_c * pow(g0 * g0, 1.0 - omega);
  R->gmax = (float*)malloc(sizeof(float) * R->Nc);
  for (int64_t c = 0; c < R->Nc; c++) R->gmax[c] = (float)sg0;
  /* inflow face cells on x- (reading R8) */
  R->open_face = (uint8_t*)calloc((size_t)p->ny * p->nz, 1);
  R->face_j = (int32_t*)malloc(sizeof(int32_t) * (size_t)p->ny * p->nz);
  R->face_k = (int32_t*)malloc(sizeof(int32_t) * (size_t)p->ny * p->nz);
  R->n_face = 0;
  for (int32_t k = 0; k < p->nz; k++)
    for (int32_t j = 0; j < p->ny; j++) {
      int open = 0;
      if (p->orifice_on) {
        double dy = j + 0.5 - p->orifice_cy, dz = k + 0.5 - p->orifice_cz;
        open = dy * dy + dz * dz <= p->orifice_r * p->orifice_r;
        R->open_face[(size_t)k * p->ny + j] = (uint8_t)open;
      }
      int face = (p->inflow_kind == ORC_INFLOW_GHOST) || (p->inflow_kind == ORC_INFLOW_EFFUSIVE && open);
      if (face) { R->face_j[R->n_face] = j; R->face_k[R->n_face] = k; R->n_face++; }
    }
  R->ghost_w = (p->inflow_U + 6.0 * sqrt(p->inflow_T)) * p->dt;
  R->ghost_x = p->inflow_n * R->ghost_w;
  if (p->inflow_kind == ORC_INFLOW_GHOST) R->insert_bound = (int64_t)R->n_face * (int64_t)ceil(R->ghost_x);
  else if (p->inflow_kind == ORC_INFLOW_EFFUSIVE) R->insert_bound = (int64_t)R->n_face * p->inflow_count;
  else R->insert_bound = 0;
  for (int a = 0; a < 3; a++) {
    R->x[a] = (float*)calloc((size_t)R->cap, sizeof(float));
    R->v[a] = (float*)calloc((size_t)R->cap, sizeof(float));
  }
  R->alive = (uint8_t*)calloc((size_t)R->cap, 1);
  R->cell = (int32_t*)malloc(sizeof(int32_t) * (size_t)R->cap);
  R->lcr = (int64_t*)malloc(sizeof(int64_t) * (size_t)R->cap);
  R->count = (int64_t*)calloc((size_t)R->Nc, sizeof(int64_t));
  R->start = (int64_t*)calloc((size_t)R->Nc, sizeof(int64_t));
  R->cand = (int64_t*)calloc((size_t)R->Nc, sizeof(int64_t));
  R->acc = (int32_t*)calloc((size_t)R->Nc, sizeof(int32_t));
  R->snap = (double*)calloc((size_t)R->n_slots * 5 * (size_t)R->Nc, sizeof(double));
  R->snap_done = (int32_t*)calloc((size_t)R->n_slots, sizeof(int32_t));
  return R;
}

void orc_destroy(orc_run* R) {
  if (!R) return;
  for (int a = 0; a < 3; a++) { free(R->x[a]); free(R->v[a]); }
  free(R->alive); free(R->cell); free(R->lcr); free(R->count); free(R->start); free(R->cand);
  free(R->acc); free(R->gmax); free(R->snap); free(R->snap_done); free(R->open_face);
  free(R->face_j); free(R->face_k);
  free(R);
}

/* Fault latch (reading R24): keep the most severe fault seen so far,
 * ENONFINITE > EINDEX > ECELL > EBOUNCE > ECAP, so the reported code does not
 * depend on the order in which particles or cells are visited. */
static int fault_rank(int32_t code) {
  switch (code) {
    case ORC_ENONFINITE: return 5;
    case ORC_EINDEX: return 4;
    case ORC_ECELL: return 3;
    case ORC_EBOUNCE: return 2;
    case ORC_ECAP: return 1;
    default: return 0;
  }
}
static void latch(orc_run* R, int32_t code) { if (fault_rank(code) > fault_rank(R->status)) R->status = code; }

/* --------------------------------------------------------- Generation -- */
/* Initial fill (SURVEY C-3): cells in increasing flat index,
 * exactly ppc particles each, store order (cell, k). */
int32_t orc_fill_initial(orc_run* R) {
  const orc_problem* p = &R->p;
  R->n = 0;
  for (int64_t c = 0; c < R->Nc; c++) {
    int32_t ix = (int32_t)(c % p->nx), iy = (int32_t)((c / p->nx) % p->ny), iz = (int32_t)(c / ((int64_t)p->nx * p->ny));
    int32_t ic[3] = {ix, iy, iz};
    const orc_fill* F = NULL;
    for (int k = 0; k < p->n_fill && !F; k++) {
      const orc_fill* G = &p->fill[k];
      int in = 1;
      for (int a = 0; a < 3; a++) in = in && ic[a] >= G->lo[a] && ic[a] < G->hi[a];
      if (in) F = G;
    }
    if (!F) continue;
    double sq = sqrt(F->T);
    for (int32_t k = 0; k < F->ppc; k++) {
      if (R->n >= R->cap) { latch(R, ORC_ECAP); return R->status; }
      uint32_t w[4], u[4];
      draw(R, (uint32_t)c, FILL_STEP, TAG_FILL, (uint32_t)k, 0, w);
      draw(R, (uint32_t)c, FILL_STEP, TAG_FILL, (uint32_t)k, 1, u);
      int64_t i = R->n++;
      for (int a = 0; a < 3; a++) R->x[a][i] = a < p->dim ? place(ic[a], w[a]) : 0.0f;
      double n1, n2, n3, n4;
      box_muller(u[0], u[1], &n1, &n2);
      box_muller(u[2], u[3], &n3, &n4);
      R->v[0][i] = (float)(F->u[0] + sq * n1);
      R->v[1][i] = (float)(F->u[1] + sq * n2);
      R->v[2][i] = (float)(F->u[2] + sq * n3);
      R->alive[i] = 1;
    }
  }
  return R->status;
}

/* Per-step Generation at the x- inflow face ("generate
 * particles at input boundaries"; SURVEY C-4, reading R8).  New particles are
 * appended at the tail in (face cell, k) order with their partial flight
 * already done; Motion does not move them again this step. */
int64_t orc_inflow_count(const orc_run* R, int32_t f, int32_t s) {
  if (R->p.inflow_kind == ORC_INFLOW_EFFUSIVE) return R->p.inflow_count;
  if (R->p.inflow_kind != ORC_INFLOW_GHOST) return 0;
  uint32_t w[4];
  draw(R, (uint32_t)f, (uint32_t)s, TAG_INFLOW_COUNT, 0, 0, w);
  return (int64_t)floor(R->ghost_x + u_co_d(w[0]));
}

int32_t orc_n_face(const orc_run* R) { return R->n_face; }

static void generation(orc_run* R, int32_t s) {
  const orc_problem* p = &R->p;
  if (p->inflow_kind == ORC_INFLOW_NONE) return;
  double sq = sqrt(p->inflow_T);
  float w_f = (float)R->ghost_w;
  for (int32_t f = 0; f < R->n_face; f++) {
    int64_t cnt = orc_inflow_count(R, f, s);
    for (int64_t k = 0; k < cnt; k++) {
      uint32_t a[4], b[4];
      draw(R, (uint32_t)f, (uint32_t)s, TAG_INFLOW_PARTICLE, (uint32_t)k, 0, a);
      draw(R, (uint32_t)f, (uint32_t)s, TAG_INFLOW_PARTICLE, (uint32_t)k, 1, b);
      double n1, n2, n3, n4;
      box_muller(b[0], b[1], &n1, &n2);
      box_muller(b[2], b[3], &n3, &n4);
      float x0[3], v[3], tau;
      x0[1] = place(R->face_j[f], a[1]);
      x0[2] = place(R->face_k[f], a[2]);
      if (p->inflow_kind == ORC_INFLOW_GHOST) {
        x0[0] = -(w_f * (float)u_oc_d(a[0]));
        v[0] = (float)(p->inflow_U + sq * n1);
        v[1] = (float)(0.0 + sq * n2);
        v[2] = (float)(0.0 + sq * n3);
        tau = R->dt_f;
      } else {
        x0[0] = 0.0f;
        v[0] = (float)(sq * sqrt(-2.0 * log(u_oc_d(a[3]))));
        v[1] = (float)(0.0 + sq * n1);
        v[2] = (float)(0.0 + sq * n2);
        tau = u_co(a[0]) * R->dt_f;
      }
      float xn[3];
      int kept = 1;
      for (int d = 0; d < 3; d++) {
        xn[d] = d < p->dim ? fmaf(v[d], tau, x0[d]) : 0.0f;
        if (d < p->dim && !(xn[d] >= 0.0f && xn[d] <= (float)axis_n(p, d))) kept = 0;
      }
      if (!kept) continue;
      if (R->n >= R->cap) { latch(R, ORC_ECAP); continue; }
      int64_t i = R->n++;
      for (int d = 0; d < 3; d++) { R->x[d][i] = xn[d]; R->v[d][i] = v[d]; }
      R->alive[i] = 1;
      R->inserted++;
    }
  }
}

/* ------------------------------------------------------------- Motion -- */
/* Full-accommodation diffuse re-emission (SURVEY C-5): normal speed
 * Rayleigh(sqrt(Tw)) into the domain, tangential N(0, Tw). */
void orc_diffuse_velocity(const orc_run* R, int32_t a, int32_t sign, double Tw, uint32_t idx,
                          uint32_t step, uint32_t bounce, float v[3]) {
  uint32_t w[4];
  draw(R, idx, step, TAG_WALL, bounce, 0, w);
  double sq = sqrt(Tw);
  double vn = sq * sqrt(-2.0 * log(u_oc_d(w[0])));
  double t1, t2;
  box_muller(w[1], w[2], &t1, &t2);
  int c1 = a == 0 ? 1 : 0;
  int c2 = a == 2 ? 1 : 2;
  v[a] = (float)(sign > 0 ? vn : -vn);
  v[c1] = (float)(0.0 + sq * t1);
  v[c2] = (float)(0.0 + sq * t2);
}

/* One particle, Motion with surface interaction (
 * reading R10 = SURVEY C-5): free flight x = fmaf(v, tau, x); the earliest
 * crossing of a non-specular, non-periodic face or of the plate is resolved
 * first (ties: lower axis, lower face, plate last); outflow kills; diffuse
 * re-emits and flies the remaining time; specular / periodic are applied per
 * axis to the final position.  Returns 1 if the particle died. */
static int motion_one(orc_run* R, int64_t i, int32_t s) {
  const orc_problem* p = &R->p;
  const int D = p->dim;
  float x[3], v[3];
  for (int a = 0; a < 3; a++) { x[a] = R->x[a][i]; v[a] = R->v[a][i]; }
  float tau = R->dt_f;
  for (int b = 0;; b++) {
    float x1[3] = {x[0], x[1], x[2]};
    for (int a = 0; a < D; a++) x1[a] = fmaf(v[a], tau, x[a]);
    int ev = -1;
    float tbest = INFINITY;
    for (int a = 0; a < D; a++)
      for (int f = 0; f < 2; f++) {
        int bc = p->bc[2 * a + f];
        if (bc == ORC_SPECULAR || bc == ORC_PERIODIC) continue;
        float L = f ? (float)axis_n(p, a) : 0.0f;
        int crossed = f ? (x1[a] > L) : (x1[a] < L);
        if (crossed) {
          float t = (L - x[a]) / v[a];
          if (t < tbest) { tbest = t; ev = 2 * a + f; }
        }
      }
    int s0 = 0;
    if (p->plate_on) {
      int pa = p->plate_axis, qa = p->plate_span_axis;
      float pc = (float)p->plate_pos;
      s0 = x[pa] >= pc;
      int s1 = x1[pa] >= pc;
      if (s0 != s1) {
        float t = (pc - x[pa]) / v[pa];
        float xq = fmaf(v[qa], t, x[qa]);
        if (xq >= (float)p->plate_lo && xq <= (float)p->plate_hi && t < tbest) { tbest = t; ev = 6; }
      }
    }
    if (ev < 0) { for (int a = 0; a < D; a++) x[a] = x1[a]; break; }
    float t = tbest < tau ? tbest : tau;
    if (ev < 6) {
      int a = ev / 2, f = ev % 2, bc = p->bc[ev];
      if (bc == ORC_OUTFLOW || bc == ORC_INFLOW) return 1;
      for (int c = 0; c < D; c++) if (c != a) x[c] = fmaf(v[c], t, x[c]);
      x[a] = f ? (float)axis_n(p, a) : 0.0f;
      if (p->orifice_on && a == 0 && f == 0) {
        int32_t j = (int32_t)floorf(x[1]), k = (int32_t)floorf(x[2]);
        if (j < 0) j = 0;
        if (j > p->ny - 1) j = p->ny - 1;
        if (k < 0) k = 0;
        if (k > p->nz - 1) k = p->nz - 1;
        if (R->open_face[(size_t)k * p->ny + j]) return 1;
      }
      if (b == MAX_BOUNCE) { latch(R, ORC_EBOUNCE); break; }
      orc_diffuse_velocity(R, a, f ? -1 : 1, p->bc_T[ev], (uint32_t)i, (uint32_t)s, (uint32_t)b, v);
    } else {
      int pa = p->plate_axis;
      float pc = (float)p->plate_pos;
      for (int c = 0; c < D; c++) if (c != pa) x[c] = fmaf(v[c], t, x[c]);
      x[pa] = s0 ? pc : nextafterf(pc, -INFINITY);
      if (b == MAX_BOUNCE) { latch(R, ORC_EBOUNCE); break; }
      orc_diffuse_velocity(R, pa, s0 ? 1 : -1, p->plate_T, (uint32_t)i, (uint32_t)s, (uint32_t)b, v);
    }
    tau = tau - t;
  }
  for (int a = 0; a < D; a++) {
    float L = (float)axis_n(p, a);
    if (p->bc[2 * a] == ORC_PERIODIC) {
      if (x[a] >= L) x[a] = x[a] - L;
      else if (x[a] < 0.0f) { x[a] = x[a] + L; if (x[a] >= L) x[a] = 0.0f; }
    } else {
      if (x[a] < 0.0f && p->bc[2 * a] == ORC_SPECULAR) { x[a] = -x[a]; v[a] = -v[a]; }
      else if (x[a] > L && p->bc[2 * a + 1] == ORC_SPECULAR) { x[a] = 2.0f * L - x[a]; v[a] = -v[a]; }
    }
  }
  for (int a = 0; a < 3; a++) { R->x[a][i] = x[a]; R->v[a][i] = v[a]; }
  return 0;
}

static void motion(orc_run* R, int32_t s, int64_t n_prev) {
  for (int64_t i = 0; i < n_prev; i++) {
    if (!R->alive[i]) continue;
    if (motion_one(R, i, s)) { R->alive[i] = 0; R->removed++; }
  }
}

/* ----------------------------------------------- Enumeration, Indexing -- */
/* Enumeration: cell = floor(x) per axis, clamped to the
 * grid (half-open cells, upper face of the domain belongs to the last cell). */
static void enumeration(orc_run* R) {
  const orc_problem* p = &R->p;
  for (int64_t i = 0; i < R->n; i++) {
    if (!R->alive[i]) { R->cell[i] = -1; continue; }
    int32_t ic[3] = {0, 0, 0};
    for (int a = 0; a < p->dim; a++) {
      float xa = R->x[a][i];
      int32_t L = axis_n(p, a);
      if (!(xa >= 0.0f && xa <= (float)L)) latch(R, ORC_EINDEX);
      int32_t c = xa >= 0.0f ? (int32_t)floorf(xa) : 0;
      if (!(xa >= 0.0f)) c = 0;
      if (c > L - 1) c = L - 1;
      ic[a] = c;
    }
    for (int a = 0; a < 3; a++)
      if (!isfinite(R->v[a][i])) latch(R, ORC_ENONFINITE);
    R->cell[i] = ic[0] + p->nx * (ic[1] + p->ny * ic[2]);
  }
}

/* Indexing: the readdressing array LCR
 * as a stable counting sort; within a cell, ascending store index (R11). */
static void indexing(orc_run* R) {
  memset(R->count, 0, sizeof(int64_t) * (size_t)R->Nc);
  for (int64_t i = 0; i < R->n; i++) if (R->cell[i] >= 0) R->count[R->cell[i]]++;
  int64_t acc = 0;
  for (int64_t c = 0; c < R->Nc; c++) { R->start[c] = acc; acc += R->count[c]; }
  int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)R->Nc);
  memcpy(cursor, R->start, sizeof(int64_t) * (size_t)R->Nc);
  for (int64_t i = 0; i < R->n; i++) if (R->cell[i] >= 0) R->lcr[cursor[R->cell[i]]++] = i;
  free(cursor);
}

/* ------------------------------------------------------- Interaction -- */
/* Isotropic unit vector, Marsaglia (1972) (reading R14): (p, q) = 2u - 1,
 * rejected while rho = p^2 + q^2 >= 1.  The first try uses words 2 and 3 of
 * the candidate's pair block w; further tries come two per COLL_DIR block. */
static void marsaglia(const orc_run* R, uint32_t c, uint32_t s, uint32_t k, const uint32_t w_pair[4], float e[3]) {
  uint32_t w[4] = {0, 0, w_pair[2], w_pair[3]};
  int h0 = 1;                                   /* the pair block offers one try: (w2, w3) */
  for (int32_t blk = -1; blk < 64; blk++) {
    if (blk >= 0) { draw(R, c, s, TAG_COLL_DIR, k, (uint32_t)blk, w); h0 = 0; }
    for (int h = h0; h < 2; h++) {
      float pp = 2.0f * u_co(w[2 * h]) - 1.0f;
      float qq = 2.0f * u_co(w[2 * h + 1]) - 1.0f;
      float rho = pp * pp + qq * qq;
      if (rho < 1.0f) {
        float sr = sqrtf(1.0f - rho);
        e[0] = 2.0f * pp * sr;
        e[1] = 2.0f * qq * sr;
        e[2] = 1.0f - 2.0f * rho;
        return;
      }
    }
  }
  e[0] = 0.0f; e[1] = 0.0f; e[2] = 1.0f;
}

/* NTC collisions in one cell (Bird's no-time-counter scheme, cited by the
 * paper at PAPER.md:48,93; readings R12-R15 = SURVEY C-8, R13 as amended):
 *   M = floor(1/2 N (N-1) F_N/V_c (sigma g)_max dt + u)
 *   candidate k, pair block (w0..w3): m = w0 N; i = m >> 32,
 *   j = lemire(m mod 2^32, N-1) (+1 if >= i); u = w1; Marsaglia's first
 *   try from (w2, w3), then COLL_DIR blocks;
 *   accept with probability sigma(g) g / (sigma g)_max, decided in fp64:
 *     HS : (u * ghat)^2 < g^2, ghat = (sigma g)_max / (pi d^2)   [no sqrt]
 *     VHS: u (sigma g)_max < sigma_c (g^2)^(1-omega)
 *   (sigma g)_max is frozen during the step; afterwards it becomes
 *   max((sigma g)_max, sigma g(max g^2)) (sigma g is monotone in g^2).
 * vel[] are the cell's particles in canonical order; returns accepted count. */
static int64_t interact(orc_run* R, int64_t c, int32_t s, int32_t N, float* vx, float* vy, float* vz,
                        float* gmax_c, int32_t* pairs, int64_t max_pairs, int64_t* n_cand) {
  *n_cand = 0;
  if (N < 2) return 0;
  double gm = (double)*gmax_c;
  double x = ((double)((int64_t)N * (N - 1)) * 0.5) * R->coef * gm;
  uint32_t w[4];
  draw(R, (uint32_t)c, (uint32_t)s, TAG_COLL_COUNT, 0, 0, w);
  int64_t M = (int64_t)floor(x + u_co_d(w[0]));
  if (M > 0xFFFFFF) { latch(R, ORC_ECELL); M = 0xFFFFFF; }
  *n_cand = M;
  const double ghat = gm / R->sigma_c;
  float maxg2 = 0.0f;
  int64_t acc = 0;
  for (int64_t k = 0; k < M; k++) {
    draw(R, (uint32_t)c, (uint32_t)s, TAG_COLL_PAIR, (uint32_t)k, 0, w);
    /* the pair from word 0 alone: i = floor(w0 N / 2^32), and j from the low
     * 32 bits of that product scaled to N - 1 (R13) */
    const uint64_t m = (uint64_t)w[0] * (uint64_t)N;
    int64_t i = (int64_t)(m >> 32);
    int64_t j = lemire((uint32_t)m, N - 1);
    if (j >= i) j++;
    float dx = vx[i] - vx[j], dy = vy[i] - vy[j], dz = vz[i] - vz[j];
    float g2 = (dx * dx + dy * dy) + dz * dz;
    if (g2 > maxg2) maxg2 = g2;
    int accept;
    if (R->p.model == ORC_HS) {
      double lhs = u_co_d(w[1]) * ghat;
      accept = lhs * lhs < (double)g2;
    } else {
      accept = u_co_d(w[1]) * gm < sigma_g(R, g2);
    }
    if (accept) {
      float e[3];
      marsaglia(R, (uint32_t)c, (uint32_t)s, (uint32_t)k, w, e);
      float cmx = (vx[i] + vx[j]) * 0.5f, cmy = (vy[i] + vy[j]) * 0.5f, cmz = (vz[i] + vz[j]) * 0.5f;
      float h = 0.5f * sqrtf(g2);
      vx[i] = cmx + h * e[0]; vy[i] = cmy + h * e[1]; vz[i] = cmz + h * e[2];
      vx[j] = cmx - h * e[0]; vy[j] = cmy - h * e[1]; vz[j] = cmz - h * e[2];
      if (pairs && acc < max_pairs) { pairs[2 * acc] = (int32_t)i; pairs[2 * acc + 1] = (int32_t)j; }
      acc++;
    }
  }
  if (M > 0) {
    double sgmax = sigma_g(R, maxg2);
    if (sgmax > gm) *gmax_c = (float)sgmax;
  }
  return acc;
}

int64_t orc_interact_cell(orc_run* R, int64_t c, int32_t step, int32_t N, float* vx, float* vy, float* vz,
                          float* gmax_inout, int32_t* pairs, int64_t max_pairs, int64_t* n_cand) {
  return interact(R, c, step, N, vx, vy, vz, gmax_inout, pairs, max_pairs, n_cand);
}

static void interaction(orc_run* R, int32_t s) {
  int64_t maxN = 0;
  for (int64_t c = 0; c < R->Nc; c++) if (R->count[c] > maxN) maxN = R->count[c];
  float* vx = (float*)malloc(sizeof(float) * (size_t)(maxN + 1));
  float* vy = (float*)malloc(sizeof(float) * (size_t)(maxN + 1));
  float* vz = (float*)malloc(sizeof(float) * (size_t)(maxN + 1));
  for (int64_t c = 0; c < R->Nc; c++) {
    int32_t N = (int32_t)R->count[c];
    const int64_t* L = R->lcr + R->start[c];
    for (int32_t q = 0; q < N; q++) { vx[q] = R->v[0][L[q]]; vy[q] = R->v[1][L[q]]; vz[q] = R->v[2][L[q]]; }
    int64_t nc;
    int64_t acc = interact(R, c, s, N, vx, vy, vz, &R->gmax[c], NULL, 0, &nc);
    for (int32_t q = 0; q < N; q++) { R->v[0][L[q]] = vx[q]; R->v[1][L[q]] = vy[q]; R->v[2][L[q]] = vz[q]; }
    R->cand[c] = nc;
    R->acc[c] = (int32_t)acc;
    R->candidates += nc;
    R->accepted += acc;
  }
  free(vx); free(vy); free(vz);
}

/* ------------------------------------------------------------ Sampling -- */
/* Sampling (array C, 121-123): per cell N, sum v,
 * sum |v|^2 in fp64, summed sequentially in LCR (canonical) order.  add = 1:
 * the sums are added to the slot's -- time averaging over Delta t_av >> Delta t
 * for steady problems -- and its sample count grows by one. */
static void sampling(orc_run* R, int32_t slot, int add) {
  double* S = R->snap + (size_t)slot * 5 * (size_t)R->Nc;
  for (int64_t c = 0; c < R->Nc; c++) {
    double sn = 0, sx = 0, sy = 0, sz = 0, se = 0;
    for (int64_t q = R->start[c]; q < R->start[c] + R->count[c]; q++) {
      int64_t i = R->lcr[q];
      double vx = (double)R->v[0][i], vy = (double)R->v[1][i], vz = (double)R->v[2][i];
      sn += 1.0; sx += vx; sy += vy; sz += vz;
      se += (vx * vx + vy * vy) + vz * vz;
    }
    if (add) {
      S[0 * R->Nc + c] += sn; S[1 * R->Nc + c] += sx; S[2 * R->Nc + c] += sy;
      S[3 * R->Nc + c] += sz; S[4 * R->Nc + c] += se;
    } else {
      S[0 * R->Nc + c] = sn; S[1 * R->Nc + c] = sx; S[2 * R->Nc + c] = sy;
      S[3 * R->Nc + c] = sz; S[4 * R->Nc + c] = se;
    }
  }
  R->snap_done[slot] = add ? R->snap_done[slot] + 1 : 1;
}

int32_t orc_sample(orc_run* R, int32_t slot) {
  if (slot < 0 || slot >= R->n_slots) return ORC_ESCHED;
  enumeration(R);
  indexing(R);
  sampling(R, slot, 0);
  return R->status;
}

int32_t orc_sample_add(orc_run* R, int32_t slot) {
  if (slot < 0 || slot >= R->n_slots) return ORC_ESCHED;
  if (!R->snap_done[slot]) memset(R->snap + (size_t)slot * 5 * (size_t)R->Nc, 0, sizeof(double) * 5 * (size_t)R->Nc);
  enumeration(R);
  indexing(R);
  sampling(R, slot, 1);
  return R->status;
}

int32_t orc_snap_count(const orc_run* R, int32_t slot) {
  if (slot < 0 || slot >= R->n_slots) return -1;
  return R->snap_done[slot];
}

/* ------------------------------------------------------------- Reorder -- */
/* Physical reordering of P in LCR order ("rearrange"),
 * dead particles dropped (reading R16). */
static void reorder(orc_run* R) {
  int64_t live = 0;
  for (int64_t c = 0; c < R->Nc; c++) live += R->count[c];
  for (int a = 0; a < 3; a++) {
    float* nx_ = (float*)malloc(sizeof(float) * (size_t)R->cap);
    float* nv_ = (float*)malloc(sizeof(float) * (size_t)R->cap);
    for (int64_t q = 0; q < live; q++) { nx_[q] = R->x[a][R->lcr[q]]; nv_[q] = R->v[a][R->lcr[q]]; }
    free(R->x[a]); free(R->v[a]);
    R->x[a] = nx_; R->v[a] = nv_;
  }
  memset(R->alive, 0, (size_t)R->cap);
  memset(R->alive, 1, (size_t)live);
  R->n = live;
}

/* ---------------------------------------------------------------- step -- */
int32_t orc_step(orc_run* R) {
  int32_t s = R->step;
  int64_t n_prev = R->n;
  generation(R, s);
  motion(R, s, n_prev);
  enumeration(R);
  indexing(R);
  interaction(R, s);
  if ((s + 1) % R->sample_every == 0) {
    int32_t slot = (s + 1) / R->sample_every - 1;
    if (slot < R->n_slots) sampling(R, slot, 0);
  }
  int K = R->p.reorder_every;
  if ((K > 0 && (s + 1) % K == 0) || R->cap - R->n < R->insert_bound) reorder(R);
  R->step = s + 1;
  return R->status;
}

int32_t orc_steps(orc_run* R, int32_t k) {
  for (int32_t q = 0; q < k; q++) orc_step(R);
  return R->status;
}

/* ------------------------------------------------------------ access -- */
int64_t orc_n_store(const orc_run* R) { return R->n; }
int32_t orc_step_index(const orc_run* R) { return R->step; }
int32_t orc_status(const orc_run* R) { return R->status; }
void orc_counters(const orc_run* R, int64_t out[4]) {
  out[0] = R->inserted; out[1] = R->removed; out[2] = R->candidates; out[3] = R->accepted;
}

int32_t orc_get_state(const orc_run* R, float* x, float* y, float* z, float* vx, float* vy, float* vz,
                      uint8_t* alive) {
  size_t n = (size_t)R->n;
  memcpy(x, R->x[0], n * 4); memcpy(y, R->x[1], n * 4); memcpy(z, R->x[2], n * 4);
  memcpy(vx, R->v[0], n * 4); memcpy(vy, R->v[1], n * 4); memcpy(vz, R->v[2], n * 4);
  memcpy(alive, R->alive, n);
  return 0;
}

int32_t orc_set_state(orc_run* R, int64_t n, const float* x, const float* y, const float* z, const float* vx,
                      const float* vy, const float* vz, const uint8_t* alive, int32_t step) {
  if (n < 0 || n > R->cap) return ORC_ECAP;
  size_t b = (size_t)n * 4;
  memcpy(R->x[0], x, b); memcpy(R->x[1], y, b); memcpy(R->x[2], z, b);
  memcpy(R->v[0], vx, b); memcpy(R->v[1], vy, b); memcpy(R->v[2], vz, b);
  memcpy(R->alive, alive, (size_t)n);
  R->n = n;
  R->step = step;
  return 0;
}

void orc_get_gmax(const orc_run* R, float* out) { memcpy(out, R->gmax, sizeof(float) * (size_t)R->Nc); }
void orc_set_gmax(orc_run* R, const float* in) { memcpy(R->gmax, in, sizeof(float) * (size_t)R->Nc); }

int64_t orc_get_index(const orc_run* R, int32_t* cell, int64_t* count, int64_t* start, int64_t* lcr) {
  int64_t live = 0;
  for (int64_t c = 0; c < R->Nc; c++) live += R->count[c];
  if (cell) memcpy(cell, R->cell, sizeof(int32_t) * (size_t)R->n);
  if (count) memcpy(count, R->count, sizeof(int64_t) * (size_t)R->Nc);
  if (start) memcpy(start, R->start, sizeof(int64_t) * (size_t)R->Nc);
  if (lcr) memcpy(lcr, R->lcr, sizeof(int64_t) * (size_t)live);
  return live;
}

void orc_get_cell_stats(const orc_run* R, int64_t* cand, int32_t* acc) {
  if (cand) memcpy(cand, R->cand, sizeof(int64_t) * (size_t)R->Nc);
  if (acc) memcpy(acc, R->acc, sizeof(int32_t) * (size_t)R->Nc);
}

int32_t orc_get_snap(const orc_run* R, int32_t slot, double* out) {
  if (slot < 0 || slot >= R->n_slots || !R->snap_done[slot]) return ORC_ESCHED;
  memcpy(out, R->snap + (size_t)slot * 5 * (size_t)R->Nc, sizeof(double) * 5 * (size_t)R->Nc);
  return 0;
}

/* ------------------------------------------------------------ Ensemble -- */
/* Pooled ratio estimates over runs, folded in ascending run id (reading
 * R18): rho = S_N F_N/V_c / n, u = S_v / S_N, T = (S_E/S_N - |u|^2)/3 (m=k=1,
 * 3 translational degrees of freedom); SE = leave-one-run-out jackknife. */
static void moments(double sn, double sx, double sy, double sz, double se, double fnum_vc, double nr,
                    double out[5]) {
  out[0] = sn * fnum_vc / nr;
  if (sn > 0) {
    double ux = sx / sn, uy = sy / sn, uz = sz / sn;
    out[1] = ux; out[2] = uy; out[3] = uz;
    out[4] = (se / sn - (ux * ux + uy * uy + uz * uz)) / 3.0;
  } else {
    out[1] = out[2] = out[3] = out[4] = NAN;
  }
}

/* Ensemble of one slot over runs (reading R18), each run's
 * sums holding m samples (m = 1: a snapshot; m > 1: time averaged):
 * density = S_N F_N/V_c / (n m). */
void orc_ensemble_m(int32_t n_runs, int64_t Nc, const double* sums, double fnum_vc, int32_t m, double* out) {
  const double mm = m > 0 ? (double)m : 1.0;
  for (int64_t c = 0; c < Nc; c++) {
    double tot[5] = {0, 0, 0, 0, 0};
    for (int32_t r = 0; r < n_runs; r++)
      for (int q = 0; q < 5; q++) tot[q] += sums[((size_t)r * 5 + q) * (size_t)Nc + c];
    double full[5];
    moments(tot[0], tot[1], tot[2], tot[3], tot[4], fnum_vc, (double)n_runs * mm, full);
    double* o = out + (size_t)c * 10;
    for (int q = 0; q < 5; q++) o[q] = full[q];
    if (n_runs < 2) { for (int q = 0; q < 5; q++) o[5 + q] = 0.0; continue; }
    double mean[5] = {0, 0, 0, 0, 0}, loo[5];
    double* th = (double*)malloc(sizeof(double) * 5 * (size_t)n_runs);
    for (int32_t r = 0; r < n_runs; r++) {
      double part[5];
      for (int q = 0; q < 5; q++) part[q] = tot[q] - sums[((size_t)r * 5 + q) * (size_t)Nc + c];
      moments(part[0], part[1], part[2], part[3], part[4], fnum_vc, (double)(n_runs - 1) * mm, loo);
      for (int q = 0; q < 5; q++) { th[r * 5 + q] = loo[q]; mean[q] += loo[q]; }
    }
    for (int q = 0; q < 5; q++) mean[q] /= (double)n_runs;
    for (int q = 0; q < 5; q++) {
      double ss = 0;
      for (int32_t r = 0; r < n_runs; r++) { double d = th[r * 5 + q] - mean[q]; ss += d * d; }
      o[5 + q] = sqrt((double)(n_runs - 1) / (double)n_runs * ss);
    }
    free(th);
  }
}

void orc_ensemble(int32_t n_runs, int64_t Nc, const double* sums, double fnum_vc, double* out) {
  orc_ensemble_m(n_runs, Nc, sums, fnum_vc, 1, out);
}
