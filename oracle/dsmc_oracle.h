/*
 * dsmc_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, sequential CPU oracle of the per-time-step unsteady DSMC update
 * of Bogdanov et al. (§1.1, Fig. 1, lines 93-130).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  It shares no code with the CUDA path (paper_cs_9902024_b200/):
 * its own Philox, its own structs, its own motion/indexing/collision/sampling.
 *
 * One oracle "run" is one statistically independent run i of the outer loop
 * (2) of Fig. 1; the RNG "shift" is the key (seed, run id).
 *
 * Parity status per function: see DESIGN.md §"Oracle pins".  Functions whose
 * full-physics result has no closed form (shock tube plateau, plate, jet) are
 * pinned only through invariants; DESIGN.md lists them as "parity unpinned"
 * beyond those invariants.
 */
#ifndef DSMC_ORACLE_H
#define DSMC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_SPECULAR = 0, ORC_PERIODIC = 1, ORC_DIFFUSE = 2, ORC_OUTFLOW = 3, ORC_INFLOW = 4 };
enum { ORC_HS = 0, ORC_VHS = 1 };
enum { ORC_INFLOW_NONE = 0, ORC_INFLOW_GHOST = 1, ORC_INFLOW_EFFUSIVE = 2 };
/* error / fault codes (same meaning as the product ABI, defined independently) */
enum { ORC_OK = 0, ORC_EINVAL = -1, ORC_ECLOCK = -2, ORC_EPARAM = -3, ORC_ECAP = -4,
       ORC_EINDEX = -5, ORC_ENONFINITE = -6, ORC_ESCHED = -8, ORC_EBOUNCE = -9, ORC_ECELL = -10 };
/* Run-time faults are latched by precedence, not by arrival (DESIGN.md reading
 * R24): the latched code is the most severe one seen so far, in the order
 * ENONFINITE > EINDEX > ECELL > EBOUNCE > ECAP. */

typedef struct {
  int32_t lo[3], hi[3];  /* cell box [lo, hi) per axis */
  int32_t ppc;           /* exact particles per cell */
  double T;              /* temperature (k = m = 1) */
  double u[3];           /* drift velocity */
} orc_fill;

typedef struct {
  int32_t dim, nx, ny, nz;
  double fnum_vc;                       /* F_N / V_c */
  int32_t model; double d_ref, omega, T_ref, mass;
  int32_t bc[6]; double bc_T[6];        /* faces x-,x+,y-,y+,z-,z+ */
  int32_t plate_on, plate_axis, plate_span_axis;
  double plate_pos, plate_lo, plate_hi, plate_T;
  int32_t orifice_on; double orifice_cy, orifice_cz, orifice_r;
  int32_t inflow_kind; double inflow_n, inflow_T, inflow_U; int32_t inflow_count;
  int32_t n_fill; orc_fill fill[4];
  double dt, dt_s, dt_L;
  uint32_t seed; int32_t n_runs, run_id0, reorder_every; int64_t cap_per_run;
} orc_problem;

typedef struct orc_run orc_run;

/* Philox4x32-10 block function (Salmon et al. 2011), written out here. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

orc_run* orc_create(const orc_problem* p, int32_t run_id, int32_t* err);
void     orc_destroy(orc_run* r);
int32_t  orc_fill_initial(orc_run* r);             /* Generation, initial fill */
int32_t  orc_step(orc_run* r);                     /* one Fig. 1 inner-loop step */
int32_t  orc_steps(orc_run* r, int32_t k);
int32_t  orc_sample(orc_run* r, int32_t slot);     /* explicit Sampling of current state */
int32_t  orc_sample_add(orc_run* r, int32_t slot); /* add current state's sums to the slot (time averaging) */
int32_t  orc_snap_count(const orc_run* r, int32_t slot); /* samples in the slot (0: never written) */

int64_t  orc_n_store(const orc_run* r);
int32_t  orc_step_index(const orc_run* r);
int32_t  orc_status(const orc_run* r);
void     orc_counters(const orc_run* r, int64_t out[4]); /* inserted, removed, candidates, accepted */
int32_t  orc_get_state(const orc_run* r, float* x, float* y, float* z,
                       float* vx, float* vy, float* vz, uint8_t* alive);
int32_t  orc_set_state(orc_run* r, int64_t n, const float* x, const float* y, const float* z,
                       const float* vx, const float* vy, const float* vz, const uint8_t* alive,
                       int32_t step);
void     orc_get_gmax(const orc_run* r, float* out);
void     orc_set_gmax(orc_run* r, const float* in);
/* last step's Enumeration/Indexing/Interaction (before any reorder) */
int64_t  orc_get_index(const orc_run* r, int32_t* cell_of_particle, int64_t* count,
                       int64_t* start, int64_t* lcr);
void     orc_get_cell_stats(const orc_run* r, int64_t* cand, int32_t* acc);
int32_t  orc_get_snap(const orc_run* r, int32_t slot, double* out /* [5][Nc] */);

/* single-cell Interaction on caller-given velocities in canonical order
 * (tests: NTC pair law).  Writes accepted pairs (i,j) into pairs[2*k]. */
int64_t  orc_interact_cell(orc_run* r, int64_t cell, int32_t step, int32_t N,
                           float* vx, float* vy, float* vz, float* gmax_inout,
                           int32_t* pairs, int64_t max_pairs, int64_t* n_cand);
/* diffuse re-emission draw (tests: KS against Rayleigh / normal) */
void     orc_diffuse_velocity(const orc_run* r, int32_t axis, int32_t sign, double Tw,
                              uint32_t idx, uint32_t step, uint32_t bounce, float v[3]);
/* inflow count of one face cell at one step (tests: flux formula) */
int64_t  orc_inflow_count(const orc_run* r, int32_t face, int32_t step);
int32_t  orc_n_face(const orc_run* r);

/* Ensemble over runs ("one processor analyzes the results"):
 * sums [n_runs][5][Nc] -> out [Nc][10] = rho,ux,uy,uz,T, then jackknife SEs. */
void     orc_ensemble_m(int32_t n_runs, int64_t Nc, const double* sums, double fnum_vc, int32_t m,
                        double* out /* [Nc][10] */);
void     orc_ensemble(int32_t n_runs, int64_t Nc, const double* sums, double fnum_vc,
                      double* out);

#ifdef __cplusplus
}
#endif
#endif
