/*
 * dsmc.h -- C ABI of libdsmc.so, the B200 (sm_100a) batched unsteady-DSMC step.
 *
 * What it computes: the inner loop (1) of the paper's Fig. 1 (PAPER.md:93-116,
 * §1.1) -- Generation, Motion with surface interaction, Enumeration and
 * Indexing into the readdressing array LCR, Interaction (per cell), Sampling
 * of cell macroparameters into the array C -- for n statistically independent
 * runs at once (the outer loop (2), becomes a batch axis).
 * The random number generator is "shifted" per run (PAPER.md:113-115,
 * 435-437) by keying a counter-based Philox4x32-10 with (seed, run id).
 * The exact semantics of every step are DESIGN.md readings R1-R24.
 *
 * Conventions for every entry point:
 *   - Return value: DSMC_OK (0) or a negative dsmc_rc code.  No C++
 *     exception, abort or CUDA error escapes the boundary; the message of the
 *     last failure on the calling thread is dsmc_last_error().
 *   - Device buffers are allocated and owned by the CALLER (the Python binding
 *     uses torch), sized by dsmc_query_sizes(); the library borrows them from
 *     dsmc_create() until dsmc_destroy() and allocates no device memory on the
 *     DSMC path.  A context owns its CUDA graph (and graph exec), a capture
 *     stream, a second stream and two events for the graph's heavy-tile branch,
 *     released by dsmc_destroy.  The one exception is the test hook
 *     dsmc_selftest_philox, which allocates and frees its own scratch buffers.
 *   - All calls are asynchronous on the caller's CUDA stream except those
 *     marked SYNC, which synchronise that stream.  Device-side faults
 *     (capacity, indexing, non-finite velocity, bounce limit, cell size) are
 *     latched in the control block and returned by the next SYNC call; when
 *     several occur the most severe is kept, ENONFINITE > EINDEX > ECELL >
 *     EBOUNCE > ECAP (reading R24), so the code does not depend on thread order.
 *   - Store order: run r owns particle slots [r*stride, r*stride + cap) of each
 *     SoA array (x, y, z, vx, vy, vz); "store index" i of run r is the offset
 *     inside that window.  Host arrays passed to the test/checkpoint hooks are
 *     in store order.
 *   - Thread safety: a dsmc_ctx is used by one host thread at a time.
 *   - Environment switches read by dsmc_create (measurement A/B only; results are
 *     bit-identical with or without them): DSMC_STATIC_CELLS=1 disables the
 *     heavy-tile queue (static block-per-tile mapping, NEXT-1); DSMC_CAPW=<n>
 *     overrides the warp-tile staging capacity; DSMC_CARVEOUT=<percent> sets the
 *     collide kernel's preferred shared-memory carveout; DSMC_COMPACT=0/1 forces
 *     the sparse-problem tile list (k_collide_triage) off or on; DSMC_NO_BRANCH=1
 *     keeps the heavy tiers on the main stream of the graph.
 */
#ifndef DSMC_H
#define DSMC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DSMC_OK = 0,
  DSMC_EINVAL = -1,    /* null pointer, bad dim/grid/run range, stride overflow */
  DSMC_ECLOCK = -2,    /* need 0 < dt <= dt_s <= dt_L, dt_s = k dt, dt_L = k' dt_s (Fig. 1 caption) */
  DSMC_EPARAM = -3,    /* T <= 0, omega outside [1/2, 1], bad boundary combination */
  DSMC_ECAP = -4,      /* capacity exceeded (latched: insertions beyond cap are dropped) */
  DSMC_EINDEX = -5,    /* live particle outside the domain after Motion (latched) */
  DSMC_ENONFINITE = -6,/* non-finite velocity (latched) */
  DSMC_ECUDA = -7,     /* CUDA runtime error (message in dsmc_last_error) */
  DSMC_ESCHED = -8,    /* reading an unwritten sample slot / slot out of range */
  DSMC_EBOUNCE = -9,   /* more than 8 diffuse bounces in one step (latched) */
  DSMC_ECELL = -10     /* a cell holds more particles than the collide path supports (latched) */
} dsmc_rc;

/* boundary kinds per face (x-, x+, y-, y+, z-, z+) */
enum { DSMC_SPECULAR = 0, DSMC_PERIODIC = 1, DSMC_DIFFUSE = 2, DSMC_OUTFLOW = 3, DSMC_INFLOW = 4 };
/* collision models: hard sphere, variable hard sphere (Bird) */
enum { DSMC_HS = 0, DSMC_VHS = 1 };
/* Generation at the x- face: none, drifting-Maxwellian ghost buffer, fixed-count effusion */
enum { DSMC_INFLOW_NONE = 0, DSMC_INFLOW_GHOST = 1, DSMC_INFLOW_EFFUSIVE = 2 };

typedef struct {
  int32_t lo[3], hi[3];  /* cell box [lo, hi) per axis */
  int32_t ppc;           /* exact particles per cell (reading R7) */
  double T;              /* temperature, k = m = 1 */
  double u[3];           /* drift velocity */
} dsmc_fill_region;

/* The problem statement: grid and cells, the clock
 * (dt, dt_s, dt_L), n runs, the physics the paper leaves to Bird (model),
 * boundaries, initial fill and inflow.  Passed by pointer, copied and
 * validated in dsmc_create. */
typedef struct {
  int32_t dim, nx, ny, nz;                 /* 1..3 spatial dims, unit cells; ny = nz = 1 below dim */
  double fnum_vc;                          /* F_N / V_c: the only scale NTC needs (0 = collisionless) */
  int32_t model; double d_ref, omega, T_ref, mass;
  int32_t bc[6]; double bc_T[6];           /* per face kind and wall temperature */
  int32_t plate_on, plate_axis, plate_span_axis;   /* zero-thickness diffuse plate (dim 2) */
  double plate_pos, plate_lo, plate_hi, plate_T;
  int32_t orifice_on; double orifice_cy, orifice_cz, orifice_r;  /* open disk in the x- wall (dim 3) */
  int32_t inflow_kind; double inflow_n, inflow_T, inflow_U; int32_t inflow_count;
  int32_t n_fill; dsmc_fill_region fill[4];
  double dt, dt_s, dt_L;                   /* time step, sample interval, run length */
  uint32_t seed; int32_t n_runs, run_id0;  /* batch run r uses Philox key (seed, run_id0 + r) */
  int32_t reorder_every; int64_t cap_per_run;  /* physical reorder period K (0 = only on capacity), P rows per run */
} dsmc_problem;

/* Bytes of each caller-owned device buffer for a problem. */
typedef struct {
  size_t P;        /* particle array P: 2 halves x 6 fp32 SoA arrays x n_runs*stride */
  size_t key;      /* uint32 per particle slot: enumerated (run, cell) key */
  size_t lcr;      /* uint32 per particle slot: the readdressing array LCR */
  size_t cell;     /* uint32 per (run, cell): counts -> starts -> segment ends */
  size_t gmax;     /* fp32 per (run, cell): (sigma g)_max of NTC */
  size_t C;        /* fp64 [n_slots][5][n_runs*Nc]: array C of sampled sums N, Sv, S|v|^2 */
  size_t ctl;      /* control block (step, status, per-run counts/flags/counters) */
  size_t scratch;  /* scan partials, inflow counts, macro staging, debug arrays */
  int64_t stride;  /* particle slots per run window (cap rounded up to 32) */
  int64_t n_cells; /* Nc = nx*ny*nz */
  int32_t n_steps, sample_every, n_slots;
} dsmc_sizes;

typedef struct { void *P, *key, *lcr, *cell, *gmax, *C, *ctl, *scratch; } dsmc_buffers;

typedef struct dsmc_ctx dsmc_ctx;

/* Validate *prob and fill *out.  debug != 0 adds per-cell candidate/accept
 * arrays to scratch and makes the collide kernel write the canonical LCR back. */
int dsmc_query_sizes(const dsmc_problem* prob, int32_t debug, dsmc_sizes* out);

/* Create a context on the caller's stream (cudaStream_t as void*; NULL = legacy
 * default stream) over caller-owned device buffers; initialises the control
 * block, (sigma g)_max = sigma(g0) g0 (reading R13) and captures the step graph.
 * Ownership of *ctx passes to the caller (release with dsmc_destroy). */
int dsmc_create(const dsmc_problem* prob, const dsmc_buffers* buf, int32_t debug, void* stream,
                dsmc_ctx** ctx);

/* Generation, initial fill (reading R7): every run's store is
 * rebuilt with exactly ppc particles per filled cell in (cell, k) order;
 * resets the step counter, counters and sample slots. */
int dsmc_generate(dsmc_ctx* ctx);

/* nsteps inner-loop steps of Fig. 1 for all runs: inflow
 * Generation, Motion + surface interaction, Enumeration, Indexing (LCR),
 * Interaction (NTC), Sampling into slot k when (s+1) dt = k dt_s, physical
 * reorder every reorder_every steps.  One CUDA-graph launch per step. */
int dsmc_step(dsmc_ctx* ctx, int32_t nsteps);

/* Explicit Sampling of the current state into slot (re-enumerates; no collisions). */
int dsmc_sample(dsmc_ctx* ctx, int32_t slot);

/* Time averaging for steady problems ("we have to increase the
 * time interval of averaging ... after steady state is achieved", Delta t_av >>
 * Delta t): ADDS the current state's per-cell sums (N, sum v, sum |v|^2, fp64)
 * to slot `slot` of array C and counts one more sample in it; a slot never
 * written before starts from zero.  dsmc_read_macros then divides the density by
 * n_runs * m (m = samples in the slot); velocity and temperature are pooled
 * ratios of the accumulated sums (reading R18).  A scheduled Sampling of the
 * unsteady clock, or dsmc_sample, overwrites the slot (m = 1).  Asynchronous;
 * DSMC_ESCHED for a slot out of range. */
int dsmc_sample_add(dsmc_ctx* ctx, int32_t slot);

/* SYNC. Samples accumulated in slot (0: never written; 1: a snapshot). */
int dsmc_slot_samples(dsmc_ctx* ctx, int32_t slot, int32_t* out);

/* SYNC. Ensemble analysis of one slot: per cell, pooled
 * over runs in ascending run id, rho, ux, uy, uz, T then their leave-one-run-
 * out jackknife standard errors -> host out[Nc][10] (fp64). */
int dsmc_read_macros(dsmc_ctx* ctx, int32_t slot, double* out);

/* SYNC. Raw per-run sums of one slot -> host out[5][n_runs*Nc] (fp64). */
int dsmc_read_sums(dsmc_ctx* ctx, int32_t slot, double* out);

/* The paper's single exchange across processors ("the data
 * exchange between processors goes after all calculation are finished. Only one
 * processor sequentially analyzes the results"), for a job whose runs are
 * sharded over several contexts (one per GPU).
 *
 * dsmc_slot_sums_ptr: DEVICE pointer (borrowed, valid until dsmc_destroy; the
 * caller-owned C buffer) to slot `slot`'s sums, [5][n_runs*Nc] fp64 -- the
 * send buffer of a collective (an all-gather over NVLink) without a host copy.
 * Asynchronous-safe: no stream work.  DSMC_ESCHED for a slot out of range.
 *
 * dsmc_read_macros_gathered: SYNC.  Ensemble analysis of one slot over
 * n_blocks * n_runs runs.  sums_dev: DEVICE array [n_blocks][5][n_runs*Nc]
 * fp64; block b holds the slot sums of the context with runs
 * [b*n_runs, (b+1)*n_runs) of the job (every context built with the same
 * problem, n_runs and schedule; the blocks in ascending run id, i.e. rank
 * order).  The fold over runs is in ascending global run id, exactly as
 * dsmc_read_macros folds one context's runs, so the result is bit-identical to
 * one context holding all the runs.  Samples per run (m, R23) are this
 * context's for the slot.  out: host [Nc][10] as dsmc_read_macros.  Borrowed
 * sums_dev is only read, on this context's stream; DSMC_EINVAL if it is not
 * device memory or n_blocks < 1; DSMC_ESCHED if the slot is unwritten here. */
int dsmc_slot_sums_ptr(dsmc_ctx* ctx, int32_t slot, const double** out);
int dsmc_read_macros_gathered(dsmc_ctx* ctx, int32_t slot, const double* sums_dev, int32_t n_blocks,
                              double* out);

/* SYNC. Returns the latched device fault (or OK); counters_out (may be NULL)
 * receives per run {inserted, removed, candidates, accepted, n_store, step,
 * live, particle_steps, max_ppc} as int64[n_runs][DSMC_STATUS_COLS];
 * particle_steps accumulates, per step, the live particles after Generation
 * (the bench metric's numerator); max_ppc is the largest particle count of one
 * cell at the last Indexing (the cell-occupancy skew). */
#define DSMC_STATUS_COLS 9
int dsmc_status(dsmc_ctx* ctx, int64_t* counters_out);

/* SYNC. Checkpoint / test hooks, host arrays in store order of run `run`.
 * get_state: n_out receives the store length; arrays need cap entries;
 * alive[i] = 0 for removed slots not yet compacted. */
int dsmc_get_state(dsmc_ctx* ctx, int32_t run, int64_t* n_out, float* x, float* y, float* z,
                   float* vx, float* vy, float* vz, uint8_t* alive);
/* set_state: replaces run `run`'s store (n <= cap) and sets the batch step
 * counter.  alive may be NULL (all live): the copies then read the caller's
 * arrays directly (pinned host memory gives full-speed H2D). */
int dsmc_set_state(dsmc_ctx* ctx, int32_t run, int64_t n, const float* x, const float* y,
                   const float* z, const float* vx, const float* vy, const float* vz,
                   const uint8_t* alive, int32_t step);
int dsmc_get_gmax(dsmc_ctx* ctx, int32_t run, float* out /* [Nc] */);
int dsmc_set_gmax(dsmc_ctx* ctx, int32_t run, const float* in /* [Nc] */);
/* Last step's index of run `run` (debug contexts only): count[Nc], start[Nc]
 * (relative to the run), canonical lcr[live] as run-local store indices,
 * cand[Nc] NTC candidates and acc[Nc] accepted pairs per cell; returns live
 * count via *live_out. */
int dsmc_get_index(dsmc_ctx* ctx, int32_t run, int64_t* live_out, int64_t* count, int64_t* start,
                   int64_t* lcr, int64_t* cand, int32_t* acc);

/* SYNC. Test-only: n Philox4x32-10 blocks on the device for counters
 * ctr[4n], key (k0,k1) -> out[4n]; and the same through cuRAND's
 * curand_Philox4x32_10 -> out_ref[4n] (may be NULL). Host arrays. */
int dsmc_selftest_philox(int64_t n, const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out,
                         uint32_t* out_ref);

/* Number of kernel launches one dsmc_step issues (graph nodes that are kernels). */
int dsmc_kernels_per_step(dsmc_ctx* ctx, int32_t* out);

/* SYNC per step. Same work as dsmc_step, issued kernel by kernel (no graph)
 * with a CUDA event pair around each launch on the context stream; adds each
 * launch's duration in ms to ms_accum[slot] where slot = dsmc_kernel_name
 * index (ms_accum needs DSMC_MAX_KERNELS entries, zeroed by the caller). */
#define DSMC_MAX_KERNELS 16
int dsmc_step_timed(dsmc_ctx* ctx, int32_t nsteps, double* ms_accum, int64_t* launches);
/* Name of kernel slot k (0 <= k < DSMC_MAX_KERNELS) or "" if unused. */
const char* dsmc_kernel_name(int32_t k);

int dsmc_destroy(dsmc_ctx* ctx);
const char* dsmc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
