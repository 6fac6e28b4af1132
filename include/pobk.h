/*
 * pobk.h -- C ABI of libpobk.so, the B200 (sm_100a) implementation of the hot path of the
 * preprocessed orthogonal block Kaczmarz method (POBK), arXiv 2401.00672.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (the paper's LaTeX source);
 * readings of the paper that this library implements are listed in DESIGN.md §3 and
 * SURVEY.md §8(c) (Z1-Z20).
 *
 * What the library computes (Alg 5, at row granularity):
 *   preprocess:  P from Reverse Cuthill-McKee, A~ = P A P^T (Eq 3.1),
 *                rows of A~ partitioned into categories of pairwise-orthogonal rows by the
 *                first-orthogonal rule iterated to maximal classes; schedule =
 *                Oclass categories (>= 2 rows) in ascending colour, then Nclass rows ascending.
 *   solve:       sweeps over the schedule; each category applies the block step Eq 1.3
 *                (P:34-37), which for pairwise-orthogonal rows collapses by Lemma 1
 *                 into simultaneous row projections Eq 1.2:
 *                    r_i = f~_i - a~_i . x~,  alpha_i = r_i / ||a~_i||^2,  x~ += alpha_i a~_i^T;
 *                stop when RSE = ||x - x*|| / ||x*|| < tol or at max_sweeps; then
 *                x = P^T x~.
 *   residual:    ||f - A x||_2 (the fused SpMV + norm of the convergence check).
 *
 * Conventions (all functions):
 *   - Every function returns pobk_status (0 = POBK_OK).  No C++ exception crosses the ABI.
 *     On error, pobk_last_error() returns a thread-local message naming the offending item.
 *   - Host input arrays are caller-owned, read-only and copied; the library keeps no pointer.
 *   - Device pointers ("_dev") are caller-owned allocations on the plan's device (e.g. torch
 *     tensors); the library never frees them.  Vectors are fp64, length m, in the USER frame.
 *   - The plan owns every internal host and device buffer; pobk_plan_destroy frees them.
 *   - A plan is not re-entrant: one solve at a time per plan.  Distinct plans are independent
 *     and may be used from different host threads.
 *   - Calls that touch the GPU set the plan's device and restore the caller's current device.
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).  Calls
 *     that return results to the host synchronise that stream before returning.
 */
#ifndef POBK_H_
#define POBK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POBK_ABI_VERSION 3

typedef struct pobk_plan_s* pobk_plan_t;
typedef int32_t pobk_status;

enum {
  POBK_OK = 0,
  POBK_ERR_ARG = 1,          /* NULL pointer, m < 1, bad option value, plan without device */
  POBK_ERR_BAD_CSR = 2,      /* row_ptr not monotone / row_ptr[0] != 0, column out of range,
                                columns unsorted or duplicated within a row */
  POBK_ERR_ZERO_ROW = 3,     /* ||a_i|| = 0 after dropping explicit zeros: Eq 1.2 undefined */
  POBK_ERR_UNSTABLE_THR = 4, /* thr > 0 and a row fails the Gershgorin guard (opts.guard = 1) */
  POBK_ERR_CUDA = 5,         /* a CUDA runtime call failed (message names it) */
  POBK_ERR_OOM = 6,          /* host or device allocation failed */
  POBK_ERR_NO_DEVICE = 7     /* operation needs a device plan (device >= 0) */
};

enum { POBK_TERM_CONVERGED = 0, POBK_TERM_MAX_SWEEPS = 1, POBK_TERM_NONFINITE = 2 };

enum {
  POBK_STOP_RSE = 0,    /* RSE = ||x~ - x~*|| / ||x~*||; needs xstar */
  POBK_STOP_RELRES = 1, /* ||f~ - A~ x~|| / ||f~|| (fused SpMV + norm every check) */
  POBK_STOP_NONE = 2    /* run exactly max_sweeps sweeps, no check (fixed-count parity) */
};

/* Sweep kernel families.  AUTO picks by size and thr. */
enum {
  POBK_KERNEL_AUTO = 0,
  POBK_KERNEL_LAUNCH = 1,    /* K1: one launch per category step, device-driven CUDA-graph loop */
  POBK_KERNEL_WAVEFRONT = 2, /* K2: persistent tiled wavefront, x~ tile-private in shared memory */
  POBK_KERNEL_SMEM = 3,      /* K3: one CTA, whole system resident in shared memory */
  POBK_KERNEL_CLUSTER = 4,   /* K4: one thread-block cluster, system in distributed shared memory */
  POBK_KERNEL_BLOCKS = 5     /* K5: the paper-literal k-block iteration (pobk_blocks_preprocess only) */
};

typedef struct {
  double thr;        /* 0 (default): structural orthogonality (disjoint supports, Z5/Z7);
                        > 0: |cos(a_i, a_l)| < thr counts as orthogonal, categories
                        may overlap and use the simultaneous update: every alpha of the step
                        at the same x, then per column x_c += alpha_i a_ic in ascending row
                        order (the oracle's order: bitwise; environment POBK_THR_ATOMIC=1:
                        fp64 atomics, order nondeterministic) -- K1/K3 only */
  int32_t reorder;   /* 1 (default): RCM; 0: identity (narrow-band matrices) */
  int32_t kernel;    /* POBK_KERNEL_*; default AUTO */
  int32_t tile_rows; /* K2 target rows per tile; 0 = auto */
  int32_t guard;     /* thr > 0 only: 1 = fail with POBK_ERR_UNSTABLE_THR when some row has
                        sum_{l in its category, l != i} |cos(a_i, a_l)| >= 1; default 0 */
} pobk_preprocess_opts;

typedef struct {
  double tol;           /* default 1e-6; stop when value < tol (strict) */
  int64_t max_sweeps;   /* default 500000: cap on the TOTAL sweep count, sweep_offset
                           included (the paper's "number of iterations exceeds 5e+5") */
  int32_t stop;         /* POBK_STOP_*; default POBK_STOP_RSE */
  int32_t check_every;  /* check after every k-th sweep; default 1 (needed for +-1 parity) */
  int64_t sweep_offset; /* resume: sweeps already applied to x0 by earlier calls (default 0).  The
                           sweeps of this call are numbered from sweep_offset + 1, so checks fall
                           on the same sweep numbers (multiples of check_every) and the cap on the
                           same total as in one uninterrupted solve; >= 0 */
  int32_t order;        /* POBK_ORDER_SCHEDULE (default): the paper's cyclic schedule (Alg 5 loop,
                           P:236-243); POBK_ORDER_RESIDUAL: every sweep applies the steps by
                           decreasing ||f~_K - A~_K x~||^2 / ||A~_K||_F^2 taken at the sweep start
                           (ties: ascending step), the greedy largest-residual rule of GRBK/GRMK
                            that POBK itself avoids; thr = 0 row-level plans,
                           runs on the launch path (reading R-G) */
} pobk_solve_opts;

enum { POBK_ORDER_SCHEDULE = 0, POBK_ORDER_RESIDUAL = 1 };

typedef struct {
  int64_t sweeps;        /* sweeps performed by this call */
  int32_t termination;   /* POBK_TERM_* (MAX_SWEEPS: the paper's "Inf"/"NAN" record) */
  int32_t kernel;        /* POBK_KERNEL_* actually used */
  double final_value;    /* last checked RSE or RELRES (NaN with POBK_STOP_NONE) */
  double solve_seconds;  /* CUDA-event time of the whole solve on `stream` (permute in .. out) */
  double sweep_seconds;  /* CUDA-event time of the sweep kernel(s) alone */
  int64_t launches;      /* kernels launched by this call (graph-launched nodes included) */
  int64_t sweeps_total;  /* sweep_offset + sweeps (the paper's iteration count IT) */
  double final_rse;      /* last checked RSE; NaN unless stop = POBK_STOP_RSE */
  double final_relres;   /* last checked ||f - A x|| / ||f||; NaN unless stop = POBK_STOP_RELRES */
} pobk_report;

void pobk_preprocess_opts_default(pobk_preprocess_opts* o);
void pobk_solve_opts_default(pobk_solve_opts* o);

/* Alg 5 steps 1-4.  Validates the 0-based CSR (row_ptr int64[m+1], col int32[nnz],
 * val fp64[nnz]; columns strictly increasing within a row), drops explicit zeros, computes the
 * RCM permutation (George-Liu start, (degree, index) ties, components by minimum index, full
 * reversal), the first-fit partition and schedule, and builds the device layout.
 * device >= 0: upload to that CUDA device; device = -1: host-only plan (queries only, no solve).
 * *out receives a new plan (NULL on error). */
pobk_status pobk_preprocess(int64_t m, const int64_t* row_ptr, const int32_t* col, const double* val,
                            const pobk_preprocess_opts* opts, int device, pobk_plan_t* out);

/* Sizes and preprocessing statistics; any output pointer may be NULL.  nsteps = number of
 * schedule steps = ncat, the number of first-fit categories: every category is one step -- the
 * Oclass categories (>= 2 rows, n_oclass of them) and the Nclass rows (singleton categories,
 * P:220); bandwidths are max |i - j| before/after RCM (Table 1). */
pobk_status pobk_plan_info(pobk_plan_t plan, int64_t* m, int64_t* nnz, int32_t* nsteps, int32_t* n_oclass,
                           int64_t* bw_before, int64_t* bw_after, double* preprocess_seconds);

/* perm[m]: the RCM permutation, perm[new] = old (Eq 3.1: f~ = P f means f~[i] = f[perm[i]]). */
pobk_status pobk_plan_get_perm(pobk_plan_t plan, int32_t* perm);

/* color[m] (first-fit colour of each RCM-frame row), cat_ptr[nsteps+1], cat_rows[m] (RCM-frame
 * rows in schedule order).  Any pointer may be NULL. */
pobk_status pobk_plan_get_partition(pobk_plan_t plan, int32_t* color, int32_t* cat_ptr, int32_t* cat_rows);

/* The K2 tiling (for tests): ntiles, and for each RCM-frame row its tile.  Either may be NULL. */
pobk_status pobk_plan_get_tiles(pobk_plan_t plan, int32_t* ntiles, int32_t* tile_of_row);

/* Device-layout statistics: kernel family chosen, K2 tiles and chunks, fraction
 * of nonzeros whose x~ column is tile-private (shared memory) and of rows that touch only private
 * columns, bytes of the K2 chunk stream. */
typedef struct {
  int32_t kernel;
  int32_t ntiles;
  int32_t nchunks;
  int32_t threads;   /* K2: threads per CTA of the sweep kernel (256 or 512), else 0 */
  double private_nnz_frac;
  double interior_row_frac;
  int64_t stream_bytes;
} pobk_layout_stats;
pobk_status pobk_plan_get_layout_stats(pobk_plan_t plan, pobk_layout_stats* out);

/* Iterate from x0 = x_dev (in/out, user frame) until the stop rule; x_dev receives x = P^T x~.
 * f_dev: right-hand side; xstar_dev: exact solution (required for POBK_STOP_RSE, else may be
 * NULL).  Blocks until *rep is filled.  opts NULL = defaults. */
pobk_status pobk_solve(pobk_plan_t plan, const double* f_dev, double* x_dev, const double* xstar_dev,
                       const pobk_solve_opts* opts, void* stream, pobk_report* rep);

/* Same as pobk_solve with HOST vectors: copies f, x0 (and x*) to the device, solves, copies x
 * back (end-to-end path).  Host buffers may be pageable; pinned memory copies faster. */
pobk_status pobk_solve_host(pobk_plan_t plan, const double* f, double* x, const double* xstar,
                            const pobk_solve_opts* opts, void* stream, pobk_report* rep);

/* R right-hand sides of ONE plan's matrix (Ax = f for R vectors f; the north star's
 * "batches of ... right-hand sides"), 1 <= R <= 8, in one sweep loop: each schedule step reads
 * every row of A~ once for all R (x~ and f~ R-interleaved), and applies Eq 1.2 to each right-hand
 * side in the per-row contract order, so right-hand side r's iterates and stop sweep are bitwise
 * those of its own pobk_solve.  Each right-hand side stops on its own rule (POBK_STOP_RSE, needs
 * xstar[r]; or POBK_STOP_NONE); POBK_STOP_RELRES is refused.  Row-level plans with thr = 0 only.
 * Arrays of R device pointers (x distinct, in/out); reps[R]; blocks until filled. */
pobk_status pobk_solve_multi(pobk_plan_t plan, int32_t R, const double* const* f_dev, double* const* x_dev,
                             const double* const* xstar_dev, const pobk_solve_opts* opts, void* stream,
                             pobk_report* reps);

/* Alg 5 for nb independent systems (one plan each, same device; the batched
 * configuration of the north star, one shard of a multi-GPU batch): every system stops on its
 * own rule.  All arguments are checked before anything is enqueued.
 * Arrays of nb device pointers; reps[nb].  Ordered after prior work on `stream`, and `stream`
 * waits for all of them.  When every plan is a K2 (wavefront) plan and L >= 2 of their grids fit
 * the device side by side (plans built with tile_rows covering at most 1/L of the SMs), system b
 * runs on internal stream b mod L (concurrent cooperative sweep kernels); otherwise back to back
 * on `stream`.  Results are identical either way.  Blocks until reps are filled. */
pobk_status pobk_solve_batch(pobk_plan_t* plans, int32_t nb, const double* const* f_dev, double* const* x_dev,
                             const double* const* xstar_dev, const pobk_solve_opts* opts, void* stream,
                             pobk_report* reps);

/* pobk_solve_batch with HOST vectors (the batched end-to-end path): arrays of nb host pointers
 * (f, x0 in / solution out, x* for POBK_STOP_RSE), same systems, stop rules, reports and results
 * as pobk_solve_batch.  With distinct plans on one device, the host->device copies of later
 * systems and the device->host copies of finished ones run on internal copy streams while other
 * systems solve (on concurrent lanes when pobk_solve_batch would use them, else on one internal
 * stream), so only the first inputs and the last solutions are not overlapped with sweeps; a
 * batch naming a plan twice goes through pobk_solve_host back to back.  The x pointers must be
 * distinct (POBK_ERR_ARG otherwise, before anything runs).  Each plan keeps a 3m
 * staging buffer on the device.  Host buffers may be pageable; the overlap needs pinned memory.
 * Ordered after prior work on `stream`; blocks until reps are filled and x holds the solutions. */
pobk_status pobk_solve_batch_host(pobk_plan_t* plans, int32_t nb, const double* const* f, double* const* x,
                                  const double* const* xstar, const pobk_solve_opts* opts, void* stream,
                                  pobk_report* reps);

/* *out = ||f - A x||_2 in the user frame (fused SpMV + squared-norm kernel, deterministic
 * two-level reduction): the residual of Ax = f whose ratio to ||f|| is the RELRES stop
 * (SURVEY Z13), the paper's RSE needing x*.  Device vectors; result returned to the host. */
pobk_status pobk_residual_norm(pobk_plan_t plan, const double* f_dev, const double* x_dev, void* stream,
                               double* out);

/* *out = sum_{row_begin <= i < row_end} (f_i - a_i . x)^2 over USER-frame rows (the per-rank part
 * of a row-sharded residual for the convergence check; combine across ranks with an
 * all-reduce SUM, then sqrt). */
pobk_status pobk_residual_sumsq_rows(pobk_plan_t plan, int64_t row_begin, int64_t row_end, const double* f_dev,
                                     const double* x_dev, void* stream, double* out);

/* ---- The paper-literal variant: k uniform row blocks (Alg 5 as written).
 * Steps: RCM; blocks 1..k-1 take floor(m/k) consecutive rows of A~, block k the rest
 * (P:207); the centroid cosine table C(i,j) = |(A-bar_i, A-bar_j)| / (||A-bar_i|| ||A-bar_j||)
 * (absolute value: DESIGN.md §3); C(i,j) < thr counts as orthogonal and each unused block
 * pairs with the first unused later block orthogonal to it (Oclass pairs), the rest is Nclass
 * (P:220).  One iteration applies every pair (tau1 then tau2) and then every Nclass block, each
 * as the block projection x~ += A_tau^+ (f~_tau - A_tau x~) (Eq 3.3) with
 * A_tau^+ = A_tau^T (A_tau A_tau^T)^-1 (Lemma 1: full-row-rank blocks; a
 * rank-deficient block fails with POBK_ERR_ARG).  The dense Gram inverses are built once at
 * preprocessing (8 b^2 bytes per block of b rows; blocks above 20,000 rows are refused).
 * The returned plan is solved with pobk_solve / pobk_solve_host (kernel POBK_KERNEL_BLOCKS);
 * plan_get_partition reports colour = block id, cat_ptr = block boundaries. */
typedef struct {
  int32_t k;       /* number of blocks, 1 <= k <= m (the paper uses k < 20) */
  double thr;      /* orthogonality threshold on C, 0 <= thr < 1 */
  int32_t reorder; /* 1 (default): RCM; 0: identity */
} pobk_blocks_opts;

pobk_status pobk_blocks_preprocess(int64_t m, const int64_t* row_ptr, const int32_t* col, const double* val,
                                   const pobk_blocks_opts* opts, int device, pobk_plan_t* out);

/* The k-block layout: k; block_ptr[k+1] (RCM-frame row boundaries); cos_table[k*k] (row-major
 * C); pairs[2*npairs] (Oclass, 0-based block ids, in iteration order); nclass[nnclass]; the
 * Definition 1-2 diagnostics zn (orthogonality proportion) and nn (non-orthogonality severity),
 * P:512-516, on the table with entries < thr set to 0.  Array outputs may be NULL; pairs and
 * nclass need room for k entries. */
pobk_status pobk_blocks_info(pobk_plan_t plan, int32_t* k, int64_t* block_ptr, double* cos_table, int32_t* pairs,
                             int32_t* npairs, int32_t* nclass, int32_t* nnclass, double* zn, double* nn);

void pobk_plan_destroy(pobk_plan_t plan);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* pobk_last_error(void);

int32_t pobk_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* POBK_H_ */
