/*
 * rhpdhg_cuda.h — the thin C ABI between the C++ host solver (librhpdhg.so,
 * the reference-API mirror) and the CUDA device library (librhp_cuda.so).
 *
 * Plain C types only: pointers, sizes, doubles. One rhp_ctx owns one solve's
 * device state (matrices, iterate, anchor, caches, schedules, CUDA graph,
 * optional NCCL communicator) on one GPU. Host buffers passed in are always in
 * the ORIGINAL row/column order of the LP; the device stores rows and columns
 * permuted by row-length bin and the ctx maps between them.
 *
 * Which reference code each entry replaces (paths under /root/reference/proj):
 *   rhp_create          SparseMatrix ctor CSR/CSC build   src/sparse_matrix.cpp:20-65
 *   rhp_scale           ruiz_equilibrate, pock_chambolle_scale, apply_scales
 *                                                        src/scaling.cpp:10-81
 *   rhp_power_*         power_iteration_norm's loop body src/pdhg.cpp:138-152
 *   rhp_set_step        StepConfig primal/dual steps     include/rhpdhg/pdhg.hpp:14-26
 *   rhp_reset_iterate   Iterate::zeros + anchor/snapshot src/lp_problem.cpp:98-107, src/solver.cpp:91-103
 *   rhp_run_block       loop body of solve(): halpern_reflected_step -> pdhg_step
 *                       -> fixed_point_residual -> check_restart, k/total
 *                       bookkeeping                      src/solver.cpp:147-181,
 *                                                        src/restart.cpp:23-69, src/pdhg.cpp:34-115
 *   rhp_kkt             kkt_check + kkt_residuals sums   src/solver.cpp:32-49, src/termination.cpp:58-118
 *   rhp_restart         do_restart (anchor, k, residuals) src/restart.cpp:71-83
 *   rhp_spmv            SparseMatrix::multiply{,_transpose} src/sparse_matrix.cpp:67-87
 *   rhp_op_pdhg         pdhg_step, halpern_reflected_step src/pdhg.cpp:34-65, src/restart.cpp:35-52
 *   rhp_op_sums         quadratic_form / distance2 / norm2 sums src/pdhg.cpp:68-75, src/restart.cpp:8-21
 *   rhp_op_mul          unscale_iterate                   src/scaling.cpp:83-94
 * The PID weight update (src/restart.cpp:85-120), the termination test
 * (src/termination.cpp:120-124) and all exception mapping stay on the host.
 *
 * Every function returns 0 on success or an RHPDHG_E_* code (rhpdhg_c.h);
 * rhp_last_error() gives the thread-local message.
 */
#ifndef RHPDHG_CUDA_H_
#define RHPDHG_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#include "rhpdhg_c.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rhp_ctx rhp_ctx;

/* Device / distribution options. world_size > 1 row-partitions A across
 * ranks (one process per GPU); nccl_id is the 128-byte ncclUniqueId created
 * by rank 0 with rhp_nccl_unique_id() and broadcast by the caller. The LP
 * view passed to rhp_create is always the FULL problem; each rank keeps its
 * row block. */
typedef struct rhp_options {
  int32_t device;        /* CUDA device ordinal */
  int32_t rank;          /* 0 */
  int32_t world_size;    /* 1 */
  int32_t use_graph;     /* 1: CUDA graph with a conditional WHILE node per block */
  int64_t block_limit;   /* max PDHG iterations per device block (default 64) */
  const void* nccl_id;   /* 128 bytes when world_size > 1, else NULL */
  int32_t resident;      /* small-LP cluster-resident blocks: -1 auto, 0 off, 1 on */
  /* locality relabelling of rows and columns at ingest (ingest.cu
   * maybe_relabel): 0 auto (large gathered vectors, kept when it cuts the
   * gather sectors), < 0 off, > 0 forced; single-GPU contexts only. The
   * RHP_LOCALITY environment variable overrides it. */
  int32_t locality;
  /* In-process collective group (rhp_local_group_create) instead of NCCL:
   * world_size contexts of ONE process, each driven by its own host thread,
   * exchange through device memory with rank-ordered reductions. Lets the
   * row-partitioned engine run at world_size > 1 on a single GPU (tests). */
  const void* local_group;
} rhp_options;

/* Step and restart parameters of the device loop. Derived quantities are
 * computed on the host with the reference's exact expressions:
 *   tau = eta/omega, sigma = eta*omega (pdhg.hpp:18-19), sigma_inv = 1/sigma
 *   (pdhg.cpp:50), primal_scale = omega/eta, dual_scale = 1/(eta*omega)
 *   (pdhg.cpp:70-71). */
typedef struct rhp_step {
  double eta, omega, gamma;
  double tau, sigma, sigma_inv, primal_scale, dual_scale;
  double beta_sufficient, beta_necessary, beta_artificial;
  int64_t check_interval;
  int64_t iteration_limit;
  int32_t restarts_enabled;
  int32_t record_history;
} rhp_step;

/* What one device block of PDHG iterations ended with. */
typedef struct rhp_block_out {
  int64_t iterations_done; /* in this block */
  int64_t total;           /* RestartState::total */
  int64_t k;               /* RestartState::k */
  int32_t verdict;         /* RestartCondition: 0 none, 1 sufficient, 2 necessary, 3 artificial */
  int32_t check_due;       /* total % check_interval == 0 || verdict != none */
  int32_t breakdown;       /* indefinite canonical norm (pdhg.cpp:114) */
  int32_t pad_;
  double r_last;           /* fixed-point residual of the last iteration */
  double r_anchor, r_prev;
  double q_last;           /* radicand when breakdown */
  /* PID inputs for the current Halpern iterate (restart.cpp:86-91):
   * ||x - x_snapshot||^2, ||y - y_snapshot||^2, ||x||^2, ||y||^2 */
  double x_dist2, y_dist2, x_norm2, y_norm2;
} rhp_block_out;

/* Raw device sums of one KKT evaluation (termination.cpp:58-118) on the
 * original instance; the host turns them into KktResiduals. */
typedef struct rhp_kkt_sums {
  double primal_value;   /* c^T x */
  double py, pr;         /* p(-y; con bounds), p(-r; var bounds), finite terms */
  double viol2;          /* ||A x - proj_[L,U](A x)||^2 */
  double eq2, cone2;     /* dual equality / cone residual squares */
  int64_t py_inf, pr_inf;/* count of +inf terms */
  int64_t nan_x, nan_y;  /* count of NaN entries */
} rhp_kkt_sums;

/* Scaling results, for parity tests (original order). */
typedef struct rhp_scaled_out {
  double* csr_values;  /* [nnz] CSR order of the reference (row-major)       may be NULL */
  double* csc_values;  /* [nnz] CSC order of the reference (column-major)    may be NULL */
  double* row_scale;   /* [m] cumulative D_row */
  double* col_scale;   /* [n] cumulative D_col */
  double* objective;   /* [n] scaled c */
  double* var_lb;      /* [n] */
  double* var_ub;      /* [n] */
  double* con_lb;      /* [m] */
  double* con_ub;      /* [m] */
} rhp_scaled_out;

typedef struct rhp_device_info {
  char name[128];
  int32_t sm_count;
  int32_t cc_major, cc_minor;
  int64_t l2_bytes;
  int64_t mem_bytes;
  int32_t graph_supported;
  int32_t pad_;
} rhp_device_info;

/* Per-operator schedule summary, for diagnostics/benchmarks. */
typedef struct rhp_layout_info {
  int64_t m_local, n, nnz_local;
  int64_t row_bins[8];  /* rows of A per bin: widths 1,2,4,8,16,32, CTA, split */
  int64_t col_bins[8];  /* rows of A^T per bin */
  int32_t grid_a, grid_at, grid_vec;
  int32_t sm_count;
  int32_t gather_l1;    /* bit 0: A's SpMV gathers through L1, bit 1: A^T's (tuned at create) */
  int32_t pdl;          /* SpMVs use programmatic dependent launch */
  int32_t thread_rows;  /* bit 0: A uses the thread-per-row engine, bit 1: A^T (last segment);
                           bit 2: A uses the long-row (CTA row run) engine; bits 3 / 4: A / A^T
                           read a sliced (32-row, element-major) copy; bits 5 / 6: A / A^T
                           have uniform row lengths (no row-pointer reads); bits 7 / 8: A / A^T
                           run a thread-per-row row band ahead of the final pass */
  int32_t segments;     /* column segments: A's in bits 0-15, A^T's in bits 16-31 (1 = unsegmented) */
  int32_t resident;     /* blocks run as one cluster-resident kernel (small LPs) */
  int32_t partition;    /* 0 single GPU, 1 row-partitioned with replicated n-side walk
                           (Option A: allreduce / peer exchange), 2 sharded (Option B) */
  int32_t const_bounds; /* bounds constant after scaling, taken from kernel parameters instead of
                           loaded: bit 0 var_lb, 1 var_ub, 2 con_lb, 3 con_ub */
  int32_t relabel;      /* rows and columns renumbered in first-touch locality order */
  int32_t pad2_;
  double sectors[4];    /* gather sectors per nonzero (256-nonzero windows): A, A^T as given,
                           A, A^T relabelled (0 when not evaluated) */
} rhp_layout_info;

const char* rhp_last_error(void);
int rhp_device_count(int* count);
int rhp_get_device_info(int device, rhp_device_info* info);
int rhp_nccl_unique_id(void* out128);

int rhp_create(const rhpdhg_lp_view* lp, const rhp_options* opt, rhp_ctx** out);
/* In-process collective group of `world` ranks (see rhp_options.local_group);
 * destroy only after every context using it. */
int rhp_local_group_create(int world, void** out);
int rhp_local_group_destroy(void* group);
int rhp_destroy(rhp_ctx* ctx);
int rhp_layout(rhp_ctx* ctx, rhp_layout_info* info);

/* Diagonal preconditioning on the device; bitwise equal to the reference. */
int rhp_scale(rhp_ctx* ctx, int enabled, int ruiz_iterations, int pock_chambolle);
int rhp_get_scaled(rhp_ctx* ctx, const rhp_scaled_out* out);

/* Power iteration on A^T A of the current (scaled) matrix. begin uploads the
 * unit start vector (column order); step does av = A v, w = A^T av and
 * returns v.w and w.w; normalize sets v = w / wnorm. */
int rhp_power_begin(rhp_ctx* ctx, const double* v0);
int rhp_power_step(rhp_ctx* ctx, double* vw, double* ww);
int rhp_power_normalize(rhp_ctx* ctx, double wnorm);

/* out = A in (transpose 0, in[n] -> out[m]) or A^T in (transpose 1) with the
 * current device matrix (original before rhp_scale, scaled after). */
int rhp_spmv(rhp_ctx* ctx, int transpose, const double* in, double* out);

int rhp_set_step(rhp_ctx* ctx, const rhp_step* step);
int rhp_reset_iterate(rhp_ctx* ctx);
/* Overwrite the scaled iterate z (x, y) and recompute exact caches; for tests. */
int rhp_set_iterate(rhp_ctx* ctx, const double* x, const double* y);
int rhp_run_block(rhp_ctx* ctx, rhp_block_out* out);
/* Copies min(count, cap) residuals of the last block. */
int rhp_get_history(rhp_ctx* ctx, double* out, int64_t cap, int64_t* count);

/* which: 0 = current Halpern iterate z (refreshes z.ax/z.aty from exact
 * products, solver.cpp:42-44, and stores the unscaled x, y, reduced costs for
 * rhp_fetch_solution); 1 = last inner PDHG point (x+, y+), no refresh. */
int rhp_kkt(rhp_ctx* ctx, int which, rhp_kkt_sums* out);
/* kkt_residuals(problem, x, y) of given original-space vectors with the
 * ORIGINAL matrix (call before rhp_scale). */
int rhp_kkt_of(rhp_ctx* ctx, const double* x, const double* y, rhp_kkt_sums* out);
int rhp_fetch_solution(rhp_ctx* ctx, double* x, double* y, double* reduced_costs);
/* Row-partitioned contexts: *any = OR of `flag` over all ranks (keeps host
 * decisions such as the time limit identical on every rank); else *any = flag. */
int rhp_any(rhp_ctx* ctx, int flag, int* any);
/* GPU-free planning: the row partition bench/tests use (world_size+1 row
 * offsets, contiguous blocks balanced by nonzeros + rows). */
int rhp_partition_rows(const rhpdhg_lp_view* lp, int world_size, int64_t* offsets);
/* Scaled iterate (x, y, ax, aty) in original order; for tests. */
int rhp_fetch_iterate(rhp_ctx* ctx, double* x, double* y, double* ax, double* aty);

/* do_restart's device half: anchor <- z (with caches), k = 0,
 * r_anchor = r_prev = +inf; the host already updated omega via rhp_set_step. */
int rhp_restart(rhp_ctx* ctx);

/* Device time (ms, CUDA events) of the last rhp_run_block. */
int rhp_last_block_ms(rhp_ctx* ctx, double* ms);
/* Event timer on the ctx stream: start != 0 records the start event;
 * start == 0 records the stop event, synchronizes, returns elapsed ms. */
int rhp_timer(rhp_ctx* ctx, int start, double* ms);
/* Average device time (ms) of `reps` back-to-back launches of each fused
 * iteration kernel (K1 = A-side SpMV + dual/Halpern epilogue, K2 = A^T-side
 * SpMV + aty/Halpern epilogue + next primal step, K3 = block-start primal
 * step) on the live iterate. Benchmark use only: mutates the iterate. */
int rhp_time_kernels(rhp_ctx* ctx, int reps, double* ms_k1, double* ms_k2, double* ms_k3);
/* Average device ms of `reps` plain SpMVs (transpose 0: A v, 1: A^T v) on
 * the current matrix, no epilogue: the SpMV engine's own rate. */
int rhp_time_spmv(rhp_ctx* ctx, int transpose, int reps, double* ms);
/* Gather ceiling (diagnostic): best device ms over `reps` of a kernel doing
 * only the irreducible SpMV work on A's / A^T's own nonzeros (coalesced index
 * + value stream, 8-B gathers with the operator's cache policy, one FMA
 * each). Either output may be null. */
int rhp_gather_ceiling(rhp_ctx* ctx, int reps, double* ms_a, double* ms_at);
/* cudaProfilerStart (start != 0) / cudaProfilerStop: brackets the launches
 * an `ncu --profile-from-start off` capture should see. */
int rhp_profiler_range(int start);
/* Synchronize the ctx stream. */
int rhp_synchronize(rhp_ctx* ctx);


/* ---- per-operation API -------------------------------------------------
 * The reference's per-op functions (pdhg.hpp:44-58 pdhg_step / p_norm /
 * fixed_point_residual, restart.hpp:47-70 halpern_reflected_step /
 * pid_update, scaling.hpp:30-32 unscale_iterate) as device round trips of
 * host vectors in original order. A ctx passed here is a product context of
 * one matrix (never rhp_scale'd); the host library caches one per
 * SparseMatrix. Elementwise formulas are bit-identical to the reference's;
 * products and sums use the device engines (reduction-order drift only). */
typedef struct rhp_op_lp {
  const double *objective, *var_lb, *var_ub; /* [n] */
  const double *con_lb, *con_ub;             /* [m] */
} rhp_op_lp;
typedef struct rhp_op_iter {
  const double *x, *y, *ax, *aty; /* x, aty: [n]; y, ax: [m] */
} rhp_op_iter;
typedef struct rhp_op_out {
  double *x, *y, *ax, *aty;
} rhp_op_out;
/* tau = eta/omega, sigma = eta*omega, sigma_inv = 1/sigma (pdhg.cpp:35-50);
 * a = (k+1)/(k+2), b = 1/(k+2), gamma (restart.cpp:38-40). */
typedef struct rhp_op_params {
  double tau, sigma, sigma_inv, gamma, a, b;
} rhp_op_params;

/* pdhg_step (pdhg.cpp:34-65) of z: inner = (x+, y+, A x+, A^T y+),
 * dx = x - x+, dy = y - y+ (dx/dy may be NULL). With anchor != NULL it is
 * halpern_reflected_step (restart.cpp:35-52): znew = a((1+g) inner - g z)
 * + b anchor for x, y, ax and aty. */
int rhp_op_pdhg(rhp_ctx* ctx, const rhp_op_params* p, const rhp_op_lp* lp, const rhp_op_iter* z,
                const rhp_op_iter* anchor, const rhp_op_out* inner, double* dx, double* dy,
                const rhp_op_out* znew);
/* CSC-order values of the matrix (the reference's csc_values(), which for a
 * matrix produced by a scaling differ from the CSR values in the last ulp):
 * scale_source 0 — A^T products of this (unscaled) ctx use them;
 * scale_source 1 — rhp_scale applies its A^T scales to them (scaling.cpp:17
 * matrix.scaled() scales each layout from its own values). */
int rhp_set_csc_values(rhp_ctx* ctx, const double* csc_values, int scale_source);
/* Replaces the objective and bounds of an unscaled ctx (kkt_residuals of a
 * problem whose matrix has a cached product context). */
int rhp_set_vectors(rhp_ctx* ctx, const rhp_op_lp* lp);
/* Sums on the device (fixed order, run-to-run identical):
 * out[0] = sum (p - pm)^2 (pm NULL: sum p^2), out[1] = sum q^2,
 * out[2] = sum q (r - rs) (r NULL: 0, rs NULL: sum q r), out[3] = sum p^2. */
int rhp_op_sums(int device, int64_t n, const double* p, const double* pm, int64_t m,
                const double* q, const double* r, const double* rs, double* out4);
/* out = s * v elementwise (unscale_iterate, scaling.cpp:83-94). */
int rhp_op_mul(int device, int64_t n, const double* s, const double* v, double* out);

#ifdef __cplusplus
}
#endif
#endif /* RHPDHG_CUDA_H_ */
