/*
 * rhpdhg_c.h — flat C ABI of the rhpdhg solver (FFI entry point).
 *
 * The reference ships no FFI: its boundary is the C++ API in
 * proj/include/rhpdhg (LpProblem, SolverConfig, solve(), SolutionReport).
 * This header is the C-ABI a foreign binding (ctypes, cgo, JNI, N-API) binds
 * instead of that C++ API; every struct below mirrors one reference type
 * field-for-field so the binding is mechanical:
 *
 *   rhpdhg_lp_view     <- struct LpProblem          proj/include/rhpdhg/lp_problem.hpp:18-36
 *                         (matrix as CSR: SparseMatrix::row_ptr/col_index/csr_values,
 *                          proj/include/rhpdhg/sparse_matrix.hpp:58-60; Index = int64)
 *   rhpdhg_config_c    <- struct SolverConfig       proj/include/rhpdhg/config.hpp:12-40
 *   rhpdhg_kkt_c       <- struct KktResiduals       proj/include/rhpdhg/termination.hpp:12-22
 *   rhpdhg_report_c    <- struct SolutionReport     proj/include/rhpdhg/report.hpp:19-42
 *   rhpdhg_solve_csr   <- SolutionReport solve(const LpProblem&, const SolverConfig&)
 *                                                   proj/include/rhpdhg/solver.hpp:13
 *   status codes       <- exception taxonomy        proj/include/rhpdhg/errors.hpp:9-37
 *
 * The implementation (librhpdhg.so) is the C++ host solver of this repo; it
 * drives the CUDA device library through include/rhpdhg_cuda.h. There is no
 * CPU fallback: without a usable CUDA device every solve returns
 * RHPDHG_E_DEVICE.
 */
#ifndef RHPDHG_C_H_
#define RHPDHG_C_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RHPDHG_C_ABI_VERSION 1

/* Status codes: 0 = success; the others map 1:1 to the reference exceptions. */
enum {
  RHPDHG_OK = 0,
  RHPDHG_E_USAGE = 1,           /* rhpdhg::UsageError              errors.hpp:10-13 */
  RHPDHG_E_INVALID_PROBLEM = 2, /* rhpdhg::InvalidProblemError     errors.hpp:16-19 */
  RHPDHG_E_PARSE = 3,           /* rhpdhg::ParseError              errors.hpp:22-31 */
  RHPDHG_E_BREAKDOWN = 4,       /* rhpdhg::NumericalBreakdownError errors.hpp:34-37 */
  RHPDHG_E_DEVICE = 5,          /* CUDA / NCCL failure (no reference equivalent) */
  RHPDHG_E_INTERNAL = 6
};

/* SolveStatus (report.hpp:13). */
enum { RHPDHG_OPTIMAL = 0, RHPDHG_ITERATION_LIMIT = 1, RHPDHG_TIME_LIMIT = 2 };

/* Borrowed view of an LP in the reference's two-sided form
 *   min c^T x + offset  s.t.  con_lb <= A x <= con_ub,  var_lb <= x <= var_ub
 * with the reference convention that maximization instances already carry a
 * negated objective/offset (lp_problem.hpp:9-11). A is CSR with int64 indices,
 * columns strictly increasing inside a row, no explicit zeros required (they
 * are dropped like SparseMatrix's ctor, sparse_matrix.cpp:31). Bounds may be
 * +-inf. */
typedef struct rhpdhg_lp_view {
  int64_t num_cons; /* m */
  int64_t num_vars; /* n */
  int64_t nnz;
  const int64_t* row_ptr;   /* [m+1] */
  const int64_t* col_index; /* [nnz] */
  const double* values;     /* [nnz] */
  const double* objective;  /* [n] */
  double objective_offset;
  const double* var_lb; /* [n] */
  const double* var_ub; /* [n] */
  const double* con_lb; /* [m] */
  const double* con_ub; /* [m] */
  int32_t maximization;
} rhpdhg_lp_view;

/* SolverConfig (config.hpp:12-40); rhpdhg_config_default() fills the shipped
 * defaults. Integer booleans are 0/1. */
typedef struct rhpdhg_config_c {
  int32_t scaling_enabled;     /* scaling.enabled       = 1    */
  int32_t ruiz_iterations;     /* scaling.ruiz_iters    = 10   */
  int32_t pock_chambolle;      /* scaling.pock_chambolle= 1    */
  int32_t restarts_enabled;    /* restart.enabled       = 1    */
  double stepsize_multiplier;  /* stepsize.multiplier   = 0.99 */
  double power_tol;            /* power.tol             = 1e-4 */
  int64_t power_max_iters;     /* power.max_iters       = 5000 */
  uint64_t power_seed;         /* power.seed            = 0    */
  double beta_sufficient;      /* 0.2  */
  double beta_necessary;       /* 0.8  */
  double beta_artificial;      /* 0.36 */
  double reflection_gamma;     /* 1.0  */
  double pid_kp;               /* 0.5  */
  double pid_ki;               /* 0.0  */
  double pid_kd;               /* 0.0  */
  double initial_weight;       /* 1.0  */
  double epsilon;              /* tol.epsilon = 1e-4 */
  int64_t check_interval;      /* tol.check_interval = 64 */
  double time_limit_seconds;   /* +inf */
  int64_t iteration_limit;     /* INT64_MAX */
  int32_t verbosity;           /* 0 */
  int32_t record_residual_history; /* 0 */
} rhpdhg_config_c;

/* KktResiduals (termination.hpp:12-22). */
typedef struct rhpdhg_kkt_c {
  double gap_abs, gap_rel;
  double primal_inf, primal_rel;
  double dual_eq, dual_cone;
  double gap_denom, primal_denom, dual_denom;
} rhpdhg_kkt_c;

/* SolutionReport (report.hpp:19-42) minus the vectors, which are written to
 * caller buffers. The timing split (setup/loop) and device info are
 * extensions that the reference does not report. */
typedef struct rhpdhg_report_c {
  int32_t status;
  int32_t has_inner_residuals;
  double objective;
  rhpdhg_kkt_c residuals;
  int64_t iterations;
  int64_t restart_count;
  double wall_time_seconds;
  double final_fixed_point_residual;
  double final_primal_weight;
  double matrix_norm_estimate;
  int64_t power_iterations;
  uint64_t spmv_loop;
  uint64_t spmv_checks;
  uint64_t spmv_setup;
  int64_t kkt_checks;
  rhpdhg_kkt_c inner_residuals;
  int64_t history_len;        /* entries of fixed_point_residual_history */
  /* extensions */
  double setup_seconds;       /* upload + scaling + power iteration */
  double loop_seconds;        /* iteration loop incl. KKT checks */
  int64_t device_blocks;      /* graph blocks launched */
} rhpdhg_report_c;

int rhpdhg_config_default(rhpdhg_config_c* cfg);

/* solve(): x/y/reduced_costs may be NULL (then not returned); they receive
 * n, m and n doubles in original space and sense like SolutionReport. history
 * receives min(history_len, history_cap) residuals when
 * record_residual_history is set. Returns a status code; on error
 * rhpdhg_last_error() holds the exception message. */
int rhpdhg_solve_csr(const rhpdhg_lp_view* lp, const rhpdhg_config_c* cfg,
                     rhpdhg_report_c* report, double* x, double* y,
                     double* reduced_costs, double* history, int64_t history_cap);

/* kkt_residuals(problem, x, y) on the device (termination.hpp:41-42). */
int rhpdhg_kkt_residuals(const rhpdhg_lp_view* lp, const double* x, const double* y,
                         rhpdhg_kkt_c* out);

/* An owned LpProblem: parse_mps_file (mps.hpp:21-25). `warnings` (may be
 * NULL) receives the parser warnings joined by '\n', truncated to cap-1. */
typedef struct rhpdhg_lp rhpdhg_lp;
int rhpdhg_lp_read_mps(const char* path, rhpdhg_lp** out, char* warnings, int64_t warnings_cap);
/* Borrowed view of an owned LP (valid until rhpdhg_lp_free). */
int rhpdhg_lp_view_of(const rhpdhg_lp* lp, rhpdhg_lp_view* view);
void rhpdhg_lp_free(rhpdhg_lp* lp);

/* Thread-local message of the last failing call on this thread. */
const char* rhpdhg_last_error(void);

/* Selects the CUDA device used by subsequent solves in this process. */
int rhpdhg_set_device(int device);
/* Device runtime knobs (not SolverConfig keys): CUDA-graph blocks on/off and
 * the maximum PDHG iterations per device block (default 1, 64). */
int rhpdhg_set_device_options(int device, int use_graph, int64_t block_limit);
/* Row-partitioned multi-GPU solves (one process per GPU): subsequent solves
 * of this process act as `rank` of `world_size`, joined through rank 0's
 * 128-byte NCCL unique id (rhp_nccl_unique_id in rhpdhg_cuda.h). nccl_id NULL
 * with world_size 1 restores single-GPU solves. */
int rhpdhg_set_distributed(int rank, int world_size, const void* nccl_id);
/* Same with an in-process collective group (rhp_local_group_create in
 * rhpdhg_cuda.h) instead of NCCL: world_size threads of this process, each
 * calling this with its rank, solve one LP together. Device options are per
 * thread. */
int rhpdhg_set_local_group(int rank, int world_size, const void* group);
/* Directory benchmark (rhpdhg::run_benchmark, reference bench.cpp:171-266):
 * solves every *.mps / *.mps.gz in `dir` on the GPU(s) (workers > 1: that
 * many concurrent solves, worker w on GPU w % device_count), scores unsolved
 * instances at their class time limit, writes the reference's JSON schema to
 * json_path (if non-empty) and the per-instance table + SGM10 summary to
 * `table` (NUL-terminated, truncated to table_cap). */
int rhpdhg_run_benchmark(const char* dir, const rhpdhg_config_c* cfg, double small_limit_seconds,
                         double large_limit_seconds, int workers, const char* json_path,
                         char* table, int64_t table_cap);
/* Small-LP cluster-resident device blocks: -1 auto (default), 0 off, 1 on. */
int rhpdhg_set_resident(int mode);
/* First-touch locality relabelling of rows and columns at device ingest (the
 * calling thread's solves): 0 auto (default: large gathered vectors, kept
 * only when it cuts the SpMV gather sectors), -1 off, 1 forced. Results come
 * back in the original order either way. */
int rhpdhg_set_locality(int mode);

/* Resumable solve (extension used by benchmarks and long-running callers):
 * create = validation + upload + scaling + power iteration + initial KKT
 * check; advance runs device blocks (with their KKT checks and restarts)
 * until at least `iterations` more PDHG iterations are done or the solve is
 * decided; finish completes the solve and fills the report like
 * rhpdhg_solve_csr. The session BORROWS the view's arrays (no host copy of
 * the LP): they must stay valid and unchanged until rhpdhg_session_destroy.
 * The matrix is validated by the device ingest with the same status codes
 * and messages as rhpdhg_solve_csr. */
typedef struct rhpdhg_session rhpdhg_session;
int rhpdhg_session_create(const rhpdhg_lp_view* lp, const rhpdhg_config_c* cfg,
                          rhpdhg_session** out);
int rhpdhg_session_advance(rhpdhg_session* s, int64_t iterations, int32_t* running);
int rhpdhg_session_info(rhpdhg_session* s, int64_t* total_iterations, int64_t* restarts,
                        rhpdhg_kkt_c* last_residuals, double* setup_seconds,
                        int64_t* device_blocks, int64_t* kkt_checks);
/* start != 0: record a CUDA event on the solve's stream; start == 0: record
 * the stop event, synchronize and return the elapsed device milliseconds. */
int rhpdhg_session_timer(rhpdhg_session* s, int start, double* ms);
/* Benchmark hook: average device ms of the fused iteration kernels over
 * `reps` launches (rhp_time_kernels); mutates the iterate, so call it only
 * after the measured work. ms3 = {K1, K2, K3}. */
int rhpdhg_session_time_kernels(rhpdhg_session* s, int reps, double* ms3);
/* Benchmark hook: gather ceilings of A and A^T (rhp_gather_ceiling), ms2 =
 * {A, A^T}. */
int rhpdhg_session_gather_ceiling(rhpdhg_session* s, int reps, double* ms2);
/* Device layout summary: m, n, nnz, then rows of A and of A^T per schedule
 * bin (8 each), the grids of the A, A^T and vector kernels, the SM count,
 * the gather cache policy (bit 0: A through L1, bit 1: A^T) and whether the
 * SpMVs use programmatic dependent launch, then the engine bits (bit 0: A
 * uses the thread-per-row engine, bit 1: A^T, bit 2: A uses the long-row
 * engine, bits 3 / 4: A / A^T read their sliced copy, bits 5 / 6: A / A^T
 * have uniform row lengths, bits 7 / 8: A / A^T run a thread-per-row row
 * band), then the column segment
 * counts (A's in bits 0-15, A^T's in bits 16-31), then 1 when blocks run as
 * the cluster-resident kernel, then the partition mode (0 single GPU,
 * 1 row-partitioned with a replicated n-side walk, 2 sharded), then the
 * constant-bound bits (bit 0 var_lb, 1 var_ub, 2 con_lb, 3 con_ub). */
int rhpdhg_session_layout(rhpdhg_session* s, int64_t* out30);
int rhpdhg_session_finish(rhpdhg_session* s, rhpdhg_report_c* report, double* x, double* y,
                          double* reduced_costs, double* history, int64_t history_cap);
void rhpdhg_session_destroy(rhpdhg_session* s);

#ifdef __cplusplus
}
#endif
#endif /* RHPDHG_C_H_ */
