/*
 * rhpdhg_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference hot path (restarted reflected
 * Halpern PDHG, cuPDLP+ arXiv 2507.14051, as shipped in
 * /root/reference/proj/src). It exists to check the CUDA product; only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it, and never as the thing measured or shipped.
 *
 * Every function follows the reference's formula shapes and summation order
 * (and is compiled with -ffp-contract=off like the reference's x86-64
 * baseline build), so on the same inputs it reproduces the reference
 * bit-for-bit; tests/test_oracle_vs_ref.py pins that against the reference
 * library compiled from its own sources (oracle/_ref) and against the
 * golden counters of SURVEY.md Appendix A (tests/golden/).
 *
 * Structs are the flat ones of the product C ABI (include/rhpdhg_c.h) so the
 * same test code drives the product, the reference and this oracle.
 */
#ifndef RHPDHG_ORACLE_H_
#define RHPDHG_ORACLE_H_

#include <stdint.h>

#include "../include/rhpdhg_c.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* solve()  — solver.cpp:63-238 */
int orc_solve_csr(const rhpdhg_lp_view* lp, const rhpdhg_config_c* cfg, rhpdhg_report_c* rep,
                  double* x, double* y, double* reduced_costs, double* history,
                  int64_t history_cap);

/* solve() with iterate snapshots: after the iteration that brings the total
 * count to ks[i], the unscaled iterate (x, y) is written to xs + i*n,
 * ys + i*m (the x, y solve() would report with iteration_limit = ks[i]). */
int orc_solve_snapshots(const rhpdhg_lp_view* lp, const rhpdhg_config_c* cfg,
                        rhpdhg_report_c* rep, const int64_t* ks, int nk, double* xs, double* ys);

/* SparseMatrix::multiply / multiply_transpose — sparse_matrix.cpp:67-87 */
int orc_spmv(const rhpdhg_lp_view* lp, const double* in, double* out, int transpose);

/* ruiz_equilibrate + pock_chambolle_scale — scaling.cpp:46-81, sparse_matrix.cpp:101-136 */
int orc_scale(const rhpdhg_lp_view* lp, int ruiz_iters, int pock_chambolle, double* csr_vals,
              double* csc_vals, double* row_scale, double* col_scale, double* c_s,
              double* var_lb_s, double* var_ub_s, double* con_lb_s, double* con_ub_s);

/* power_iteration_norm — pdhg.cpp:117-170 */
int orc_power_iteration(const rhpdhg_lp_view* lp, double tol, int64_t max_iters, uint64_t seed,
                        double* value, int64_t* iterations, int32_t* converged);

/* kkt_residuals(problem, x, y) — termination.cpp:49-118 */
int orc_kkt_residuals(const rhpdhg_lp_view* lp, const double* x, const double* y,
                      rhpdhg_kkt_c* out);

/* The power-iteration start vector v_j = 2*U53 - 1 from mt19937_64(seed),
 * normalised (pdhg.cpp:126-133). */
void orc_power_start(int64_t n, uint64_t seed, double* v);

#ifdef __cplusplus
}
#endif
#endif
