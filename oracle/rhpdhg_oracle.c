/*
 * rhpdhg_oracle.c — TEST INFRASTRUCTURE ONLY (see rhpdhg_oracle.h).
 *
 * Plain-C restatement of the reference's restarted reflected-Halpern PDHG
 * (/root/reference/proj/src). Written from the algorithm, not translated
 * line by line, but keeping every floating-point expression in the
 * reference's evaluation order so results agree bit-for-bit (compiled with
 * -ffp-contract=off, like the reference's x86-64 baseline build without FMA).
 * Each function names the reference lines it restates.
 */
#include "rhpdhg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* std::max / std::min semantics (returns the first argument on ties/NaN). */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }

/* ---------------------------------------------------------------- matrix -- */
/* CSR + CSC pair (sparse_matrix.hpp:30-76); explicit zeros dropped like the
 * ctor (sparse_matrix.cpp:31); CSC filled in row order (:53-64). */
typedef struct {
  int64_t m, n, nnz;
  int64_t *rp, *ci, *cp, *ri;
  double *v, *vt;
} Mat;

static void mat_free(Mat* a) {
  free(a->rp); free(a->ci); free(a->cp); free(a->ri); free(a->v); free(a->vt);
  memset(a, 0, sizeof *a);
}

static void mat_build_csc(Mat* a) {
  a->cp = calloc((size_t)a->n + 1, sizeof(int64_t));
  a->ri = malloc(((size_t)a->nnz + 1) * sizeof(int64_t));
  a->vt = malloc(((size_t)a->nnz + 1) * sizeof(double));
  for (int64_t e = 0; e < a->nnz; ++e) a->cp[a->ci[e] + 1]++;
  for (int64_t j = 0; j < a->n; ++j) a->cp[j + 1] += a->cp[j];
  int64_t* next = malloc(((size_t)a->n + 1) * sizeof(int64_t));
  memcpy(next, a->cp, (size_t)a->n * sizeof(int64_t));
  for (int64_t i = 0; i < a->m; ++i)
    for (int64_t e = a->rp[i]; e < a->rp[i + 1]; ++e) {
      const int64_t s = next[a->ci[e]]++;
      a->ri[s] = i;
      a->vt[s] = a->v[e];
    }
  free(next);
}

static int mat_from_view(const rhpdhg_lp_view* lp, Mat* a) {
  memset(a, 0, sizeof *a);
  a->m = lp->num_cons;
  a->n = lp->num_vars;
  a->rp = calloc((size_t)a->m + 1, sizeof(int64_t));
  a->ci = malloc(((size_t)lp->nnz + 1) * sizeof(int64_t));
  a->v = malloc(((size_t)lp->nnz + 1) * sizeof(double));
  int64_t k = 0;
  for (int64_t i = 0; i < a->m; ++i) {
    for (int64_t e = lp->row_ptr[i]; e < lp->row_ptr[i + 1]; ++e) {
      const double v = lp->values[e];
      const int64_t j = lp->col_index[e];
      if (j < 0 || j >= a->n) return fail(RHPDHG_E_USAGE, "matrix entry out of bounds");
      if (!isfinite(v)) return fail(RHPDHG_E_INVALID_PROBLEM, "matrix entry is not finite");
      if (v == 0.0) continue;
      if (k > a->rp[i] && a->ci[k - 1] >= j)
        return fail(RHPDHG_E_INVALID_PROBLEM, "columns not strictly increasing in a row");
      a->ci[k] = j;
      a->v[k] = v;
      ++k;
    }
    a->rp[i + 1] = k;
  }
  a->nnz = k;
  mat_build_csc(a);
  return 0;
}

/* out = A x, sequential row sums (sparse_matrix.cpp:67-76). Rows are
 * independent, so the OpenMP row split (bench-size parity tests) leaves every
 * row sum, and so every result, bit-identical to the sequential loop. */
static void mat_mul(const Mat* a, const double* x, double* out) {
#pragma omp parallel for schedule(static, 4096)
  for (int64_t i = 0; i < a->m; ++i) {
    double acc = 0.0;
    for (int64_t e = a->rp[i]; e < a->rp[i + 1]; ++e) acc += a->v[e] * x[a->ci[e]];
    out[i] = acc;
  }
}

/* out = A^T y over the CSC copy (sparse_matrix.cpp:78-87). */
static void mat_mul_t(const Mat* a, const double* y, double* out) {
#pragma omp parallel for schedule(static, 4096)
  for (int64_t j = 0; j < a->n; ++j) {
    double acc = 0.0;
    for (int64_t e = a->cp[j]; e < a->cp[j + 1]; ++e) acc += a->vt[e] * y[a->ri[e]];
    out[j] = acc;
  }
}

/* In-place D_row A D_col with the reference's two multiplication orders:
 * CSR (r_i a) c_j, CSC (c_j a) r_i (sparse_matrix.cpp:101-114). Both copies
 * are rebuilt from the given (unscaled-by-this-call) values. */
static void mat_scale(Mat* a, const double* rs, const double* cs) {
#pragma omp parallel for schedule(static, 4096)
  for (int64_t i = 0; i < a->m; ++i)
    for (int64_t e = a->rp[i]; e < a->rp[i + 1]; ++e) a->v[e] = rs[i] * a->v[e] * cs[a->ci[e]];
#pragma omp parallel for schedule(static, 4096)
  for (int64_t j = 0; j < a->n; ++j)
    for (int64_t e = a->cp[j]; e < a->cp[j + 1]; ++e) a->vt[e] = cs[j] * a->vt[e] * rs[a->ri[e]];
}

/* --------------------------------------------------------------- problem -- */
typedef struct {
  Mat A;
  int64_t m, n;
  double *c, *vl, *vu, *cl, *cu;
  double offset;
  int maxi;
} Lp;

static void lp_free(Lp* p) {
  mat_free(&p->A);
  free(p->c); free(p->vl); free(p->vu); free(p->cl); free(p->cu);
}

static double* dup(const double* s, int64_t k) {
  double* d = malloc(((size_t)k + 1) * sizeof(double));
  if (k) memcpy(d, s, (size_t)k * sizeof(double));
  return d;
}

/* LpProblem::validate (lp_problem.cpp:30-46, check_bound_pair :15-27). */
static int bound_pair_ok(const double* lb, const double* ub, int64_t k) {
  for (int64_t i = 0; i < k; ++i) {
    if (isnan(lb[i]) || isnan(ub[i])) return 0;
    if (lb[i] > ub[i]) return 0;
    if (lb[i] == INFINITY || ub[i] == -INFINITY) return 0;
  }
  return 1;
}

static int lp_from_view(const rhpdhg_lp_view* v, Lp* p) {
  memset(p, 0, sizeof *p);
  int rc = mat_from_view(v, &p->A);
  if (rc) return rc;
  p->m = v->num_cons;
  p->n = v->num_vars;
  p->c = dup(v->objective, p->n);
  p->vl = dup(v->var_lb, p->n);
  p->vu = dup(v->var_ub, p->n);
  p->cl = dup(v->con_lb, p->m);
  p->cu = dup(v->con_ub, p->m);
  p->offset = v->objective_offset;
  p->maxi = v->maximization;
  for (int64_t j = 0; j < p->n; ++j)
    if (!isfinite(p->c[j])) return fail(RHPDHG_E_INVALID_PROBLEM, "objective not finite");
  if (!isfinite(p->offset)) return fail(RHPDHG_E_INVALID_PROBLEM, "offset not finite");
  if (!bound_pair_ok(p->vl, p->vu, p->n)) return fail(RHPDHG_E_INVALID_PROBLEM, "variable bounds");
  if (!bound_pair_ok(p->cl, p->cu, p->m)) return fail(RHPDHG_E_INVALID_PROBLEM, "constraint bounds");
  return 0;
}

/* apply_scales (scaling.cpp:10-34): c <- c_j c, var bounds / c_j, con bounds r_i *. */
static void lp_apply_scales(Lp* p, const double* rs, const double* cs) {
  mat_scale(&p->A, rs, cs);
  for (int64_t j = 0; j < p->n; ++j) {
    p->c[j] = cs[j] * p->c[j];
    p->vl[j] = p->vl[j] / cs[j];
    p->vu[j] = p->vu[j] / cs[j];
  }
  for (int64_t i = 0; i < p->m; ++i) {
    p->cl[i] = rs[i] * p->cl[i];
    p->cu[i] = rs[i] * p->cu[i];
  }
}

/* Scaled copy of the instance plus the cumulative scales (solver.cpp:72-78).
 * Ruiz (scaling.cpp:46-68): max-abs on the iteratively divided values, sqrt,
 * value /= (rmax*cmax), scale /= max; the final instance is apply_scales of
 * the ORIGINAL data. Pock-Chambolle (scaling.cpp:70-81): 1/sqrt of the row
 * and column 1-norms of the Ruiz-scaled CSR values, summed in row-major order
 * (sparse_matrix.cpp:127-136), applied to the Ruiz-scaled instance. */
static void lp_scale(const Lp* orig, int ruiz_iters, int pc, Lp* out, double* rs, double* cs) {
  const int64_t m = orig->m, n = orig->n, nz = orig->A.nnz;
  for (int64_t i = 0; i < m; ++i) rs[i] = 1.0;
  for (int64_t j = 0; j < n; ++j) cs[j] = 1.0;
  double* w = dup(orig->A.v, nz);
  double* rmax = malloc(((size_t)m + 1) * sizeof(double));
  double* cmax = malloc(((size_t)n + 1) * sizeof(double));
  for (int pass = 0; pass < ruiz_iters; ++pass) {
    for (int64_t i = 0; i < m; ++i) rmax[i] = 0.0;
    for (int64_t j = 0; j < n; ++j) cmax[j] = 0.0;
    for (int64_t i = 0; i < m; ++i)
      for (int64_t e = orig->A.rp[i]; e < orig->A.rp[i + 1]; ++e) {
        const double a = fabs(w[e]);
        if (a > rmax[i]) rmax[i] = a;
        if (a > cmax[orig->A.ci[e]]) cmax[orig->A.ci[e]] = a;
      }
    for (int64_t i = 0; i < m; ++i) rmax[i] = rmax[i] > 0.0 ? sqrt(rmax[i]) : 1.0;
    for (int64_t j = 0; j < n; ++j) cmax[j] = cmax[j] > 0.0 ? sqrt(cmax[j]) : 1.0;
    for (int64_t i = 0; i < m; ++i)
      for (int64_t e = orig->A.rp[i]; e < orig->A.rp[i + 1]; ++e)
        w[e] /= rmax[i] * cmax[orig->A.ci[e]];
    for (int64_t i = 0; i < m; ++i) rs[i] /= rmax[i];
    for (int64_t j = 0; j < n; ++j) cs[j] /= cmax[j];
  }
  free(w);
  /* deep copy + apply */
  memset(out, 0, sizeof *out);
  out->m = m;
  out->n = n;
  out->offset = orig->offset;
  out->maxi = orig->maxi;
  out->A.m = m;
  out->A.n = n;
  out->A.nnz = nz;
  out->A.rp = malloc(((size_t)m + 1) * sizeof(int64_t));
  memcpy(out->A.rp, orig->A.rp, ((size_t)m + 1) * sizeof(int64_t));
  out->A.ci = malloc(((size_t)nz + 1) * sizeof(int64_t));
  if (nz) memcpy(out->A.ci, orig->A.ci, (size_t)nz * sizeof(int64_t));
  out->A.cp = malloc(((size_t)n + 1) * sizeof(int64_t));
  memcpy(out->A.cp, orig->A.cp, ((size_t)n + 1) * sizeof(int64_t));
  out->A.ri = malloc(((size_t)nz + 1) * sizeof(int64_t));
  if (nz) memcpy(out->A.ri, orig->A.ri, (size_t)nz * sizeof(int64_t));
  out->A.v = dup(orig->A.v, nz);
  out->A.vt = dup(orig->A.vt, nz);
  out->c = dup(orig->c, n);
  out->vl = dup(orig->vl, n);
  out->vu = dup(orig->vu, n);
  out->cl = dup(orig->cl, m);
  out->cu = dup(orig->cu, m);
  lp_apply_scales(out, rs, cs);
  if (pc) {
    for (int64_t i = 0; i < m; ++i) rmax[i] = 0.0;
    for (int64_t j = 0; j < n; ++j) cmax[j] = 0.0;
    for (int64_t i = 0; i < m; ++i)
      for (int64_t e = out->A.rp[i]; e < out->A.rp[i + 1]; ++e) {
        const double a = fabs(out->A.v[e]);
        rmax[i] += a;
        cmax[out->A.ci[e]] += a;
      }
    for (int64_t i = 0; i < m; ++i) rmax[i] = rmax[i] > 0.0 ? 1.0 / sqrt(rmax[i]) : 1.0;
    for (int64_t j = 0; j < n; ++j) cmax[j] = cmax[j] > 0.0 ? 1.0 / sqrt(cmax[j]) : 1.0;
    lp_apply_scales(out, rmax, cmax);
    for (int64_t i = 0; i < m; ++i) rs[i] *= rmax[i];
    for (int64_t j = 0; j < n; ++j) cs[j] *= cmax[j];
  }
  free(rmax);
  free(cmax);
}

/* ------------------------------------------------------------ mt19937_64 -- */
typedef struct {
  uint64_t mt[312];
  int idx;
} Mt64;

static void mt_seed(Mt64* g, uint64_t s) {
  g->mt[0] = s;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt_next(Mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

static double dot(const double* a, const double* b, int64_t k) {
  double acc = 0.0;
  for (int64_t i = 0; i < k; ++i) acc += a[i] * b[i];
  return acc;
}

void orc_power_start(int64_t n, uint64_t seed, double* v) {
  Mt64 g;
  mt_seed(&g, seed);
  for (int64_t j = 0; j < n; ++j) v[j] = 2.0 * ((double)(mt_next(&g) >> 11) * 0x1.0p-53) - 1.0;
  const double nv = sqrt(dot(v, v, n));
  for (int64_t j = 0; j < n; ++j) v[j] /= nv;
}

/* power_iteration_norm (pdhg.cpp:117-170). */
static void power_iter(const Mat* a, double tol, int64_t max_iters, uint64_t seed, double* value,
                       int64_t* iters, int* conv) {
  *value = 0.0;
  *iters = 0;
  *conv = 0;
  if (a->nnz == 0) {
    *conv = 1;
    return;
  }
  const int64_t n = a->n;
  double* v = malloc((size_t)n * sizeof(double));
  double* w = malloc((size_t)n * sizeof(double));
  double* av = malloc(((size_t)a->m + 1) * sizeof(double));
  orc_power_start(n, seed, v);
  double sigma_prev = 0.0, change_prev = INFINITY;
  for (int64_t it = 1; it <= max_iters; ++it) {
    mat_mul(a, v, av);
    mat_mul_t(a, av, w);
    const double lambda = dot(v, w, n);
    const double sigma = lambda > 0.0 ? sqrt(lambda) : 0.0;
    *iters = it;
    *value = sigma;
    const double wn = sqrt(dot(w, w, n));
    if (wn == 0.0) {
      *conv = 1;
      break;
    }
    for (int64_t j = 0; j < n; ++j) v[j] = w[j] / wn;
    const double change = fabs(sigma - sigma_prev);
    if (it >= 3 && change <= tol * smax(sigma, 1e-300)) {
      const double ratio = smin(change / smax(change_prev, 1e-300), 0.999);
      const double tail = change * ratio / (1.0 - ratio);
      if (tail <= tol * smax(sigma, 1e-300)) {
        *conv = 1;
        break;
      }
    }
    sigma_prev = sigma;
    change_prev = change;
  }
  free(v);
  free(w);
  free(av);
}

/* ------------------------------------------------------------ termination -- */
/* clip_to_sign_cone (termination.cpp:24-31). */
static double clip_sign(double s, double lb, double ub) {
  const int lf = lb > -INFINITY, uf = ub < INFINITY;
  if (lf && uf) return s;
  if (lf) return smax(s, 0.0);
  if (uf) return smin(s, 0.0);
  return 0.0;
}

/* p_support (lp_problem.cpp:72-87) evaluated on -y; +inf when a dual sign is
 * infeasible against an infinite bound. */
static double p_support_neg(const double* y, const double* lb, const double* ub, int64_t k) {
  double total = 0.0;
  for (int64_t i = 0; i < k; ++i) {
    const double v = -y[i];
    const double yp = smax(v, 0.0);
    const double yn = smax(-v, 0.0);
    const double up = yp == 0.0 ? 0.0 : ub[i] * yp;
    const double lo = yn == 0.0 ? 0.0 : lb[i] * yn;
    if (up == INFINITY || lo == -INFINITY) return INFINITY;
    total += up - lo;
  }
  return total;
}

/* kkt_residuals with given products (termination.cpp:58-118). */
static int kkt(const Lp* p, const double* x, const double* y, const double* ax, const double* aty,
               rhpdhg_kkt_c* res) {
  for (int64_t j = 0; j < p->n; ++j)
    if (isnan(x[j])) return fail(RHPDHG_E_BREAKDOWN, "NaN in primal iterate");
  for (int64_t i = 0; i < p->m; ++i)
    if (isnan(y[i])) return fail(RHPDHG_E_BREAKDOWN, "NaN in dual iterate");
  double* r = malloc(((size_t)p->n + 1) * sizeof(double));
  for (int64_t j = 0; j < p->n; ++j) r[j] = clip_sign(p->c[j] - aty[j], p->vl[j], p->vu[j]);
  const double py = p_support_neg(y, p->cl, p->cu, p->m);
  const double pr = p_support_neg(r, p->vl, p->vu, p->n);
  const double p_terms = py + pr;
  const double primal_value = dot(p->c, x, p->n);
  if (p_terms == INFINITY) {
    res->gap_abs = res->gap_denom = res->gap_rel = INFINITY;
  } else {
    res->gap_abs = fabs(primal_value + p_terms);
    res->gap_denom = 1.0 + fabs(p_terms) + fabs(primal_value);
    res->gap_rel = res->gap_abs / res->gap_denom;
  }
  double viol2 = 0.0, bound2 = 0.0;
  for (int64_t i = 0; i < p->m; ++i) {
    const double proj = smin(smax(ax[i], p->cl[i]), p->cu[i]);
    const double d = ax[i] - proj;
    viol2 += d * d;
    if (isfinite(p->cl[i])) bound2 += p->cl[i] * p->cl[i];
    if (isfinite(p->cu[i])) bound2 += p->cu[i] * p->cu[i];
  }
  res->primal_inf = sqrt(viol2);
  res->primal_denom = 1.0 + sqrt(bound2);
  res->primal_rel = res->primal_inf / res->primal_denom;
  double eq2 = 0.0, cone2 = 0.0;
  for (int64_t j = 0; j < p->n; ++j) {
    const double d = p->c[j] - aty[j] - r[j];
    eq2 += d * d;
    const double c = r[j] - clip_sign(r[j], p->vl[j], p->vu[j]);
    cone2 += c * c;
  }
  res->dual_eq = sqrt(eq2);
  res->dual_cone = sqrt(cone2);
  res->dual_denom = 1.0 + sqrt(dot(p->c, p->c, p->n));
  free(r);
  return 0;
}

/* is_optimal (termination.cpp:120-124), non-strict. */
static int is_optimal(const rhpdhg_kkt_c* r, double eps) {
  return r->gap_rel <= eps && r->primal_rel <= eps && r->dual_eq <= eps * r->dual_denom &&
         r->dual_cone <= eps * r->dual_denom;
}

/* ------------------------------------------------------------------ solve -- */
typedef struct {
  double *x, *y, *ax, *aty;
} It;

static void it_alloc(It* z, int64_t m, int64_t n) {
  z->x = calloc((size_t)n + 1, sizeof(double));
  z->aty = calloc((size_t)n + 1, sizeof(double));
  z->y = calloc((size_t)m + 1, sizeof(double));
  z->ax = calloc((size_t)m + 1, sizeof(double));
}
static void it_free(It* z) { free(z->x); free(z->y); free(z->ax); free(z->aty); }
static void it_copy(It* d, const It* s, int64_t m, int64_t n) {
  memcpy(d->x, s->x, (size_t)n * sizeof(double));
  memcpy(d->aty, s->aty, (size_t)n * sizeof(double));
  memcpy(d->y, s->y, (size_t)m * sizeof(double));
  memcpy(d->ax, s->ax, (size_t)m * sizeof(double));
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* kkt_check (solver.cpp:32-49): unscale, exact products on the ORIGINAL
 * matrix, refresh the scaled caches, residuals. xo/yo/axo/atyo receive the
 * original-space iterate and products. */
static int kkt_check(It* z, const Lp* orig, const double* rs, const double* cs, double* xo,
                     double* yo, double* axo, double* atyo, rhpdhg_kkt_c* res) {
  for (int64_t j = 0; j < orig->n; ++j) xo[j] = cs[j] * z->x[j];
  for (int64_t i = 0; i < orig->m; ++i) yo[i] = rs[i] * z->y[i];
  mat_mul(&orig->A, xo, axo);
  mat_mul_t(&orig->A, yo, atyo);
  for (int64_t i = 0; i < orig->m; ++i) z->ax[i] = rs[i] * axo[i];
  for (int64_t j = 0; j < orig->n; ++j) z->aty[j] = cs[j] * atyo[j];
  return kkt(orig, xo, yo, axo, atyo, res);
}

/* SolverConfig::validate (config.cpp:50-69). */
static int cfg_ok(const rhpdhg_config_c* c) {
  if (c->ruiz_iterations < 0) return 0;
  if (!(c->stepsize_multiplier > 0.0 && c->stepsize_multiplier <= 0.99)) return 0;
  if (!(c->power_tol > 0.0)) return 0;
  if (c->power_max_iters < 1) return 0;
  if (!(c->beta_sufficient > 0.0 && c->beta_sufficient < c->beta_necessary &&
        c->beta_necessary < 1.0))
    return 0;
  if (!(c->beta_artificial > 0.0 && c->beta_artificial < 1.0)) return 0;
  if (!(c->reflection_gamma >= 0.0 && c->reflection_gamma <= 1.0)) return 0;
  if (!(c->initial_weight > 0.0) || !isfinite(c->initial_weight)) return 0;
  if (!(c->epsilon > 0.0)) return 0;
  if (c->check_interval < 1) return 0;
  if (c->time_limit_seconds < 0.0 || isnan(c->time_limit_seconds)) return 0;
  if (c->iteration_limit < 0) return 0;
  return 1;
}

/* pid_update (restart.cpp:85-120). */
typedef struct {
  double kp, ki, kd, integral, prev_error, omega;
} Pid;

static double pid_update(Pid* pid, const It* z, const double* sx, const double* sy, int64_t m,
                         int64_t n) {
  double ax2 = 0.0, ay2 = 0.0, nx2 = 0.0, ny2 = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    const double d = z->x[j] - sx[j];
    ax2 += d * d;
  }
  for (int64_t i = 0; i < m; ++i) {
    const double d = z->y[i] - sy[i];
    ay2 += d * d;
  }
  for (int64_t j = 0; j < n; ++j) nx2 += z->x[j] * z->x[j];
  for (int64_t i = 0; i < m; ++i) ny2 += z->y[i] * z->y[i];
  const double dx = sqrt(ax2), dy = sqrt(ay2);
  double error = 0.0;
  if (dx > 1e-10 * (1.0 + sqrt(nx2)) && dy > 1e-10 * (1.0 + sqrt(ny2)))
    error = log(pid->omega) + log(dx) - log(dy);
  pid->integral += error;
  double delta = -(pid->kp * error + pid->ki * pid->integral + pid->kd * (error - pid->prev_error));
  pid->prev_error = error;
  int clamped = 0;
  const double max_step = log(10.0);
  if (delta > max_step) {
    delta = max_step;
    clamped = 1;
  } else if (delta < -max_step) {
    delta = -max_step;
    clamped = 1;
  }
  double omega = delta == 0.0 ? pid->omega : exp(log(pid->omega) + delta);
  if (omega < 1e-8) {
    omega = 1e-8;
    clamped = 1;
  } else if (omega > 1e8) {
    omega = 1e8;
    clamped = 1;
  }
  if (clamped) pid->integral = 0.0;
  pid->omega = omega;
  return omega;
}

/* Snapshot request of orc_solve_snapshots (test infrastructure, one solve at
 * a time): after the iteration that brings `total` to ks[i], the unscaled
 * Halpern iterate (x = D_col x_bar, y = D_row y_bar) goes to xs + i*n,
 * ys + i*m. */
static const int64_t* g_snap_k = NULL;
static int g_snap_nk = 0;
static double *g_snap_x = NULL, *g_snap_y = NULL;

int orc_solve_csr(const rhpdhg_lp_view* lpv, const rhpdhg_config_c* cfg, rhpdhg_report_c* rep,
                  double* x_out, double* y_out, double* rc_out, double* hist, int64_t hist_cap) {
  if (!cfg_ok(cfg)) return fail(RHPDHG_E_USAGE, "invalid solver configuration");
  Lp orig;
  int rc = lp_from_view(lpv, &orig);
  if (rc) {
    lp_free(&orig);
    return rc;
  }
  const double t0 = now_s();
  const int64_t m = orig.m, n = orig.n;
  double* rs = malloc(((size_t)m + 1) * sizeof(double));
  double* cs = malloc(((size_t)n + 1) * sizeof(double));
  Lp sc;
  if (cfg->scaling_enabled) {
    lp_scale(&orig, cfg->ruiz_iterations, cfg->pock_chambolle, &sc, rs, cs);
  } else {
    lp_scale(&orig, 0, 0, &sc, rs, cs); /* identity scales: exact copy */
  }
  /* (2) step size from the scaled norm (solver.cpp:81-88) */
  double norm;
  int64_t piters;
  int pconv;
  power_iter(&sc.A, cfg->power_tol, cfg->power_max_iters, cfg->power_seed, &norm, &piters, &pconv);
  const double eta = norm == 0.0 ? 1.0 : cfg->stepsize_multiplier / norm;
  if (norm > 0.0 && eta * norm > 0.99 * (1.0 + 1e-9)) {
    lp_free(&orig); lp_free(&sc); free(rs); free(cs);
    return fail(RHPDHG_E_USAGE, "step size violates the PSD margin");
  }
  double omega = cfg->initial_weight;
  const double gamma = cfg->reflection_gamma;

  memset(rep, 0, sizeof *rep);
  rep->matrix_norm_estimate = norm;
  rep->power_iterations = piters;
  rep->spmv_setup = 2ULL * (uint64_t)piters;

  It z, anc, nx, inner;
  it_alloc(&z, m, n);
  it_alloc(&anc, m, n);
  it_alloc(&nx, m, n);
  it_alloc(&inner, m, n); /* x_next, y_next, ax_next, aty_next */
  double* sx = calloc((size_t)n + 1, sizeof(double));
  double* sy = calloc((size_t)m + 1, sizeof(double));
  double* xo = calloc((size_t)n + 1, sizeof(double));
  double* yo = calloc((size_t)m + 1, sizeof(double));
  double* axo = calloc((size_t)m + 1, sizeof(double));
  double* atyo = calloc((size_t)n + 1, sizeof(double));
  Pid pid = {cfg->pid_kp, cfg->pid_ki, cfg->pid_kd, 0.0, 0.0, cfg->initial_weight};
  int64_t k = 0, total = 0, restarts = 0, checks = 0, hist_len = 0;
  double r_anchor = INFINITY, r_prev = INFINITY, last_fpr = INFINITY;
  int have_inner = 0, status = RHPDHG_ITERATION_LIMIT, decided = 0;
  rhpdhg_kkt_c res;

  rc = kkt_check(&z, &orig, rs, cs, xo, yo, axo, atyo, &res);
  ++checks;
  if (rc) goto done;
  if (is_optimal(&res, cfg->epsilon)) {
    status = RHPDHG_OPTIMAL;
    decided = 1;
  }
  while (!decided) {
    if (total >= cfg->iteration_limit) {
      status = RHPDHG_ITERATION_LIMIT;
      break;
    }
    if (now_s() - t0 >= cfg->time_limit_seconds) {
      status = RHPDHG_TIME_LIMIT;
      break;
    }
    /* pdhg_step (pdhg.cpp:34-65) */
    const double tau = eta / omega, sigma = eta * omega;
    for (int64_t j = 0; j < n; ++j) {
      const double t = z.x[j] - tau * (sc.c[j] - z.aty[j]);
      inner.x[j] = smin(smax(t, sc.vl[j]), sc.vu[j]);
    }
    mat_mul(&sc.A, inner.x, inner.ax);
    const double sigma_inv = 1.0 / sigma;
    for (int64_t i = 0; i < m; ++i) {
      const double amid = 2.0 * inner.ax[i] - z.ax[i];
      const double v = sigma_inv * z.y[i] - amid;
      const double proj = smin(smax(v, -sc.cu[i]), -sc.cl[i]);
      inner.y[i] = z.y[i] - sigma * amid - sigma * proj;
    }
    mat_mul_t(&sc.A, inner.y, inner.aty);
    /* halpern_reflected_step / affine_combine (restart.cpp:23-52) */
    const double a = (double)(k + 1) / (double)(k + 2);
    const double b = 1.0 / (double)(k + 2);
    for (int64_t j = 0; j < n; ++j) {
      nx.x[j] = a * ((1.0 + gamma) * inner.x[j] - gamma * z.x[j]) + b * anc.x[j];
      nx.aty[j] = a * ((1.0 + gamma) * inner.aty[j] - gamma * z.aty[j]) + b * anc.aty[j];
    }
    for (int64_t i = 0; i < m; ++i) {
      nx.y[i] = a * ((1.0 + gamma) * inner.y[i] - gamma * z.y[i]) + b * anc.y[i];
      nx.ax[i] = a * ((1.0 + gamma) * inner.ax[i] - gamma * z.ax[i]) + b * anc.ax[i];
    }
    /* fixed_point_residual (pdhg.cpp:101-115) */
    double xx = 0.0, yy = 0.0, yax = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      const double d = z.x[j] - inner.x[j];
      xx += d * d;
    }
    for (int64_t i = 0; i < m; ++i) {
      const double d = z.y[i] - inner.y[i];
      yy += d * d;
    }
    for (int64_t i = 0; i < m; ++i) {
      const double d = z.y[i] - inner.y[i];
      const double dax = z.ax[i] - inner.ax[i];
      yax += d * dax;
    }
    const double ps = omega / eta, ds = 1.0 / (eta * omega);
    const double diag = ps * xx + ds * yy;
    const double q = diag + 2.0 * yax;
    double r;
    if (q >= 0.0) {
      r = sqrt(q);
    } else if (q >= -1e-12 * smax(diag, 1e-300)) {
      r = 0.0;
    } else {
      const double scale = ps * dot(z.x, z.x, n) + ds * dot(z.y, z.y, m);
      if (q >= -1e-24 * (1.0 + scale)) {
        r = 0.0;
      } else {
        rc = fail(RHPDHG_E_BREAKDOWN, "canonical norm radicand is negative beyond roundoff");
        goto done;
      }
    }
    /* restart verdict (solver.cpp:162-169, restart.cpp:54-69) */
    int verdict = 0;
    if (k == 0) {
      r_anchor = r;
      r_prev = r;
    } else {
      if (k >= 1 && isfinite(r_anchor)) {
        if (r <= cfg->beta_sufficient * r_anchor)
          verdict = 1;
        else if (r <= cfg->beta_necessary * r_anchor && r > r_prev)
          verdict = 2;
        else if ((double)k >= cfg->beta_artificial * (double)total)
          verdict = 3;
      }
      r_prev = r;
    }
    if (!cfg->restarts_enabled) verdict = 0;
    { It t = z; z = nx; nx = t; }
    k += 1;
    total += 1;
    last_fpr = r;
    have_inner = 1;
    if (cfg->record_residual_history) {
      if (hist && hist_len < hist_cap) hist[hist_len] = r;
      ++hist_len;
    }
    if (total % cfg->check_interval == 0 || verdict != 0) {
      rc = kkt_check(&z, &orig, rs, cs, xo, yo, axo, atyo, &res);
      ++checks;
      if (rc) goto done;
      if (is_optimal(&res, cfg->epsilon)) {
        status = RHPDHG_OPTIMAL;
        break;
      }
    }
    if (verdict != 0) { /* do_restart (restart.cpp:71-83) */
      omega = pid_update(&pid, &z, sx, sy, m, n);
      memcpy(sx, z.x, (size_t)n * sizeof(double));
      memcpy(sy, z.y, (size_t)m * sizeof(double));
      it_copy(&anc, &z, m, n);
      k = 0;
      restarts += 1;
      r_anchor = INFINITY;
      r_prev = INFINITY;
    }
    for (int s2 = 0; s2 < g_snap_nk; ++s2)
      if (g_snap_k[s2] == total) {
        for (int64_t j = 0; j < n; ++j) g_snap_x[(size_t)s2 * n + j] = cs[j] * z.x[j];
        for (int64_t i = 0; i < m; ++i) g_snap_y[(size_t)s2 * m + i] = rs[i] * z.y[i];
      }
  }
  if (status != RHPDHG_OPTIMAL) {
    rc = kkt_check(&z, &orig, rs, cs, xo, yo, axo, atyo, &res);
    ++checks;
    if (rc) goto done;
  }
  rep->status = status;
  {
    double acc = orig.offset;
    for (int64_t j = 0; j < n; ++j) acc += orig.c[j] * xo[j];
    rep->objective = orig.maxi ? -acc : acc;
  }
  rep->residuals = res;
  rep->iterations = total;
  rep->restart_count = restarts;
  rep->final_fixed_point_residual = last_fpr;
  rep->final_primal_weight = omega;
  rep->spmv_loop = 2ULL * (uint64_t)total;
  rep->spmv_checks = 2ULL * (uint64_t)checks;
  rep->kkt_checks = checks;
  rep->history_len = hist_len;
  if (x_out) memcpy(x_out, xo, (size_t)n * sizeof(double));
  if (y_out) memcpy(y_out, yo, (size_t)m * sizeof(double));
  if (rc_out)
    for (int64_t j = 0; j < n; ++j) rc_out[j] = clip_sign(orig.c[j] - atyo[j], orig.vl[j], orig.vu[j]);
  if (have_inner) { /* inner residuals of the last PDHG point (solver.cpp:228-234) */
    for (int64_t j = 0; j < n; ++j) xo[j] = cs[j] * inner.x[j];
    for (int64_t i = 0; i < m; ++i) yo[i] = rs[i] * inner.y[i];
    mat_mul(&orig.A, xo, axo);
    mat_mul_t(&orig.A, yo, atyo);
    rc = kkt(&orig, xo, yo, axo, atyo, &rep->inner_residuals);
    rep->has_inner_residuals = rc == 0;
  }
  rep->wall_time_seconds = now_s() - t0;
done:
  it_free(&z); it_free(&anc); it_free(&nx); it_free(&inner);
  free(sx); free(sy); free(xo); free(yo); free(axo); free(atyo); free(rs); free(cs);
  lp_free(&orig);
  lp_free(&sc);
  return rc;
}

int orc_solve_snapshots(const rhpdhg_lp_view* lp, const rhpdhg_config_c* cfg,
                        rhpdhg_report_c* rep, const int64_t* ks, int nk, double* xs, double* ys) {
  g_snap_k = ks;
  g_snap_nk = nk;
  g_snap_x = xs;
  g_snap_y = ys;
  const int rc = orc_solve_csr(lp, cfg, rep, NULL, NULL, NULL, NULL, 0);
  g_snap_k = NULL;
  g_snap_nk = 0;
  g_snap_x = g_snap_y = NULL;
  return rc;
}

/* ---------------------------------------------------------- per-op entry -- */
int orc_spmv(const rhpdhg_lp_view* lp, const double* in, double* out, int transpose) {
  Mat a;
  int rc = mat_from_view(lp, &a);
  if (!rc) {
    if (transpose)
      mat_mul_t(&a, in, out);
    else
      mat_mul(&a, in, out);
  }
  mat_free(&a);
  return rc;
}

int orc_scale(const rhpdhg_lp_view* lp, int ruiz_iters, int pc, double* csr_vals,
              double* csc_vals, double* row_scale, double* col_scale, double* c_s,
              double* var_lb_s, double* var_ub_s, double* con_lb_s, double* con_ub_s) {
  Lp o, s;
  int rc = lp_from_view(lp, &o);
  if (rc) {
    lp_free(&o);
    return rc;
  }
  lp_scale(&o, ruiz_iters, pc, &s, row_scale, col_scale);
  memcpy(csr_vals, s.A.v, (size_t)s.A.nnz * sizeof(double));
  memcpy(csc_vals, s.A.vt, (size_t)s.A.nnz * sizeof(double));
  memcpy(c_s, s.c, (size_t)s.n * sizeof(double));
  memcpy(var_lb_s, s.vl, (size_t)s.n * sizeof(double));
  memcpy(var_ub_s, s.vu, (size_t)s.n * sizeof(double));
  memcpy(con_lb_s, s.cl, (size_t)s.m * sizeof(double));
  memcpy(con_ub_s, s.cu, (size_t)s.m * sizeof(double));
  lp_free(&o);
  lp_free(&s);
  return 0;
}

int orc_power_iteration(const rhpdhg_lp_view* lp, double tol, int64_t max_iters, uint64_t seed,
                        double* value, int64_t* iterations, int32_t* converged) {
  Mat a;
  int rc = mat_from_view(lp, &a);
  if (!rc) {
    int c;
    power_iter(&a, tol, max_iters, seed, value, iterations, &c);
    *converged = c;
  }
  mat_free(&a);
  return rc;
}

int orc_kkt_residuals(const rhpdhg_lp_view* lp, const double* x, const double* y,
                      rhpdhg_kkt_c* out) {
  Lp p;
  int rc = lp_from_view(lp, &p);
  if (!rc) {
    double* ax = calloc((size_t)p.m + 1, sizeof(double));
    double* aty = calloc((size_t)p.n + 1, sizeof(double));
    mat_mul(&p.A, x, ax);
    mat_mul_t(&p.A, y, aty);
    rc = kkt(&p, x, y, ax, aty, out);
    free(ax);
    free(aty);
  }
  lp_free(&p);
  return rc;
}
