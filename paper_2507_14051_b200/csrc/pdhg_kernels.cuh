// pdhg_kernels.cuh — the fused PDHG iteration, KKT, power-iteration and
// scaling kernels of the device library.
//
// One restarted reflected-Halpern PDHG iteration (reference solver.cpp:158-181)
// is two launches on one GPU:
//
//   K1 = spmv_fused<EpiDual> over A (rows = constraints):
//        ax+ = A x+ (row sum), then per row, in one HBM pass
//          amid = 2 ax+ - ax, v = y/sigma - amid, y+ = y - sigma amid - sigma proj
//                                                     (pdhg.cpp:49-56)
//          y  <- a((1+g) y+  - g y ) + b y0          (restart.cpp:44-45)
//          ax <- a((1+g) ax+ - g ax) + b ax0         (restart.cpp:47)
//        and block partials of ||dy||^2, dy.(ax-ax+), ||y-y0||^2, ||y||^2,
//        ||y_old||^2. The last block to finish reduces them together with the
//        primal partials, evaluates the fixed-point residual with its clamp
//        rules (pdhg.cpp:101-115), the restart verdict (restart.cpp:54-69,
//        solver.cpp:162-169), the k/total bookkeeping and the block-stop
//        condition, and sets the CUDA-graph WHILE condition.
//   K2 = spmv_fused<EpiAty> over A^T (rows = variables):
//        aty+ = A^T y+, aty <- a((1+g) aty+ - g aty) + b aty0 (restart.cpp:48),
//        then, unless the block stops, the NEXT iteration's primal step in the
//        same pass: x+ = clamp(x - tau(c - aty), l, u) (pdhg.cpp:41-45) and
//        x <- a'((1+g) x+ - g x) + b' x0 with partials ||dx||^2, ||x-x0||^2,
//        ||x||^2, ||x_old||^2.
//   K3 = primal_init: the primal step of a block's first iteration (after a
//        KKT check or restart changed aty, tau or the anchor).
#pragma once

#include "spmv.cuh"

namespace rhp {

// ------------------------------------------------------------ primal step --
struct PrimalArgs {
  double* x;
  double* xplus;
  const double* x0;
  const double* c;
  const double* vl;
  const double* vu;
};

// pdhg.cpp:41-45 + restart.cpp:44 for one column; acc gets the residual and
// PID partials of this column.
__device__ __forceinline__ void primal_col(const PrimalArgs& p, int64_t j, double atyj, double tau,
                                           double a, double opg, double g, double b,
                                           double (&acc)[4]) {
  const double xj = p.x[j];
  const double t = sub(xj, mul(tau, sub(p.c[j], atyj)));
  const double xp = smin(smax(t, p.vl[j]), p.vu[j]);
  p.xplus[j] = xp;
  const double x0j = p.x0[j];
  const double xn = affine(a, opg, g, b, xp, xj, x0j);
  p.x[j] = xn;
  const double dx = sub(xj, xp);
  const double d0 = sub(xn, x0j);
  acc[0] = fma(dx, dx, acc[0]);
  acc[1] = fma(d0, d0, acc[1]);
  acc[2] = fma(xn, xn, acc[2]);
  acc[3] = fma(xj, xj, acc[3]);
}

__device__ __forceinline__ double halpern_a(int64_t k) {
  return static_cast<double>(k + 1) / static_cast<double>(k + 2);
}
__device__ __forceinline__ double halpern_b(int64_t k) { return 1.0 / static_cast<double>(k + 2); }

// K3: first primal step of a block. Also resets the block counters.
__global__ void __launch_bounds__(kBlock) primal_init(Ctl* ctl, PrimalArgs p, const double* aty,
                                                      int64_t n, double* part3) {
  const int64_t k = ctl->k;
  const double a = halpern_a(k), b = halpern_b(k);
  const double g = ctl->gamma, opg = 1.0 + g, tau = ctl->tau;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t j = blockIdx.x * (int64_t)kBlock + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kBlock)
    primal_col(p, j, aty[j], tau, a, opg, g, b, acc);
  block_reduce_store<4>(acc, part3, gridDim.x, blockIdx.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->stop = 0;
    ctl->block_iters = 0;
    ctl->k1_token = -1;
  }
}

// ------------------------------------------------------------------- K1 ----
struct EpiDual {
  static constexpr int NRED = 5;
  static constexpr bool REDUCE = true;
  static constexpr bool FINAL = true;
  Ctl* ctl;
  double* y;
  double* ax;
  double* yplus;
  const double* y0;
  const double* ax0;
  const double* cl;
  const double* cu;
  const double* part3;  // primal partials [4][grid3]
  int grid3;
  int token;            // launch index inside a plain (non-graph) block
  // per-thread scalars loaded in enter()
  double sigma, sigma_inv, a, b, g, opg;

  __device__ bool enter() {
    if (!ctl->graph_mode && ctl->stop && !ctl->bench) return false;
    sigma = ctl->sigma;
    sigma_inv = ctl->sigma_inv;
    const int64_t k = ctl->k;
    a = halpern_a(k);
    b = halpern_b(k);
    g = ctl->gamma;
    opg = 1.0 + g;
    return true;
  }

  __device__ void row(int64_t i, double axp, double (&acc)[NRED]) {
    const double yi = y[i], axi = ax[i];
    const double amid = sub(mul(2.0, axp), axi);
    const double v = sub(mul(sigma_inv, yi), amid);
    const double proj = smin(smax(v, -cu[i]), -cl[i]);
    const double yp = sub(sub(yi, mul(sigma, amid)), mul(sigma, proj));
    yplus[i] = yp;
    const double y0i = y0[i];
    const double yn = affine(a, opg, g, b, yp, yi, y0i);
    y[i] = yn;
    ax[i] = affine(a, opg, g, b, axp, axi, ax0[i]);
    const double dy = sub(yi, yp);
    const double dax = sub(axi, axp);
    const double d0 = sub(yn, y0i);
    acc[0] = fma(dy, dy, acc[0]);
    acc[1] = fma(dy, dax, acc[1]);
    acc[2] = fma(d0, d0, acc[2]);
    acc[3] = fma(yn, yn, acc[3]);
    acc[4] = fma(yi, yi, acc[4]);
  }

  // Last block: fixed-point residual, restart verdict, counters, stop flag.
  __device__ void finalize(const Sched& s, const double* part, int grid) {
    double t1[5], t3[4];
    block_sum_partials<5>(part, grid, grid, t1);
    add_long_slots<5>(s, t1);
    block_sum_partials<4>(part3, grid3, grid3, t3);
    if (threadIdx.x != 0) return;
    const double ps = ctl->primal_scale, ds = ctl->dual_scale;
    // quadratic_form(dx, dy, d_ax) (pdhg.cpp:68-75)
    const double diag = add(mul(ps, t3[0]), mul(ds, t1[0]));
    const double q = add(diag, mul(2.0, t1[1]));
    double r = 0.0;
    int breakdown = 0;
    if (q >= 0.0) {
      r = sqrt(q);
    } else if (q >= -1e-12 * smax(diag, 1e-300)) {
      r = 0.0;
    } else {
      const double scale = add(mul(ps, t3[3]), mul(ds, t1[4]));
      if (q >= -1e-24 * (1.0 + scale)) r = 0.0;
      else breakdown = 1;
    }
    int64_t k = ctl->k, total = ctl->total;
    int verdict = 0;
    double r_anchor = ctl->r_anchor, r_prev = ctl->r_prev;
    if (k == 0) {
      r_anchor = r;
      r_prev = r;
    } else {
      if (k >= 1 && isfinite(r_anchor)) {
        if (r <= ctl->beta_s * r_anchor) verdict = 1;
        else if (r <= ctl->beta_n * r_anchor && r > r_prev) verdict = 2;
        else if (static_cast<double>(k) >= ctl->beta_a * static_cast<double>(total)) verdict = 3;
      }
      r_prev = r;
    }
    if (!ctl->restarts_enabled) verdict = 0;
    k += 1;
    total += 1;
    const int64_t bi = ctl->block_iters;
    if (ctl->record_history) ctl->hist[bi] = r;
    const int check_due = (total % ctl->check_interval == 0) || verdict != 0;
    const int stop = check_due || breakdown || total >= ctl->iteration_limit ||
                     bi + 1 >= ctl->block_limit;
    ctl->k = k;
    ctl->total = total;
    ctl->block_iters = bi + 1;
    ctl->r_anchor = r_anchor;
    ctl->r_prev = r_prev;
    ctl->r_last = r;
    ctl->q_last = q;
    ctl->verdict = verdict;
    ctl->check_due = check_due;
    ctl->breakdown = breakdown;
    ctl->stop = stop;
    ctl->k1_token = token;
    ctl->x_dist2 = t3[1];
    ctl->x_norm2 = t3[2];
    ctl->y_dist2 = t1[2];
    ctl->y_norm2 = t1[3];
    if (ctl->graph_mode) cudaGraphSetConditional(ctl->cond_handle, stop ? 0u : 1u);
  }
};

// ------------------------------------------------------------------- K2 ----
struct EpiAty {
  static constexpr int NRED = 4;
  static constexpr bool REDUCE = true;
  static constexpr bool FINAL = false;
  Ctl* ctl;
  double* aty;
  const double* aty0;
  PrimalArgs p;
  int token;
  double a, b, a2, b2, g, opg, tau;
  int stop;

  __device__ bool enter() {
    if (!ctl->graph_mode && ctl->k1_token != token && !ctl->bench) return false;
    const int64_t k = ctl->k;  // already incremented by K1's finalize
    a = halpern_a(k - 1);
    b = halpern_b(k - 1);
    a2 = halpern_a(k);
    b2 = halpern_b(k);
    g = ctl->gamma;
    opg = 1.0 + g;
    tau = ctl->tau;
    stop = ctl->stop;
    return true;
  }

  __device__ void row(int64_t j, double atyp, double (&acc)[NRED]) {
    const double atyn = affine(a, opg, g, b, atyp, aty[j], aty0[j]);
    aty[j] = atyn;
    if (!stop) primal_col(p, j, atyn, tau, a2, opg, g, b2, acc);
  }
  __device__ void finalize(const Sched&, const double*, int) {}
};

// ------------------------------------------------------------ plain store --
struct EpiStore {
  static constexpr int NRED = 1;
  static constexpr bool REDUCE = false;
  static constexpr bool FINAL = false;
  double* out;
  __device__ bool enter() { return true; }
  __device__ void row(int64_t i, double s, double (&)[NRED]) { out[i] = s; }
  __device__ void finalize(const Sched&, const double*, int) {}
};

// w = A^T (A v): store w, reduce v.w and w.w (pdhg.cpp:141-146)
struct EpiPowerW {
  static constexpr int NRED = 2;
  static constexpr bool REDUCE = true;
  static constexpr bool FINAL = true;
  Ctl* ctl;
  const double* v;
  double* w;
  __device__ bool enter() { return true; }
  __device__ void row(int64_t j, double s, double (&acc)[NRED]) {
    w[j] = s;
    acc[0] = fma(v[j], s, acc[0]);
    acc[1] = fma(s, s, acc[1]);
  }
  __device__ void finalize(const Sched& sc, const double* part, int grid) {
    double t[2];
    block_sum_partials<2>(part, grid, grid, t);
    add_long_slots<2>(sc, t);
    if (threadIdx.x == 0) {
      ctl->pw_vw = t[0];
      ctl->pw_ww = t[1];
    }
  }
};

// --------------------------------------------------------------- KKT -------
// p_support term of one coordinate of -v (lp_problem.cpp:72-87); returns
// false for a +inf term.
__device__ __forceinline__ bool p_term(double v_neg_src, double lb, double ub, double* term) {
  const double v = -v_neg_src;
  const double yp = smax(v, 0.0);
  const double yn = smax(-v, 0.0);
  const double up = yp == 0.0 ? 0.0 : mul(ub, yp);
  const double lo = yn == 0.0 ? 0.0 : mul(lb, yn);
  if (up == CUDART_INF || lo == -CUDART_INF) return false;
  *term = sub(up, lo);
  return true;
}

// clip_to_sign_cone (termination.cpp:24-31)
__device__ __forceinline__ double clip_sign(double s, double lb, double ub) {
  const bool lf = lb > -CUDART_INF, uf = ub < CUDART_INF;
  if (lf && uf) return s;
  if (lf) return smax(s, 0.0);
  if (uf) return smin(s, 0.0);
  return 0.0;
}

// Over A: products of the scaled matrix give the original ones as
// (A_orig x_orig)_i = (Abar xbar)_i / D_row_i; refresh z.ax = Abar xbar
// (solver.cpp:42); primal violation and p(-y) (termination.cpp:69-103).
struct EpiKktRow {
  static constexpr int NRED = 4;
  static constexpr bool REDUCE = true;
  static constexpr bool FINAL = false;
  double* ax_refresh;   // may be null
  const double* y;      // scaled y
  const double* rs;     // D_row
  const double* clo;    // original con bounds
  const double* cuo;
  double* yout;         // may be null
  __device__ bool enter() { return true; }
  __device__ void row(int64_t i, double s, double (&acc)[NRED]) {
    if (ax_refresh) ax_refresh[i] = s;
    const double ri = rs[i];
    const double ao = s / ri;
    const double yo = mul(ri, y[i]);
    if (yout) yout[i] = yo;
    if (isnan(yo)) acc[0] += 1.0;
    const double lo = clo[i], up = cuo[i];
    const double proj = smin(smax(ao, lo), up);
    const double d = sub(ao, proj);
    acc[1] = fma(d, d, acc[1]);
    double t;
    if (p_term(yo, lo, up, &t)) acc[3] += t;
    else acc[2] += 1.0;
  }
  __device__ void finalize(const Sched&, const double*, int) {}
};

struct EpiKktCol {
  static constexpr int NRED = 6;
  static constexpr bool REDUCE = true;
  static constexpr bool FINAL = true;
  Ctl* ctl;
  double* aty_refresh;  // may be null
  const double* x;      // scaled x
  const double* cs;     // D_col
  const double* co;     // original c, var bounds
  const double* vlo;
  const double* vuo;
  double* xout;         // may be null
  double* rcout;        // may be null
  const double* part_row;  // EpiKktRow partials [4][grid_row]
  int grid_row;
  int n_multi_row;
  const double* long_red_row;

  __device__ bool enter() { return true; }
  __device__ void row(int64_t j, double s, double (&acc)[NRED]) {
    if (aty_refresh) aty_refresh[j] = s;
    const double cj = cs[j];
    const double ato = s / cj;
    const double xo = mul(cj, x[j]);
    if (xout) xout[j] = xo;
    if (isnan(xo)) acc[0] += 1.0;
    const double c = co[j], lb = vlo[j], ub = vuo[j];
    const double slack = sub(c, ato);
    const double r = clip_sign(slack, lb, ub);
    if (rcout) rcout[j] = r;
    double t;
    if (p_term(r, lb, ub, &t)) acc[2] += t;
    else acc[1] += 1.0;
    const double d = sub(slack, r);
    acc[3] = fma(d, d, acc[3]);
    const double cc = sub(r, clip_sign(r, lb, ub));
    acc[4] = fma(cc, cc, acc[4]);
    acc[5] = fma(c, xo, acc[5]);
  }
  __device__ void finalize(const Sched& sc, const double* part, int grid) {
    double tc[6], tr[4];
    block_sum_partials<6>(part, grid, grid, tc);
    add_long_slots<6>(sc, tc);
    block_sum_partials<4>(part_row, grid_row, grid_row, tr);
    // multi-chunk rows of the A pass
    __shared__ double lr[4];
    if (threadIdx.x < 4) {
      double v = 0.0;
      for (int i = 0; i < n_multi_row; ++i) v += __ldcg(long_red_row + (size_t)i * 16 + threadIdx.x);
      lr[threadIdx.x] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      ctl->kkt_nan_y = tr[0] + lr[0];
      ctl->kkt_viol2 = tr[1] + lr[1];
      ctl->kkt_py_inf = tr[2] + lr[2];
      ctl->kkt_py = tr[3] + lr[3];
      ctl->kkt_nan_x = tc[0];
      ctl->kkt_pr_inf = tc[1];
      ctl->kkt_pr = tc[2];
      ctl->kkt_eq2 = tc[3];
      ctl->kkt_cone2 = tc[4];
      ctl->kkt_cx = tc[5];
    }
  }
};

// ------------------------------------------------------------- scaling -----
// Per-row max |a| -> sqrt or 1 (scaling.cpp:56-61). Max is order-free.
__global__ void k_row_absmax_sqrt(const int64_t* rp, const double* w, int64_t rows, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * kBlock) {
    double mx = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const double a = fabs(w[e]);
      if (a > mx) mx = a;
    }
    out[i] = mx > 0.0 ? sqrt(mx) : 1.0;
  }
}

// w /= rmax_row * cmax_col (scaling.cpp:62), for an operator whose rows carry
// `row_fac` and columns `col_fac`; `row_first` keeps the reference's factor
// order rmax*cmax (multiplication is commutative, so both orders agree).
__global__ void k_ruiz_divide(const int64_t* rp, const int32_t* ci, double* w, int64_t rows,
                              const double* row_fac, const double* col_fac) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * kBlock) {
    const double fr = row_fac[i];
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) w[e] = __ddiv_rn(w[e], mul(fr, col_fac[ci[e]]));
  }
}

__global__ void k_vec_div(double* s, const double* by, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kBlock)
    s[i] = __ddiv_rn(s[i], by[i]);
}

__global__ void k_vec_mul(double* s, const double* by, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kBlock)
    s[i] = mul(s[i], by[i]);
}

// out_e = (f_row * a_e) * f_col (sparse_matrix.cpp:109 for CSR with
// f_row = r, f_col = c; :112 for CSC with f_row = c, f_col = r).
__global__ void k_scale_values(const int64_t* rp, const int32_t* ci, const double* src,
                               double* dst, int64_t rows, const double* f_row,
                               const double* f_col) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * kBlock) {
    const double fr = f_row[i];
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) dst[e] = mul(mul(fr, src[e]), f_col[ci[e]]);
  }
}

// Row 1-norms of the CSR values, sequential per row (sparse_matrix.cpp:130-133):
// out = 1/sqrt(norm) or 1 (scaling.cpp:73).
__global__ void k_pc_rows(const int64_t* rp, const double* v, int64_t rows, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * kBlock) {
    double acc = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) acc = add(acc, fabs(v[e]));
    out[i] = acc > 0.0 ? __ddiv_rn(1.0, sqrt(acc)) : 1.0;
  }
}

// Column 1-norms as the reference accumulates them: for column j, the CSR
// values (r_i a_ij) c_j added in ascending row order (sparse_matrix.cpp:134).
// Walks row j of A^T (ascending original rows) recomputing the CSR value
// from the original a_ij.
__global__ void k_pc_cols(const int64_t* rp, const int32_t* ci, const double* a_orig,
                          int64_t rows, const double* rs, const double* cs, double* out) {
  for (int64_t j = blockIdx.x * (int64_t)kBlock + threadIdx.x; j < rows;
       j += (int64_t)gridDim.x * kBlock) {
    const double cj = cs[j];
    double acc = 0.0;
    for (int64_t e = rp[j]; e < rp[j + 1]; ++e) acc = add(acc, fabs(mul(mul(rs[ci[e]], a_orig[e]), cj)));
    out[j] = acc > 0.0 ? __ddiv_rn(1.0, sqrt(acc)) : 1.0;
  }
}

// apply_scales on the vectors (scaling.cpp:21-32):
//   c <- cs*c, lb <- lb/cs, ub <- ub/cs ; con bounds <- rs*bound
__global__ void k_apply_col_scales(double* c, double* lb, double* ub, const double* cs, int64_t n) {
  for (int64_t j = blockIdx.x * (int64_t)kBlock + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kBlock) {
    const double s = cs[j];
    c[j] = mul(s, c[j]);
    lb[j] = __ddiv_rn(lb[j], s);
    ub[j] = __ddiv_rn(ub[j], s);
  }
}
__global__ void k_apply_row_scales(double* lb, double* ub, const double* rs, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * kBlock) {
    const double s = rs[i];
    lb[i] = mul(s, lb[i]);
    ub[i] = mul(s, ub[i]);
  }
}

__global__ void k_normalize(double* v, const double* w, double wn, int64_t n) {
  for (int64_t j = blockIdx.x * (int64_t)kBlock + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kBlock)
    v[j] = __ddiv_rn(w[j], wn);
}

}  // namespace rhp
