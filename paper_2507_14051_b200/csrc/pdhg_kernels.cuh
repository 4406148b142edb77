// pdhg_kernels.cuh — the fused PDHG iteration, KKT and power-iteration
// epilogues of the device library (the SpMV engine is spmv.cuh).
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
//   K3 = epilogue_walk<EpiPrimal>: the primal step of a block's first
//        iteration (after a KKT check or restart changed aty, tau or the
//        anchor), with K2's exact row->thread map so its partials are
//        bit-identical to K2's.
// The engines (spmv.cuh) call Epi::row(i, rowsum, e, stride, acc) once per
// row with the row's epilogue inputs loaded by the finishing lane: input k of
// row i is e[k*stride].
#pragma once

#include "spmv.cuh"

namespace rhp {

__device__ __forceinline__ double halpern_a(int64_t k) {
  return static_cast<double>(k + 1) / static_cast<double>(k + 2);
}
__device__ __forceinline__ double halpern_b(int64_t k) { return 1.0 / static_cast<double>(k + 2); }

// ------------------------------------------------------------ primal step --
struct PrimalOut {
  double* x;
  double* xplus;
};

// pdhg.cpp:41-45 + restart.cpp:44 for column j; acc gets the residual and PID
// partials of this column: ||x - x+||^2, ||x_new - x0||^2, ||x_new||^2, ||x||^2.
__device__ __forceinline__ void primal_col(const PrimalOut& o, int64_t j, double atyj, double xj,
                                           double cj, double lbj, double ubj, double x0j,
                                           double tau, double a, double opg, double g, double b,
                                           double* acc) {
  const double t = sub(xj, mul(tau, sub(cj, atyj)));
  const double xp = smin(smax(t, lbj), ubj);
  o.xplus[j] = xp;
  const double xn = affine(a, opg, g, b, xp, xj, x0j);
  o.x[j] = xn;
  const double dx = sub(xj, xp);
  const double d0 = sub(xn, x0j);
  acc[0] = fma(dx, dx, acc[0]);
  acc[1] = fma(d0, d0, acc[1]);
  acc[2] = fma(xn, xn, acc[2]);
  acc[3] = fma(xj, xj, acc[3]);
}

// K3 (walker): inputs aty, x, c, lb, ub, x0
struct EpiPrimal {
  static constexpr int NRED = 4;
  static constexpr int NIN = 6;
  Ctl* ctl;
  PrimalOut o;
  const double* in[NIN];
  ConstInputs cin;  // constant inputs (bounds), not loaded
  double a, b, g, opg, tau;
  __device__ bool enter() {
    const int64_t k = ctl->k;
    a = halpern_a(k);
    b = halpern_b(k);
    g = ctl->gamma;
    opg = 1.0 + g;
    tau = ctl->tau;
    return true;
  }
  __device__ void row(int64_t j, double, const double* e, int st, double (&acc)[NRED]) {
    primal_col(o, j, e[0], e[st], e[2 * st], e[3 * st], e[4 * st], e[5 * st], tau, a, opg, g, b,
               acc);
  }
  __device__ void walk_done() {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ctl->stop = 0;
      ctl->block_iters = 0;
      ctl->k1_token = -1;
    }
  }
};

// End-of-iteration control, one thread: fixed-point residual with its clamp
// rules (pdhg.cpp:101-115), restart verdict (restart.cpp:54-69,
// solver.cpp:162-169), k/total bookkeeping and the block-stop condition.
// t1 = y-side sums {||dy||^2, dy.dax, ||y-y0||^2, ||y||^2, ||y_old||^2},
// t3 = x-side sums {||dx||^2, ||x-x0||^2, ||x||^2, ||x_old||^2}.
__device__ __forceinline__ void pdhg_control(Ctl* ctl, const double* t1, const double* t3,
                                             int token) {
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
  const int stop =
      check_due || breakdown || total >= ctl->iteration_limit || bi + 1 >= ctl->block_limit;
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

// ------------------------------------------------------------------- K1 ----
// inputs: y, ax, con_lb, con_ub, y0, ax0
struct EpiDual {
  static constexpr int NRED = 5;
  static constexpr int NIN = 6;
  static constexpr bool REDUCE = true;
  static constexpr bool FINAL = true;
  Ctl* ctl;
  double* y;
  double* ax;
  double* yplus;
  const double* in[NIN];
  ConstInputs cin;  // constant inputs (bounds), not loaded
  const double* part3;     // primal partials [4][grid3]
  int grid3;
  int n_multi3;            // multi-chunk rows of the A^T schedule and their
  const double* long_red3; //   primal partial slots
  double* xchg;            // row-partitioned path: where the y-side sums go (else null)
  int token;               // launch index inside a plain (non-graph) block
  int guard;               // graph copy > 0 of an unrolled body: skip once stopped
  double sigma, sigma_inv, a, b, g, opg;

  __device__ bool enter() {
    if ((guard || !ctl->graph_mode) && ctl->stop && !ctl->bench) return false;
    sigma = ctl->sigma;
    sigma_inv = ctl->sigma_inv;
    const int64_t k = ctl->k;
    a = halpern_a(k);
    b = halpern_b(k);
    g = ctl->gamma;
    opg = 1.0 + g;
    return true;
  }

  __device__ void row(int64_t i, double axp, const double* e, int st, double (&acc)[NRED]) {
    const double yi = e[0], axi = e[st], lo = e[2 * st], hi = e[3 * st], y0i = e[4 * st],
                 ax0i = e[5 * st];
    const double amid = sub(mul(2.0, axp), axi);
    const double v = sub(mul(sigma_inv, yi), amid);
    const double proj = smin(smax(v, -hi), -lo);
    const double yp = sub(sub(yi, mul(sigma, amid)), mul(sigma, proj));
    yplus[i] = yp;
    const double yn = affine(a, opg, g, b, yp, yi, y0i);
    y[i] = yn;
    ax[i] = affine(a, opg, g, b, axp, axi, ax0i);
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
    iteration_sums<5, 4>(part, grid, s.long_red, s.n_multi, part3, grid3, long_red3, n_multi3, t1,
                         t3);
    if (threadIdx.x != 0) return;
    if (xchg) {  // row-partitioned: publish the local y-side sums, control after the allreduce
#pragma unroll
      for (int q = 0; q < 5; ++q) xchg[q] = t1[q];
      ctl->k1_token_pending = token;
      return;
    }
    pdhg_control(ctl, t1, t3, token);
  }
};

// ------------------------------------------------- row-partitioned (NCCL) --
// After the allreduce of [A_p^T y+_p partials (n) | y-side sums (5)]:
// one CTA reduces the (replicated, rank-identical) x-side partials and runs
// the control on the global sums.
// xsums: the allreduced y-side sums (5); x_sums (sharded path): the
// allreduced x-side sums (4) of the previous n-side walk, else they are
// reduced here from the (rank-identical) walker partials part3.
__global__ void __launch_bounds__(kBlock) k_dist_control(Ctl* ctl, const double* part3, int grid3,
                                                         int n_multi3, const double* long_red3,
                                                         const double* xsums, int token,
                                                         const double* x_sums) {
  if (!ctl->graph_mode && ctl->k1_token_pending != token && !ctl->bench) {
    // an iteration past the block's stop: tell the host (rhp_run_block polls)
    if (threadIdx.x == 0 && ctl->stop_mirror) reinterpret_cast<volatile int*>(ctl->stop_mirror)[token] = 1;
    return;
  }
  double t3[4];
  if (x_sums) {
    for (int q = 0; q < 4; ++q) t3[q] = __ldcg(x_sums + q);
  } else {
    block_sum_partials<4>(part3, grid3, grid3, t3);
    add_slots<4>(long_red3, n_multi3, t3);
  }
  if (threadIdx.x == 0) {
    double t1[5];
    for (int q = 0; q < 5; ++q) t1[q] = __ldcg(xsums + q);
    pdhg_control(ctl, t1, t3, token);
    if (ctl->stop_mirror) reinterpret_cast<volatile int*>(ctl->stop_mirror)[token] = ctl->stop;
  }
}

// K2c: aty Halpern update + next primal step from the allreduced A^T y+.
// inputs: aty+ (allreduced), aty, aty0, x, c, var_lb, var_ub, x0
struct EpiAtyDist {
  static constexpr int NRED = 4;
  static constexpr int NIN = 8;
  Ctl* ctl;
  double* aty;
  PrimalOut o;
  const double* in[NIN];
  ConstInputs cin;  // constant inputs (bounds), not loaded
  int token;
  double a, b, a2, b2, g, opg, tau;
  int stop;
  __device__ bool enter() {
    if (!ctl->graph_mode && ctl->k1_token != token && !ctl->bench) return false;
    const int64_t k = ctl->k;
    a = halpern_a(k - 1);
    b = halpern_b(k - 1);
    a2 = halpern_a(k);
    b2 = halpern_b(k);
    g = ctl->gamma;
    opg = 1.0 + g;
    tau = ctl->tau;
    stop = ctl->stop && !ctl->bench;
    return true;
  }
  __device__ void row(int64_t j, double, const double* e, int st, double (&acc)[NRED]) {
    const double atyn = affine(a, opg, g, b, e[0], e[st], e[2 * st]);
    aty[j] = atyn;
    if (!stop)
      primal_col(o, j, atyn, e[3 * st], e[4 * st], e[5 * st], e[6 * st], e[7 * st], tau, a2, opg,
                 g, b2, acc);
  }
  __device__ void walk_done() {}
};

// ------------------------------------------------------------------- K2 ----
// inputs: aty, aty0, x, c, var_lb, var_ub, x0
struct EpiAty {
  static constexpr int NRED = 4;
  static constexpr int NIN = 7;
  static constexpr bool REDUCE = true;
  static constexpr bool FINAL = false;
  Ctl* ctl;
  double* aty;
  PrimalOut o;
  const double* in[NIN];
  ConstInputs cin;  // constant inputs (bounds), not loaded
  int token;
  int guard;  // graph copy > 0 of an unrolled body: run only after its own K1
  double a, b, a2, b2, g, opg, tau;
  int stop;

  __device__ bool enter() {
    if ((guard || !ctl->graph_mode) && ctl->k1_token != token && !ctl->bench) return false;
    const int64_t k = ctl->k;  // already incremented by K1's finalize
    a = halpern_a(k - 1);
    b = halpern_b(k - 1);
    a2 = halpern_a(k);
    b2 = halpern_b(k);
    g = ctl->gamma;
    opg = 1.0 + g;
    tau = ctl->tau;
    stop = ctl->stop && !ctl->bench;
    return true;
  }

  __device__ void row(int64_t j, double atyp, const double* e, int st, double (&acc)[NRED]) {
    const double atyn = affine(a, opg, g, b, atyp, e[0], e[st]);
    aty[j] = atyn;
    if (!stop)
      primal_col(o, j, atyn, e[2 * st], e[3 * st], e[4 * st], e[5 * st], e[6 * st], tau, a2, opg,
                 g, b2, acc);
  }
  __device__ void finalize(const Sched&, const double*, int) {}
};

// ------------------------------------------------------------ plain store --
struct EpiStore {
  static constexpr int NRED = 1;
  static constexpr int NIN = 0;
  static constexpr bool REDUCE = false;
  static constexpr bool FINAL = false;
  double* out;
  const double* in[1];
  Ctl* ctl;   // optional guard (row-partitioned A^T pass): run only after K1 of `token`
  int token;
  __device__ bool enter() {
    return !ctl || ctl->graph_mode || ctl->bench || ctl->k1_token_pending == token;
  }
  __device__ void row(int64_t i, double s, const double*, int, double (&)[NRED]) { out[i] = s; }
  __device__ void finalize(const Sched&, const double*, int) {}
};

// Intermediate column segment of a segmented operator (rhp_cuda.cu
// launch_spmv): stores its row sums like EpiStore, but runs only when the
// final segment's epilogue `Gate` will (same enter() test, evaluated on a
// copy), so iterations past a block's stop skip every segment pass, not just
// the last.
template <class Gate>
struct EpiSegStore {
  static constexpr int NRED = 1;
  static constexpr int NIN = 0;
  static constexpr bool REDUCE = false;
  static constexpr bool FINAL = false;
  double* out;
  const double* in[1];
  Gate gate;
  __device__ bool enter() {
    Gate g = gate;
    return g.enter();
  }
  __device__ void row(int64_t i, double s, const double*, int, double (&)[NRED]) { out[i] = s; }
  __device__ void finalize(const Sched&, const double*, int) {}
};

// w = A^T (A v): store w, reduce v.w and w.w (pdhg.cpp:141-146); input: v
struct EpiPowerW {
  static constexpr int NRED = 2;
  static constexpr int NIN = 1;
  static constexpr bool REDUCE = true;
  static constexpr bool FINAL = true;
  Ctl* ctl;
  double* w;
  const double* in[NIN];
  __device__ bool enter() { return true; }
  __device__ void row(int64_t j, double s, const double* e, int, double (&acc)[NRED]) {
    w[j] = s;
    acc[0] = fma(e[0], s, acc[0]);
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
// inputs: y (scaled), D_row, con_lb, con_ub (original)
struct EpiKktRow {
  static constexpr int NRED = 4;
  static constexpr int NIN = 4;
  static constexpr bool REDUCE = true;
  static constexpr bool FINAL = false;
  double* ax_refresh;  // may be null
  double* yout;        // may be null
  const double* in[NIN];
  __device__ bool enter() { return true; }
  __device__ void row(int64_t i, double s, const double* e, int st, double (&acc)[NRED]) {
    if (ax_refresh) ax_refresh[i] = s;
    const double ri = e[st];
    const double ao = s / ri;
    const double yo = mul(ri, e[0]);
    if (yout) yout[i] = yo;
    if (isnan(yo)) acc[0] += 1.0;
    const double lo = e[2 * st], up = e[3 * st];
    const double proj = smin(smax(ao, lo), up);
    const double d = sub(ao, proj);
    acc[1] = fma(d, d, acc[1]);
    double t;
    if (p_term(yo, lo, up, &t)) acc[3] += t;
    else acc[2] += 1.0;
  }
  __device__ void finalize(const Sched&, const double*, int) {}
};

// inputs: x (scaled), D_col, c, var_lb, var_ub (original)
struct EpiKktCol {
  static constexpr int NRED = 6;
  static constexpr int NIN = 5;
  static constexpr bool REDUCE = true;
  static constexpr bool FINAL = true;
  Ctl* ctl;
  double* aty_refresh;  // may be null
  double* xout;         // may be null
  double* rcout;        // may be null
  const double* in[NIN];
  const double* part_row;  // EpiKktRow partials [4][grid_row]
  int grid_row;
  int n_multi_row;
  const double* long_red_row;

  __device__ bool enter() { return true; }
  __device__ void row(int64_t j, double s, const double* e, int st, double (&acc)[NRED]) {
    if (aty_refresh) aty_refresh[j] = s;
    const double cj = e[st];
    const double ato = s / cj;
    const double xo = mul(cj, e[0]);
    if (xout) xout[j] = xo;
    if (isnan(xo)) acc[0] += 1.0;
    const double c = e[2 * st], lb = e[3 * st], ub = e[4 * st];
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
    add_slots<4>(long_red_row, n_multi_row, tr);  // multi-chunk rows of the A pass
    if (threadIdx.x == 0) {
      ctl->kkt_nan_y = tr[0];
      ctl->kkt_viol2 = tr[1];
      ctl->kkt_py_inf = tr[2];
      ctl->kkt_py = tr[3];
      ctl->kkt_nan_x = tc[0];
      ctl->kkt_pr_inf = tc[1];
      ctl->kkt_pr = tc[2];
      ctl->kkt_eq2 = tc[3];
      ctl->kkt_cone2 = tc[4];
      ctl->kkt_cx = tc[5];
    }
  }
};

// ---------------------------------------- row-partitioned KKT and power ----
// KA (local rows): as EpiKktRow, the last block publishes the 4 row-side sums
// into the exchange buffer that is allreduced with the A^T partial.
struct EpiKktRowDist : EpiKktRow {
  static constexpr bool FINAL = true;
  double* xsums;  // 4 doubles
  __device__ void finalize(const Sched& s, const double* part, int grid) {
    double t[4];
    block_sum_partials<4>(part, grid, grid, t);
    add_long_slots<4>(s, t);
    if (threadIdx.x == 0)
      for (int q = 0; q < 4; ++q) xsums[q] = t[q];
  }
};

// KB (all columns, redundant on every rank): as EpiKktCol with the allreduced
// A^T y as input 0. inputs: aty (allreduced), x, D_col, c, var_lb, var_ub
struct EpiKktColDist {
  static constexpr int NRED = 6;
  static constexpr int NIN = 6;
  EpiKktCol col;  // row() logic; col.in[] = in[1..5]
  const double* in[NIN];
  __device__ bool enter() { return true; }
  __device__ void row(int64_t j, double, const double* e, int st, double (&acc)[NRED]) {
    col.row(j, e[0], e + st, st, acc);
  }
  __device__ void walk_done() {}
};

__global__ void __launch_bounds__(kBlock) k_kkt_dist_finalize(Ctl* ctl, const double* part,
                                                              int grid, int n_multi,
                                                              const double* long_red,
                                                              const double* xsums) {
  double tc[6];
  block_sum_partials<6>(part, grid, grid, tc);
  add_slots<6>(long_red, n_multi, tc);
  if (threadIdx.x == 0) {
    ctl->kkt_nan_y = __ldcg(xsums + 0);
    ctl->kkt_viol2 = __ldcg(xsums + 1);
    ctl->kkt_py_inf = __ldcg(xsums + 2);
    ctl->kkt_py = __ldcg(xsums + 3);
    ctl->kkt_nan_x = tc[0];
    ctl->kkt_pr_inf = tc[1];
    ctl->kkt_pr = tc[2];
    ctl->kkt_eq2 = tc[3];
    ctl->kkt_cone2 = tc[4];
    ctl->kkt_cx = tc[5];
  }
}

// power iteration, w = allreduced A^T (A_p v): inputs w, v
struct EpiPowerDist {
  static constexpr int NRED = 2;
  static constexpr int NIN = 2;
  double* w;
  const double* in[NIN];
  __device__ bool enter() { return true; }
  __device__ void row(int64_t j, double, const double* e, int st, double (&acc)[NRED]) {
    const double s = e[0];
    w[j] = s;
    acc[0] = fma(e[st], s, acc[0]);
    acc[1] = fma(s, s, acc[1]);
  }
  __device__ void walk_done() {}
};

__global__ void __launch_bounds__(kBlock) k_power_dist_finalize(Ctl* ctl, const double* part,
                                                                int grid, int n_multi,
                                                                const double* long_red) {
  double t[2];
  block_sum_partials<2>(part, grid, grid, t);
  add_slots<2>(long_red, n_multi, t);
  if (threadIdx.x == 0) {
    ctl->pw_vw = t[0];
    ctl->pw_ww = t[1];
  }
}

// ------------------------------------------------ sharded (Option B) helpers --
// One CTA: the N walker partials (fixed order) into out[0..N), this rank's
// share of the scalars the next allreduce sums.
template <int N>
__global__ void __launch_bounds__(kBlock) k_sum_partials(const double* part, int grid, double* out) {
  double t[N];
  block_sum_partials<N>(part, grid, grid, t);
  if (threadIdx.x == 0)
    for (int q = 0; q < N; ++q) out[q] = t[q];
}

// The KKT sums from the allreduced scalars: row side s[0..4), column side
// s[4..10) (layout of EpiKktRowDist / EpiKktCol partials).
__global__ void k_kkt_from_sums(Ctl* ctl, const double* s) {
  if (threadIdx.x != 0) return;
  ctl->kkt_nan_y = __ldcg(s + 0);
  ctl->kkt_viol2 = __ldcg(s + 1);
  ctl->kkt_py_inf = __ldcg(s + 2);
  ctl->kkt_py = __ldcg(s + 3);
  ctl->kkt_nan_x = __ldcg(s + 4);
  ctl->kkt_pr_inf = __ldcg(s + 5);
  ctl->kkt_pr = __ldcg(s + 6);
  ctl->kkt_eq2 = __ldcg(s + 7);
  ctl->kkt_cone2 = __ldcg(s + 8);
  ctl->kkt_cx = __ldcg(s + 9);
}

__global__ void k_power_from_sums(Ctl* ctl, const double* s) {
  if (threadIdx.x != 0) return;
  ctl->pw_vw = __ldcg(s + 0);
  ctl->pw_ww = __ldcg(s + 1);
}

}  // namespace rhp
