// ref_adapter.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" shim over the *unmodified* reference library compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/. It lets the
// Python parity tests and bench.py's CPU-baseline leg call the reference's own
// public C++ API (proj/include/rhpdhg/*.hpp) with the same flat structs as the
// product's C ABI (include/rhpdhg_c.h), so product and reference are driven
// identically:
//   ref_solve_csr          -> rhpdhg::solve                 (solver.cpp:63-238)
//   ref_kkt_residuals      -> rhpdhg::kkt_residuals         (termination.cpp:49-56)
//   ref_spmv / ref_spmv_t  -> SparseMatrix::multiply{,_transpose} (sparse_matrix.cpp:67-87)
//   ref_scale              -> ruiz_equilibrate + pock_chambolle_scale (scaling.cpp:46-81)
//   ref_power_iteration    -> power_iteration_norm          (pdhg.cpp:117-170)
//   ref_lp_from_mps        -> parse_mps_file                (mps.cpp:417-435)
//   ref_lp_random_feasible -> testutil::random_feasible_lp  (tests/oracles.hpp:61-110)
//   ref_session_*          -> setup + N loop iterations through the public
//                             per-op API (restart.hpp:47-70), timed; the
//                             current iterate in original space.
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <tuple>
#include <string>
#include <vector>

#include "oracles.hpp"
#include "rhpdhg/errors.hpp"
#include "rhpdhg/mps.hpp"
#include "rhpdhg/pdhg.hpp"
#include "rhpdhg/restart.hpp"
#include "rhpdhg/scaling.hpp"
#include "rhpdhg/solver.hpp"
#include "rhpdhg/termination.hpp"
#include "rhpdhg_c.h"

using namespace rhpdhg;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return RHPDHG_OK;
  } catch (const UsageError& e) {
    g_err = e.what();
    return RHPDHG_E_USAGE;
  } catch (const InvalidProblemError& e) {
    g_err = e.what();
    return RHPDHG_E_INVALID_PROBLEM;
  } catch (const ParseError& e) {
    g_err = e.what();
    return RHPDHG_E_PARSE;
  } catch (const NumericalBreakdownError& e) {
    g_err = e.what();
    return RHPDHG_E_BREAKDOWN;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RHPDHG_E_INTERNAL;
  }
}

LpProblem from_view(const rhpdhg_lp_view* v) {
  std::vector<Triplet> t;
  t.reserve(static_cast<std::size_t>(v->nnz));
  for (Index i = 0; i < v->num_cons; ++i)
    for (Index e = v->row_ptr[i]; e < v->row_ptr[i + 1]; ++e)
      t.push_back({i, v->col_index[e], v->values[e]});
  LpProblem p;
  p.matrix = SparseMatrix(v->num_cons, v->num_vars, std::move(t));
  const auto n = static_cast<std::size_t>(v->num_vars);
  const auto m = static_cast<std::size_t>(v->num_cons);
  p.objective.assign(v->objective, v->objective + n);
  p.objective_offset = v->objective_offset;
  p.var_lb.assign(v->var_lb, v->var_lb + n);
  p.var_ub.assign(v->var_ub, v->var_ub + n);
  p.con_lb.assign(v->con_lb, v->con_lb + m);
  p.con_ub.assign(v->con_ub, v->con_ub + m);
  p.maximization = v->maximization != 0;
  return p;
}

SolverConfig from_c(const rhpdhg_config_c* c) {
  SolverConfig s;
  s.scaling_enabled = c->scaling_enabled != 0;
  s.ruiz_iterations = c->ruiz_iterations;
  s.pock_chambolle = c->pock_chambolle != 0;
  s.restarts_enabled = c->restarts_enabled != 0;
  s.stepsize_multiplier = c->stepsize_multiplier;
  s.power_tol = c->power_tol;
  s.power_max_iters = c->power_max_iters;
  s.power_seed = c->power_seed;
  s.beta_sufficient = c->beta_sufficient;
  s.beta_necessary = c->beta_necessary;
  s.beta_artificial = c->beta_artificial;
  s.reflection_gamma = c->reflection_gamma;
  s.pid_kp = c->pid_kp;
  s.pid_ki = c->pid_ki;
  s.pid_kd = c->pid_kd;
  s.initial_weight = c->initial_weight;
  s.epsilon = c->epsilon;
  s.check_interval = c->check_interval;
  s.time_limit_seconds = c->time_limit_seconds;
  s.iteration_limit = c->iteration_limit;
  s.verbosity = c->verbosity;
  s.record_residual_history = c->record_residual_history != 0;
  return s;
}

void to_c(const KktResiduals& r, rhpdhg_kkt_c* o) {
  o->gap_abs = r.gap_abs;
  o->gap_rel = r.gap_rel;
  o->primal_inf = r.primal_inf;
  o->primal_rel = r.primal_rel;
  o->dual_eq = r.dual_eq;
  o->dual_cone = r.dual_cone;
  o->gap_denom = r.gap_denom;
  o->primal_denom = r.primal_denom;
  o->dual_denom = r.dual_denom;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_solve_csr(const rhpdhg_lp_view* lp, const rhpdhg_config_c* cfg, rhpdhg_report_c* out,
                  double* x, double* y, double* rc, double* hist, int64_t hist_cap) {
  return guarded([&] {
    const LpProblem p = from_view(lp);
    const SolutionReport r = solve(p, from_c(cfg));
    std::memset(out, 0, sizeof(*out));
    out->status = static_cast<int32_t>(r.status);
    out->objective = r.objective;
    to_c(r.residuals, &out->residuals);
    out->iterations = r.iterations;
    out->restart_count = r.restart_count;
    out->wall_time_seconds = r.wall_time_seconds;
    out->final_fixed_point_residual = r.final_fixed_point_residual;
    out->final_primal_weight = r.final_primal_weight;
    out->matrix_norm_estimate = r.matrix_norm_estimate;
    out->power_iterations = r.power_iterations;
    out->spmv_loop = r.spmv_loop;
    out->spmv_checks = r.spmv_checks;
    out->spmv_setup = r.spmv_setup;
    out->kkt_checks = r.kkt_checks;
    out->has_inner_residuals = r.inner_residuals.has_value() ? 1 : 0;
    if (r.inner_residuals) to_c(*r.inner_residuals, &out->inner_residuals);
    out->history_len = static_cast<int64_t>(r.fixed_point_residual_history.size());
    if (x) std::memcpy(x, r.x.data(), r.x.size() * sizeof(double));
    if (y) std::memcpy(y, r.y.data(), r.y.size() * sizeof(double));
    if (rc) std::memcpy(rc, r.reduced_costs.data(), r.reduced_costs.size() * sizeof(double));
    if (hist) {
      const auto k = std::min<std::size_t>(r.fixed_point_residual_history.size(),
                                           static_cast<std::size_t>(hist_cap));
      std::memcpy(hist, r.fixed_point_residual_history.data(), k * sizeof(double));
    }
  });
}

int ref_kkt_residuals(const rhpdhg_lp_view* lp, const double* x, const double* y,
                      rhpdhg_kkt_c* out) {
  return guarded([&] {
    const LpProblem p = from_view(lp);
    const auto r = kkt_residuals(
        p, std::span<const double>(x, static_cast<std::size_t>(lp->num_vars)),
        std::span<const double>(y, static_cast<std::size_t>(lp->num_cons)));
    to_c(r, out);
  });
}

int ref_spmv(const rhpdhg_lp_view* lp, const double* x, double* out, int transpose) {
  return guarded([&] {
    const LpProblem p = from_view(lp);
    const auto m = static_cast<std::size_t>(lp->num_cons);
    const auto n = static_cast<std::size_t>(lp->num_vars);
    if (transpose)
      p.matrix.multiply_transpose(std::span<const double>(x, m), std::span<double>(out, n));
    else
      p.matrix.multiply(std::span<const double>(x, n), std::span<double>(out, m));
  });
}

// Scaled instance exactly as solve() builds it (solver.cpp:72-78): CSR and
// CSC values of the scaled matrix, cumulative scales, scaled c and bounds.
int ref_scale(const rhpdhg_lp_view* lp, int ruiz_iters, int pock_chambolle, double* csr_vals,
              double* csc_vals, double* row_scale, double* col_scale, double* c_s,
              double* var_lb_s, double* var_ub_s, double* con_lb_s, double* con_ub_s) {
  return guarded([&] {
    const LpProblem p = from_view(lp);
    auto [scaled, info] = ruiz_equilibrate(p, ruiz_iters);
    if (pock_chambolle) scaled = pock_chambolle_scale(scaled, info);
    const auto cv = scaled.matrix.csr_values();
    const auto tv = scaled.matrix.csc_values();
    std::memcpy(csr_vals, cv.data(), cv.size() * sizeof(double));
    std::memcpy(csc_vals, tv.data(), tv.size() * sizeof(double));
    std::memcpy(row_scale, info.row_scale.data(), info.row_scale.size() * sizeof(double));
    std::memcpy(col_scale, info.col_scale.data(), info.col_scale.size() * sizeof(double));
    std::memcpy(c_s, scaled.objective.data(), scaled.objective.size() * sizeof(double));
    std::memcpy(var_lb_s, scaled.var_lb.data(), scaled.var_lb.size() * sizeof(double));
    std::memcpy(var_ub_s, scaled.var_ub.data(), scaled.var_ub.size() * sizeof(double));
    std::memcpy(con_lb_s, scaled.con_lb.data(), scaled.con_lb.size() * sizeof(double));
    std::memcpy(con_ub_s, scaled.con_ub.data(), scaled.con_ub.size() * sizeof(double));
  });
}

int ref_power_iteration(const rhpdhg_lp_view* lp, double tol, int64_t max_iters, uint64_t seed,
                        double* value, int64_t* iterations, int32_t* converged) {
  return guarded([&] {
    const LpProblem p = from_view(lp);
    const auto r = power_iteration_norm(p.matrix, tol, max_iters, seed);
    *value = r.value;
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
  });
}

// ---- LP handles (instances produced by the reference's own loaders) -------
void* ref_lp_from_mps(const char* path) {
  LpProblem* out = nullptr;
  const int rc = guarded([&] { out = new LpProblem(parse_mps_file(path)); });
  return rc == RHPDHG_OK ? out : nullptr;
}

void* ref_lp_random_feasible(uint64_t seed, int64_t m, int64_t n, double density) {
  LpProblem* out = nullptr;
  guarded([&] {
    testutil::Rng rng(seed);
    out = new LpProblem(testutil::random_feasible_lp(rng, m, n, density));
  });
  return out;
}

void ref_lp_dims(const void* h, int64_t* m, int64_t* n, int64_t* nnz) {
  const auto* p = static_cast<const LpProblem*>(h);
  *m = p->num_cons();
  *n = p->num_vars();
  *nnz = p->matrix.nnz();
}

void ref_lp_export(const void* h, int64_t* row_ptr, int64_t* col_index, double* values,
                   double* objective, double* offset, double* var_lb, double* var_ub,
                   double* con_lb, double* con_ub, int32_t* maximization) {
  const auto* p = static_cast<const LpProblem*>(h);
  const auto rp = p->matrix.row_ptr();
  const auto ci = p->matrix.col_index();
  const auto v = p->matrix.csr_values();
  std::memcpy(row_ptr, rp.data(), rp.size() * sizeof(int64_t));
  std::memcpy(col_index, ci.data(), ci.size() * sizeof(int64_t));
  std::memcpy(values, v.data(), v.size() * sizeof(double));
  std::memcpy(objective, p->objective.data(), p->objective.size() * sizeof(double));
  *offset = p->objective_offset;
  std::memcpy(var_lb, p->var_lb.data(), p->var_lb.size() * sizeof(double));
  std::memcpy(var_ub, p->var_ub.data(), p->var_ub.size() * sizeof(double));
  std::memcpy(con_lb, p->con_lb.data(), p->con_lb.size() * sizeof(double));
  std::memcpy(con_ub, p->con_ub.data(), p->con_ub.size() * sizeof(double));
  *maximization = p->maximization ? 1 : 0;
}

void ref_lp_free(void* h) { delete static_cast<LpProblem*>(h); }

// ---- bounded CPU samples for bench.py (cpu_baseline leg, --impl reference) --
// A resumable run of the reference solve: setup (scaling + power iteration,
// solver.cpp:72-88) in ref_session_create, then the loop body
// (solver.cpp:147-196: halpern_reflected_step, fixed_point_residual,
// check_restart, KKT check every check_interval and at restarts, do_restart)
// advanced `iters` iterations at a time through the reference's public API.
struct RefSession {
  LpProblem p;
  SolverConfig cfg;
  LpProblem scaled;
  ScalingInfo info;
  StepConfig step;
  Iterate z;
  RestartState rs;
  PidState pid;
  ToleranceConfig tol;
  double setup_seconds = 0.0;
  double last_r = 0.0;
  bool optimal = false;
  KktResiduals last;
};

void* ref_session_create(const rhpdhg_lp_view* lp, const rhpdhg_config_c* cfg_c) {
  RefSession* s = nullptr;
  guarded([&] {
    using Clock = std::chrono::steady_clock;
    auto h = std::make_unique<RefSession>();
    h->p = from_view(lp);
    h->cfg = from_c(cfg_c);
    const auto t0 = Clock::now();
    std::tie(h->scaled, h->info) = ruiz_equilibrate(h->p, h->cfg.ruiz_iterations);
    if (h->cfg.pock_chambolle) h->scaled = pock_chambolle_scale(h->scaled, h->info);
    const auto pi = power_iteration_norm(h->scaled.matrix, h->cfg.power_tol,
                                         h->cfg.power_max_iters, h->cfg.power_seed);
    h->step.matrix_norm_estimate = pi.value;
    h->step.step_size = default_stepsize(pi.value, h->cfg.stepsize_multiplier);
    h->step.primal_weight = h->cfg.initial_weight;
    h->step.reflection = h->cfg.reflection_gamma;
    h->z = Iterate::zeros(h->scaled);
    h->rs.anchor = h->z;
    h->rs.beta_sufficient = h->cfg.beta_sufficient;
    h->rs.beta_necessary = h->cfg.beta_necessary;
    h->rs.beta_artificial = h->cfg.beta_artificial;
    h->pid.kp = h->cfg.pid_kp;
    h->pid.ki = h->cfg.pid_ki;
    h->pid.kd = h->cfg.pid_kd;
    h->pid.omega = h->cfg.initial_weight;
    h->pid.snapshot_x = h->z.x;
    h->pid.snapshot_y = h->z.y;
    h->tol.epsilon = h->cfg.epsilon;
    h->setup_seconds = std::chrono::duration<double>(Clock::now() - t0).count();
    s = h.release();
  });
  return s;
}

int ref_session_advance(void* hv, int64_t iters, int32_t* running, double* seconds,
                        int64_t* total) {
  return guarded([&] {
    using Clock = std::chrono::steady_clock;
    RefSession& h = *static_cast<RefSession*>(hv);
    const auto t0 = Clock::now();
    for (int64_t it = 0; it < iters && !h.optimal; ++it) {
      auto [zn, inner] = halpern_reflected_step(h.z, h.rs.anchor, h.rs.k, h.step, h.scaled);
      h.last_r = fixed_point_residual(h.z, inner, h.step);
      RestartCondition verdict = RestartCondition::none;
      if (h.rs.k == 0) {
        h.rs.r_anchor = h.last_r;
        h.rs.r_prev = h.last_r;
      } else {
        verdict = check_restart(h.rs, h.last_r);
      }
      if (!h.cfg.restarts_enabled) verdict = RestartCondition::none;
      h.z = std::move(zn);
      h.rs.k += 1;
      h.rs.total += 1;
      if (h.rs.total % h.cfg.check_interval == 0 || verdict != RestartCondition::none) {
        Iterate o = unscale_iterate(h.z, h.info);
        o.ax = h.p.matrix.multiply(o.x);
        o.aty = h.p.matrix.multiply_transpose(o.y);
        for (std::size_t i = 0; i < h.z.ax.size(); ++i) h.z.ax[i] = h.info.row_scale[i] * o.ax[i];
        for (std::size_t j = 0; j < h.z.aty.size(); ++j)
          h.z.aty[j] = h.info.col_scale[j] * o.aty[j];
        h.last = kkt_residuals(h.p, o.x, o.y, o.ax, o.aty);
        if (is_optimal(h.last, h.tol)) h.optimal = true;
      }
      if (!h.optimal && verdict != RestartCondition::none)
        do_restart(h.rs, h.z, h.pid, h.step);
    }
    if (seconds) *seconds = std::chrono::duration<double>(Clock::now() - t0).count();
    if (running) *running = h.optimal ? 0 : 1;
    if (total) *total = h.rs.total;
  });
}

double ref_session_setup_seconds(void* hv) { return static_cast<RefSession*>(hv)->setup_seconds; }

// The current Halpern iterate in original space (unscale_iterate,
// scaling.cpp:83-94): what solve() reports for x, y after `total` iterations.
int ref_session_iterate(void* hv, double* x, double* y) {
  return guarded([&] {
    RefSession& h = *static_cast<RefSession*>(hv);
    const Iterate o = unscale_iterate(h.z, h.info);
    std::copy(o.x.begin(), o.x.end(), x);
    std::copy(o.y.begin(), o.y.end(), y);
  });
}

void ref_session_free(void* hv) { delete static_cast<RefSession*>(hv); }

}  // extern "C"
