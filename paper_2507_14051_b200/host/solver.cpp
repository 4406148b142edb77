// solver.cpp — solve(): the host orchestration of the restarted reflected
// Halpern PDHG (reference src/solver.cpp:63-238) over the device library.
//
// Host responsibilities: validation, exception mapping, the power-iteration
// stopping rule, the termination test, the PID weight update and the report.
// Everything O(nnz) or O(m+n) runs on the GPU: scaling, the products, the
// fused iteration kernels, the restart verdict and the KKT sums. The device
// runs the loop in blocks (one CUDA graph launch each) that end exactly where
// the reference loop does host-visible work: a scheduled KKT check
// (total % check_interval == 0), a restart verdict, the iteration limit or
// the block length. The time limit is therefore tested between blocks (the
// reference tests it every iteration; a zero limit still stops before the
// first iteration).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "device.hpp"
#include "kkt.hpp"
#include "rhpdhg/errors.hpp"
#include "rhpdhg/pdhg.hpp"
#include "rhpdhg/restart.hpp"
#include "rhpdhg/scaling.hpp"
#include "rhpdhg/solver.hpp"
#include "session.hpp"

namespace rhpdhg {

namespace {
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

// power_iteration_norm (pdhg.cpp:117-170): start vector and stopping rule on
// the host (bit-identical to the reference), products and dots on the device.
PowerIterationResult device_power_iteration(rhp_ctx* c, Index n, Index nnz, double tol,
                                            long max_iters, std::uint64_t seed) {
  PowerIterationResult res;
  if (nnz == 0) {
    res.converged = true;
    return res;
  }
  std::vector<double> v(static_cast<size_t>(n));
  std::mt19937_64 eng(seed);
  for (double& e : v) e = 2.0 * (static_cast<double>(eng() >> 11) * 0x1.0p-53) - 1.0;
  double nv2 = 0.0;
  for (double e : v) nv2 += e * e;
  const double nv = std::sqrt(nv2);
  for (double& e : v) e /= nv;
  detail::ok(rhp_power_begin(c, v.data()), "rhp_power_begin");
  double sigma_prev = 0.0, change_prev = std::numeric_limits<double>::infinity();
  for (long it = 1; it <= max_iters; ++it) {
    double vw = 0.0, ww = 0.0;
    detail::ok(rhp_power_step(c, &vw, &ww), "rhp_power_step");
    const double sigma = vw > 0.0 ? std::sqrt(vw) : 0.0;
    res.iterations = it;
    res.value = sigma;
    const double wn = std::sqrt(ww);
    if (wn == 0.0) {
      res.converged = true;
      return res;
    }
    detail::ok(rhp_power_normalize(c, wn), "rhp_power_normalize");
    const double change = std::abs(sigma - sigma_prev);
    if (it >= 3 && change <= tol * std::max(sigma, 1e-300)) {
      const double ratio = std::min(change / std::max(change_prev, 1e-300), 0.999);
      const double tail = change * ratio / (1.0 - ratio);
      if (tail <= tol * std::max(sigma, 1e-300)) {
        res.converged = true;
        return res;
      }
    }
    sigma_prev = sigma;
    change_prev = change;
  }
  return res;
}

rhp_step device_step(const StepConfig& s, const SolverConfig& cfg) {
  rhp_step d{};
  d.eta = s.step_size;
  d.omega = s.primal_weight;
  d.gamma = s.reflection;
  d.tau = s.primal_step();                       // pdhg.hpp:18
  d.sigma = s.dual_step();                       // pdhg.hpp:19
  d.sigma_inv = 1.0 / d.sigma;                   // pdhg.cpp:50
  d.primal_scale = s.primal_weight / s.step_size;          // pdhg.cpp:70
  d.dual_scale = 1.0 / (s.step_size * s.primal_weight);    // pdhg.cpp:71
  d.beta_sufficient = cfg.beta_sufficient;
  d.beta_necessary = cfg.beta_necessary;
  d.beta_artificial = cfg.beta_artificial;
  d.check_interval = cfg.check_interval;
  d.iteration_limit = cfg.iteration_limit;
  d.restarts_enabled = cfg.restarts_enabled ? 1 : 0;
  d.record_history = cfg.record_residual_history ? 1 : 0;
  return d;
}

void log_progress(const SolverConfig& cfg, long iter, double fpr, const KktResiduals& r,
                  double omega, long restarts) {
  if (cfg.verbosity < 1) return;
  std::fprintf(stderr,
               "iter %8ld  fpr %9.3e  gap %9.3e  primal %9.3e  dual %9.3e  omega %9.3e  "
               "restarts %ld\n",
               iter, fpr, r.gap_rel, r.primal_rel, r.dual_eq / r.dual_denom, omega, restarts);
}

}  // namespace

DeviceOptions& default_device_options() {
  thread_local DeviceOptions opts;
  return opts;
}

SolutionReport solve(const LpProblem& problem, const SolverConfig& cfg) {
  return solve(problem, cfg, default_device_options());
}

// ---------------------------------------------------------------- Session --
// solve() as a resumable state machine so callers (bench, FFI) can advance
// the loop in slices; solve() runs it to completion.
Session::Session(const LpProblem& problem, const SolverConfig& cfg, const DeviceOptions& dopt)
    : Session((cfg.validate(), problem.validate(), detail::view_of(problem)), problem.name, true, cfg,
              dopt) {}

Session::Session(const rhpdhg_lp_view& view, const SolverConfig& cfg, const DeviceOptions& dopt)
    : Session(view, std::string(), false, cfg, dopt) {}

Session::Session(const rhpdhg_lp_view& view, const std::string& name, bool validated,
                 const SolverConfig& cfg, const DeviceOptions& dopt)
    : view_(view), name_(name), cfg_(cfg) {
  cfg.validate();
  detail::NvtxRange setup_range("rhpdhg:setup");
  t0_ = Clock::now();
  // RHPDHG_SETUP_TRACE=1: per-phase setup times on stderr
  const bool trace = std::getenv("RHPDHG_SETUP_TRACE") != nullptr;
  Clock::time_point tp = t0_;
  auto phase = [&](const char* what) {
    if (!trace) return;
    const Clock::time_point now = Clock::now();
    std::fprintf(stderr, "setup %-24s %9.3f s\n", what, std::chrono::duration<double>(now - tp).count());
    tp = now;
  };
  const Index n = view.num_vars;
  if (view.num_cons < 0 || view.num_vars < 0) throw UsageError("matrix dimensions must be nonnegative");
  // the matrix is validated by the device ingest (from_csr's exceptions),
  // then the vectors (LpProblem::validate, lp_problem.cpp:30-46)
  {
    detail::NvtxRange r("rhpdhg:ingest");
    dev_ = std::make_unique<detail::Device>(view, detail::options(dopt));
  }
  rhp_ctx* c = dev_->get();
  if (!validated) detail::validate_vectors(view);
  // nonzeros after the ingest dropped explicit zeros (SparseMatrix::nnz())
  Index nnz = view.nnz;
  if (!validated) {
    rhp_layout_info li{};
    detail::ok(rhp_layout(c, &li), "rhp_layout");
    nnz = li.nnz_local;
    if (dopt.world_size > 1) {  // local count on this rank: count the global one on the host
      nnz = 0;
      if (view.num_cons > 0)
        for (Index e = view.row_ptr[0]; e < view.row_ptr[view.num_cons]; ++e) nnz += view.values[e] != 0.0;
    }
  }
  phase("device create+ingest");
  // (1) diagonal preconditioning on the device (solver.cpp:72-78)
  {
    detail::NvtxRange r("rhpdhg:scaling");
    detail::ok(rhp_scale(c, cfg.scaling_enabled ? 1 : 0, cfg.ruiz_iterations, cfg.pock_chambolle ? 1 : 0),
               "rhp_scale");
  }
  phase("scaling");
  // (2) step size from the scaled norm (solver.cpp:81-88)
  PowerIterationResult pi;
  {
    detail::NvtxRange r("rhpdhg:power_iteration");
    pi = device_power_iteration(c, n, nnz, cfg.power_tol, cfg.power_max_iters, cfg.power_seed);
  }
  phase("power iteration");
  step_.matrix_norm_estimate = pi.value;
  step_.step_size = default_stepsize(pi.value, cfg.stepsize_multiplier);
  step_.primal_weight = cfg.initial_weight;
  step_.reflection = cfg.reflection_gamma;
  step_.validate();
  report_.config = cfg;
  report_.matrix_norm_estimate = pi.value;
  report_.power_iterations = pi.iterations;
  report_.spmv_setup = 2u * static_cast<std::uint64_t>(pi.iterations);
  spmv_counter::add(report_.spmv_setup);
  if (cfg.verbosity >= 1)
    std::fprintf(stderr, "%s: %ld rows, %ld cols, %ld nonzeros, ||A|| ~ %.6e, eta %.6e\n",
                 name_.empty() ? "instance" : name_.c_str(), static_cast<long>(view.num_cons),
                 static_cast<long>(n), static_cast<long>(nnz), pi.value, step_.step_size);
  // (3) zero start, anchor = snapshot = start (solver.cpp:91-103)
  const rhp_step dstep = device_step(step_, cfg);
  detail::ok(rhp_set_step(c, &dstep), "rhp_set_step");
  detail::ok(rhp_reset_iterate(c), "rhp_reset_iterate");
  pid_.kp = cfg.pid_kp;
  pid_.ki = cfg.pid_ki;
  pid_.kd = cfg.pid_kd;
  pid_.omega = cfg.initial_weight;
  denoms_ = detail::problem_denoms(view);
  tol_.epsilon = cfg.epsilon;
  report_.setup_seconds = since(t0_);
  phase("step/iterate/denoms");
  t_loop_ = Clock::now();
  // initial check: the zero start may already be optimal (solver.cpp:136-145)
  last_ = kkt_check(0);
  if (is_optimal(last_, tol_)) {
    status_ = SolveStatus::optimal;
    decided_ = true;
  }
}

Session::~Session() = default;

KktResiduals Session::kkt_check(int which) {
  detail::NvtxRange r("rhpdhg:kkt_check");
  rhp_kkt_sums s{};
  detail::ok(rhp_kkt(dev_->get(), which, &s), "rhp_kkt");
  spmv_counter::add(2);
  if (which == 0) {
    spmv_checks_ += 2;
    ++report_.kkt_checks;
  }
  return detail::residuals_from_sums(s, denoms_);
}

// One pass of the reference loop body at block granularity
// (solver.cpp:147-196). Returns false once the solve is decided.
bool Session::step() {
  if (decided_) return false;
  rhp_ctx* c = dev_->get();
  if (total_ >= cfg_.iteration_limit) {
    status_ = SolveStatus::iteration_limit;
    decided_ = true;
    return false;
  }
  int out_of_time = since(t0_) >= cfg_.time_limit_seconds ? 1 : 0;
  detail::ok(rhp_any(c, out_of_time, &out_of_time), "rhp_any");  // same verdict on every rank
  if (out_of_time) {
    status_ = SolveStatus::time_limit;
    decided_ = true;
    return false;
  }
  rhp_block_out out{};
  {
    detail::NvtxRange r("rhpdhg:block");
    detail::ok(rhp_run_block(c, &out), "rhp_run_block");
  }
  ++report_.device_blocks;
  if (out.breakdown)
    throw NumericalBreakdownError("canonical norm radicand " + std::to_string(out.q_last) +
                                  " is negative beyond roundoff; the P matrix is indefinite");
  spmv_counter::add(2u * static_cast<std::uint64_t>(out.iterations_done));
  if (cfg_.record_residual_history && out.iterations_done > 0) {
    std::vector<double> h(static_cast<size_t>(out.iterations_done));
    int64_t got = 0;
    detail::ok(rhp_get_history(c, h.data(), out.iterations_done, &got), "rhp_get_history");
    report_.fixed_point_residual_history.insert(report_.fixed_point_residual_history.end(),
                                                h.begin(), h.begin() + got);
  }
  total_ = out.total;
  if (out.iterations_done > 0) {
    last_fpr_ = out.r_last;
    have_inner_ = true;
  }
  if (out.check_due) {
    last_ = kkt_check(0);
    log_progress(cfg_, total_, out.r_last, last_, step_.primal_weight, restarts_);
    if (is_optimal(last_, tol_)) {
      status_ = SolveStatus::optimal;
      decided_ = true;
      return false;
    }
  }
  if (out.verdict != 0) {  // do_restart (restart.cpp:71-83)
    detail::NvtxRange r("rhpdhg:restart");
    step_.primal_weight = pid_update(pid_, std::sqrt(out.x_dist2), std::sqrt(out.y_dist2),
                                     std::sqrt(out.x_norm2), std::sqrt(out.y_norm2));
    const rhp_step dstep = device_step(step_, cfg_);
    detail::ok(rhp_set_step(c, &dstep), "rhp_set_step");
    detail::ok(rhp_restart(c), "rhp_restart");
    ++restarts_;
  }
  return true;
}

bool Session::advance(long iterations) {
  const long target = total_ + iterations;
  while (!decided_ && total_ < target) step();
  return !decided_;
}

SolutionReport Session::finish() {
  while (step()) {
  }
  rhp_ctx* c = dev_->get();
  detail::NvtxRange fin("rhpdhg:finish");
  if (status_ != SolveStatus::optimal) last_ = kkt_check(0);
  report_.loop_seconds = since(t_loop_);
  const Index m = view_.num_cons, n = view_.num_vars;
  report_.status = status_;
  report_.x.resize(static_cast<size_t>(n));
  report_.y.resize(static_cast<size_t>(m));
  report_.reduced_costs.resize(static_cast<size_t>(n));
  detail::ok(rhp_fetch_solution(c, report_.x.data(), report_.y.data(), report_.reduced_costs.data()),
             "rhp_fetch_solution");
  double acc = view_.objective_offset;  // solver.cpp:211-218
  for (size_t j = 0; j < report_.x.size(); ++j) acc += view_.objective[j] * report_.x[j];
  report_.objective = view_.maximization ? -acc : acc;
  report_.residuals = last_;
  report_.iterations = total_;
  report_.restart_count = restarts_;
  report_.final_fixed_point_residual = last_fpr_;
  report_.final_primal_weight = step_.primal_weight;
  report_.spmv_loop = 2u * static_cast<std::uint64_t>(total_);
  report_.spmv_checks = spmv_checks_;
  if (have_inner_) report_.inner_residuals = kkt_check(1);  // solver.cpp:228-234
  report_.wall_time_seconds = since(t0_);
  return report_;
}

rhp_ctx* Session::device() const { return dev_->get(); }

SolutionReport solve(const LpProblem& problem, const SolverConfig& cfg, const DeviceOptions& dopt) {
  Session s(problem, cfg, dopt);
  return s.finish();
}

// ------------------------------------------------------- per-op setup API --
void StepConfig::validate() const {
  if (!(step_size > 0.0) || !std::isfinite(step_size))
    throw UsageError("step size must be positive and finite");
  if (!(primal_weight > 0.0) || !std::isfinite(primal_weight))
    throw UsageError("primal weight must be positive and finite");
  if (!(reflection >= 0.0 && reflection <= 1.0))
    throw UsageError("reflection coefficient must lie in [0, 1]");
  if (matrix_norm_estimate > 0.0 && step_size * matrix_norm_estimate > 0.99 * (1.0 + 1e-9))
    throw UsageError("step size violates the PSD margin step_size * ||A|| <= 0.99");
}

double default_stepsize(double norm_estimate, double multiplier) {
  if (norm_estimate < 0.0 || std::isnan(norm_estimate))
    throw UsageError("matrix norm estimate must be nonnegative");
  if (!(multiplier > 0.0 && multiplier <= 0.99))
    throw UsageError("stepsize multiplier must lie in (0, 0.99]");
  return norm_estimate == 0.0 ? 1.0 : multiplier / norm_estimate;
}

PowerIterationResult power_iteration_norm(const SparseMatrix& matrix, double tol, long max_iters,
                                          std::uint64_t seed) {
  PowerIterationResult r;
  if (matrix.nnz() == 0) {
    r.converged = true;
  } else {  // on the matrix's cached product context
    std::unique_lock<std::mutex> lock;
    rhp_ctx* ctx = detail::product_context(matrix, lock);
    r = device_power_iteration(ctx, matrix.cols(), matrix.nnz(), tol, max_iters, seed);
  }
  spmv_counter::add(2u * static_cast<std::uint64_t>(r.iterations));
  return r;
}

double initial_weight() { return 1.0; }

RestartCondition check_restart(RestartState& st, double r) {
  RestartCondition v = RestartCondition::none;
  if (st.k >= 1 && std::isfinite(st.r_anchor)) {
    if (r <= st.beta_sufficient * st.r_anchor) v = RestartCondition::sufficient;
    else if (r <= st.beta_necessary * st.r_anchor && r > st.r_prev)
      v = RestartCondition::necessary_no_progress;
    else if (static_cast<double>(st.k) >= st.beta_artificial * static_cast<double>(st.total))
      v = RestartCondition::artificial;
  }
  st.r_prev = r;
  return v;
}

// restart.cpp:85-120 on the four device-reduced norms.
double pid_update(PidState& pid, double dx, double dy, double x_norm, double y_norm) {
  double error = 0.0;
  if (dx > 1e-10 * (1.0 + x_norm) && dy > 1e-10 * (1.0 + y_norm))
    error = std::log(pid.omega) + std::log(dx) - std::log(dy);
  pid.integral += error;
  double delta = -(pid.kp * error + pid.ki * pid.integral + pid.kd * (error - pid.prev_error));
  pid.prev_error = error;
  const double cap = std::log(10.0);
  bool clamped = false;
  if (delta > cap) {
    delta = cap;
    clamped = true;
  } else if (delta < -cap) {
    delta = -cap;
    clamped = true;
  }
  double omega = delta == 0.0 ? pid.omega : std::exp(std::log(pid.omega) + delta);
  if (omega < 1e-8) {
    omega = 1e-8;
    clamped = true;
  } else if (omega > 1e8) {
    omega = 1e8;
    clamped = true;
  }
  if (clamped) pid.integral = 0.0;
  pid.omega = omega;
  return omega;
}

ScalingInfo ScalingInfo::identity(const LpProblem& p) {
  ScalingInfo s;
  s.row_scale.assign(static_cast<size_t>(p.num_cons()), 1.0);
  s.col_scale.assign(static_cast<size_t>(p.num_vars()), 1.0);
  s.active = false;
  return s;
}

std::pair<LpProblem, ScalingInfo> scale_problem(const LpProblem& problem, bool enabled,
                                                int ruiz_iterations, bool pock_chambolle) {
  if (!enabled) return {problem, ScalingInfo::identity(problem)};  // solver.cpp:72-78
  auto [scaled, info] = ruiz_equilibrate(problem, ruiz_iterations);
  if (pock_chambolle) scaled = pock_chambolle_scale(scaled, info);
  return {std::move(scaled), std::move(info)};
}

}  // namespace rhpdhg
