// ops.cpp — the reference's per-operation API (pdhg.hpp:30-58,
// restart.hpp:47-70, scaling.hpp:23-32) over the device library. solve()
// never calls these (it runs the fused block kernels); they serve callers
// that drive single operations, such as the reference's own unit tests.
// Every O(n + m + nnz) piece is a device round trip: the products on the
// matrix's cached product context, the elementwise updates with the
// reference's evaluation order (bit-identical per element), and the sums of
// the canonical norm and the PID movement. Scalar control (clamp rules, PID
// arithmetic) stays on the host as in the reference.
#include <cmath>
#include <string>

#include "device.hpp"
#include "rhpdhg/errors.hpp"
#include "rhpdhg/pdhg.hpp"
#include "rhpdhg/restart.hpp"
#include "rhpdhg/scaling.hpp"
#include "rhpdhg/solver.hpp"

namespace rhpdhg {

namespace {

int device_ordinal() { return default_device_options().device; }

void check_iterate(const Iterate& z, const LpProblem& p, const char* what) {
  const size_t n = static_cast<size_t>(p.num_vars()), m = static_cast<size_t>(p.num_cons());
  if (z.x.size() != n || z.aty.size() != n || z.y.size() != m || z.ax.size() != m)
    throw UsageError(std::string(what) + ": iterate sizes do not match the problem");
  if (p.objective.size() != n || p.var_lb.size() != n || p.var_ub.size() != n ||
      p.con_lb.size() != m || p.con_ub.size() != m)
    throw UsageError(std::string(what) + ": problem vector sizes do not match the matrix");
}

rhp_op_lp lp_vectors(const LpProblem& p) {
  return rhp_op_lp{p.objective.data(), p.var_lb.data(), p.var_ub.data(), p.con_lb.data(),
                   p.con_ub.data()};
}

rhp_op_iter iter_view(const Iterate& z) { return rhp_op_iter{z.x.data(), z.y.data(), z.ax.data(), z.aty.data()}; }

void size_output(PdhgStepOutput& o, size_t n, size_t m) {
  o.x_next.resize(n);
  o.aty_next.resize(n);
  o.dx.resize(n);
  o.y_next.resize(m);
  o.ax_next.resize(m);
  o.dy.resize(m);
}

// One device round trip of pdhg_step, and with an anchor of the Halpern
// combination (rhp_op_pdhg).
void device_step(const Iterate& z, const Iterate* anchor, long k, const StepConfig& cfg,
                 const LpProblem& problem, PdhgStepOutput& out, Iterate* next) {
  check_iterate(z, problem, "pdhg_step");
  if (anchor) check_iterate(*anchor, problem, "halpern_reflected_step");
  const size_t n = static_cast<size_t>(problem.num_vars()), m = static_cast<size_t>(problem.num_cons());
  size_output(out, n, m);
  rhp_op_params prm{};
  prm.tau = cfg.primal_step();         // pdhg.cpp:35
  prm.sigma = cfg.dual_step();         // pdhg.cpp:36
  prm.sigma_inv = 1.0 / prm.sigma;     // pdhg.cpp:50
  prm.gamma = cfg.reflection;
  prm.a = static_cast<double>(k + 1) / static_cast<double>(k + 2);  // restart.cpp:38
  prm.b = 1.0 / static_cast<double>(k + 2);                         // restart.cpp:39
  const rhp_op_lp lp = lp_vectors(problem);
  const rhp_op_iter zi = iter_view(z);
  rhp_op_iter ai{};
  if (anchor) ai = iter_view(*anchor);
  rhp_op_out inner{out.x_next.data(), out.y_next.data(), out.ax_next.data(), out.aty_next.data()};
  rhp_op_out zo{};
  if (next) {
    next->x.resize(n);
    next->y.resize(m);
    next->ax.resize(m);
    next->aty.resize(n);
    next->ax_valid = next->aty_valid = true;
    zo = rhp_op_out{next->x.data(), next->y.data(), next->ax.data(), next->aty.data()};
  }
  spmv_counter::add(2);  // A x+ and A^T y+ (pdhg.cpp:47, :57)
  std::unique_lock<std::mutex> lock;
  rhp_ctx* ctx = detail::product_context(problem.matrix, lock);
  detail::ok(rhp_op_pdhg(ctx, &prm, &lp, &zi, anchor ? &ai : nullptr, &inner, out.dx.data(),
                         out.dy.data(), next ? &zo : nullptr),
             "rhp_op_pdhg");
}

struct Sums {
  double p2 = 0.0;     // sum (p - pm)^2
  double q2 = 0.0;     // sum q^2
  double cross = 0.0;  // sum q (r - rs)
  double pn2 = 0.0;    // sum p^2
};

Sums device_sums(std::span<const double> p, const double* pm, std::span<const double> q,
                 const double* r, const double* rs) {
  double o[4] = {0.0, 0.0, 0.0, 0.0};
  detail::ok(rhp_op_sums(device_ordinal(), static_cast<int64_t>(p.size()), p.data(), pm,
                         static_cast<int64_t>(q.size()), q.data(), r, rs, o),
             "rhp_op_sums");
  return Sums{o[0], o[1], o[2], o[3]};
}

// quadratic_form (pdhg.cpp:68-75) from device sums: returns q, sets diag.
double quadratic_form(const Sums& s, const StepConfig& cfg, double* diag_out) {
  const double primal_scale = cfg.primal_weight / cfg.step_size;
  const double dual_scale = 1.0 / (cfg.step_size * cfg.primal_weight);
  const double diag = primal_scale * s.p2 + dual_scale * s.q2;
  if (diag_out) *diag_out = diag;
  return diag + 2.0 * s.cross;
}

[[noreturn]] void throw_indefinite(double q) {
  throw NumericalBreakdownError("canonical norm radicand " + std::to_string(q) +
                                " is negative beyond roundoff; the P matrix is indefinite");
}

}  // namespace

// ------------------------------------------------------------ pdhg.hpp --
PdhgStepOutput pdhg_step(const Iterate& z, const LpProblem& problem, const StepConfig& cfg) {
  PdhgStepOutput out;
  device_step(z, nullptr, 0, cfg, problem, out, nullptr);
  return out;
}

double p_norm(std::span<const double> x, std::span<const double> y, std::span<const double> ax,
              const StepConfig& cfg) {
  if (ax.size() != y.size()) throw UsageError("p_norm: ax and y sizes differ");
  double diag = 0.0;
  const double q = quadratic_form(device_sums(x, nullptr, y, ax.data(), nullptr), cfg, &diag);
  if (q < 0.0) {  // pdhg.cpp:87-93
    if (q >= -1e-12 * std::max(diag, 1e-300)) return 0.0;
    throw_indefinite(q);
  }
  return std::sqrt(q);
}

double p_norm(std::span<const double> x, std::span<const double> y, const StepConfig& cfg,
              const LpProblem& problem) {
  std::vector<double> ax(y.size());
  problem.matrix.multiply(x, ax);
  return p_norm(x, y, ax, cfg);
}

double fixed_point_residual(const Iterate& z, const PdhgStepOutput& out, const StepConfig& cfg) {
  if (out.dx.size() != z.x.size() || out.dy.size() != z.y.size() || out.ax_next.size() != z.ax.size())
    throw UsageError("fixed_point_residual: step output does not match the iterate");
  // dy . (ax - ax+) with A dx from the caches (pdhg.cpp:101-104)
  double diag = 0.0;
  const double q = quadratic_form(device_sums(out.dx, nullptr, out.dy, z.ax.data(), out.ax_next.data()),
                                  cfg, &diag);
  if (q >= 0.0) return std::sqrt(q);
  if (q >= -1e-12 * std::max(diag, 1e-300)) return 0.0;
  // roundoff floor of the iterate itself (pdhg.cpp:108-114)
  double iterate_scale = 0.0;
  quadratic_form(device_sums(z.x, nullptr, z.y, nullptr, nullptr), cfg, &iterate_scale);
  if (q >= -1e-24 * (1.0 + iterate_scale)) return 0.0;
  throw_indefinite(q);
}

// --------------------------------------------------------- restart.hpp --
std::pair<Iterate, PdhgStepOutput> halpern_reflected_step(const Iterate& z, const Iterate& anchor,
                                                          long k, const StepConfig& cfg,
                                                          const LpProblem& problem) {
  PdhgStepOutput out;
  Iterate next;
  device_step(z, &anchor, k, cfg, problem, out, &next);
  return {std::move(next), std::move(out)};
}

void do_restart(RestartState& state, const Iterate& z_current, PidState& pid, StepConfig& cfg) {
  cfg.primal_weight = pid_update(pid, z_current);  // restart.cpp:71-83
  pid.snapshot_x = z_current.x;
  pid.snapshot_y = z_current.y;
  state.anchor = z_current;
  state.k = 0;
  state.n += 1;
  state.restart_count += 1;
  state.r_anchor = std::numeric_limits<double>::infinity();
  state.r_prev = std::numeric_limits<double>::infinity();
}

double pid_update(PidState& pid, const Iterate& z_current) {
  if (pid.snapshot_x.size() != z_current.x.size() || pid.snapshot_y.size() != z_current.y.size())
    throw UsageError("pid_update: snapshot sizes do not match the iterate");
  // ||x - x_snap||, ||x|| and ||y - y_snap||, ||y|| on the device (restart.cpp:86-91)
  const Sums sx = device_sums(z_current.x, pid.snapshot_x.data(), std::span<const double>(), nullptr, nullptr);
  const Sums sy = device_sums(z_current.y, pid.snapshot_y.data(), std::span<const double>(), nullptr, nullptr);
  return pid_update(pid, std::sqrt(sx.p2), std::sqrt(sy.p2), std::sqrt(sx.pn2), std::sqrt(sy.pn2));
}

// --------------------------------------------------------- scaling.hpp --
namespace {

// One scaling pass on a temporary context of `problem` (rhp_scale):
// `ruiz` l-inf passes then, if `pc`, one 1-norm pass; returns the scaled
// instance (CSR and CSC values each scaled from the input's own layout, as
// sparse_matrix.cpp:101-114) and the scales of this call.
std::pair<LpProblem, ScalingInfo> device_scaling(const LpProblem& problem, int ruiz, bool pc) {
  problem.validate();
  const DeviceOptions& d = default_device_options();
  detail::Device dev(detail::view_of(problem), detail::options(d.device, false, 1));
  const Index nz = problem.matrix.nnz();
  if (nz > 0)  // the A^T apply scales the input's CSC values
    detail::ok(rhp_set_csc_values(dev.get(), problem.matrix.csc_values().data(), 1),
               "rhp_set_csc_values");
  detail::ok(rhp_scale(dev.get(), 1, ruiz, pc ? 1 : 0), "rhp_scale");
  const size_t m = static_cast<size_t>(problem.num_cons()), n = static_cast<size_t>(problem.num_vars());
  std::vector<double> csr(static_cast<size_t>(nz)), csc(static_cast<size_t>(nz));
  LpProblem out;
  out.name = problem.name;
  out.maximization = problem.maximization;
  out.objective_offset = problem.objective_offset;  // never scaled (scaling.cpp:17)
  out.objective.resize(n);
  out.var_lb.resize(n);
  out.var_ub.resize(n);
  out.con_lb.resize(m);
  out.con_ub.resize(m);
  ScalingInfo info;
  info.row_scale.resize(m);
  info.col_scale.resize(n);
  info.active = true;
  rhp_scaled_out o{csr.data(), csc.data(), info.row_scale.data(), info.col_scale.data(),
                   out.objective.data(), out.var_lb.data(), out.var_ub.data(),
                   out.con_lb.data(), out.con_ub.data()};
  detail::ok(rhp_get_scaled(dev.get(), &o), "rhp_get_scaled");
  out.matrix = detail::with_values(problem.matrix, std::move(csr), std::move(csc));
  return {std::move(out), std::move(info)};
}

}  // namespace

std::pair<LpProblem, ScalingInfo> ruiz_equilibrate(const LpProblem& problem, int iterations) {
  if (iterations < 0) throw UsageError("ruiz_equilibrate: negative iteration count");
  return device_scaling(problem, iterations, false);
}

LpProblem pock_chambolle_scale(const LpProblem& problem, ScalingInfo& info) {
  if (info.row_scale.size() != static_cast<size_t>(problem.num_cons()) ||
      info.col_scale.size() != static_cast<size_t>(problem.num_vars()))
    throw UsageError("pock_chambolle_scale: scaling info does not match the problem");
  auto [out, pc] = device_scaling(problem, 0, true);
  // compose multiplicatively (scaling.cpp:77-79)
  for (size_t i = 0; i < info.row_scale.size(); ++i) info.row_scale[i] *= pc.row_scale[i];
  for (size_t j = 0; j < info.col_scale.size(); ++j) info.col_scale[j] *= pc.col_scale[j];
  info.active = true;
  return std::move(out);
}

Iterate unscale_iterate(const Iterate& scaled, const ScalingInfo& info) {
  if (info.col_scale.size() != scaled.x.size() || info.row_scale.size() != scaled.y.size())
    throw UsageError("unscale_iterate: scaling info does not match the iterate");
  Iterate out;
  out.x.resize(scaled.x.size());
  out.y.resize(scaled.y.size());
  detail::ok(rhp_op_mul(device_ordinal(), static_cast<int64_t>(scaled.x.size()), info.col_scale.data(),
                        scaled.x.data(), out.x.data()),
             "rhp_op_mul");
  detail::ok(rhp_op_mul(device_ordinal(), static_cast<int64_t>(scaled.y.size()), info.row_scale.data(),
                        scaled.y.data(), out.y.data()),
             "rhp_op_mul");
  out.ax.assign(scaled.y.size(), 0.0);  // caches invalidated (scaling.cpp:90-93)
  out.aty.assign(scaled.x.size(), 0.0);
  out.ax_valid = false;
  out.aty_valid = false;
  return out;
}

}  // namespace rhpdhg
