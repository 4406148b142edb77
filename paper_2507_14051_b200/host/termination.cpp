// termination.cpp — relative KKT residuals (termination.cpp:24-124 of the
// reference). The O(nnz) part (two products plus the per-entry sums) runs on
// the device (EpiKktRow/EpiKktCol); this file turns the device sums into
// KktResiduals with the reference's final formulas.
#include <cmath>
#include <limits>

#include "device.hpp"
#include "kkt.hpp"
#include "rhpdhg/solver.hpp"
#include "rhpdhg/termination.hpp"

namespace rhpdhg {

namespace {
constexpr double kInf = std::numeric_limits<double>::infinity();

double clip_to_sign_cone(double s, double lb, double ub) {
  const bool lower = lb > -kInf, upper = ub < kInf;
  if (lower && upper) return s;
  if (lower) return std::max(s, 0.0);
  if (upper) return std::min(s, 0.0);
  return 0.0;
}
}  // namespace

namespace detail {

// Constant denominators, summed sequentially in the reference's order
// (termination.cpp:92-103 bound2, :116 ||c||).
Denoms problem_denoms(const LpProblem& p) {
  double bound2 = 0.0;
  for (size_t i = 0; i < p.con_lb.size(); ++i) {
    if (std::isfinite(p.con_lb[i])) bound2 += p.con_lb[i] * p.con_lb[i];
    if (std::isfinite(p.con_ub[i])) bound2 += p.con_ub[i] * p.con_ub[i];
  }
  double c2 = 0.0;
  for (double v : p.objective) c2 += v * v;
  return Denoms{1.0 + std::sqrt(bound2), 1.0 + std::sqrt(c2)};
}

Denoms problem_denoms(const rhpdhg_lp_view& v) {
  double bound2 = 0.0;
  for (int64_t i = 0; i < v.num_cons; ++i) {
    if (std::isfinite(v.con_lb[i])) bound2 += v.con_lb[i] * v.con_lb[i];
    if (std::isfinite(v.con_ub[i])) bound2 += v.con_ub[i] * v.con_ub[i];
  }
  double c2 = 0.0;
  for (int64_t j = 0; j < v.num_vars; ++j) c2 += v.objective[j] * v.objective[j];
  return Denoms{1.0 + std::sqrt(bound2), 1.0 + std::sqrt(c2)};
}

KktResiduals residuals_from_sums(const rhp_kkt_sums& s, const Denoms& d) {
  if (s.nan_x > 0) throw NumericalBreakdownError("NaN in primal iterate");
  if (s.nan_y > 0) throw NumericalBreakdownError("NaN in dual iterate");
  KktResiduals r;
  const double p_terms = (s.py_inf > 0 || s.pr_inf > 0) ? kInf : s.py + s.pr;
  if (p_terms == kInf) {
    r.gap_abs = r.gap_denom = r.gap_rel = kInf;
  } else {
    r.gap_abs = std::fabs(s.primal_value + p_terms);
    r.gap_denom = 1.0 + std::fabs(p_terms) + std::fabs(s.primal_value);
    r.gap_rel = r.gap_abs / r.gap_denom;
  }
  r.primal_inf = std::sqrt(s.viol2);
  r.primal_denom = d.primal_denom;
  r.primal_rel = r.primal_inf / r.primal_denom;
  r.dual_eq = std::sqrt(s.eq2);
  r.dual_cone = std::sqrt(s.cone2);
  r.dual_denom = d.dual_denom;
  return r;
}

}  // namespace detail

std::vector<double> reduced_costs_from_slack(const LpProblem& p, std::span<const double> aty) {
  std::vector<double> r(aty.size());
  for (size_t j = 0; j < r.size(); ++j)
    r[j] = clip_to_sign_cone(p.objective[j] - aty[j], p.var_lb[j], p.var_ub[j]);
  return r;
}

std::vector<double> reduced_costs(const LpProblem& p, std::span<const double> y) {
  std::vector<double> aty(static_cast<size_t>(p.num_vars()));
  p.matrix.multiply_transpose(y, aty);
  return reduced_costs_from_slack(p, aty);
}

KktResiduals kkt_residuals(const LpProblem& p, std::span<const double> x,
                           std::span<const double> y) {
  if (static_cast<Index>(x.size()) != p.num_vars() || static_cast<Index>(y.size()) != p.num_cons())
    throw UsageError("kkt_residuals: size mismatch");
  if (static_cast<Index>(p.objective.size()) != p.num_vars() ||
      static_cast<Index>(p.var_lb.size()) != p.num_vars() ||
      static_cast<Index>(p.var_ub.size()) != p.num_vars() ||
      static_cast<Index>(p.con_lb.size()) != p.num_cons() ||
      static_cast<Index>(p.con_ub.size()) != p.num_cons())
    throw UsageError("kkt_residuals: problem vector sizes do not match the matrix");
  spmv_counter::add(2);
  // on the matrix's cached product context, with this problem's vectors
  std::unique_lock<std::mutex> lock;
  rhp_ctx* ctx = detail::product_context(p.matrix, lock);
  const rhp_op_lp vec{p.objective.data(), p.var_lb.data(), p.var_ub.data(), p.con_lb.data(),
                      p.con_ub.data()};
  detail::ok(rhp_set_vectors(ctx, &vec), "rhp_set_vectors");
  rhp_kkt_sums s{};
  detail::ok(rhp_kkt_of(ctx, x.data(), y.data(), &s), "rhp_kkt_of");
  return detail::residuals_from_sums(s, detail::problem_denoms(p));
}

// Residuals from caller-supplied products: no products spent, host sums.
KktResiduals kkt_residuals(const LpProblem& p, std::span<const double> x,
                           std::span<const double> y, std::span<const double> ax,
                           std::span<const double> aty) {
  rhp_kkt_sums s{};
  for (double v : x) s.nan_x += std::isnan(v) ? 1 : 0;
  for (double v : y) s.nan_y += std::isnan(v) ? 1 : 0;
  const std::vector<double> r = reduced_costs_from_slack(p, aty);
  for (size_t i = 0; i < y.size(); ++i) {
    const double v = -y[i], pos = std::max(v, 0.0), neg = std::max(-v, 0.0);
    const double up = pos == 0.0 ? 0.0 : p.con_ub[i] * pos;
    const double lo = neg == 0.0 ? 0.0 : p.con_lb[i] * neg;
    if (up == kInf || lo == -kInf) s.py_inf++;
    else s.py += up - lo;
    const double proj = std::min(std::max(ax[i], p.con_lb[i]), p.con_ub[i]);
    s.viol2 += (ax[i] - proj) * (ax[i] - proj);
  }
  for (size_t j = 0; j < x.size(); ++j) {
    const double v = -r[j], pos = std::max(v, 0.0), neg = std::max(-v, 0.0);
    const double up = pos == 0.0 ? 0.0 : p.var_ub[j] * pos;
    const double lo = neg == 0.0 ? 0.0 : p.var_lb[j] * neg;
    if (up == kInf || lo == -kInf) s.pr_inf++;
    else s.pr += up - lo;
    const double d = p.objective[j] - aty[j] - r[j];
    s.eq2 += d * d;
    const double cc = r[j] - clip_to_sign_cone(r[j], p.var_lb[j], p.var_ub[j]);
    s.cone2 += cc * cc;
    s.primal_value += p.objective[j] * x[j];
  }
  return detail::residuals_from_sums(s, detail::problem_denoms(p));
}

bool is_optimal(const KktResiduals& r, const ToleranceConfig& tol) {
  const double eps = tol.epsilon;
  return r.gap_rel <= eps && r.primal_rel <= eps && r.dual_eq <= eps * r.dual_denom &&
         r.dual_cone <= eps * r.dual_denom;
}

}  // namespace rhpdhg
