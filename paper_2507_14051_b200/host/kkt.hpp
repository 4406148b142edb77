// kkt.hpp — internal: device KKT sums -> KktResiduals.
#pragma once

#include "rhpdhg/lp_problem.hpp"
#include "rhpdhg/termination.hpp"
#include "rhpdhg_cuda.h"

namespace rhpdhg::detail {

struct Denoms {
  double primal_denom;  // 1 + ||(L, U) finite||_2
  double dual_denom;    // 1 + ||c||_2
};

Denoms problem_denoms(const LpProblem& p);
Denoms problem_denoms(const rhpdhg_lp_view& v);
KktResiduals residuals_from_sums(const rhp_kkt_sums& s, const Denoms& d);

}  // namespace rhpdhg::detail
