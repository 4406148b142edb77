// scaling.hpp — diagonal preconditioning state. Mirrors
// /root/reference/proj/include/rhpdhg/scaling.hpp:13-19. Ruiz and
// Pock-Chambolle run on the device inside solve() (rhp_scale).
#pragma once

#include <vector>

#include "rhpdhg/lp_problem.hpp"

namespace rhpdhg {

struct ScalingInfo {
  std::vector<double> row_scale;
  std::vector<double> col_scale;
  bool active = false;

  static ScalingInfo identity(const LpProblem& problem);
};

/// The scaled instance and cumulative scales exactly as solve() builds them
/// (ruiz_equilibrate then pock_chambolle_scale, scaling.cpp:46-81), computed
/// on the device.
std::pair<LpProblem, ScalingInfo> scale_problem(const LpProblem& problem, bool enabled,
                                                int ruiz_iterations, bool pock_chambolle);

}  // namespace rhpdhg
