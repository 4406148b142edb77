// scaling.hpp — diagonal preconditioning. Same declarations as
// /root/reference/proj/include/rhpdhg/scaling.hpp:13-32. Ruiz and
// Pock-Chambolle run on the device (rhp_scale), bit-identical to the
// reference; inside solve() they run on the solve's own context.
#pragma once

#include <utility>
#include <vector>

#include "rhpdhg/lp_problem.hpp"

namespace rhpdhg {

struct ScalingInfo {
  std::vector<double> row_scale;
  std::vector<double> col_scale;
  bool active = false;

  static ScalingInfo identity(const LpProblem& problem);
};

/// `iterations` l-inf equilibration passes (scaling.cpp:46-68).
std::pair<LpProblem, ScalingInfo> ruiz_equilibrate(const LpProblem& problem, int iterations);

/// One 1-norm pass composed into `info` (scaling.cpp:70-81).
LpProblem pock_chambolle_scale(const LpProblem& problem, ScalingInfo& info);

/// x = D_col x_bar, y = D_row y_bar; caches invalidated (scaling.cpp:83-94).
Iterate unscale_iterate(const Iterate& scaled, const ScalingInfo& info);

/// Extension: the scaled instance and cumulative scales exactly as solve()
/// builds them (ruiz_equilibrate then pock_chambolle_scale) in one device pass.
std::pair<LpProblem, ScalingInfo> scale_problem(const LpProblem& problem, bool enabled,
                                                int ruiz_iterations, bool pock_chambolle);

}  // namespace rhpdhg
