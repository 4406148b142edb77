// session.hpp — internal: the solve() state machine (setup in the ctor,
// one device block + host control per step(), report in finish()).
#pragma once

#include <chrono>
#include <memory>
#include <string>

#include "device.hpp"
#include "kkt.hpp"
#include "rhpdhg/config.hpp"
#include "rhpdhg/pdhg.hpp"
#include "rhpdhg/report.hpp"
#include "rhpdhg/restart.hpp"
#include "rhpdhg/solver.hpp"

namespace rhpdhg {

using Clock = std::chrono::steady_clock;

namespace detail {
// NVTX range for the duration of a scope (host/nvtx.cpp; header-only NVTX3,
// no-op unless a profiler such as nsys / ncu --nvtx is attached). Names:
// rhpdhg:setup / :ingest / :scaling / :power_iteration, :block, :kkt_check,
// :restart, :finish.
class NvtxRange {
 public:
  explicit NvtxRange(const char* name);
  ~NvtxRange();
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace detail

class Session {
 public:
  Session(const LpProblem& problem, const SolverConfig& cfg, const DeviceOptions& dopt);
  // Zero-copy: the view's arrays are borrowed and must outlive the session.
  // The matrix is validated by the device ingest (same exception classes and
  // messages as SparseMatrix::from_csr), the vectors as LpProblem::validate.
  Session(const rhpdhg_lp_view& view, const SolverConfig& cfg, const DeviceOptions& dopt);
  ~Session();
  bool step();                   // false once decided
  bool advance(long iterations); // runs blocks until >= iterations more are done or decided
  SolutionReport finish();
  long total() const { return total_; }
  bool decided() const { return decided_; }
  long restarts() const { return restarts_; }
  long device_blocks() const { return report_.device_blocks; }
  long kkt_checks() const { return report_.kkt_checks; }
  const KktResiduals& last_residuals() const { return last_; }
  double setup_seconds() const { return report_.setup_seconds; }
  rhp_ctx* device() const;

 private:
  Session(const rhpdhg_lp_view& view, const std::string& name, bool validated,
          const SolverConfig& cfg, const DeviceOptions& dopt);
  KktResiduals kkt_check(int which);

  rhpdhg_lp_view view_{};  // the problem's arrays (borrowed)
  std::string name_;
  SolverConfig cfg_;
  std::unique_ptr<detail::Device> dev_;
  Clock::time_point t0_, t_loop_;
  StepConfig step_;
  PidState pid_;
  detail::Denoms denoms_{1.0, 1.0};
  ToleranceConfig tol_;
  SolutionReport report_;
  KktResiduals last_;
  SolveStatus status_ = SolveStatus::iteration_limit;
  bool decided_ = false, have_inner_ = false;
  long total_ = 0, restarts_ = 0;
  std::uint64_t spmv_checks_ = 0;
  double last_fpr_ = std::numeric_limits<double>::infinity();
};

}  // namespace rhpdhg
