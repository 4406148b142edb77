// solver.hpp — the solve() entry point. Mirrors
// /root/reference/proj/include/rhpdhg/solver.hpp:13; the pipeline (scaling,
// power iteration, restarted reflected-Halpern loop, KKT checks) runs on the
// GPU through the device library (include/rhpdhg_cuda.h).
#pragma once

#include <vector>

#include "rhpdhg/config.hpp"
#include "rhpdhg/lp_problem.hpp"
#include "rhpdhg/report.hpp"

namespace rhpdhg {

/// Device-side runtime knobs (not SolverConfig file keys, so the config echo
/// stays identical to the reference).
struct DeviceOptions {
  int device = 0;
  bool use_graph = true;   // CUDA graph with a conditional WHILE node per block
  long block_limit = 64;   // PDHG iterations per device block at most
  int resident = -1;       // small LPs: one cluster runs whole blocks (-1 auto, 0 off, 1 on)
  int locality = 0;        // first-touch row/column relabelling (0 auto, -1 off, 1 forced)
  // Row-partitioned multi-GPU solve (one process per GPU): every rank calls
  // solve() on the FULL problem with the same config; rank 0's 128-byte
  // ncclUniqueId (rhp_nccl_unique_id) is shared out of band. An id with
  // world_size == 1 runs the same partitioned code path on one GPU.
  int rank = 0;
  int world_size = 1;
  std::vector<char> nccl_id;  // empty: single-GPU path
  // Instead of NCCL: an in-process collective group (rhp_local_group_create)
  // shared by world_size threads of this process, one rank each.
  const void* local_group = nullptr;
};

/// The calling thread's default device options (used by solve(problem, cfg));
/// per thread so threads of one process can act as different ranks.
DeviceOptions& default_device_options();

SolutionReport solve(const LpProblem& problem, const SolverConfig& cfg);
SolutionReport solve(const LpProblem& problem, const SolverConfig& cfg, const DeviceOptions& dev);

}  // namespace rhpdhg
