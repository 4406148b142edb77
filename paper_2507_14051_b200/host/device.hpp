// device.hpp — RAII handle over the device C ABI (include/rhpdhg_cuda.h)
// that turns status codes back into the rhpdhg exception types.
#pragma once

#include <memory>
#include <mutex>
#include <string>

#include "rhpdhg/errors.hpp"
#include "rhpdhg/lp_problem.hpp"
#include "rhpdhg_cuda.h"

namespace rhpdhg::detail {

[[noreturn]] inline void throw_status(int rc, const std::string& where) {
  const std::string msg = where + ": " + rhp_last_error();
  switch (rc) {
    case RHPDHG_E_USAGE: throw UsageError(msg);
    case RHPDHG_E_INVALID_PROBLEM: throw InvalidProblemError(msg);
    case RHPDHG_E_PARSE: throw ParseError(msg, 0);
    case RHPDHG_E_BREAKDOWN: throw NumericalBreakdownError(msg);
    default: throw DeviceError(msg);
  }
}

inline void ok(int rc, const char* where) {
  if (rc != RHPDHG_OK) throw_status(rc, where);
}

/// Borrowed C view of an LpProblem (CSR of its matrix).
// LpProblem::validate's vector checks on a borrowed view (model.cpp).
void validate_vectors(const rhpdhg_lp_view& v);

inline rhpdhg_lp_view view_of(const LpProblem& p) {
  rhpdhg_lp_view v{};
  v.num_cons = p.num_cons();
  v.num_vars = p.num_vars();
  v.nnz = p.matrix.nnz();
  v.row_ptr = p.matrix.row_ptr().data();
  v.col_index = p.matrix.col_index().data();
  v.values = p.matrix.csr_values().data();
  v.objective = p.objective.data();
  v.objective_offset = p.objective_offset;
  v.var_lb = p.var_lb.data();
  v.var_ub = p.var_ub.data();
  v.con_lb = p.con_lb.data();
  v.con_ub = p.con_ub.data();
  v.maximization = p.maximization ? 1 : 0;
  return v;
}

class Device {
 public:
  Device(const rhpdhg_lp_view& v, const rhp_options& opt) { ok(rhp_create(&v, &opt, &ctx_), "rhp_create"); }
  ~Device() { rhp_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  rhp_ctx* get() const { return ctx_; }

 private:
  rhp_ctx* ctx_ = nullptr;
};

inline rhp_options options(int device, bool use_graph, long block_limit) {
  rhp_options o{};
  o.device = device;
  o.rank = 0;
  o.world_size = 1;
  o.use_graph = use_graph ? 1 : 0;
  o.block_limit = block_limit;
  o.nccl_id = nullptr;
  o.local_group = nullptr;
  o.resident = 0;  // per-op contexts (products, KKT, scaling) never use resident blocks
  o.locality = -1;  // nor a relabelled layout (CSC values keep the reference's element order)
  return o;
}

// Full options of a solve, including the row-partitioned multi-GPU fields
// (the id buffer must outlive rhp_create).
template <class DeviceOptionsT>
inline rhp_options options(const DeviceOptionsT& d) {
  rhp_options o = options(d.device, d.use_graph, d.block_limit);
  o.resident = d.resident;
  o.locality = d.locality;
  o.rank = d.rank;
  o.world_size = d.world_size;
  if (!d.nccl_id.empty()) {
    if (d.nccl_id.size() != 128) throw UsageError("nccl_id must be 128 bytes");
    o.nccl_id = d.nccl_id.data();
  } else if (d.local_group) {
    o.local_group = d.local_group;
  } else if (d.world_size > 1) {
    throw UsageError("world_size > 1 needs the NCCL unique id of rank 0 or a local group");
  }
  return o;
}

// A SparseMatrix's cached product context (sparse_matrix.hpp dev_): built on
// first use from the matrix's CSR (and CSC values when they were set
// explicitly), with zero objective/bounds; the per-op API uploads the
// vectors it needs with each call. `mu` serialises its users.
struct DeviceCache {
  std::mutex mu;
  std::unique_ptr<Device> dev;
};

// Locks the matrix's cache and returns its context (created on first use).
rhp_ctx* product_context(const SparseMatrix& a, std::unique_lock<std::mutex>& lock);

}  // namespace rhpdhg::detail
