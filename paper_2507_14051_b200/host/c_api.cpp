// c_api.cpp — the flat C ABI of include/rhpdhg_c.h over the C++ API.
#include <cstring>
#include <memory>
#include <exception>
#include <sstream>
#include <string>

#include "device.hpp"
#include "rhpdhg/errors.hpp"
#include "rhpdhg/solver.hpp"
#include "rhpdhg/mps.hpp"
#include "rhpdhg/termination.hpp"
#include "rhpdhg/bench.hpp"
#include "rhpdhg_c.h"
#include "session.hpp"

using namespace rhpdhg;

namespace {
thread_local std::string g_msg;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return RHPDHG_OK;
  } catch (const UsageError& e) {
    g_msg = e.what();
    return RHPDHG_E_USAGE;
  } catch (const InvalidProblemError& e) {
    g_msg = e.what();
    return RHPDHG_E_INVALID_PROBLEM;
  } catch (const ParseError& e) {
    g_msg = e.what();
    return RHPDHG_E_PARSE;
  } catch (const NumericalBreakdownError& e) {
    g_msg = e.what();
    return RHPDHG_E_BREAKDOWN;
  } catch (const DeviceError& e) {
    g_msg = e.what();
    return RHPDHG_E_DEVICE;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return RHPDHG_E_INTERNAL;
  }
}

LpProblem to_problem(const rhpdhg_lp_view* v) {
  if (!v) throw UsageError("null LP view");
  if (v->num_cons < 0 || v->num_vars < 0) throw UsageError("matrix dimensions must be nonnegative");
  const size_t m = static_cast<size_t>(v->num_cons), n = static_cast<size_t>(v->num_vars);
  const Index nz = (v->num_cons > 0 && v->row_ptr) ? v->row_ptr[v->num_cons] : 0;
  std::vector<Index> rp = v->row_ptr ? std::vector<Index>(v->row_ptr, v->row_ptr + m + 1)
                                     : std::vector<Index>(m + 1, 0);
  LpProblem p;
  p.matrix = SparseMatrix::from_csr(v->num_cons, v->num_vars, std::move(rp),
                                    std::vector<Index>(v->col_index, v->col_index + nz),
                                    std::vector<double>(v->values, v->values + nz));
  p.objective.assign(v->objective, v->objective + n);
  p.objective_offset = v->objective_offset;
  p.var_lb.assign(v->var_lb, v->var_lb + n);
  p.var_ub.assign(v->var_ub, v->var_ub + n);
  p.con_lb.assign(v->con_lb, v->con_lb + m);
  p.con_ub.assign(v->con_ub, v->con_ub + m);
  p.maximization = v->maximization != 0;
  return p;
}

SolverConfig to_config(const rhpdhg_config_c* c) {
  SolverConfig s;
  if (!c) return s;
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
  *o = rhpdhg_kkt_c{r.gap_abs,    r.gap_rel,   r.primal_inf, r.primal_rel,  r.dual_eq,
                    r.dual_cone,  r.gap_denom, r.primal_denom, r.dual_denom};
}

void fill_report(const SolutionReport& r, rhpdhg_report_c* out, double* x, double* y, double* rc,
                 double* hist, int64_t hist_cap);
}  // namespace

struct rhpdhg_session {
  LpProblem problem;
  std::unique_ptr<Session> session;
};

struct rhpdhg_lp {
  LpProblem problem;
};

extern "C" {

const char* rhpdhg_last_error(void) { return g_msg.c_str(); }

int rhpdhg_lp_read_mps(const char* path, rhpdhg_lp** out, char* warnings, int64_t cap) {
  *out = nullptr;
  return guarded([&] {
    std::vector<std::string> w;
    auto h = std::make_unique<rhpdhg_lp>();
    h->problem = parse_mps_file(path, &w);
    if (warnings && cap > 0) {
      std::string joined;
      for (const std::string& s : w) joined += (joined.empty() ? "" : "\n") + s;
      const size_t k = std::min<size_t>(joined.size(), static_cast<size_t>(cap - 1));
      std::memcpy(warnings, joined.data(), k);
      warnings[k] = '\0';
    }
    *out = h.release();
  });
}

int rhpdhg_lp_view_of(const rhpdhg_lp* lp, rhpdhg_lp_view* v) {
  return guarded([&] { *v = detail::view_of(lp->problem); });
}

void rhpdhg_lp_free(rhpdhg_lp* lp) { delete lp; }

int rhpdhg_config_default(rhpdhg_config_c* c) {
  return guarded([&] {
    const SolverConfig s;
    std::memset(c, 0, sizeof(*c));
    c->scaling_enabled = s.scaling_enabled;
    c->ruiz_iterations = s.ruiz_iterations;
    c->pock_chambolle = s.pock_chambolle;
    c->restarts_enabled = s.restarts_enabled;
    c->stepsize_multiplier = s.stepsize_multiplier;
    c->power_tol = s.power_tol;
    c->power_max_iters = s.power_max_iters;
    c->power_seed = s.power_seed;
    c->beta_sufficient = s.beta_sufficient;
    c->beta_necessary = s.beta_necessary;
    c->beta_artificial = s.beta_artificial;
    c->reflection_gamma = s.reflection_gamma;
    c->pid_kp = s.pid_kp;
    c->pid_ki = s.pid_ki;
    c->pid_kd = s.pid_kd;
    c->initial_weight = s.initial_weight;
    c->epsilon = s.epsilon;
    c->check_interval = s.check_interval;
    c->time_limit_seconds = s.time_limit_seconds;
    c->iteration_limit = s.iteration_limit;
    c->verbosity = s.verbosity;
    c->record_residual_history = s.record_residual_history;
  });
}

int rhpdhg_set_device(int device) {
  return guarded([&] { default_device_options().device = device; });
}

int rhpdhg_set_device_options(int device, int use_graph, int64_t block_limit) {
  return guarded([&] {
    if (block_limit < 1) throw UsageError("block_limit must be >= 1");
    DeviceOptions& d = default_device_options();
    d.device = device;
    d.use_graph = use_graph != 0;
    d.block_limit = static_cast<long>(block_limit);
  });
}

int rhpdhg_set_resident(int mode) {
  return guarded([&] { default_device_options().resident = mode < 0 ? -1 : (mode ? 1 : 0); });
}

int rhpdhg_set_locality(int mode) {
  return guarded([&] { default_device_options().locality = mode < 0 ? -1 : (mode ? 1 : 0); });
}

int rhpdhg_set_distributed(int rank, int world_size, const void* nccl_id) {
  return guarded([&] {
    if (world_size < 1 || rank < 0 || rank >= world_size) throw UsageError("bad rank/world_size");
    if (world_size > 1 && !nccl_id) throw UsageError("world_size > 1 needs an NCCL unique id");
    DeviceOptions& d = default_device_options();
    d.rank = rank;
    d.world_size = world_size;
    if (nccl_id) {
      const char* p = static_cast<const char*>(nccl_id);
      d.nccl_id.assign(p, p + 128);
    } else {
      d.nccl_id.clear();
    }
    d.local_group = nullptr;
  });
}

int rhpdhg_set_local_group(int rank, int world_size, const void* group) {
  return guarded([&] {
    if (world_size < 1 || rank < 0 || rank >= world_size) throw UsageError("bad rank/world_size");
    if (!group) throw UsageError("rhpdhg_set_local_group: null group");
    DeviceOptions& d = default_device_options();
    d.rank = rank;
    d.world_size = world_size;
    d.nccl_id.clear();
    d.local_group = group;
  });
}

int rhpdhg_solve_csr(const rhpdhg_lp_view* lp, const rhpdhg_config_c* cfg, rhpdhg_report_c* out,
                     double* x, double* y, double* rc, double* hist, int64_t hist_cap) {
  return guarded([&] {
    const LpProblem p = to_problem(lp);
    fill_report(solve(p, to_config(cfg)), out, x, y, rc, hist, hist_cap);
  });
}

int rhpdhg_session_create(const rhpdhg_lp_view* lp, const rhpdhg_config_c* cfg,
                          rhpdhg_session** out) {
  *out = nullptr;
  return guarded([&] {
    if (!lp) throw UsageError("null LP view");
    auto h = std::make_unique<rhpdhg_session>();
    const bool complete = lp->num_cons >= 0 && lp->num_vars >= 0 &&
                          (lp->num_cons == 0 || lp->row_ptr) &&
                          (lp->num_cons == 0 || lp->row_ptr[lp->num_cons] == lp->row_ptr[0] ||
                           (lp->col_index && lp->values));
    if (complete) {  // zero-copy: the caller's arrays are borrowed until destroy
      h->session = std::make_unique<Session>(*lp, to_config(cfg), default_device_options());
    } else {
      h->problem = to_problem(lp);
      h->session = std::make_unique<Session>(h->problem, to_config(cfg), default_device_options());
    }
    *out = h.release();
  });
}

int rhpdhg_session_advance(rhpdhg_session* s, int64_t iterations, int32_t* running) {
  return guarded([&] {
    const bool r = s->session->advance(static_cast<long>(iterations));
    if (running) *running = r ? 1 : 0;
  });
}

int rhpdhg_session_info(rhpdhg_session* s, int64_t* total, int64_t* restarts, rhpdhg_kkt_c* last,
                        double* setup_seconds, int64_t* blocks, int64_t* checks) {
  return guarded([&] {
    if (total) *total = s->session->total();
    if (restarts) *restarts = s->session->restarts();
    if (last) to_c(s->session->last_residuals(), last);
    if (setup_seconds) *setup_seconds = s->session->setup_seconds();
    if (blocks) *blocks = s->session->device_blocks();
    if (checks) *checks = s->session->kkt_checks();
  });
}

int rhpdhg_session_timer(rhpdhg_session* s, int start, double* ms) {
  return guarded([&] { detail::ok(rhp_timer(s->session->device(), start, ms), "rhp_timer"); });
}

int rhpdhg_session_time_kernels(rhpdhg_session* s, int reps, double* ms3) {
  return guarded([&] {
    detail::ok(rhp_time_kernels(s->session->device(), reps, &ms3[0], &ms3[1], &ms3[2]),
               "rhp_time_kernels");
  });
}

int rhpdhg_session_gather_ceiling(rhpdhg_session* s, int reps, double* ms2) {
  return guarded([&] {
    detail::ok(rhp_gather_ceiling(s->session->device(), reps, &ms2[0], &ms2[1]), "rhp_gather_ceiling");
  });
}

int rhpdhg_session_layout(rhpdhg_session* s, int64_t* o) {
  return guarded([&] {
    rhp_layout_info li{};
    detail::ok(rhp_layout(s->session->device(), &li), "rhp_layout");
    o[0] = li.m_local;
    o[1] = li.n;
    o[2] = li.nnz_local;
    for (int k = 0; k < 8; ++k) {
      o[3 + k] = li.row_bins[k];
      o[11 + k] = li.col_bins[k];
    }
    o[19] = li.grid_a;
    o[20] = li.grid_at;
    o[21] = li.grid_vec;
    o[22] = li.sm_count;
    o[23] = li.gather_l1;
    o[24] = li.pdl;
    o[25] = li.thread_rows;
    o[26] = li.segments;
    o[27] = li.resident;
    o[28] = li.partition;
    o[29] = li.const_bounds;
    o[30] = li.relabel;
    for (int k = 0; k < 4; ++k) std::memcpy(&o[31 + k], &li.sectors[k], sizeof(double));
  });
}

int rhpdhg_session_finish(rhpdhg_session* s, rhpdhg_report_c* out, double* x, double* y,
                          double* rc, double* hist, int64_t hist_cap) {
  return guarded([&] { fill_report(s->session->finish(), out, x, y, rc, hist, hist_cap); });
}

void rhpdhg_session_destroy(rhpdhg_session* s) { delete s; }

}  // extern "C"

namespace {
void fill_report(const SolutionReport& r, rhpdhg_report_c* out, double* x, double* y, double* rc,
                 double* hist, int64_t hist_cap) {
  {
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
    out->has_inner_residuals = r.inner_residuals ? 1 : 0;
    if (r.inner_residuals) to_c(*r.inner_residuals, &out->inner_residuals);
    out->history_len = static_cast<int64_t>(r.fixed_point_residual_history.size());
    out->setup_seconds = r.setup_seconds;
    out->loop_seconds = r.loop_seconds;
    out->device_blocks = r.device_blocks;
    if (x) std::memcpy(x, r.x.data(), r.x.size() * sizeof(double));
    if (y) std::memcpy(y, r.y.data(), r.y.size() * sizeof(double));
    if (rc) std::memcpy(rc, r.reduced_costs.data(), r.reduced_costs.size() * sizeof(double));
    if (hist && hist_cap > 0) {
      const size_t k = std::min<size_t>(r.fixed_point_residual_history.size(),
                                        static_cast<size_t>(hist_cap));
      std::memcpy(hist, r.fixed_point_residual_history.data(), k * sizeof(double));
    }
  }
}
}  // namespace

extern "C" {

int rhpdhg_run_benchmark(const char* dir, const rhpdhg_config_c* cfg, double small_limit_seconds,
                         double large_limit_seconds, int workers, const char* json_path,
                         char* table, int64_t table_cap) {
  return guarded([&] {
    BenchmarkOptions opts;
    opts.small_limit_seconds = small_limit_seconds;
    opts.large_limit_seconds = large_limit_seconds;
    opts.workers = workers;
    const SolverConfig c = to_config(cfg);
    std::ostringstream log;
    const BenchmarkReport rep = run_benchmark(dir, c, opts, &log);
    if (json_path && *json_path) write_benchmark_json(rep, c.epsilon, json_path);
    std::ostringstream os;
    os << log.str();
    write_benchmark_table(rep, os);
    if (table && table_cap > 0) {
      const std::string t = os.str();
      const size_t k = std::min<size_t>(t.size(), static_cast<size_t>(table_cap - 1));
      std::memcpy(table, t.data(), k);
      table[k] = '\0';
    }
  });
}

int rhpdhg_kkt_residuals(const rhpdhg_lp_view* lp, const double* x, const double* y,
                         rhpdhg_kkt_c* out) {
  return guarded([&] {
    const LpProblem p = to_problem(lp);
    const KktResiduals r = kkt_residuals(
        p, std::span<const double>(x, static_cast<size_t>(p.num_vars())),
        std::span<const double>(y, static_cast<size_t>(p.num_cons())));
    to_c(r, out);
  });
}

}  // extern "C"
