"""ctypes mirror of the C ABIs in include/rhpdhg_c.h and include/rhpdhg_cuda.h.

Structs are field-for-field copies of the C declarations; `load_*` functions
open the in-tree shared libraries and fail loudly when they are missing
(there is no CPU fallback in the product).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
# RHPDHG_LIB_DIR selects an alternative in-tree build (kernel experiments)
LIB_DIR = Path(os.environ.get("RHPDHG_LIB_DIR", str(PKG_DIR / "lib"))).resolve()

OK, E_USAGE, E_INVALID_PROBLEM, E_PARSE, E_BREAKDOWN, E_DEVICE, E_INTERNAL = range(7)
OPTIMAL, ITERATION_LIMIT, TIME_LIMIT = range(3)
STATUS_NAMES = {OPTIMAL: "optimal", ITERATION_LIMIT: "iteration_limit", TIME_LIMIT: "time_limit"}

c_double_p = C.POINTER(C.c_double)
c_int64_p = C.POINTER(C.c_int64)


class LpView(C.Structure):
    """rhpdhg_lp_view <- struct LpProblem (lp_problem.hpp:18-36)."""

    _fields_ = [
        ("num_cons", C.c_int64),
        ("num_vars", C.c_int64),
        ("nnz", C.c_int64),
        ("row_ptr", c_int64_p),
        ("col_index", c_int64_p),
        ("values", c_double_p),
        ("objective", c_double_p),
        ("objective_offset", C.c_double),
        ("var_lb", c_double_p),
        ("var_ub", c_double_p),
        ("con_lb", c_double_p),
        ("con_ub", c_double_p),
        ("maximization", C.c_int32),
    ]


class ConfigC(C.Structure):
    """rhpdhg_config_c <- struct SolverConfig (config.hpp:12-40)."""

    _fields_ = [
        ("scaling_enabled", C.c_int32),
        ("ruiz_iterations", C.c_int32),
        ("pock_chambolle", C.c_int32),
        ("restarts_enabled", C.c_int32),
        ("stepsize_multiplier", C.c_double),
        ("power_tol", C.c_double),
        ("power_max_iters", C.c_int64),
        ("power_seed", C.c_uint64),
        ("beta_sufficient", C.c_double),
        ("beta_necessary", C.c_double),
        ("beta_artificial", C.c_double),
        ("reflection_gamma", C.c_double),
        ("pid_kp", C.c_double),
        ("pid_ki", C.c_double),
        ("pid_kd", C.c_double),
        ("initial_weight", C.c_double),
        ("epsilon", C.c_double),
        ("check_interval", C.c_int64),
        ("time_limit_seconds", C.c_double),
        ("iteration_limit", C.c_int64),
        ("verbosity", C.c_int32),
        ("record_residual_history", C.c_int32),
    ]


class KktC(C.Structure):
    """rhpdhg_kkt_c <- struct KktResiduals (termination.hpp:12-22)."""

    _fields_ = [
        (n, C.c_double)
        for n in ("gap_abs", "gap_rel", "primal_inf", "primal_rel", "dual_eq", "dual_cone",
                  "gap_denom", "primal_denom", "dual_denom")
    ]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class ReportC(C.Structure):
    """rhpdhg_report_c <- struct SolutionReport (report.hpp:19-42)."""

    _fields_ = [
        ("status", C.c_int32),
        ("has_inner_residuals", C.c_int32),
        ("objective", C.c_double),
        ("residuals", KktC),
        ("iterations", C.c_int64),
        ("restart_count", C.c_int64),
        ("wall_time_seconds", C.c_double),
        ("final_fixed_point_residual", C.c_double),
        ("final_primal_weight", C.c_double),
        ("matrix_norm_estimate", C.c_double),
        ("power_iterations", C.c_int64),
        ("spmv_loop", C.c_uint64),
        ("spmv_checks", C.c_uint64),
        ("spmv_setup", C.c_uint64),
        ("kkt_checks", C.c_int64),
        ("inner_residuals", KktC),
        ("history_len", C.c_int64),
        ("setup_seconds", C.c_double),
        ("loop_seconds", C.c_double),
        ("device_blocks", C.c_int64),
    ]


# ----------------------------------------------------------- rhpdhg_cuda.h --
class RhpOptions(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("rank", C.c_int32),
        ("world_size", C.c_int32),
        ("use_graph", C.c_int32),
        ("block_limit", C.c_int64),
        ("nccl_id", C.c_void_p),
        ("resident", C.c_int32),
        ("locality", C.c_int32),
        ("local_group", C.c_void_p),
    ]


class RhpStep(C.Structure):
    _fields_ = [
        ("eta", C.c_double), ("omega", C.c_double), ("gamma", C.c_double),
        ("tau", C.c_double), ("sigma", C.c_double), ("sigma_inv", C.c_double),
        ("primal_scale", C.c_double), ("dual_scale", C.c_double),
        ("beta_sufficient", C.c_double), ("beta_necessary", C.c_double),
        ("beta_artificial", C.c_double),
        ("check_interval", C.c_int64), ("iteration_limit", C.c_int64),
        ("restarts_enabled", C.c_int32), ("record_history", C.c_int32),
    ]


class RhpBlockOut(C.Structure):
    _fields_ = [
        ("iterations_done", C.c_int64), ("total", C.c_int64), ("k", C.c_int64),
        ("verdict", C.c_int32), ("check_due", C.c_int32), ("breakdown", C.c_int32),
        ("pad_", C.c_int32),
        ("r_last", C.c_double), ("r_anchor", C.c_double), ("r_prev", C.c_double),
        ("q_last", C.c_double),
        ("x_dist2", C.c_double), ("y_dist2", C.c_double), ("x_norm2", C.c_double),
        ("y_norm2", C.c_double),
    ]


class RhpKktSums(C.Structure):
    _fields_ = [
        ("primal_value", C.c_double), ("py", C.c_double), ("pr", C.c_double),
        ("viol2", C.c_double), ("eq2", C.c_double), ("cone2", C.c_double),
        ("py_inf", C.c_int64), ("pr_inf", C.c_int64), ("nan_x", C.c_int64),
        ("nan_y", C.c_int64),
    ]


class RhpScaledOut(C.Structure):
    _fields_ = [(n, c_double_p) for n in (
        "csr_values", "csc_values", "row_scale", "col_scale", "objective", "var_lb",
        "var_ub", "con_lb", "con_ub")]


class RhpDeviceInfo(C.Structure):
    _fields_ = [
        ("name", C.c_char * 128), ("sm_count", C.c_int32), ("cc_major", C.c_int32),
        ("cc_minor", C.c_int32), ("l2_bytes", C.c_int64), ("mem_bytes", C.c_int64),
        ("graph_supported", C.c_int32), ("pad_", C.c_int32),
    ]


class RhpLayoutInfo(C.Structure):
    _fields_ = [
        ("m_local", C.c_int64), ("n", C.c_int64), ("nnz_local", C.c_int64),
        ("row_bins", C.c_int64 * 8), ("col_bins", C.c_int64 * 8),
        ("grid_a", C.c_int32), ("grid_at", C.c_int32), ("grid_vec", C.c_int32),
        ("sm_count", C.c_int32), ("gather_l1", C.c_int32), ("pdl", C.c_int32),
        ("thread_rows", C.c_int32), ("segments", C.c_int32),
        ("resident", C.c_int32), ("partition", C.c_int32), ("const_bounds", C.c_int32),
        ("relabel", C.c_int32), ("pad2_", C.c_int32), ("sectors", C.c_double * 4),
    ]


# The C-ABI symbols each library exports (checked by the CPU test suite).
CUDA_SYMBOLS = [
    "rhp_last_error", "rhp_device_count", "rhp_get_device_info", "rhp_nccl_unique_id",
    "rhp_create", "rhp_destroy", "rhp_layout", "rhp_scale", "rhp_get_scaled",
    "rhp_power_begin", "rhp_power_step", "rhp_power_normalize", "rhp_spmv", "rhp_set_step",
    "rhp_reset_iterate", "rhp_set_iterate", "rhp_run_block", "rhp_get_history", "rhp_kkt",
    "rhp_kkt_of", "rhp_fetch_solution", "rhp_fetch_iterate", "rhp_restart", "rhp_any",
    "rhp_partition_rows",
    "rhp_last_block_ms", "rhp_timer", "rhp_time_kernels", "rhp_time_spmv", "rhp_gather_ceiling", "rhp_profiler_range",
    "rhp_synchronize",
    "rhp_op_pdhg", "rhp_set_vectors", "rhp_set_csc_values", "rhp_op_sums", "rhp_op_mul",
    "rhp_local_group_create", "rhp_local_group_destroy",
]
HOST_SYMBOLS = [
    "rhpdhg_config_default", "rhpdhg_solve_csr", "rhpdhg_kkt_residuals", "rhpdhg_last_error",
    "rhpdhg_set_device", "rhpdhg_set_device_options", "rhpdhg_set_distributed",
    "rhpdhg_set_resident", "rhpdhg_set_locality", "rhpdhg_set_local_group", "rhpdhg_run_benchmark",
    "rhpdhg_session_create",
    "rhpdhg_session_advance", "rhpdhg_session_info", "rhpdhg_session_timer",
    "rhpdhg_session_finish", "rhpdhg_session_destroy", "rhpdhg_session_time_kernels",
    "rhpdhg_session_gather_ceiling",
    "rhpdhg_session_layout", "rhpdhg_lp_read_mps", "rhpdhg_lp_view_of", "rhpdhg_lp_free",
]

_cache: dict[str, C.CDLL] = {}


def _open(path: Path) -> C.CDLL:
    key = str(path)
    if key not in _cache:
        if not path.exists():
            raise RuntimeError(
                f"{path} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()' or `make`). "
                "There is no CPU fallback.")
        _cache[key] = C.CDLL(key, mode=os.RTLD_NOW | os.RTLD_LOCAL)
    return _cache[key]


def load_cuda() -> C.CDLL:
    lib = _open(LIB_DIR / "librhp_cuda.so")
    if not getattr(lib, "_typed", False):
        P = C.c_void_p
        lib.rhp_last_error.restype = C.c_char_p
        sig = {
            "rhp_device_count": [C.POINTER(C.c_int)],
            "rhp_get_device_info": [C.c_int, C.POINTER(RhpDeviceInfo)],
            "rhp_nccl_unique_id": [P],
            "rhp_create": [C.POINTER(LpView), C.POINTER(RhpOptions), C.POINTER(P)],
            "rhp_destroy": [P],
            "rhp_layout": [P, C.POINTER(RhpLayoutInfo)],
            "rhp_scale": [P, C.c_int, C.c_int, C.c_int],
            "rhp_get_scaled": [P, C.POINTER(RhpScaledOut)],
            "rhp_power_begin": [P, c_double_p],
            "rhp_power_step": [P, c_double_p, c_double_p],
            "rhp_power_normalize": [P, C.c_double],
            "rhp_spmv": [P, C.c_int, c_double_p, c_double_p],
            "rhp_set_step": [P, C.POINTER(RhpStep)],
            "rhp_reset_iterate": [P],
            "rhp_set_iterate": [P, c_double_p, c_double_p],
            "rhp_run_block": [P, C.POINTER(RhpBlockOut)],
            "rhp_get_history": [P, c_double_p, C.c_int64, c_int64_p],
            "rhp_kkt": [P, C.c_int, C.POINTER(RhpKktSums)],
            "rhp_kkt_of": [P, c_double_p, c_double_p, C.POINTER(RhpKktSums)],
            "rhp_fetch_solution": [P, c_double_p, c_double_p, c_double_p],
            "rhp_fetch_iterate": [P, c_double_p, c_double_p, c_double_p, c_double_p],
            "rhp_restart": [P],
            "rhp_any": [P, C.c_int, C.POINTER(C.c_int)],
            "rhp_partition_rows": [C.POINTER(LpView), C.c_int, c_int64_p],
            "rhp_last_block_ms": [P, c_double_p],
            "rhp_timer": [P, C.c_int, c_double_p],
            "rhp_time_kernels": [P, C.c_int, c_double_p, c_double_p, c_double_p],
            "rhp_profiler_range": [C.c_int],
            "rhp_time_spmv": [P, C.c_int, C.c_int, c_double_p],
            "rhp_gather_ceiling": [P, C.c_int, c_double_p, c_double_p],
            "rhp_synchronize": [P],
            "rhp_op_pdhg": [P, P, P, P, P, P, c_double_p, c_double_p, P],
            "rhp_set_vectors": [P, P],
            "rhp_set_csc_values": [P, c_double_p, C.c_int],
            "rhp_op_sums": [C.c_int, C.c_int64, c_double_p, c_double_p, C.c_int64, c_double_p,
                            c_double_p, c_double_p, c_double_p],
            "rhp_op_mul": [C.c_int, C.c_int64, c_double_p, c_double_p, c_double_p],
            "rhp_local_group_create": [C.c_int, C.POINTER(P)],
            "rhp_local_group_destroy": [P],
        }
        for name, args in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        lib._typed = True
    return lib


def load_host() -> C.CDLL:
    load_cuda()  # dependency, loaded from the same directory
    lib = _open(LIB_DIR / "librhpdhg.so")
    if not getattr(lib, "_typed", False):
        lib.rhpdhg_last_error.restype = C.c_char_p
        lib.rhpdhg_config_default.argtypes = [C.POINTER(ConfigC)]
        lib.rhpdhg_config_default.restype = C.c_int
        lib.rhpdhg_set_device.argtypes = [C.c_int]
        lib.rhpdhg_set_device.restype = C.c_int
        lib.rhpdhg_solve_csr.argtypes = [
            C.POINTER(LpView), C.POINTER(ConfigC), C.POINTER(ReportC), c_double_p, c_double_p,
            c_double_p, c_double_p, C.c_int64]
        lib.rhpdhg_solve_csr.restype = C.c_int
        lib.rhpdhg_kkt_residuals.argtypes = [C.POINTER(LpView), c_double_p, c_double_p,
                                             C.POINTER(KktC)]
        lib.rhpdhg_kkt_residuals.restype = C.c_int
        P = C.c_void_p
        sig = {
            "rhpdhg_set_device_options": [C.c_int, C.c_int, C.c_int64],
            "rhpdhg_set_distributed": [C.c_int, C.c_int, C.c_void_p],
            "rhpdhg_set_local_group": [C.c_int, C.c_int, C.c_void_p],
            "rhpdhg_run_benchmark": [C.c_char_p, C.POINTER(ConfigC), C.c_double, C.c_double,
                                     C.c_int, C.c_char_p, C.c_char_p, C.c_int64],
            "rhpdhg_set_resident": [C.c_int],
            "rhpdhg_set_locality": [C.c_int],
            "rhpdhg_session_create": [C.POINTER(LpView), C.POINTER(ConfigC), C.POINTER(P)],
            "rhpdhg_session_advance": [P, C.c_int64, C.POINTER(C.c_int32)],
            "rhpdhg_session_info": [P, c_int64_p, c_int64_p, C.POINTER(KktC), c_double_p,
                                    c_int64_p, c_int64_p],
            "rhpdhg_session_timer": [P, C.c_int, c_double_p],
            "rhpdhg_session_time_kernels": [P, C.c_int, c_double_p],
            "rhpdhg_session_gather_ceiling": [P, C.c_int, c_double_p],
            "rhpdhg_session_layout": [P, c_int64_p],
            "rhpdhg_session_finish": [P, C.POINTER(ReportC), c_double_p, c_double_p, c_double_p,
                                      c_double_p, C.c_int64],
        }
        for name, args in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
        lib.rhpdhg_session_destroy.argtypes = [P]
        lib.rhpdhg_session_destroy.restype = None
        lib.rhpdhg_lp_read_mps.argtypes = [C.c_char_p, C.POINTER(P), C.c_char_p, C.c_int64]
        lib.rhpdhg_lp_read_mps.restype = C.c_int
        lib.rhpdhg_lp_view_of.argtypes = [P, C.POINTER(LpView)]
        lib.rhpdhg_lp_view_of.restype = C.c_int
        lib.rhpdhg_lp_free.argtypes = [P]
        lib.rhpdhg_lp_free.restype = None
        lib._typed = True
    return lib


def default_config() -> ConfigC:
    """SolverConfig defaults (config.hpp:12-40) without needing the library."""
    c = ConfigC()
    c.scaling_enabled = 1
    c.ruiz_iterations = 10
    c.pock_chambolle = 1
    c.restarts_enabled = 1
    c.stepsize_multiplier = 0.99
    c.power_tol = 1e-4
    c.power_max_iters = 5000
    c.power_seed = 0
    c.beta_sufficient = 0.2
    c.beta_necessary = 0.8
    c.beta_artificial = 0.36
    c.reflection_gamma = 1.0
    c.pid_kp = 0.5
    c.pid_ki = 0.0
    c.pid_kd = 0.0
    c.initial_weight = 1.0
    c.epsilon = 1e-4
    c.check_interval = 64
    c.time_limit_seconds = float("inf")
    c.iteration_limit = 2**63 - 1
    c.verbosity = 0
    c.record_residual_history = 0
    return c
