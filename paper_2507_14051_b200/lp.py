"""Python mirror of the reference's solver API (proj/include/rhpdhg).

    LpProblem       <- struct LpProblem      lp_problem.hpp:18-36 (CSR arrays, int64 indices)
    SolverConfig    <- struct SolverConfig   config.hpp:12-40 (same names and defaults)
    SolutionReport  <- struct SolutionReport report.hpp:19-42
    solve()         <- rhpdhg::solve         solver.hpp:13
    kkt_residuals() <- rhpdhg::kkt_residuals termination.hpp:41-42

Every call goes through the C ABI of librhpdhg.so (include/rhpdhg_c.h), i.e.
the C++ host solver driving the CUDA device library. Errors come back as the
reference's exception types (errors.hpp:9-37).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from dataclasses import dataclass, field

import numpy as np

from . import capi

INF = float("inf")


class RhpdhgError(RuntimeError):
    """Base of the exception taxonomy."""


class UsageError(RhpdhgError, ValueError):
    pass


class InvalidProblemError(RhpdhgError):
    pass


class ParseError(RhpdhgError):
    pass


class NumericalBreakdownError(RhpdhgError):
    pass


class DeviceError(RhpdhgError):
    pass


_ERRORS = {
    capi.E_USAGE: UsageError,
    capi.E_INVALID_PROBLEM: InvalidProblemError,
    capi.E_PARSE: ParseError,
    capi.E_BREAKDOWN: NumericalBreakdownError,
    capi.E_DEVICE: DeviceError,
    capi.E_INTERNAL: RhpdhgError,
}


def raise_status(rc: int, msg: str):
    if rc != capi.OK:
        raise _ERRORS.get(rc, RhpdhgError)(msg)


def _f64(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.shape != (n,):
        raise UsageError(f"expected length {n}, got {a.shape}")
    return a


@dataclass
class LpProblem:
    """min c^T x + offset s.t. con_lb <= A x <= con_ub, var_lb <= x <= var_ub.

    A is CSR (row_ptr[m+1], col_index[nnz], values[nnz], int64 indices).
    Maximization instances store the negated objective, like the reference.
    """

    num_cons: int
    num_vars: int
    row_ptr: np.ndarray
    col_index: np.ndarray
    values: np.ndarray
    objective: np.ndarray
    var_lb: np.ndarray
    var_ub: np.ndarray
    con_lb: np.ndarray
    con_ub: np.ndarray
    objective_offset: float = 0.0
    maximization: bool = False
    name: str = ""

    def __post_init__(self):
        m, n = int(self.num_cons), int(self.num_vars)
        self.num_cons, self.num_vars = m, n
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_index = np.ascontiguousarray(self.col_index, dtype=np.int64)
        self.values = _f64(self.values)
        self.objective = _f64(self.objective, n)
        self.var_lb = _f64(self.var_lb, n)
        self.var_ub = _f64(self.var_ub, n)
        self.con_lb = _f64(self.con_lb, m)
        self.con_ub = _f64(self.con_ub, m)
        if self.row_ptr.shape != (m + 1,):
            raise UsageError("row_ptr must have num_cons+1 entries")

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if self.num_cons else 0

    @classmethod
    def from_triplets(cls, m, n, rows, cols, vals, **kw):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        rp = np.zeros(m + 1, dtype=np.int64)
        np.add.at(rp, rows + 1, 1)
        return cls(m, n, np.cumsum(rp), cols, vals, **kw)

    def view(self) -> capi.LpView:
        """Borrowed C view; keep `self` alive while the view is in use."""
        v = capi.LpView()
        v.num_cons = self.num_cons
        v.num_vars = self.num_vars
        v.nnz = self.nnz
        v.row_ptr = self.row_ptr.ctypes.data_as(capi.c_int64_p)
        v.col_index = self.col_index.ctypes.data_as(capi.c_int64_p)
        v.values = self.values.ctypes.data_as(capi.c_double_p)
        v.objective = self.objective.ctypes.data_as(capi.c_double_p)
        v.objective_offset = float(self.objective_offset)
        v.var_lb = self.var_lb.ctypes.data_as(capi.c_double_p)
        v.var_ub = self.var_ub.ctypes.data_as(capi.c_double_p)
        v.con_lb = self.con_lb.ctypes.data_as(capi.c_double_p)
        v.con_ub = self.con_ub.ctypes.data_as(capi.c_double_p)
        v.maximization = 1 if self.maximization else 0
        return v

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.num_cons, self.num_vars))
        for i in range(self.num_cons):
            s, e = self.row_ptr[i], self.row_ptr[i + 1]
            d[i, self.col_index[s:e]] = self.values[s:e]
        return d


@dataclass
class SolverConfig:
    """SolverConfig (config.hpp:12-40) with the shipped defaults."""

    scaling_enabled: bool = True
    ruiz_iterations: int = 10
    pock_chambolle: bool = True
    stepsize_multiplier: float = 0.99
    power_tol: float = 1e-4
    power_max_iters: int = 5000
    power_seed: int = 0
    restarts_enabled: bool = True
    beta_sufficient: float = 0.2
    beta_necessary: float = 0.8
    beta_artificial: float = 0.36
    reflection_gamma: float = 1.0
    pid_kp: float = 0.5
    pid_ki: float = 0.0
    pid_kd: float = 0.0
    initial_weight: float = 1.0
    epsilon: float = 1e-4
    check_interval: int = 64
    time_limit_seconds: float = INF
    iteration_limit: int = 2**63 - 1
    verbosity: int = 0
    record_residual_history: bool = False

    def to_c(self) -> capi.ConfigC:
        c = capi.ConfigC()
        for f in dataclasses.fields(self):
            v = getattr(self, f.name)
            setattr(c, f.name, int(v) if isinstance(v, bool) else v)
        return c


@dataclass
class KktResiduals:
    gap_abs: float = 0.0
    gap_rel: float = 0.0
    primal_inf: float = 0.0
    primal_rel: float = 0.0
    dual_eq: float = 0.0
    dual_cone: float = 0.0
    gap_denom: float = 1.0
    primal_denom: float = 1.0
    dual_denom: float = 1.0

    @classmethod
    def from_c(cls, k: capi.KktC) -> "KktResiduals":
        return cls(**k.as_dict())


@dataclass
class SolutionReport:
    status: str
    x: np.ndarray
    y: np.ndarray
    reduced_costs: np.ndarray
    objective: float
    residuals: KktResiduals
    iterations: int
    restart_count: int
    wall_time_seconds: float
    final_fixed_point_residual: float
    final_primal_weight: float
    matrix_norm_estimate: float
    power_iterations: int
    spmv_loop: int
    spmv_checks: int
    spmv_setup: int
    kkt_checks: int
    inner_residuals: KktResiduals | None
    fixed_point_residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    setup_seconds: float = 0.0
    loop_seconds: float = 0.0
    device_blocks: int = 0


def run_solve_fn(fn, err_fn, lp: LpProblem, cfg: SolverConfig | None = None,
                 history_cap: int = 1 << 20) -> SolutionReport:
    """Calls any function with the rhpdhg_solve_csr signature (the product,
    and in tests the oracle and the reference adapter)."""
    cfg = cfg or SolverConfig()
    rep = capi.ReportC()
    x = np.zeros(lp.num_vars)
    y = np.zeros(lp.num_cons)
    rc_ = np.zeros(lp.num_vars)
    cap = history_cap if cfg.record_residual_history else 0
    hist = np.zeros(max(cap, 1))
    view = lp.view()
    cc = cfg.to_c()
    rc = fn(C.byref(view), C.byref(cc), C.byref(rep), x.ctypes.data_as(capi.c_double_p),
            y.ctypes.data_as(capi.c_double_p), rc_.ctypes.data_as(capi.c_double_p),
            hist.ctypes.data_as(capi.c_double_p), C.c_int64(cap))
    raise_status(rc, (err_fn() or b"").decode(errors="replace"))
    hl = min(int(rep.history_len), cap)
    return SolutionReport(
        status=capi.STATUS_NAMES[rep.status], x=x, y=y, reduced_costs=rc_,
        objective=rep.objective, residuals=KktResiduals.from_c(rep.residuals),
        iterations=rep.iterations, restart_count=rep.restart_count,
        wall_time_seconds=rep.wall_time_seconds,
        final_fixed_point_residual=rep.final_fixed_point_residual,
        final_primal_weight=rep.final_primal_weight,
        matrix_norm_estimate=rep.matrix_norm_estimate, power_iterations=rep.power_iterations,
        spmv_loop=rep.spmv_loop, spmv_checks=rep.spmv_checks, spmv_setup=rep.spmv_setup,
        kkt_checks=rep.kkt_checks,
        inner_residuals=KktResiduals.from_c(rep.inner_residuals) if rep.has_inner_residuals else None,
        fixed_point_residual_history=hist[:hl].copy(),
        setup_seconds=rep.setup_seconds, loop_seconds=rep.loop_seconds,
        device_blocks=rep.device_blocks)


def solve(lp: LpProblem, cfg: SolverConfig | None = None) -> SolutionReport:
    """rhpdhg::solve on the GPU (librhpdhg.so -> librhp_cuda.so)."""
    lib = capi.load_host()
    return run_solve_fn(lib.rhpdhg_solve_csr, lib.rhpdhg_last_error, lp, cfg)


def kkt_residuals(lp: LpProblem, x, y) -> KktResiduals:
    """rhpdhg::kkt_residuals(problem, x, y) with the products on the GPU."""
    lib = capi.load_host()
    x = _f64(x, lp.num_vars)
    y = _f64(y, lp.num_cons)
    out = capi.KktC()
    view = lp.view()
    rc = lib.rhpdhg_kkt_residuals(C.byref(view), x.ctypes.data_as(capi.c_double_p),
                                  y.ctypes.data_as(capi.c_double_p), C.byref(out))
    raise_status(rc, lib.rhpdhg_last_error().decode(errors="replace"))
    return KktResiduals.from_c(out)


def set_device(device: int) -> None:
    lib = capi.load_host()
    raise_status(lib.rhpdhg_set_device(device), lib.rhpdhg_last_error().decode())


def read_mps(path: str) -> tuple[LpProblem, list[str]]:
    """rhpdhg::parse_mps_file (host C++; '.gz' accepted) -> (LpProblem, warnings)."""
    lib = capi.load_host()
    h = C.c_void_p()
    buf = C.create_string_buffer(1 << 16)
    raise_status(lib.rhpdhg_lp_read_mps(str(path).encode(), C.byref(h), buf, len(buf)),
                 lib.rhpdhg_last_error().decode(errors="replace"))
    try:
        v = capi.LpView()
        raise_status(lib.rhpdhg_lp_view_of(h, C.byref(v)), lib.rhpdhg_last_error().decode())
        m, n = v.num_cons, v.num_vars
        nnz = v.row_ptr[m] if m else 0

        def arr(p, k, dt=np.float64):
            return np.ctypeslib.as_array(p, shape=(k,)).astype(dt, copy=True) if k else np.zeros(0, dt)

        lp = LpProblem(m, n, arr(v.row_ptr, m + 1, np.int64), arr(v.col_index, nnz, np.int64),
                       arr(v.values, nnz), arr(v.objective, n), arr(v.var_lb, n),
                       arr(v.var_ub, n), arr(v.con_lb, m), arr(v.con_ub, m),
                       objective_offset=v.objective_offset, maximization=bool(v.maximization))
    finally:
        lib.rhpdhg_lp_free(h)
    warnings = [w for w in buf.value.decode(errors="replace").split("\n") if w]
    return lp, warnings


def write_mps(lp: LpProblem, path: str) -> None:
    """Free-format MPS of an LpProblem (minimisation form as stored; bounds
    written explicitly, two-sided rows as E/L/G + RANGES)."""
    def num(v):
        return repr(float(v))

    m, n = lp.num_cons, lp.num_vars
    lines = [f"NAME {lp.name or 'LP'}", "ROWS", " N OBJ"]
    kinds, rhs, rng = [], [], []
    for i in range(m):
        lo, hi = lp.con_lb[i], lp.con_ub[i]
        if lo == hi:
            kinds.append("E"); rhs.append(lo); rng.append(None)
        elif np.isinf(lo) and np.isinf(hi):
            raise UsageError("free rows have no MPS row sense here")
        elif np.isinf(lo):
            kinds.append("L"); rhs.append(hi); rng.append(None)
        elif np.isinf(hi):
            kinds.append("G"); rhs.append(lo); rng.append(None)
        else:
            kinds.append("G"); rhs.append(lo); rng.append(hi - lo)
        lines.append(f" {kinds[-1]} R{i}")
    cols = [[] for _ in range(n)]
    for i in range(m):
        for e in range(lp.row_ptr[i], lp.row_ptr[i + 1]):
            cols[lp.col_index[e]].append((i, lp.values[e]))
    lines.append("COLUMNS")
    for j in range(n):
        lines.append(f" X{j} OBJ {num(lp.objective[j])}")
        for i, v in cols[j]:
            lines.append(f" X{j} R{i} {num(v)}")
    lines.append("RHS")
    if lp.objective_offset != 0.0:
        lines.append(f" RHS OBJ {num(-lp.objective_offset)}")
    for i in range(m):
        lines.append(f" RHS R{i} {num(rhs[i])}")
    if any(r is not None for r in rng):
        lines.append("RANGES")
        for i in range(m):
            if rng[i] is not None:
                lines.append(f" RNG R{i} {num(rng[i])}")
    lines.append("BOUNDS")
    for j in range(n):
        lo, hi = lp.var_lb[j], lp.var_ub[j]
        if np.isinf(lo) and np.isinf(hi):
            lines.append(f" FR BND X{j}")
            continue
        if np.isinf(lo):
            lines.append(f" MI BND X{j}")
        else:
            lines.append(f" LO BND X{j} {num(lo)}")
        if not np.isinf(hi):
            lines.append(f" UP BND X{j} {num(hi)}")
    lines.append("ENDATA")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def run_benchmark(directory: str, cfg: SolverConfig | None = None,
                  small_limit_seconds: float = 3600.0, large_limit_seconds: float = 18000.0,
                  workers: int = 1, json_path: str | None = None) -> str:
    """rhpdhg::run_benchmark over a directory of *.mps / *.mps.gz on the GPU(s)
    (reference bench.cpp:171-266): returns the per-instance table with the
    SGM10 summary; writes the reference's JSON report to json_path."""
    lib = capi.load_host()
    cc = (cfg or SolverConfig()).to_c()
    buf = C.create_string_buffer(1 << 20)
    raise_status(lib.rhpdhg_run_benchmark(str(directory).encode(), C.byref(cc),
                                          small_limit_seconds, large_limit_seconds, workers,
                                          (json_path or "").encode(), buf, len(buf)),
                 lib.rhpdhg_last_error().decode(errors="replace"))
    return buf.value.decode(errors="replace")


def set_device_options(device: int = 0, use_graph: bool = True, block_limit: int = 64) -> None:
    lib = capi.load_host()
    raise_status(lib.rhpdhg_set_device_options(device, int(use_graph), block_limit),
                 lib.rhpdhg_last_error().decode())


def set_resident(mode: int = -1) -> None:
    """Small-LP cluster-resident device blocks: -1 auto, 0 off, 1 on."""
    lib = capi.load_host()
    raise_status(lib.rhpdhg_set_resident(mode), lib.rhpdhg_last_error().decode())


def set_locality(mode: int = 0) -> None:
    """First-touch row/column relabelling at device ingest: 0 auto, -1 off, 1 forced."""
    lib = capi.load_host()
    raise_status(lib.rhpdhg_set_locality(mode), lib.rhpdhg_last_error().decode())


def nccl_unique_id() -> bytes:
    """rank 0: a fresh 128-byte ncclUniqueId to share with the other ranks."""
    lib = capi.load_cuda()
    buf = C.create_string_buffer(128)
    raise_status(lib.rhp_nccl_unique_id(buf), lib.rhp_last_error().decode(errors="replace"))
    return buf.raw


def set_distributed(rank: int = 0, world_size: int = 1, nccl_id: bytes | None = None) -> None:
    """Row-partitioned multi-GPU solves: this process is `rank` of
    `world_size`; every rank solves the FULL problem with the same config."""
    lib = capi.load_host()
    idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
    raise_status(lib.rhpdhg_set_distributed(rank, world_size, idbuf),
                 lib.rhpdhg_last_error().decode(errors="replace"))


class LocalGroup:
    """In-process collective group (rhp_local_group_create): `world` threads
    of this process, each calling set_local_group(rank, world, group) and
    then solving the same LP, run the row-partitioned engine together; their
    exchanges go through device memory with rank-ordered reductions."""

    def __init__(self, world: int):
        self._lib = capi.load_cuda()
        h = C.c_void_p()
        raise_status(self._lib.rhp_local_group_create(world, C.byref(h)),
                     self._lib.rhp_last_error().decode(errors="replace"))
        self.handle = h
        self.world = world

    def close(self):
        if self.handle:
            self._lib.rhp_local_group_destroy(self.handle)
            self.handle = None


def set_local_group(rank: int, world_size: int, group: "LocalGroup") -> None:
    """This THREAD acts as `rank` of an in-process group (device options are
    per thread)."""
    lib = capi.load_host()
    raise_status(lib.rhpdhg_set_local_group(rank, world_size, group.handle),
                 lib.rhpdhg_last_error().decode(errors="replace"))


def partition_rows(lp: LpProblem, world_size: int) -> np.ndarray:
    """The row partition the multi-GPU path uses (GPU-free host logic)."""
    lib = capi.load_cuda()
    out = np.zeros(world_size + 1, dtype=np.int64)
    view = lp.view()
    raise_status(lib.rhp_partition_rows(C.byref(view), world_size,
                                        out.ctypes.data_as(capi.c_int64_p)),
                 lib.rhp_last_error().decode(errors="replace"))
    return out


class Session:
    """Resumable solve (rhpdhg_session_*): setup in the constructor, then
    advance() in slices of PDHG iterations, then finish() -> SolutionReport."""

    def __init__(self, lp: LpProblem, cfg: SolverConfig | None = None):
        self._lib = capi.load_host()
        self._lp = lp
        self._cfg = cfg or SolverConfig()
        h = C.c_void_p()
        view = lp.view()
        cc = self._cfg.to_c()
        self._check(self._lib.rhpdhg_session_create(C.byref(view), C.byref(cc), C.byref(h)))
        self._h = h

    def _check(self, rc):
        raise_status(rc, self._lib.rhpdhg_last_error().decode(errors="replace"))

    def advance(self, iterations: int) -> bool:
        running = C.c_int32(0)
        self._check(self._lib.rhpdhg_session_advance(self._h, iterations, C.byref(running)))
        return bool(running.value)

    def info(self):
        total, restarts, setup = C.c_int64(), C.c_int64(), C.c_double()
        blocks, checks = C.c_int64(), C.c_int64()
        k = capi.KktC()
        self._check(self._lib.rhpdhg_session_info(self._h, C.byref(total), C.byref(restarts),
                                                  C.byref(k), C.byref(setup), C.byref(blocks),
                                                  C.byref(checks)))
        return {"total": total.value, "restarts": restarts.value, "setup_seconds": setup.value,
                "residuals": KktResiduals.from_c(k), "device_blocks": blocks.value,
                "kkt_checks": checks.value}

    def timer_start(self):
        self._check(self._lib.rhpdhg_session_timer(self._h, 1, None))

    def timer_stop(self) -> float:
        ms = C.c_double()
        self._check(self._lib.rhpdhg_session_timer(self._h, 0, C.byref(ms)))
        return ms.value

    def time_kernels(self, reps: int = 20) -> dict:
        """Average device ms of K1/K2/K3 (mutates the iterate; call last)."""
        ms = (C.c_double * 3)()
        self._check(self._lib.rhpdhg_session_time_kernels(self._h, reps, ms))
        return {"k1_dual_spmv_ms": ms[0], "k2_aty_spmv_primal_ms": ms[1], "k3_primal_ms": ms[2]}

    def gather_ceiling(self, reps: int = 5) -> dict:
        """Best device ms of the pure-gather probe over A and A^T."""
        ms = (C.c_double * 2)()
        self._check(self._lib.rhpdhg_session_gather_ceiling(self._h, reps, ms))
        return {"A": ms[0], "At": ms[1]}

    def layout(self) -> dict:
        o = (C.c_int64 * 35)()
        self._check(self._lib.rhpdhg_session_layout(self._h, o))
        return {"m": o[0], "n": o[1], "nnz": o[2], "row_bins": list(o[3:11]),
                "col_bins": list(o[11:19]), "grid_a": o[19], "grid_at": o[20],
                "grid_vec": o[21], "sm_count": o[22],
                "gather_l1": {"A": bool(o[23] & 1), "At": bool(o[23] & 2)}, "pdl": bool(o[24]),
                "thread_rows": {"A": bool(o[25] & 1), "At": bool(o[25] & 2)},
                "cta_rows": {"A": bool(o[25] & 4)},
                "sliced": {"A": bool(o[25] & 8), "At": bool(o[25] & 16)},
                "uniform_rows": {"A": bool(o[25] & 32), "At": bool(o[25] & 64)},
                "row_band": {"A": bool(o[25] & 128), "At": bool(o[25] & 256)},
                "segments": {"A": int(o[26] & 0xffff), "At": int(o[26] >> 16)},
                "resident": bool(o[27]),
                "partition": {0: "single", 1: "replicated", 2: "sharded"}[int(o[28])],
                "const_bounds": [k for b, k in enumerate(("var_lb", "var_ub", "con_lb", "con_ub"))
                                 if (o[29] >> b) & 1],
                "relabel": bool(o[30]),
                "gather_sectors_per_nnz": [C.cast(C.pointer(C.c_int64(o[31 + k])),
                                                  C.POINTER(C.c_double))[0] for k in range(4)]}

    def finish(self) -> SolutionReport:
        def fn(view, cc, rep, x, y, rc_, hist, cap):
            return self._lib.rhpdhg_session_finish(self._h, rep, x, y, rc_, hist, cap)
        return run_solve_fn(fn, self._lib.rhpdhg_last_error, self._lp, self._cfg)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.rhpdhg_session_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
