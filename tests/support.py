"""Test infrastructure: loaders for the checkers (oracle/liboracle.so, my C
restatement; oracle/_ref/librhpdhg_ref.so, the reference compiled from its
own sources) and for the committed golden fixtures under tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from pathlib import Path

import numpy as np

from paper_2507_14051_b200 import capi
from paper_2507_14051_b200.lp import LpProblem, SolverConfig, run_solve_fn

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "librhpdhg_ref.so"
GOLDEN = ROOT / "tests" / "golden"

_libs: dict[str, C.CDLL] = {}

D = capi.c_double_p


def _type_common(lib, prefix):
    getattr(lib, f"{prefix}_last_error").restype = C.c_char_p
    lib.__dict__["_prefix"] = prefix
    solve = getattr(lib, f"{prefix}_solve_csr")
    solve.argtypes = [C.POINTER(capi.LpView), C.POINTER(capi.ConfigC), C.POINTER(capi.ReportC),
                      D, D, D, D, C.c_int64]
    solve.restype = C.c_int
    spmv = getattr(lib, f"{prefix}_spmv")
    spmv.argtypes = [C.POINTER(capi.LpView), D, D, C.c_int]
    spmv.restype = C.c_int
    scale = getattr(lib, f"{prefix}_scale")
    scale.argtypes = [C.POINTER(capi.LpView), C.c_int, C.c_int] + [D] * 9
    scale.restype = C.c_int
    pw = getattr(lib, f"{prefix}_power_iteration")
    pw.argtypes = [C.POINTER(capi.LpView), C.c_double, C.c_int64, C.c_uint64, D,
                   C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    pw.restype = C.c_int
    kk = getattr(lib, f"{prefix}_kkt_residuals")
    kk.argtypes = [C.POINTER(capi.LpView), D, D, C.POINTER(capi.KktC)]
    kk.restype = C.c_int


def oracle():
    if "orc" not in _libs:
        if not ORACLE_SO.exists():
            raise RuntimeError(f"{ORACLE_SO} missing: run `make oracle`")
        lib = C.CDLL(str(ORACLE_SO))
        _type_common(lib, "orc")
        lib.orc_power_start.argtypes = [C.c_int64, C.c_uint64, D]
        lib.orc_power_start.restype = None
        lib.orc_solve_snapshots.argtypes = [C.POINTER(capi.LpView), C.POINTER(capi.ConfigC),
                                            C.POINTER(capi.ReportC), capi.c_int64_p, C.c_int,
                                            D, D]
        lib.orc_solve_snapshots.restype = C.c_int
        _libs["orc"] = lib
    return _libs["orc"]


def ref_available() -> bool:
    return REF_SO.exists()


def ref():
    if "ref" not in _libs:
        if not REF_SO.exists():
            raise RuntimeError(f"{REF_SO} missing: run `make ref` where /root/reference exists")
        lib = C.CDLL(str(REF_SO))
        _type_common(lib, "ref")
        lib.ref_lp_from_mps.argtypes = [C.c_char_p]
        lib.ref_lp_from_mps.restype = C.c_void_p
        lib.ref_lp_random_feasible.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_double]
        lib.ref_lp_random_feasible.restype = C.c_void_p
        lib.ref_lp_dims.argtypes = [C.c_void_p] + [C.POINTER(C.c_int64)] * 3
        lib.ref_lp_dims.restype = None
        lib.ref_lp_export.argtypes = [C.c_void_p, capi.c_int64_p, capi.c_int64_p, D, D, D, D, D,
                                      D, D, C.POINTER(C.c_int32)]
        lib.ref_lp_export.restype = None
        lib.ref_lp_free.argtypes = [C.c_void_p]
        lib.ref_lp_free.restype = None
        lib.ref_session_create.argtypes = [C.POINTER(capi.LpView), C.POINTER(capi.ConfigC)]
        lib.ref_session_create.restype = C.c_void_p
        lib.ref_session_advance.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int32), D,
                                            C.POINTER(C.c_int64)]
        lib.ref_session_advance.restype = C.c_int
        lib.ref_session_setup_seconds.argtypes = [C.c_void_p]
        lib.ref_session_setup_seconds.restype = C.c_double
        lib.ref_session_free.argtypes = [C.c_void_p]
        lib.ref_session_free.restype = None
        lib.ref_session_iterate.argtypes = [C.c_void_p, D, D]
        lib.ref_session_iterate.restype = C.c_int
        _libs["ref"] = lib
    return _libs["ref"]


def _err(lib):
    return getattr(lib, f"{lib._prefix}_last_error")


def check(lib, rc):
    if rc != 0:
        raise RuntimeError(f"{lib._prefix}: status {rc}: {_err(lib)().decode(errors='replace')}")


def solve_with(lib, lp: LpProblem, cfg: SolverConfig | None = None):
    return run_solve_fn(getattr(lib, f"{lib._prefix}_solve_csr"), _err(lib), lp, cfg)


def spmv_with(lib, lp: LpProblem, vec, transpose=False):
    out = np.zeros(lp.num_vars if transpose else lp.num_cons)
    v = np.ascontiguousarray(vec, dtype=np.float64)
    view = lp.view()
    check(lib, getattr(lib, f"{lib._prefix}_spmv")(C.byref(view), v.ctypes.data_as(D),
                                                   out.ctypes.data_as(D), int(transpose)))
    return out


def scale_with(lib, lp: LpProblem, ruiz=10, pc=True):
    m, n, nz = lp.num_cons, lp.num_vars, lp.nnz
    out = {k: np.zeros(s) for k, s in (("csr", nz), ("csc", nz), ("row_scale", m),
                                        ("col_scale", n), ("c", n), ("var_lb", n), ("var_ub", n),
                                        ("con_lb", m), ("con_ub", m))}
    view = lp.view()
    check(lib, getattr(lib, f"{lib._prefix}_scale")(
        C.byref(view), ruiz, int(pc), *[out[k].ctypes.data_as(D) for k in
                                        ("csr", "csc", "row_scale", "col_scale", "c", "var_lb",
                                         "var_ub", "con_lb", "con_ub")]))
    return out


def power_with(lib, lp: LpProblem, tol=1e-4, max_iters=5000, seed=0):
    val, its, conv = C.c_double(), C.c_int64(), C.c_int32()
    view = lp.view()
    check(lib, getattr(lib, f"{lib._prefix}_power_iteration")(
        C.byref(view), tol, max_iters, seed, C.byref(val), C.byref(its), C.byref(conv)))
    return val.value, its.value, bool(conv.value)


def kkt_with(lib, lp: LpProblem, x, y):
    out = capi.KktC()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    view = lp.view()
    check(lib, getattr(lib, f"{lib._prefix}_kkt_residuals")(
        C.byref(view), x.ctypes.data_as(D), y.ctypes.data_as(D), C.byref(out)))
    return out.as_dict()


def oracle_snapshots(lp: LpProblem, cfg: SolverConfig, ks):
    """Unscaled iterates (x, y) after each iteration count in ks, from ONE
    oracle solve (orc_solve_snapshots; OpenMP row-parallel products, results
    bit-identical to the sequential oracle)."""
    lib = oracle()
    ks = np.ascontiguousarray(ks, dtype=np.int64)
    xs = np.zeros((len(ks), lp.num_vars))
    ys = np.zeros((len(ks), lp.num_cons))
    view = lp.view()
    cc = cfg.to_c()
    rep = capi.ReportC()
    check(lib, lib.orc_solve_snapshots(C.byref(view), C.byref(cc), C.byref(rep),
                                       ks.ctypes.data_as(capi.c_int64_p), len(ks),
                                       xs.ctypes.data_as(D), ys.ctypes.data_as(D)))
    return xs, ys


def ref_lp_from_handle(h) -> LpProblem:
    lib = ref()
    if not h:
        raise RuntimeError(_err(lib)().decode())
    m, n, nz = C.c_int64(), C.c_int64(), C.c_int64()
    lib.ref_lp_dims(h, C.byref(m), C.byref(n), C.byref(nz))
    m, n, nz = m.value, n.value, nz.value
    rp = np.zeros(m + 1, dtype=np.int64)
    ci = np.zeros(nz, dtype=np.int64)
    v = np.zeros(nz)
    c = np.zeros(n)
    vl, vu, cl, cu = np.zeros(n), np.zeros(n), np.zeros(m), np.zeros(m)
    off = C.c_double()
    mx = C.c_int32()
    lib.ref_lp_export(h, rp.ctypes.data_as(capi.c_int64_p), ci.ctypes.data_as(capi.c_int64_p),
                      v.ctypes.data_as(D), c.ctypes.data_as(D), C.byref(off), vl.ctypes.data_as(D),
                      vu.ctypes.data_as(D), cl.ctypes.data_as(D), cu.ctypes.data_as(D),
                      C.byref(mx))
    lib.ref_lp_free(h)
    return LpProblem(m, n, rp, ci, v, c, vl, vu, cl, cu, objective_offset=off.value,
                     maximization=bool(mx.value))


class RefSession:
    """The reference's solve loop advanced in slices (oracle/ref_adapter.cpp)."""

    def __init__(self, lp: LpProblem, cfg: SolverConfig):
        self.lib = ref()
        self._lp = lp
        view = lp.view()
        cc = cfg.to_c()
        self.h = self.lib.ref_session_create(C.byref(view), C.byref(cc))
        if not self.h:
            raise RuntimeError(self.lib.ref_last_error().decode(errors="replace"))
        self.setup_seconds = self.lib.ref_session_setup_seconds(self.h)

    def advance(self, iters: int):
        running, secs, total = C.c_int32(), C.c_double(), C.c_int64()
        check(self.lib, self.lib.ref_session_advance(self.h, iters, C.byref(running),
                                                     C.byref(secs), C.byref(total)))
        return bool(running.value), secs.value, total.value

    def iterate(self):
        """Current Halpern iterate in original space (x, y)."""
        x = np.zeros(self._lp.num_vars)
        y = np.zeros(self._lp.num_cons)
        check(self.lib, self.lib.ref_session_iterate(self.h, x.ctypes.data_as(D),
                                                     y.ctypes.data_as(D)))
        return x, y

    def close(self):
        if self.h:
            self.lib.ref_session_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


# ------------------------------------------------------------------ golden --
def lp_to_json(lp: LpProblem) -> dict:
    return {
        "m": lp.num_cons, "n": lp.num_vars, "row_ptr": lp.row_ptr.tolist(),
        "col_index": lp.col_index.tolist(), "values": lp.values.tolist(),
        "objective": lp.objective.tolist(), "offset": lp.objective_offset,
        "var_lb": lp.var_lb.tolist(), "var_ub": lp.var_ub.tolist(),
        "con_lb": lp.con_lb.tolist(), "con_ub": lp.con_ub.tolist(),
        "maximization": lp.maximization, "name": lp.name,
    }


def lp_from_json(d: dict) -> LpProblem:
    return LpProblem(d["m"], d["n"], d["row_ptr"], d["col_index"], d["values"], d["objective"],
                     d["var_lb"], d["var_ub"], d["con_lb"], d["con_ub"],
                     objective_offset=d["offset"], maximization=d["maximization"],
                     name=d.get("name", ""))


def load_golden(name: str) -> dict:
    with open(GOLDEN / name) as f:
        return json.load(f)


def report_summary(r) -> dict:
    return {
        "status": r.status, "objective": r.objective, "iterations": r.iterations,
        "restart_count": r.restart_count, "kkt_checks": r.kkt_checks,
        "final_primal_weight": r.final_primal_weight,
        "matrix_norm_estimate": r.matrix_norm_estimate,
        "power_iterations": r.power_iterations, "spmv_loop": r.spmv_loop,
        "spmv_checks": r.spmv_checks, "spmv_setup": r.spmv_setup,
        "final_fixed_point_residual": r.final_fixed_point_residual,
        "residuals": vars(r.residuals).copy(),
        "x": r.x.tolist(), "y": r.y.tolist(),
    }


def have_gpu() -> bool:
    if os.environ.get("RHPDHG_FORCE_NO_GPU"):
        return False
    try:
        lib = capi.load_cuda()
    except Exception:
        return False
    cnt = C.c_int(0)
    return lib.rhp_device_count(C.byref(cnt)) == 0 and cnt.value > 0
