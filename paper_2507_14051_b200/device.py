"""Python handle on one device context (include/rhpdhg_cuda.h): the per-op
surface used by the parity tests and the kernel benchmarks."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from .lp import LpProblem, raise_status

D = capi.c_double_p


def _p(a):
    return a.ctypes.data_as(D)


class DeviceContext:
    def __init__(self, lp: LpProblem, device: int = 0, use_graph: bool = True,
                 block_limit: int = 64, resident: int = 0, locality: int = -1):
        self.lib = capi.load_cuda()
        self.lp = lp
        opt = capi.RhpOptions(device=device, rank=0, world_size=1, use_graph=int(use_graph),
                              block_limit=block_limit, nccl_id=None, resident=resident,
                              locality=locality)
        h = C.c_void_p()
        self._view = lp.view()
        self._ok(self.lib.rhp_create(C.byref(self._view), C.byref(opt), C.byref(h)))
        self.h = h

    def _ok(self, rc):
        raise_status(rc, self.lib.rhp_last_error().decode(errors="replace"))

    def close(self):
        if getattr(self, "h", None):
            self.lib.rhp_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- operators ------------------------------------------------------------
    def spmv(self, vec, transpose=False):
        v = np.ascontiguousarray(vec, dtype=np.float64)
        out = np.zeros(self.lp.num_vars if transpose else self.lp.num_cons)
        self._ok(self.lib.rhp_spmv(self.h, int(transpose), _p(v), _p(out)))
        return out

    def layout(self):
        info = capi.RhpLayoutInfo()
        self._ok(self.lib.rhp_layout(self.h, C.byref(info)))
        return {"m_local": info.m_local, "n": info.n, "nnz_local": info.nnz_local,
                "row_bins": list(info.row_bins), "col_bins": list(info.col_bins),
                "grid_a": info.grid_a, "grid_at": info.grid_at, "grid_vec": info.grid_vec,
                "sm_count": info.sm_count,
                "gather_l1": {"A": bool(info.gather_l1 & 1), "At": bool(info.gather_l1 & 2)},
                "pdl": bool(info.pdl),
                "thread_rows": {"A": bool(info.thread_rows & 1), "At": bool(info.thread_rows & 2)},
                "sliced": {"A": bool(info.thread_rows & 8), "At": bool(info.thread_rows & 16)},
                "uniform_rows": {"A": bool(info.thread_rows & 32),
                                 "At": bool(info.thread_rows & 64)},
                "row_band": {"A": bool(info.thread_rows & 128), "At": bool(info.thread_rows & 256)},
                "segments": {"A": info.segments & 0xffff, "At": info.segments >> 16},
                "resident": bool(info.resident),
                "const_bounds": [k for b, k in enumerate(("var_lb", "var_ub", "con_lb", "con_ub"))
                                 if (info.const_bounds >> b) & 1],
                "relabel": bool(info.relabel), "sectors": list(info.sectors)}

    def scale(self, enabled=True, ruiz=10, pock_chambolle=True):
        self._ok(self.lib.rhp_scale(self.h, int(enabled), ruiz, int(pock_chambolle)))

    def get_scaled(self):
        lp = self.lp
        m, n, nz = lp.num_cons, lp.num_vars, lp.nnz
        out = {k: np.zeros(s) for k, s in (("csr", nz), ("csc", nz), ("row_scale", m),
                                            ("col_scale", n), ("c", n), ("var_lb", n),
                                            ("var_ub", n), ("con_lb", m), ("con_ub", m))}
        so = capi.RhpScaledOut(*[_p(out[k]) for k in ("csr", "csc", "row_scale", "col_scale",
                                                       "c", "var_lb", "var_ub", "con_lb",
                                                       "con_ub")])
        self._ok(self.lib.rhp_get_scaled(self.h, C.byref(so)))
        return out

    def power_begin(self, v0):
        v = np.ascontiguousarray(v0, dtype=np.float64)
        self._ok(self.lib.rhp_power_begin(self.h, _p(v)))

    def power_step(self):
        vw, ww = C.c_double(), C.c_double()
        self._ok(self.lib.rhp_power_step(self.h, C.byref(vw), C.byref(ww)))
        return vw.value, ww.value

    def power_normalize(self, wn):
        self._ok(self.lib.rhp_power_normalize(self.h, wn))

    def set_step(self, **kw):
        self._ok(self.lib.rhp_set_step(self.h, C.byref(capi.RhpStep(**kw))))

    def reset_iterate(self):
        self._ok(self.lib.rhp_reset_iterate(self.h))

    def set_iterate(self, x, y):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        self._ok(self.lib.rhp_set_iterate(self.h, _p(x), _p(y)))

    def run_block(self):
        out = capi.RhpBlockOut()
        self._ok(self.lib.rhp_run_block(self.h, C.byref(out)))
        return {n: getattr(out, n) for n, _ in capi.RhpBlockOut._fields_ if n != "pad_"}

    def kkt(self, which=0):
        s = capi.RhpKktSums()
        self._ok(self.lib.rhp_kkt(self.h, which, C.byref(s)))
        return {n: getattr(s, n) for n, _ in capi.RhpKktSums._fields_}

    def kkt_of(self, x, y):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        s = capi.RhpKktSums()
        self._ok(self.lib.rhp_kkt_of(self.h, _p(x), _p(y), C.byref(s)))
        return {n: getattr(s, n) for n, _ in capi.RhpKktSums._fields_}

    def fetch_iterate(self):
        lp = self.lp
        x, y, ax, aty = (np.zeros(lp.num_vars), np.zeros(lp.num_cons), np.zeros(lp.num_cons),
                         np.zeros(lp.num_vars))
        self._ok(self.lib.rhp_fetch_iterate(self.h, _p(x), _p(y), _p(ax), _p(aty)))
        return x, y, ax, aty

    def restart(self):
        self._ok(self.lib.rhp_restart(self.h))

    def timer_start(self):
        self._ok(self.lib.rhp_timer(self.h, 1, None))

    def timer_stop(self) -> float:
        ms = C.c_double()
        self._ok(self.lib.rhp_timer(self.h, 0, C.byref(ms)))
        return ms.value

    def time_spmv(self, transpose=False, reps=20) -> float:
        ms = C.c_double()
        self._ok(self.lib.rhp_time_spmv(self.h, int(transpose), reps, C.byref(ms)))
        return ms.value

    def last_block_ms(self) -> float:
        ms = C.c_double()
        self._ok(self.lib.rhp_last_block_ms(self.h, C.byref(ms)))
        return ms.value


def device_info(device: int = 0) -> dict:
    lib = capi.load_cuda()
    info = capi.RhpDeviceInfo()
    raise_status(lib.rhp_get_device_info(device, C.byref(info)),
                 lib.rhp_last_error().decode(errors="replace"))
    return {"name": info.name.decode(), "sm_count": info.sm_count,
            "cc": f"{info.cc_major}.{info.cc_minor}", "l2_bytes": info.l2_bytes,
            "mem_bytes": info.mem_bytes, "graph_supported": bool(info.graph_supported)}
