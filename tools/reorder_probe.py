"""Probe: does a locality relabelling of rows/columns speed up the loop?

Builds a config's LP, relabels its columns (and optionally rows) in
first-touch order (numpy, host), and times the device loop (iter/s, K1/K2,
gather ceiling) on the original and the relabelled LP. Experiment driver,
not product code.

  python tools/reorder_probe.py c4 [passes...]
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2507_14051_b200 import generators  # noqa: E402
from paper_2507_14051_b200.lp import LpProblem, Session, SolverConfig, set_device_options  # noqa: E402


def first_touch(idx, size):
    """label[j] = rank of index j by its first position in idx (unseen last)."""
    first = np.full(size, np.iinfo(np.int64).max, np.int64)
    pos = np.arange(len(idx), dtype=np.int64)
    # positions are increasing: the first write per index wins if we go in reverse
    first[idx[::-1]] = pos[::-1]
    order = np.argsort(first, kind="stable")
    lab = np.empty(size, np.int64)
    lab[order] = np.arange(size)
    return lab


def relabel(lp, passes):
    m, n = lp.num_cons, lp.num_vars
    rp = np.asarray(lp.row_ptr, np.int64)
    ci = np.asarray(lp.col_index, np.int64)
    v = np.asarray(lp.values)
    rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(rp))
    cperm = np.arange(n)  # new label of original column
    rperm = np.arange(m)
    for p in passes:
        if p == "c":
            lab = first_touch(ci, n)
            ci = lab[ci]
            cperm = lab[cperm]
        elif p == "r":
            # first touch of rows scanning columns in (new) column order
            o = np.argsort(ci, kind="stable")
            rl = first_touch(rows[o], m)
            rows = rl[rows]
            rperm = rl[rperm]
            o2 = np.argsort(rows, kind="stable")  # keeps element order inside a row
            rows, ci, v = rows[o2], ci[o2], v[o2]
    o3 = np.lexsort((ci, rows))  # columns ascending inside a row (CSR validation)
    rows, ci, v = rows[o3], ci[o3], v[o3]
    rp2 = np.zeros(m + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=m), out=rp2[1:])
    cinv = np.empty(n, np.int64)
    cinv[cperm] = np.arange(n)
    rinv = np.empty(m, np.int64)
    rinv[rperm] = np.arange(m)
    return LpProblem(m, n, rp2, ci, v, np.asarray(lp.objective)[cinv], np.asarray(lp.var_lb)[cinv],
                     np.asarray(lp.var_ub)[cinv], np.asarray(lp.con_lb)[rinv],
                     np.asarray(lp.con_ub)[rinv], name=lp.name + "_ft")


def timeit(lp, steps=10, warm=3):
    s = Session(lp, SolverConfig(epsilon=1e-300))
    lay = s.layout()
    for _ in range(warm):
        s.advance(64)
    a = s.info()["total"]
    s.timer_start()
    for _ in range(steps):
        s.advance(64)
    ms = s.timer_stop()
    it = s.info()["total"] - a
    gc = s.gather_ceiling(reps=5)
    kt = s.time_kernels(reps=10)
    s.close()
    return {"iter_s": it / (ms / 1e3), "k1_us": kt["k1_dual_spmv_ms"] * 1e3,
            "k2_us": kt["k2_aty_spmv_primal_ms"] * 1e3, "k3_us": kt["k3_primal_ms"] * 1e3,
            "gc_a_us": gc["A"] * 1e3, "gc_at_us": gc["At"] * 1e3,
            "segments": lay.get("segments"), "row_band": lay.get("row_band"),
            "thread_rows": lay.get("thread_rows")}


def main():
    cfg = sys.argv[1]
    variants = sys.argv[2:] or ["", "c", "cr", "crcr"]
    set_device_options(0, True, 64)
    lp = generators.CONFIGS[cfg]()
    for var in variants:
        t = time.perf_counter()
        l2 = relabel(lp, list(var)) if var else lp
        tr = time.perf_counter() - t
        r = timeit(l2)
        r["variant"] = var or "orig"
        r["relabel_s"] = tr
        print(json.dumps(r), flush=True)
        del l2


if __name__ == "__main__":
    main()
