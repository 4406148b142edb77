"""SpMV engine probe (run on the GPU box): device time of plain A x and A^T y
for matrices that differ only in row-length distribution and column
locality, reported against their streamed bytes (12 B/nnz + row pointers +
vectors) and the MEASURED_PEAKS HBM figure.

    python tools/spmv_probe.py [--out gpurun_out/spmv_probe.json]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2507_14051_b200 import LpProblem  # noqa: E402
from paper_2507_14051_b200.device import DeviceContext  # noqa: E402
from paper_2507_14051_b200.generators import _csr_from_rows, c2_powerlaw, c3_transport, lomax_lengths  # noqa: E402


def lp_from_csr(m, n, rp, ci, v):
    return LpProblem(m, n, rp, ci, v, np.zeros(n), np.full(n, -np.inf), np.full(n, np.inf),
                     np.zeros(m), np.zeros(m))


def make(kind, m=500_000, n=1_000_000, seed=3):
    rng = np.random.default_rng(seed)
    if kind == "c2":
        return c2_powerlaw()
    if kind == "c3":
        return c3_transport()
    L = lomax_lengths(rng, m) if "pow" in kind else np.full(m, 20, dtype=np.int64)
    row_of = np.repeat(np.arange(m, dtype=np.int64), L)
    if "rand" in kind:
        col = rng.integers(0, n, row_of.size)
    else:  # banded: columns near 2*i (perfect gather locality)
        col = (2 * row_of + rng.integers(0, 64, row_of.size)) % n
    rp, ci, v = _csr_from_rows(m, n, row_of, col, rng.uniform(-2, 2, row_of.size))
    return lp_from_csr(m, n, rp, ci, v)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    ap.add_argument("--kinds", default="c2,pow_rand,uni_rand,pow_band,uni_band,c3")
    a = ap.parse_args()
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    res = []
    for kind in a.kinds.split(","):
        lp = make(kind)
        m, n, nnz = lp.num_cons, lp.num_vars, lp.nnz
        with DeviceContext(lp) as dev:
            dev.spmv(np.ones(n))  # warm
            t_ax = dev.time_spmv(False, 20)
            t_aty = dev.time_spmv(True, 20)
            lay = dev.layout()
        b_ax = 12 * nnz + 8 * (m + 1) + 8 * n + 8 * m
        b_aty = 12 * nnz + 8 * (n + 1) + 8 * m + 8 * n
        r = {"kind": kind, "m": m, "n": n, "nnz": nnz, "ax_us": t_ax * 1e3,
             "ax_gbs": b_ax / t_ax / 1e6, "aty_us": t_aty * 1e3, "aty_gbs": b_aty / t_aty / 1e6,
             "ax_frac": b_ax / t_ax / 1e6 / peak, "aty_frac": b_aty / t_aty / 1e6 / peak,
             "grid_a": lay["grid_a"], "grid_at": lay["grid_at"]}
        print(json.dumps(r), flush=True)
        res.append(r)
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
