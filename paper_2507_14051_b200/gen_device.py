"""GPU-side generator for the billion-nonzero configuration (BASELINE.json
configs[4], C5: "synthetic row-partitioned LP at ~1B nnz").

numpy cannot build a 1B-nonzero CSR in reasonable time or memory (the host
generators sort (row, col) keys), so C5 is generated with torch on the GPU —
benchmark infrastructure, not the product path — and handed to the product as
ordinary host CSR arrays (the e2e path then uploads them through the C ABI
like any other LP).

Distributions follow generators._finish: row lengths
discrete Lomax(alpha=2), mean 20, capped; a_ij ~ U(-2,2); columns of a row of
length L are stratified: one uniformly random column in each of the L integer
bands [floor(k n/L), floor((k+1) n/L)), k < L — strictly
increasing (sorted, no duplicates) and spread over all of x, so the gather
pattern is as random as C2's. Variables: 70% boxed, 20% lower-only, 10% free;
rows 30% equalities, the rest finite two-sided ranges around A x0 for an
interior x0; c = A^T y0 + s sign-matched to the variable type (bounded LP).
All reductions are deterministic (segment sums over sorted keys), so a seed
gives the same LP bit for bit.

    c5_rowpart(seed, m=50M, n=20M)   ~1.0B nonzeros, ~24 GB of device matrices
"""
from __future__ import annotations

import numpy as np

from .lp import LpProblem


def _segment_sum(vals, lengths):
    import torch

    return torch.segment_reduce(vals, "sum", lengths=lengths, unsafe=True)


def c5_rowpart(seed: int = 20240822, m: int = 50_000_000, n: int = 20_000_000,
               mean_row: float = 20.0, cap: int = 10_000, chunk: int = 1 << 27,
               device: str = "cuda") -> LpProblem:
    import torch

    dev = torch.device(device)
    f64, i64 = torch.float64, torch.int64
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    alpha = 2.0
    scale = (mean_row - 0.5) * (alpha - 1.0)
    u = torch.rand(m, generator=g, device=dev, dtype=f64)
    L = (1.0 + torch.floor(scale * (u.pow(-1.0 / alpha) - 1.0))).clamp_(max=float(min(cap, n)))
    L = L.to(i64)
    del u
    rp = torch.zeros(m + 1, dtype=i64, device=dev)
    torch.cumsum(L, 0, out=rp[1:])
    nnz = int(rp[-1])
    # columns and values, in chunks of elements (bounded temporaries)
    ci = torch.empty(nnz, dtype=i64, device=dev)
    v = torch.empty(nnz, dtype=f64, device=dev)
    rows_all = torch.arange(m, device=dev, dtype=i64)
    for s in range(0, nnz, chunk):
        e = min(nnz, s + chunk)
        pos = torch.arange(s, e, device=dev, dtype=i64)
        row = torch.searchsorted(rp, pos, right=True) - 1
        k = pos - rp[row]
        w = float(n) / L[row].to(f64)  # band width >= 1
        kf = k.to(f64)
        lo = torch.floor(kf * w)
        hi = torch.floor((kf + 1.0) * w)  # integer bands [lo, hi): disjoint, non-empty
        uu = torch.rand(e - s, generator=g, device=dev, dtype=f64)
        ci[s:e] = torch.minimum(lo + torch.floor(uu * (hi - lo)), hi - 1.0).to(i64)
        vv = torch.rand(e - s, generator=g, device=dev, dtype=f64) * 4.0 - 2.0
        vv[vv == 0.0] = 1.0
        v[s:e] = vv
        del pos, row, k, w, kf, lo, hi, uu, vv
    del rows_all
    # variables and an interior point
    kind = torch.rand(n, generator=g, device=dev, dtype=f64)
    boxed = kind < 0.7
    lower = (kind >= 0.7) & (kind < 0.9)
    free = ~(boxed | lower)
    lb = torch.rand(n, generator=g, device=dev, dtype=f64) * -3.0
    ub = lb + 0.5 + 4.5 * torch.rand(n, generator=g, device=dev, dtype=f64)
    t1 = 0.2 + 0.6 * torch.rand(n, generator=g, device=dev, dtype=f64)
    t2 = 0.1 + 1.9 * torch.rand(n, generator=g, device=dev, dtype=f64)
    t3 = -2.0 + 4.0 * torch.rand(n, generator=g, device=dev, dtype=f64)
    x0 = torch.where(boxed, lb + t1 * (ub - lb), torch.where(lower, lb + t2, t3))
    var_lb = torch.where(free, torch.full_like(lb, -np.inf), lb)
    var_ub = torch.where(boxed, ub, torch.full_like(ub, np.inf))
    # A x0 (row segment sums) and the row bounds around it
    ax0 = torch.empty(m, dtype=f64, device=dev)
    r0 = 0
    while r0 < m:  # row chunks of about `chunk` elements
        r1 = int(torch.searchsorted(rp, rp[r0] + chunk, right=True)) - 1
        r1 = min(m, max(r1, r0 + 1))
        a, b = int(rp[r0]), int(rp[r1])
        ax0[r0:r1] = _segment_sum(v[a:b] * x0[ci[a:b]], L[r0:r1])
        r0 = r1
    eq = torch.rand(m, generator=g, device=dev, dtype=f64) < 0.3
    lo_s = 0.1 + 1.9 * torch.rand(m, generator=g, device=dev, dtype=f64)
    hi_s = 0.1 + 1.9 * torch.rand(m, generator=g, device=dev, dtype=f64)
    con_lb = torch.where(eq, ax0, ax0 - lo_s)
    con_ub = torch.where(eq, ax0, ax0 + hi_s)
    del lo_s, hi_s, eq
    # c = A^T y0 + s: column segment sums over a stable sort by column
    y0 = torch.rand(m, generator=g, device=dev, dtype=f64) * 2.0 - 1.0
    order = torch.argsort(ci, stable=True)
    col_cnt = torch.bincount(ci, minlength=n)
    row_of = torch.searchsorted(rp, order, right=True) - 1
    aty0 = _segment_sum(v[order] * y0[row_of], col_cnt)
    del order, row_of
    s_b = torch.rand(n, generator=g, device=dev, dtype=f64) * 2.0 - 1.0
    s_l = torch.rand(n, generator=g, device=dev, dtype=f64)
    c = aty0 + torch.where(boxed, s_b, torch.where(lower, s_l, torch.zeros_like(s_l)))
    host = {k: t.cpu().numpy() for k, t in
            dict(rp=rp, ci=ci, v=v, c=c, var_lb=var_lb, var_ub=var_ub, con_lb=con_lb,
                 con_ub=con_ub).items()}
    del rp, ci, v
    torch.cuda.empty_cache()
    return LpProblem(m, n, host["rp"], host["ci"], host["v"], host["c"], host["var_lb"],
                     host["var_ub"], host["con_lb"], host["con_ub"], name="c5_rowpart")
