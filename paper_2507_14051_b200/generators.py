"""Seeded synthetic LP generators for the BASELINE.json configurations.

Shapes and value distributions follow BASELINE.md §3 / SURVEY.md §8(d):
a_ij ~ U(-2,2); variables a mix of boxed (l ~ U(-3,0), u = l + U(0.5,5)),
lower-only and free; rows are equalities or FINITE two-sided ranges placed
around A x0 for an interior x0 (one-sided rows trip the reference's +inf
duality-gap defect); c = A^T y0 + s with s sign-matched
to the variable type so the LP is dual feasible (bounded).

    c1_small(seed)            m=1k, n=2k, ~10k nnz
    c2_powerlaw(seed, scale)  m=500k, n=1M, ~10M nnz, Lomax(alpha=2) row lengths
    c3_transport(seed, S, T)  S supplies x T demands, n=S*T, nnz=2n (rows of length T and S)
    c4_multicommodity(...)    K commodities on a random graph, conservation
                              equalities + [0, cap] capacity rows
    c5_rowpart(...)           m=50M, n=20M, ~1B nnz (GPU-generated, gen_device.py)
Generation is vectorised numpy with numpy.random.Generator(PCG64(seed)).
"""
from __future__ import annotations

import numpy as np

from .lp import LpProblem

INF = np.inf


def _csr_from_rows(m, n, row_of, col_of, vals):
    """CSR with columns sorted inside rows and duplicate (row, col) dropped."""
    key = row_of.astype(np.int64) * n + col_of.astype(np.int64)
    order = np.argsort(key, kind="stable")
    key = key[order]
    keep = np.ones(key.shape[0], dtype=bool)
    keep[1:] = key[1:] != key[:-1]
    key = key[keep]
    vals = vals[order][keep]
    rows = key // n
    cols = key % n
    rp = np.zeros(m + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    return np.cumsum(rp), cols.astype(np.int64), vals.astype(np.float64)


def _spmv(rp, ci, v, x, m):
    rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(rp))
    return np.bincount(rows, weights=v * x[ci], minlength=m)


def _spmv_t(rp, ci, v, y, m, n):
    rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(rp))
    return np.bincount(ci, weights=v * y[rows], minlength=n)


def _finish(rng, m, n, rp, ci, v, frac_boxed=0.7, frac_lower=0.2, frac_eq=0.3, name=""):
    kind = rng.random(n)
    boxed = kind < frac_boxed
    lower = (kind >= frac_boxed) & (kind < frac_boxed + frac_lower)
    free = ~(boxed | lower)
    lb = rng.uniform(-3.0, 0.0, n)
    ub = lb + rng.uniform(0.5, 5.0, n)
    x0 = np.where(boxed, lb + rng.uniform(0.2, 0.8, n) * (ub - lb),
                  np.where(lower, lb + rng.uniform(0.1, 2.0, n), rng.uniform(-2.0, 2.0, n)))
    var_lb = np.where(free, -INF, lb)
    var_ub = np.where(boxed, ub, INF)
    ax0 = _spmv(rp, ci, v, x0, m)
    eq = rng.random(m) < frac_eq
    con_lb = np.where(eq, ax0, ax0 - rng.uniform(0.1, 2.0, m))
    con_ub = np.where(eq, ax0, ax0 + rng.uniform(0.1, 2.0, m))
    y0 = rng.uniform(-1.0, 1.0, m)
    s = np.where(boxed, rng.uniform(-1.0, 1.0, n), np.where(lower, rng.uniform(0.0, 1.0, n), 0.0))
    c = _spmv_t(rp, ci, v, y0, m, n) + s
    return LpProblem(m, n, rp, ci, v, c, var_lb, var_ub, con_lb, con_ub, name=name)


def random_rows_lp(seed: int, m: int, n: int, row_lengths: np.ndarray, name: str = "",
                   **kw) -> LpProblem:
    rng = np.random.default_rng(seed)
    L = np.minimum(np.asarray(row_lengths, dtype=np.int64), n)
    row_of = np.repeat(np.arange(m, dtype=np.int64), L)
    col_of = rng.integers(0, n, size=row_of.shape[0], dtype=np.int64)
    vals = rng.uniform(-2.0, 2.0, row_of.shape[0])
    vals[vals == 0.0] = 1.0
    rp, ci, v = _csr_from_rows(m, n, row_of, col_of, vals)
    return _finish(rng, m, n, rp, ci, v, name=name, **kw)


def c1_small(seed: int = 20240818, m: int = 1000, n: int = 2000, per_row: int = 10) -> LpProblem:
    """C1: m=1k, n=2k, ~10k nnz, equality/two-sided rows."""
    return random_rows_lp(seed, m, n, np.full(m, per_row), name="c1_small")


def lomax_lengths(rng, m, mean=20.0, alpha=2.0, cap=100_000):
    """Discrete Lomax (Pareto II) lengths >= 1 with the given mean and tail."""
    scale = (mean - 0.5) * (alpha - 1.0)
    u = rng.random(m)
    L = 1 + np.floor(scale * (u ** (-1.0 / alpha) - 1.0))
    return np.minimum(L, cap).astype(np.int64)


def c2_powerlaw(seed: int = 20240819, m: int = 500_000, n: int = 1_000_000,
                mean_row: float = 20.0) -> LpProblem:
    """C2: MIPLIB-relaxation-like, power-law (alpha=2) row lengths, ~10M nnz."""
    rng = np.random.default_rng(seed + 7)
    L = lomax_lengths(rng, m, mean=mean_row, cap=min(100_000, n))
    return random_rows_lp(seed, m, n, L, name="c2_powerlaw")


def c3_transport(seed: int = 20240820, S: int = 1000, T: int = 1000) -> LpProblem:
    """C3: balanced transportation LP, x_st >= 0, supply and demand equalities."""
    rng = np.random.default_rng(seed)
    n, m = S * T, S + T
    supply = rng.uniform(1.0, 100.0, S)
    demand = rng.uniform(1.0, 100.0, T)
    demand *= supply.sum() / demand.sum()
    # row s: columns s*T .. s*T+T-1 ; row S+t: columns t, T+t, ...
    rp = np.concatenate([np.arange(0, S * T, T, dtype=np.int64),
                         S * T + np.arange(0, S * T + 1, S, dtype=np.int64)])
    ci = np.concatenate([np.arange(S * T, dtype=np.int64),
                         (np.arange(S, dtype=np.int64)[None, :] * T +
                          np.arange(T, dtype=np.int64)[:, None]).ravel()])
    v = np.ones(2 * n)
    c = rng.uniform(1.0, 100.0, n)
    rhs = np.concatenate([supply, demand])
    return LpProblem(m, n, rp, ci, v, c, np.zeros(n), np.full(n, INF), rhs, rhs.copy(),
                     name="c3_transport")


def c4_multicommodity(seed: int = 20240821, V: int = 200_000, E: int = 1_000_000,
                      K: int = 25, terminals: int = 40) -> LpProblem:
    """C4: K-commodity min-cost flow with shared arc and node capacities.

    Random directed graph: V nodes, E arcs (a Hamiltonian cycle + E-V random
    arcs). Variables x_ke >= 0, n = K*E, commodity-major (column k*E + e).
    Rows (m = K*V + E + V, nnz = 4*K*E):
      * conservation per (k, v): sum_{e out of v} x_ke - sum_{e into v} x_ke = b_kv
        (equality); commodity k has `terminals` sources and as many sinks with
        supplies U(1,10), balanced;
      * joint arc capacity per arc e: 0 <= sum_k x_ke <= cap_e, with
        cap_e ~ U(1,6) on the random arcs (tight: they bind) and the total
        demand on the cycle arcs (so the cycle alone routes everything: the LP
        is feasible);
      * node inflow capacity per node v: 0 <= sum_k sum_{e into v} x_ke <= ncap_v,
        ncap_v = U(1,2) * total demand.
    Costs: U(1,10) per arc, the cycle arcs U(20,40) (expensive detour).
    All rows are equalities or finite two-sided ranges.
    The CSR is built directly from the per-commodity pattern (no global sort).
    """
    rng = np.random.default_rng(seed)
    perm = rng.permutation(V)
    tail = np.concatenate([perm, rng.integers(0, V, E - V)])
    head = np.concatenate([np.roll(perm, -1), rng.integers(0, V, E - V)])
    same = tail == head
    head[same] = (head[same] + 1) % V
    cyc = np.zeros(E, dtype=bool)
    cyc[:V] = True
    cost = np.where(cyc, rng.uniform(20.0, 40.0, E), rng.uniform(1.0, 10.0, E))
    # supplies: per commodity `terminals` distinct sources and sinks
    b = np.zeros((K, V))
    for k in range(K):
        nodes = rng.choice(V, 2 * terminals, replace=False)
        s = rng.uniform(1.0, 10.0, terminals)
        d = rng.uniform(1.0, 10.0, terminals)
        d *= s.sum() / d.sum()
        b[k, nodes[:terminals]] += s
        b[k, nodes[terminals:]] -= d
    total = float(np.abs(b).sum()) / 2.0
    cap = np.where(cyc, total, rng.uniform(1.0, 6.0, E))
    ncap = rng.uniform(1.0, 2.0, V) * total
    n = K * E
    m1 = K * V
    m = m1 + E + V
    # base conservation pattern (commodity 0): row v holds +1 at its out-arcs
    # and -1 at its in-arcs, columns ascending
    br = np.concatenate([tail, head]).astype(np.int64)
    bc = np.concatenate([np.arange(E), np.arange(E)]).astype(np.int64)
    bv = np.concatenate([np.ones(E), -np.ones(E)])
    order = np.lexsort((bc, br))
    br, bc, bv = br[order], bc[order], bv[order]
    blen = np.bincount(br, minlength=V).astype(np.int64)
    # node inflow pattern (commodity 0): row v holds its in-arcs ascending
    ir = head.astype(np.int64)
    ic = np.arange(E, dtype=np.int64)
    o2 = np.lexsort((ic, ir))
    ic = ic[o2]
    ilen = np.bincount(ir, minlength=V).astype(np.int64)
    nnz = 2 * E * K + E * K + E * K
    lens = np.concatenate([np.tile(blen, K), np.full(E, K, dtype=np.int64), ilen * K])
    rp = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    assert rp[-1] == nnz
    ci = np.empty(nnz, dtype=np.int64)
    v = np.empty(nnz, dtype=np.float64)
    for k in range(K):  # conservation block of commodity k
        lo = 2 * E * k
        ci[lo:lo + 2 * E] = bc + k * E
        v[lo:lo + 2 * E] = bv
    lo = 2 * E * K  # arc capacity rows: columns e, E+e, ..., (K-1)E+e
    ci[lo:lo + E * K] = (np.arange(E, dtype=np.int64)[:, None] +
                         E * np.arange(K, dtype=np.int64)[None, :]).ravel()
    v[lo:lo + E * K] = 1.0
    lo += E * K  # node inflow rows: for k: in-arcs of v shifted by k*E
    istart = np.zeros(V + 1, dtype=np.int64)
    np.cumsum(ilen, out=istart[1:])
    # element j of node row v (length ilen[v]*K): k = j // ilen[v], arc = ic[istart[v] + j % ilen[v]]
    rows = np.repeat(np.arange(V, dtype=np.int64), ilen * K)
    j = np.arange(E * K, dtype=np.int64) - np.repeat(istart[:-1] * K, ilen * K)
    L = ilen[rows]
    ci[lo:] = ic[istart[rows] + j % L] + (j // L) * E
    v[lo:] = 1.0
    del rows, j, L
    con_lb = np.concatenate([b.ravel(), np.zeros(E), np.zeros(V)])
    con_ub = np.concatenate([b.ravel(), cap, ncap])
    c = np.tile(cost, K)
    return LpProblem(m, n, rp, ci, v, c, np.zeros(n), np.full(n, INF), con_lb, con_ub,
                     name="c4_multicommodity")


def c5_rowpart(**kw) -> LpProblem:
    """C5: ~1B-nonzero C2-like LP (m=50M, n=20M), generated on the GPU
    (gen_device.py: a host numpy build of 1B nonzeros is impractical)."""
    from .gen_device import c5_rowpart as gen

    return gen(**kw)


CONFIGS = {
    "c1": c1_small,
    "c2": c2_powerlaw,
    "c3": c3_transport,
    "c4": c4_multicommodity,
    "c5": c5_rowpart,
}
