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
                      K: int = 20) -> LpProblem:
    """C4: K-commodity min-cost flow on a random directed graph (V nodes, E
    arcs incl. a Hamiltonian cycle for connectivity). Variables x_ke >= 0
    (n = K*E); rows: conservation per (k, v) (equality, m1 = K*V) and shared
    capacity per arc as [0, cap_e] (m2 = E). nnz = 3*K*E."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(V)
    tail = np.concatenate([perm, rng.integers(0, V, E - V)])
    head = np.concatenate([np.roll(perm, -1), rng.integers(0, V, E - V)])
    same = tail == head
    head[same] = (head[same] + 1) % V
    cost = rng.uniform(1.0, 10.0, E)
    # each commodity: one source/sink pair with demand d_k routed along
    src = rng.integers(0, V, K)
    dst = (src + 1 + rng.integers(0, V - 1, K)) % V
    dem = rng.uniform(1.0, 10.0, K)
    cap = rng.uniform(1.0, 2.0, E) * dem.sum()  # the Hamiltonian cycle alone is feasible
    n = K * E
    m1 = K * V
    m = m1 + E
    k_of = np.repeat(np.arange(K, dtype=np.int64), E)
    e_of = np.tile(np.arange(E, dtype=np.int64), K)
    var = np.arange(n, dtype=np.int64)
    rows = np.concatenate([k_of * V + tail[e_of], k_of * V + head[e_of], m1 + e_of])
    cols = np.concatenate([var, var, var])
    vals = np.concatenate([np.ones(n), -np.ones(n), np.ones(n)])
    rp, ci, v = _csr_from_rows(m, n, rows, cols, vals)
    b = np.zeros(m1)
    b[np.arange(K) * V + src] += dem
    b[np.arange(K) * V + dst] -= dem
    con_lb = np.concatenate([b, np.zeros(E)])
    con_ub = np.concatenate([b, cap])
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
