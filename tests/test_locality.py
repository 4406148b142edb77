"""Locality relabelling (ingest.cu maybe_relabel) on the GPU (-m gpu).

The device may renumber rows and columns in first-touch order at ingest; the
order maps must make that invisible at the boundary: products, iterates and
solutions come back in the caller's order and match the oracle (which knows
nothing of it) within the usual tolerances. Forced on small LPs here
(locality=1); the auto rule (large gathered vectors, fewer gather sectors)
is exercised at bench size by test_bench_parity.py (C4).
"""
import numpy as np
import pytest

import support
from paper_2507_14051_b200 import SolverConfig, solve
from paper_2507_14051_b200.device import DeviceContext
from paper_2507_14051_b200.generators import c1_small, c3_transport, c4_multicommodity, random_rows_lp
from paper_2507_14051_b200.lp import set_locality, set_resident

pytestmark = pytest.mark.gpu


def lps():
    rng = np.random.default_rng(5)
    lengths = rng.integers(0, 40, 3000)
    lengths[::97] = 0
    return [c4_multicommodity(V=300, E=1500, K=4, terminals=5), c1_small(m=500, n=900),
            c3_transport(S=40, T=70), random_rows_lp(9, lengths.size, 5000, lengths, name="ragged_small")]


LPS = lps()
IDS = [lp.name for lp in LPS]


@pytest.mark.parametrize("lp", LPS, ids=IDS)
def test_relabelled_products_in_caller_order(gpu, lp):
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, lp.num_vars)
    y = rng.uniform(-1, 1, lp.num_cons)
    with DeviceContext(lp, locality=1) as dev:
        lay = dev.layout()
        ax, aty = dev.spmv(x), dev.spmv(y, transpose=True)
    assert lay["relabel"]
    assert all(s > 0 for s in lay["sectors"])
    orc = support.oracle()
    ax_ref = support.spmv_with(orc, lp, x)
    aty_ref = support.spmv_with(orc, lp, y, transpose=True)
    assert np.max(np.abs(ax - ax_ref)) <= 1e-13 * max(1.0, np.max(np.abs(ax_ref)))
    assert np.max(np.abs(aty - aty_ref)) <= 1e-13 * max(1.0, np.max(np.abs(aty_ref)))


def test_relabel_is_a_permutation(gpu):
    """Row r of the relabelled operator is some original row: A x with
    x = e_j lands on exactly the original rows of column j."""
    lp = LPS[0]
    A = lp.to_dense()
    with DeviceContext(lp, locality=1) as dev:
        for j in (0, 7, lp.num_vars // 2, lp.num_vars - 1):
            e = np.zeros(lp.num_vars)
            e[j] = 1.0
            assert np.array_equal(dev.spmv(e), A[:, j])


def test_auto_rule_leaves_small_lps_alone(gpu):
    with DeviceContext(LPS[0], locality=0) as dev:
        assert not dev.layout()["relabel"]


@pytest.mark.parametrize("lp", LPS, ids=IDS)
def test_relabelled_solve_matches_oracle(gpu, lp):
    cfg = SolverConfig(epsilon=1e-6)
    try:
        set_locality(1)
        set_resident(0)  # the multi-CTA engine (the resident kernel holds the whole LP anyway)
        got = solve(lp, cfg)
    finally:
        set_locality(0)
        set_resident(-1)
    want = support.solve_with(support.oracle(), lp, cfg)
    assert got.status == want.status
    if want.status == "optimal":
        rel = abs(got.objective - want.objective) / max(1.0, abs(want.objective))
        assert rel <= 1e-6, rel
        # the returned point, in the caller's order, re-checked by the oracle
        k = support.kkt_with(support.oracle(), lp, got.x, got.y)
        assert k["gap_rel"] <= 2e-6 and k["primal_rel"] <= 2e-6


def test_relabelled_first_iterates(gpu):
    """First iterates of the relabelled solve against the oracle's (only the
    reduction orders moved: 1e-10 relative, as test_bench_parity.py)."""
    lp = LPS[0]
    ks = [1, 10, 64, 65, 100]
    xs, ys = support.oracle_snapshots(lp, SolverConfig(epsilon=1e-300, iteration_limit=max(ks)), ks)
    try:
        set_locality(1)
        set_resident(0)
        for i, k in enumerate(ks):
            rep = solve(lp, SolverConfig(epsilon=1e-300, iteration_limit=k))
            assert rep.iterations == k
            x, y = np.asarray(rep.x), np.asarray(rep.y)
            dx = np.max(np.abs(x - xs[i])) / max(1e-300, np.max(np.abs(xs[i])))
            dy = np.max(np.abs(y - ys[i])) / max(1e-300, np.max(np.abs(ys[i])))
            assert dx <= 1e-10 and dy <= 1e-10, (k, dx, dy)
    finally:
        set_locality(0)
        set_resident(-1)


def test_matrix_values_of_a_relabelled_layout_are_refused(gpu):
    """The per-op API's CSR/CSC value exchange is in the reference's element
    order, which only an unrelabelled layout has: refused, not reordered."""
    with DeviceContext(LPS[0], locality=1) as dev:
        dev.scale()
        with pytest.raises(Exception, match="relabelled"):
            dev.get_scaled()
