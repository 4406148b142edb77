"""The row-partitioned engine at world size > 1 on ONE GPU.

NCCL refuses two ranks on one device, so these tests join the ranks through
the in-process collective group of comm.cuh (rhp_local_group_create): one
host thread per rank, each with its own device context, stream and row
block, exchanging A_p^T y_p partials, y-side sums, scaling maxima / 1-norms,
power-iteration and KKT sums and the y gather through device memory with
rank-ordered reductions. Everything the multi-GPU path runs on the device —
non-zero row offsets, the distributed scaling, power iteration and KKT
checks, gather_rows, the stop polling of partitioned plain blocks — runs
here for real; only the transport differs from NCCL.

Both exchanges of SURVEY.md §8(e) run: Option B (the default at world > 1:
reduce-scatter of A^T y, n-side walk on the owned column slice, all-gather
of x+) and Option A (RHP_DIST_REPLICATED=1: allreduce, replicated walk).

Checks: every rank reports the same solve (bitwise); the first iterates
equal the single-GPU path's within 1e-12 relative (the only difference is
the summation order of A^T y across row blocks); solves match the single
GPU and the oracle's objective and pass the oracle's KKT check.
"""
import threading

import numpy as np
import pytest

import support
from paper_2507_14051_b200 import SolverConfig, solve
from paper_2507_14051_b200.generators import c1_small, c3_transport, random_rows_lp
from paper_2507_14051_b200.lp import LocalGroup, partition_rows, set_local_group, set_resident

pytestmark = pytest.mark.gpu


def ragged():
    L = np.random.default_rng(5).integers(0, 60, 700)
    L[::97] = 3000  # long rows (split rows in the merge-path schedule)
    return random_rows_lp(17, 700, 900, L)


LPS = {"c1_small": lambda: c1_small(m=400, n=700), "ragged_long_rows": ragged,
       "transport": lambda: c3_transport(S=40, T=70)}


def solve_ranks(lp, cfg, world):
    """All ranks of one in-process group solve lp together; per-rank reports."""
    group = LocalGroup(world)
    reps, errs = [None] * world, []

    def worker(r):
        try:
            set_local_group(r, world, group)
            reps[r] = solve(lp, cfg)
        except Exception as e:  # surfaced below
            errs.append((r, e))

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    group.close()
    assert not errs, errs
    return reps


def single(lp, cfg):
    try:
        set_resident(0)  # the multi-CTA engine the partitioned path shares
        return solve(lp, cfg)
    finally:
        set_resident(-1)


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300))


@pytest.fixture(params=["sharded", "replicated"])
def exchange(request, monkeypatch):
    """Option B (reduce-scatter + all-gather, n-side walk on the owned column
    slice; the default at world > 1) or Option A (allreduce, replicated
    n-side walk; RHP_DIST_REPLICATED=1)."""
    if request.param == "replicated":
        monkeypatch.setenv("RHP_DIST_REPLICATED", "1")
    return request.param


@pytest.mark.parametrize("name", sorted(LPS))
@pytest.mark.parametrize("world", [2, 3])
def test_ranks_agree_and_match_single_gpu(gpu, name, world, exchange):
    lp = LPS[name]()
    off = partition_rows(lp, world)
    assert np.all(np.diff(off) > 0)  # every rank owns rows (non-zero row_begin)
    cfg = SolverConfig(epsilon=1e-7)
    reps = solve_ranks(lp, cfg, world)
    for r in reps[1:]:  # identical decisions and results on every rank
        assert r.status == reps[0].status and r.iterations == reps[0].iterations
        assert r.objective == reps[0].objective
        assert np.array_equal(r.x, reps[0].x) and np.array_equal(r.y, reps[0].y)
    ref = single(lp, cfg)
    got = reps[0]
    assert got.status == ref.status == "optimal"
    assert abs(got.objective - ref.objective) <= 1e-6 * max(1.0, abs(ref.objective))
    assert abs(got.matrix_norm_estimate - ref.matrix_norm_estimate) <= 1e-12 * ref.matrix_norm_estimate
    orc = support.solve_with(support.oracle(), lp, cfg)
    assert abs(got.objective - orc.objective) <= 1e-6 * max(1.0, abs(orc.objective))
    k = support.kkt_with(support.oracle(), lp, got.x, got.y)
    assert k["gap_rel"] <= 1e-7 and k["primal_rel"] <= 1e-7
    assert k["dual_eq"] <= 1e-7 * k["dual_denom"]


@pytest.mark.parametrize("name", sorted(LPS))
def test_first_iterates_match_single_gpu(gpu, name, exchange):
    lp = LPS[name]()
    for k in (1, 10, 64, 65, 100):
        cfg = SolverConfig(epsilon=1e-300, iteration_limit=k)
        got = solve_ranks(lp, cfg, 2)[0]
        want = single(lp, cfg)
        assert got.iterations == want.iterations == k
        assert rel(got.x, want.x) <= 1e-12, (k, rel(got.x, want.x))
        assert rel(got.y, want.y) <= 1e-12, (k, rel(got.y, want.y))


def test_partitioned_with_column_segments(gpu, monkeypatch, exchange):
    """Forced 1 KB column segments on every rank's operators."""
    monkeypatch.setenv("RHP_SEG_BYTES", "1024")
    monkeypatch.setenv("RHP_SEG_FORCE", "1")
    lp = ragged()
    cfg = SolverConfig(epsilon=1e-7)
    got = solve_ranks(lp, cfg, 2)[0]
    ref = single(lp, cfg)
    assert got.status == ref.status == "optimal"
    assert abs(got.objective - ref.objective) <= 1e-6 * max(1.0, abs(ref.objective))


def test_iteration_limit_and_restart_stops_are_exact(gpu, exchange):
    """Blocks that stop on the device mid-block (restart verdicts) and at the
    iteration limit: the stop polling issues no extra iteration (counts equal
    the single-GPU path's)."""
    lp = c1_small(m=400, n=700)
    for limit in (3, 64, 130, 777):
        cfg = SolverConfig(epsilon=1e-300, iteration_limit=limit)
        reps = solve_ranks(lp, cfg, 2)
        ref = single(lp, cfg)
        assert [r.iterations for r in reps] == [limit, limit]
        assert reps[0].restart_count == ref.restart_count
        assert reps[0].kkt_checks == ref.kkt_checks


def test_sharded_more_ranks_than_slices_of_work(gpu):
    """World 4 on a tiny LP: uneven and empty column slices (n = 5)."""
    from paper_2507_14051_b200 import LpProblem

    lp = LpProblem(4, 5, [0, 2, 4, 6, 7], [0, 3, 1, 4, 0, 2, 3], [1.0, 2.0, -1.0, 1.0, 3.0, 1.0, 1.0],
                   [1.0, -1.0, 2.0, 0.5, -0.5], [0.0] * 5, [4.0] * 5, [1.0, -1.0, 0.0, 0.5],
                   [2.0, 1.0, 3.0, 0.5])
    cfg = SolverConfig(epsilon=1e-8)
    reps = solve_ranks(lp, cfg, 4)
    ref = single(lp, cfg)
    assert all(r.status == ref.status for r in reps)
    assert abs(reps[0].objective - ref.objective) <= 1e-6 * max(1.0, abs(ref.objective))
