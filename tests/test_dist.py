"""Row-partitioned multi-GPU path.

CPU (gloo, world_size 2): the partition the device path uses
(rhp_partition_rows, host code) covers the rows exactly once with balanced
nonzeros, and the exchange algebra of one PDHG iteration — local A_p x, the
allreduce of the A_p^T y_p partials plus the y-side sums, the column-max and
1-norm allreduces of the scaling — reproduces the single-process quantities
(oracle arithmetic on each rank's row block).

GPU (-m gpu): the partitioned device path (K1d / A_p^T / NCCL allreduce /
control / K2c, distributed scaling, power iteration and KKT) run with one
NCCL rank is bit-identical to the single-GPU path.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import support
from paper_2507_14051_b200 import LpProblem, SolverConfig, solve
from paper_2507_14051_b200.generators import c1_small, random_rows_lp
from paper_2507_14051_b200.lp import (nccl_unique_id, partition_rows, set_distributed,
                                      set_resident)


def block(lp: LpProblem, r0: int, r1: int) -> LpProblem:
    """Rows [r0, r1) of lp as their own LP (the rank-local operator)."""
    b, e = lp.row_ptr[r0], lp.row_ptr[r1]
    return LpProblem(r1 - r0, lp.num_vars, lp.row_ptr[r0:r1 + 1] - b, lp.col_index[b:e],
                     lp.values[b:e], lp.objective, lp.var_lb, lp.var_ub, lp.con_lb[r0:r1],
                     lp.con_ub[r0:r1])


def ragged():
    L = np.random.default_rng(5).integers(0, 60, 700)
    L[::97] = 3000  # long rows
    return random_rows_lp(17, 700, 900, L)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_covers_rows_and_balances_nnz(world):
    lp = ragged()
    off = partition_rows(lp, world)
    assert off[0] == 0 and off[-1] == lp.num_cons and np.all(np.diff(off) >= 0)
    w = np.diff(lp.row_ptr) + 1
    per = [w[off[r]:off[r + 1]].sum() for r in range(world)]
    assert max(per) <= w.sum() / world + w.max() + 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O = support.oracle()
        lp = ragged()
        off = partition_rows(lp, world)
        loc = block(lp, int(off[rank]), int(off[rank + 1]))
        rng = np.random.default_rng(0)
        x = rng.uniform(-1, 1, lp.num_vars)  # replicated
        y = rng.uniform(-1, 1, lp.num_cons)
        y_loc = y[off[rank]:off[rank + 1]]
        # A x is local; A^T y = sum of the ranks' partials (one allreduce)
        ax_loc = support.spmv_with(O, loc, x)
        xchg = torch.from_numpy(np.concatenate([support.spmv_with(O, loc, y_loc, True),
                                                [float(np.dot(y_loc, y_loc))]]))
        dist.all_reduce(xchg)
        # scaling: column maxima (max-allreduce) and column 1-norms (sum)
        cmax = torch.zeros(lp.num_vars, dtype=torch.float64)
        cnorm = torch.zeros(lp.num_vars, dtype=torch.float64)
        for i in range(loc.num_cons):
            s, e = loc.row_ptr[i], loc.row_ptr[i + 1]
            cols, vals = loc.col_index[s:e], np.abs(loc.values[s:e])
            cmax[cols] = torch.maximum(cmax[cols], torch.from_numpy(vals))
            cnorm[cols] += torch.from_numpy(vals)
        dist.all_reduce(cmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(cnorm)
        q.put((rank, int(off[rank]), ax_loc, xchg.numpy(), cmax.numpy(), cnorm.numpy()))
    finally:
        dist.destroy_process_group()


def test_row_partition_exchange_matches_single_process_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lp = ragged()
    O = support.oracle()
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, lp.num_vars)
    y = rng.uniform(-1, 1, lp.num_cons)
    ax = np.concatenate([r[2] for r in res])
    assert np.array_equal(ax, support.spmv_with(O, lp, x))  # local rows: same sums
    aty = support.spmv_with(O, lp, y, True)
    for _, _, _, xchg, cmax, cnorm in res:
        assert np.array_equal(xchg, res[0][3])  # identical on every rank
        assert np.allclose(xchg[:-1], aty, rtol=1e-13, atol=1e-13)
        assert xchg[-1] == pytest.approx(float(np.dot(y, y)), rel=1e-14)
        A = lp.to_dense()
        assert np.array_equal(cmax, np.abs(A).max(axis=0))  # exact
        assert np.allclose(cnorm, np.abs(A).sum(axis=0), rtol=1e-14)


@pytest.mark.gpu
@pytest.mark.parametrize("maker", [lambda: c1_small(m=400, n=700), ragged,
                                   lambda: support.lp_from_json(
                                       support.load_golden("random_feasible.json")
                                       ["instances"][-1]["lp"])],
                         ids=["c1_small", "ragged_long_rows", "rfl_5002"])
@pytest.mark.parametrize("segments", [False, True], ids=["whole", "column_segments"])
@pytest.mark.parametrize("exchange", ["nccl", "peer"])
def test_partitioned_path_one_rank_is_bitwise_single_gpu(gpu, maker, segments, exchange,
                                                         monkeypatch):
    """One rank of the row-partitioned engine (NCCL allreduce, or the
    NVLink peer-memory exchange of peer.cuh with the rank as its own peer)
    reproduces the single-GPU solve bit for bit."""
    if segments:  # both paths with forced 1 KB column segments
        monkeypatch.setenv("RHP_SEG_BYTES", "1024")
        monkeypatch.setenv("RHP_SEG_FORCE", "1")
    if exchange == "peer":
        monkeypatch.setenv("RHP_PEER_EXCHANGE", "1")
    lp = maker()
    cfg = SolverConfig(epsilon=1e-7, record_residual_history=True)
    try:
        set_resident(0)  # compare against the multi-CTA single-GPU path
        single = solve(lp, cfg)
        set_distributed(0, 1, nccl_unique_id())
        part = solve(lp, cfg)
    finally:
        set_distributed(0, 1, None)
        set_resident(-1)
    assert part.status == single.status
    assert part.iterations == single.iterations and part.restart_count == single.restart_count
    assert part.objective == single.objective
    assert np.array_equal(part.x, single.x) and np.array_equal(part.y, single.y)
    assert np.array_equal(part.fixed_point_residual_history, single.fixed_point_residual_history)
    assert part.matrix_norm_estimate == single.matrix_norm_estimate


def _peer_worker(rank, world, port, q):
    """The peer-memory exchange of peer.cuh restated over gloo: every rank
    publishes its partial, reduces the columns it owns (slice n*r/P ..
    n*(r+1)/P, the formula of owned_slice) over all partials in rank order,
    and gathers every owner's slice."""
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O = support.oracle()
        lp = ragged()
        off = partition_rows(lp, world)
        loc = block(lp, int(off[rank]), int(off[rank + 1]))
        y = np.random.default_rng(1).uniform(-1, 1, lp.num_cons)
        y_loc = y[off[rank]:off[rank + 1]]
        n = lp.num_vars
        part = torch.from_numpy(np.concatenate([support.spmv_with(O, loc, y_loc, True),
                                                [float(np.dot(y_loc, y_loc))]]))
        # phase 1: every rank can read every partial (peer loads)
        parts = [torch.zeros_like(part) for _ in range(world)]
        dist.all_gather(parts, part)
        lo, hi = n * rank // world, n * (rank + 1) // world
        own = parts[0][lo:hi].clone()
        for p in parts[1:]:
            own += p[lo:hi]  # rank order
        ysum = parts[0][n:].clone()
        for p in parts[1:]:
            ysum += p[n:]
        # phase 2: gather the owners' slices (variable sizes: pad to the largest)
        width = -(-n // world) + 1
        padded = torch.zeros(width, dtype=torch.float64)
        padded[:hi - lo] = own
        slices = [torch.zeros_like(padded) for _ in range(world)]
        dist.all_gather(slices, padded)
        full = torch.cat([slices[r][:n * (r + 1) // world - n * r // world] for r in range(world)])
        ref = part.clone()
        dist.all_reduce(ref)
        q.put((rank, torch.cat([full, ysum]).numpy(), ref.numpy()))
    finally:
        dist.destroy_process_group()


def test_peer_exchange_protocol_gloo():
    """Every rank ends with the same reduced vector (bitwise), equal to the
    allreduce up to summation order and to the single-process A^T y."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, full, ref in res:
        assert np.array_equal(full, res[0][1])  # identical on every rank
        assert np.allclose(full, ref, rtol=1e-13, atol=1e-13)
    lp = ragged()
    y = np.random.default_rng(1).uniform(-1, 1, lp.num_cons)
    aty = support.spmv_with(support.oracle(), lp, y, True)
    assert np.allclose(res[0][1][:-1], aty, rtol=1e-12, atol=1e-12)
