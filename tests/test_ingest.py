"""Device-side ingest (paper_2507_14051_b200/csrc/ingest.cu) and the C5
generator.

GPU: a CSR with explicit zeros (leading, trailing, whole rows) is compacted on
the device exactly like the reference's SparseMatrix (sparse_matrix.cpp:23-31
drops them): the device operators, A x, A^T y and the bit-exact scaling all
equal the oracle's on the zero-free matrix; invalid CSR input is rejected by
rhp_create with the reference's exception classes and messages.
CPU: the GPU C5 generator's structure (sorted unique columns, determinism,
solvability) at a small size on torch's CPU backend.
"""
import numpy as np
import pytest

import support
from paper_2507_14051_b200 import LpProblem, SolverConfig
from paper_2507_14051_b200.generators import random_rows_lp


def with_zeros(seed=5):
    """A random LP whose CSR carries explicit zeros, and its zero-free twin."""
    base = random_rows_lp(seed, 60, 45, np.random.default_rng(seed).integers(0, 12, 60))
    rng = np.random.default_rng(seed + 1)
    rp, ci, v = base.row_ptr, base.col_index, base.values.copy()
    # zero out ~25% of the entries, one whole row, and each row's first/last entry of a few rows
    z = rng.random(v.size) < 0.25
    r_full = int(np.argmax(np.diff(rp) > 3))
    z[rp[r_full]:rp[r_full + 1]] = True
    for r in range(0, 60, 7):
        if rp[r + 1] > rp[r]:
            z[rp[r]] = True
            z[rp[r + 1] - 1] = True
    v[z] = 0.0
    dirty = LpProblem(base.num_cons, base.num_vars, rp, ci, v, base.objective, base.var_lb,
                      base.var_ub, base.con_lb, base.con_ub, name="with_zeros")
    keep = v != 0.0
    row = np.repeat(np.arange(base.num_cons), np.diff(rp))
    rp2 = np.zeros(base.num_cons + 1, dtype=np.int64)
    np.add.at(rp2, row[keep] + 1, 1)
    clean = LpProblem(base.num_cons, base.num_vars, np.cumsum(rp2), ci[keep], v[keep], base.objective,
                      base.var_lb, base.var_ub, base.con_lb, base.con_ub, name="clean")
    return dirty, clean, int(z.sum())


@pytest.mark.gpu
def test_device_ingest_drops_explicit_zeros(gpu):
    from paper_2507_14051_b200.device import DeviceContext

    dirty, clean, nzero = with_zeros()
    assert nzero > 0
    o = support.oracle()
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, clean.num_vars)
    y = rng.uniform(-1, 1, clean.num_cons)
    with DeviceContext(dirty) as dev:
        assert dev.layout()["nnz_local"] == clean.nnz
        ax, aty = dev.spmv(x), dev.spmv(y, transpose=True)
        dev.scale(True, 10, True)
        got = dev.get_scaled()
    want_ax = support.spmv_with(o, clean, x)
    want_aty = support.spmv_with(o, clean, y, transpose=True)
    assert np.max(np.abs(ax - want_ax)) <= 1e-13 * max(1.0, np.max(np.abs(want_ax)))
    assert np.max(np.abs(aty - want_aty)) <= 1e-13 * max(1.0, np.max(np.abs(want_aty)))
    want = support.scale_with(o, clean, 10, True)
    for k in ("csr", "csc"):  # the dirty LP's buffers are longer: compacted prefix
        assert np.array_equal(got[k][:clean.nnz], want[k]), k  # bit-identical, as without zeros
    for k in ("row_scale", "col_scale", "c", "con_lb"):
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("case,exc,msg", [
    ("col_range", "UsageError", "out of bounds"),
    ("nonfinite", "InvalidProblemError", "is not finite"),
    ("unsorted", "InvalidProblemError", "duplicate or unsorted"),
    ("duplicate", "InvalidProblemError", "duplicate or unsorted"),
])
def test_device_ingest_rejects_invalid_csr(gpu, case, exc, msg):
    import paper_2507_14051_b200 as pkg
    from paper_2507_14051_b200.device import DeviceContext

    rp = np.array([0, 2, 4, 6], dtype=np.int64)
    ci = np.array([0, 2, 1, 3, 0, 1], dtype=np.int64)
    v = np.array([1.0, 2.0, 3.0, 4.0, 5.0, 6.0])
    bad_at = 3  # row 1, second entry
    if case == "col_range":
        ci[bad_at] = 9
    elif case == "nonfinite":
        v[bad_at] = np.inf
    elif case == "unsorted":
        ci[bad_at] = 0
    else:
        ci[bad_at] = 1
    # straight to rhp_create (no host SparseMatrix): the device must catch it
    lp = LpProblem(3, 4, rp, ci, v, np.zeros(4), np.full(4, -1.0), np.full(4, 1.0), np.zeros(3),
                   np.ones(3), name=case)
    with pytest.raises(getattr(pkg, exc), match=msg) as e:
        DeviceContext(lp)
    assert "(1," in str(e.value)  # the first offending entry, in row-major order


def test_c5_generator_structure_small():
    torch = pytest.importorskip("torch")
    del torch
    from paper_2507_14051_b200.gen_device import c5_rowpart

    lp = c5_rowpart(m=4000, n=3000, device="cpu", chunk=20000)
    rp, ci = lp.row_ptr, lp.col_index
    assert rp[0] == 0 and rp[-1] == ci.size and np.all(np.diff(rp) >= 1)
    start = np.zeros(ci.size, dtype=bool)
    start[rp[:-1]] = True
    assert np.all((np.diff(ci) > 0) | start[1:]), "columns strictly increasing inside rows"
    assert ci.min() >= 0 and ci.max() < lp.num_vars
    assert np.all(lp.values != 0.0) and np.all(np.abs(lp.values) <= 2.0)
    assert np.all(lp.con_lb <= lp.con_ub) and np.all(np.isfinite(lp.con_lb))
    again = c5_rowpart(m=4000, n=3000, device="cpu", chunk=20000)  # seeded: same LP
    for a, b in ((lp.col_index, again.col_index), (lp.objective, again.objective),
                 (lp.con_lb, again.con_lb), (lp.var_ub, again.var_ub)):
        assert np.array_equal(a, b)
    rep = support.solve_with(support.oracle(), lp, SolverConfig(epsilon=1e-4, iteration_limit=50_000))
    assert rep.status == "optimal"
