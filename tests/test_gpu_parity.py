"""GPU parity suite (-m gpu): the CUDA product, driven through its C ABIs,
against the oracle (oracle/rhpdhg_oracle.c, bit-identical to the reference,
see test_oracle.py) and against the golden fixtures generated from the
reference (tests/golden/).

Tolerances (BASELINE.json north star):
  * SpMV: |gpu - ref| <= 1e-14 * (|A| |x|)_i  (sum-order/FMA drift only)
  * scaling (Ruiz + Pock-Chambolle): bit-identical
  * first 100 iterates: max |dz| <= 1e-10 * max(1, max |z_ref|)
  * final objective: 1e-6 relative; KKT of the returned point at the solve's
    epsilon (re-evaluated by the oracle); status equal.
"""
import math

import numpy as np
import pytest

import support
from paper_2507_14051_b200 import LpProblem, SolverConfig, kkt_residuals, set_device_options, solve
from paper_2507_14051_b200.device import DeviceContext
from paper_2507_14051_b200.generators import c1_small, c3_transport, random_rows_lp

pytestmark = pytest.mark.gpu

RANDOM = support.load_golden("random_feasible.json")["instances"]
ANALYTIC = support.load_golden("analytic_lps.json")["instances"]
SUITE = support.load_golden("random_suite.json")["instances"]
INF = math.inf


def ragged_lp():
    """Every bin of the schedule: empty rows, 1-nnz rows, each sub-warp width,
    CTA rows (>512) and multi-chunk rows (>8192 nnz)."""
    lengths = np.array([0, 1, 2, 3, 4, 5, 8, 9, 16, 17, 32, 33, 64, 65, 300, 512, 513, 700, 4000,
                        8192, 8193, 20000] + [7] * 300 + [0] * 20 + [1] * 50)
    rng = np.random.default_rng(11)
    rng.shuffle(lengths)
    return random_rows_lp(21, lengths.size, 25000, lengths, name="ragged")


def cases():
    out = [support.lp_from_json(i["lp"]) for i in RANDOM]
    out += [ragged_lp(), c1_small(m=500, n=900), c3_transport(S=40, T=70),
            LpProblem(3, 4, [0, 0, 0, 0], [], [], np.ones(4), np.zeros(4), np.ones(4),
                      np.zeros(3), np.ones(3), name="empty"),
            LpProblem(0, 3, [0], [], [], [2.0, -1.0, 0.5], [-1.0, -2.0, 0.25], [4.0, 3.0, 5.0],
                      [], [], name="rowless")]
    return out


CASES = cases()


def max_rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


@pytest.mark.parametrize("lp", CASES, ids=[c.name or str(i) for i, c in enumerate(CASES)])
def test_spmv_matches_oracle(gpu, lp):
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, lp.num_vars)
    y = rng.uniform(-1, 1, lp.num_cons)
    absA = LpProblem(lp.num_cons, lp.num_vars, lp.row_ptr, lp.col_index, np.abs(lp.values),
                     lp.objective, lp.var_lb, lp.var_ub, lp.con_lb, lp.con_ub)
    O = support.oracle()
    with DeviceContext(lp) as dev:
        ax, aty = dev.spmv(x), dev.spmv(y, True)
    bound_ax = support.spmv_with(O, absA, np.abs(x)) * 1e-14 + 1e-300
    bound_aty = support.spmv_with(O, absA, np.abs(y), True) * 1e-14 + 1e-300
    assert np.all(np.abs(ax - support.spmv_with(O, lp, x)) <= bound_ax)
    assert np.all(np.abs(aty - support.spmv_with(O, lp, y, True)) <= bound_aty)


@pytest.mark.parametrize("inst", RANDOM, ids=[i["name"] for i in RANDOM])
def test_spmv_matches_reference_golden(gpu, inst):
    lp = support.lp_from_json(inst["lp"])
    sp = inst["spmv"]
    with DeviceContext(lp) as dev:
        assert max_rel(dev.spmv(sp["x"]), sp["ax"]) <= 1e-14
        assert max_rel(dev.spmv(sp["y"], True), sp["aty"]) <= 1e-14


@pytest.mark.parametrize("lp", CASES[:-2], ids=[c.name or str(i) for i, c in enumerate(CASES[:-2])])
def test_scaling_bitwise_equal_to_oracle(gpu, lp):
    for ruiz, pc in ((10, True), (10, False), (0, True), (3, True)):
        want = support.scale_with(support.oracle(), lp, ruiz, pc)
        with DeviceContext(lp) as dev:
            dev.scale(True, ruiz, pc)
            got = dev.get_scaled()
        for k in want:
            assert np.array_equal(got[k], want[k]), (k, ruiz, pc)


@pytest.mark.parametrize("inst", RANDOM, ids=[i["name"] for i in RANDOM])
def test_scaling_matches_reference_golden(gpu, inst):
    lp = support.lp_from_json(inst["lp"])
    with DeviceContext(lp) as dev:
        dev.scale()
        got = dev.get_scaled()
    for k, v in inst["scaling"].items():
        assert got[k].tolist() == v, k


@pytest.mark.parametrize("inst", RANDOM, ids=[i["name"] for i in RANDOM])
def test_first_100_iterates_match_reference(gpu, inst):
    """Iterates after k = 1..100 iterations (full pipeline incl. scaling,
    power iteration, restarts, KKT cache refreshes at 64) agree with the
    reference within 1e-10 relative."""
    lp = support.lp_from_json(inst["lp"])
    for k, snap in inst["snapshots"].items():
        r = solve(lp, SolverConfig(epsilon=1e-300, iteration_limit=int(k)))
        if r.status == "optimal" and r.iterations < int(k):
            # eps=1e-300 can only be met by EXACTLY zero residuals: a tiny LP
            # whose KKT sums cancel to 0.0 in the device's summation order
            # stops at that check; the reference (other order) runs on.
            assert r.residuals.gap_rel == r.residuals.primal_rel == r.residuals.dual_eq == 0.0
            break
        assert r.iterations == int(k)
        assert max_rel(r.x, snap["x"]) <= 1e-10, k
        assert max_rel(r.y, snap["y"]) <= 1e-10, k


@pytest.mark.parametrize("inst", ANALYTIC, ids=[i["name"] for i in ANALYTIC])
@pytest.mark.parametrize("eps", ["0.0001", "1e-08"])
def test_analytic_fixtures_match_reference(gpu, inst, eps):
    lp = support.lp_from_json(inst["lp"])
    want = inst["results"][eps]
    r = solve(lp, SolverConfig(epsilon=float(eps)))
    assert r.status == want["status"] == "optimal"
    assert abs(r.objective - want["objective"]) <= 1e-6 * max(1.0, abs(want["objective"]))
    assert r.matrix_norm_estimate == pytest.approx(want["matrix_norm_estimate"], rel=1e-12)
    assert r.power_iterations == want["power_iterations"]
    # tiny analytic LPs have <= 3 terms per row: the trajectory is reproduced
    assert (r.iterations, r.restart_count, r.kkt_checks) == \
        (want["iterations"], want["restart_count"], want["kkt_checks"])


@pytest.mark.parametrize("inst", SUITE, ids=[i["name"] for i in SUITE])
def test_random_suite_objective_and_kkt(gpu, inst):
    lp = support.lp_from_json(inst["lp"])
    want = inst["result_1e-8_cap20k"]
    r = solve(lp, SolverConfig(epsilon=1e-8, iteration_limit=20000))
    assert r.status == want["status"] == "optimal"
    assert abs(r.objective - want["objective"]) <= 1e-6 * max(1.0, abs(want["objective"]))
    h = inst["highs_objective"]
    assert abs(r.objective - h) <= 1e-5 * max(1.0, abs(h))
    k = support.kkt_with(support.oracle(), lp, r.x, r.y)
    assert k["gap_rel"] <= 1e-8 and k["primal_rel"] <= 1e-8
    assert k["dual_eq"] <= 1e-8 * k["dual_denom"]


def test_solver_parity_c1(gpu):
    lp = c1_small()
    for eps in (1e-4, 1e-8):
        cfg = SolverConfig(epsilon=eps)
        g = solve(lp, cfg)
        o = support.solve_with(support.oracle(), lp, cfg)
        assert g.status == o.status == "optimal"
        assert abs(g.objective - o.objective) <= 1e-6 * max(1.0, abs(o.objective))
        k = support.kkt_with(support.oracle(), lp, g.x, g.y)
        assert k["gap_rel"] <= eps and k["primal_rel"] <= eps
        assert k["dual_eq"] <= eps * k["dual_denom"]
        assert g.matrix_norm_estimate == pytest.approx(o.matrix_norm_estimate, rel=1e-12)


def test_solves_are_bitwise_deterministic(gpu):
    lp = c1_small(m=300, n=500)
    a = solve(lp, SolverConfig(epsilon=1e-8))
    b = solve(lp, SolverConfig(epsilon=1e-8))
    assert a.iterations == b.iterations and a.restart_count == b.restart_count
    assert a.objective == b.objective
    assert np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y)


def test_graph_and_plain_launch_modes_agree_bitwise(gpu):
    lp = support.lp_from_json(RANDOM[-1]["lp"])
    cfg = SolverConfig(epsilon=1e-8, record_residual_history=True)
    try:
        set_device_options(0, True, 64)
        a = solve(lp, cfg)
        set_device_options(0, False, 64)
        b = solve(lp, cfg)
        set_device_options(0, True, 7)
        c = solve(lp, cfg)
    finally:
        set_device_options(0, True, 64)
    for r in (b, c):
        assert r.iterations == a.iterations and r.objective == a.objective
        assert np.array_equal(r.x, a.x) and np.array_equal(r.y, a.y)
        assert np.array_equal(r.fixed_point_residual_history, a.fixed_point_residual_history)


@pytest.mark.parametrize("mode", [0, 1], ids=["multi_cta", "cluster_resident"])
def test_both_block_engines_match_oracle(gpu, mode):
    """The multi-CTA K1/K2 path and the small-LP cluster-resident block
    kernel each reproduce the reference solve (objective 1e-6, KKT at eps)
    and the first iterates (1e-10)."""
    from paper_2507_14051_b200.lp import set_resident

    lp = c1_small(m=300, n=500)
    try:
        set_resident(mode)
        for eps in (1e-4, 1e-8):
            cfg = SolverConfig(epsilon=eps)
            g = solve(lp, cfg)
            o = support.solve_with(support.oracle(), lp, cfg)
            assert g.status == o.status == "optimal"
            assert abs(g.objective - o.objective) <= 1e-6 * max(1.0, abs(o.objective))
            k = support.kkt_with(support.oracle(), lp, g.x, g.y)
            assert k["gap_rel"] <= eps and k["primal_rel"] <= eps
        for it in (1, 5, 30, 64, 100):
            cfg = SolverConfig(epsilon=1e-300, iteration_limit=it)
            g = solve(lp, cfg)
            o = support.solve_with(support.oracle(), lp, cfg)
            assert max_rel(g.x, o.x) <= 1e-10 and max_rel(g.y, o.y) <= 1e-10
        a = solve(lp, SolverConfig(epsilon=1e-8, record_residual_history=True))
        b = solve(lp, SolverConfig(epsilon=1e-8, record_residual_history=True))
        assert np.array_equal(a.x, b.x) and a.iterations == b.iterations  # deterministic
    finally:
        set_resident(-1)


ENGINE_LPS = [c3_transport(S=40, T=70), c1_small(m=300, n=500), ragged_lp()]


@pytest.mark.parametrize("lp", ENGINE_LPS, ids=[c.name for c in ENGINE_LPS])
def test_spmv_engines_and_gather_policies(gpu, lp, monkeypatch):
    """Both SpMV engines (merge-path warps; thread per row, chosen for
    operators whose rows all have <= 8 nonzeros) under both gather cache
    policies: SpMV within 1e-14 of the oracle (bit-exact for the
    thread-per-row engine, which sums in the reference's order), solves that
    match the reference, and gather policies that never change a result."""
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, lp.num_vars)
    y = rng.uniform(-1, 1, lp.num_cons)
    O = support.oracle()
    ref_ax, ref_aty = support.spmv_with(O, lp, x), support.spmv_with(O, lp, y, True)
    cfg = SolverConfig(epsilon=1e-8)
    o = support.solve_with(O, lp, cfg)
    longest_t = int(np.max(np.bincount(lp.col_index, minlength=lp.num_vars))) if lp.nnz else 0
    for rows in ("0", "1"):
        results = []
        for l1 in ("0", "1"):
            monkeypatch.setenv("RHP_THREAD_ROWS", rows)
            monkeypatch.setenv("RHP_L1_GATHER", l1)
            with DeviceContext(lp) as dev:
                lay = dev.layout()
                ax, aty = dev.spmv(x), dev.spmv(y, True)
            assert lay["gather_l1"] == {"A": l1 == "1", "At": l1 == "1"}
            assert lay["thread_rows"]["At"] == (rows == "1" and longest_t <= 64)
            for got, ref, row_engine in ((ax, ref_ax, lay["thread_rows"]["A"]),
                                         (aty, ref_aty, lay["thread_rows"]["At"])):
                if row_engine:
                    assert np.array_equal(got, ref)
                else:
                    assert max_rel(got, ref) <= 1e-13
            g = solve(lp, cfg)
            assert g.status == o.status == "optimal"
            assert abs(g.objective - o.objective) <= 1e-6 * max(1.0, abs(o.objective))
            g30 = solve(lp, SolverConfig(epsilon=1e-300, iteration_limit=30))
            o30 = support.solve_with(O, lp, SolverConfig(epsilon=1e-300, iteration_limit=30))
            assert max_rel(g30.x, o30.x) <= 1e-10 and max_rel(g30.y, o30.y) <= 1e-10
            results.append(g)
        a, b = results
        assert a.iterations == b.iterations and np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y)


SEG_LPS = [c1_small(m=300, n=500), c3_transport(S=40, T=70)]


@pytest.mark.parametrize("band", [None, (0.3, 0.7), (0.0, 0.25), (0.8, 1.0)],
                         ids=["all_rows", "mid_band", "head_band", "tail_band"])
@pytest.mark.parametrize("lp", SEG_LPS, ids=[c.name for c in SEG_LPS])
def test_column_segments_match_oracle(gpu, lp, band, monkeypatch):
    """Column-segmented operators (built after scaling when the gathered
    vector exceeds RHP_SEG_BYTES; forced here with a 1 KB segment): SpMV
    within 1e-13 of the oracle, solves that match the reference (objective
    1e-6, KKT at eps, first iterates 1e-10) and stay deterministic."""
    monkeypatch.setenv("RHP_SEG_BYTES", "1024")
    monkeypatch.setenv("RHP_SEG_FORCE", "1")
    if band is not None:  # only this row band (rows of A; A^T reads it as its own rows)
        monkeypatch.setenv("RHP_SEG_BAND", f"{int(band[0] * lp.num_cons)},{int(band[1] * lp.num_cons)}")
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, lp.num_vars)
    y = rng.uniform(-1, 1, lp.num_cons)
    O = support.oracle()
    with DeviceContext(lp) as dev:
        dev.scale(enabled=False)
        lay = dev.layout()
        ax, aty = dev.spmv(x), dev.spmv(y, True)
    assert lay["segments"]["A"] == -(-lp.num_vars * 8 // 1024)
    assert lay["segments"]["At"] == max(1, -(-lp.num_cons * 8 // 1024))
    assert max_rel(ax, support.spmv_with(O, lp, x)) <= 1e-13
    assert max_rel(aty, support.spmv_with(O, lp, y, True)) <= 1e-13
    cfg = SolverConfig(epsilon=1e-8)
    g = solve(lp, cfg)
    o = support.solve_with(O, lp, cfg)
    assert g.status == o.status == "optimal"
    assert abs(g.objective - o.objective) <= 1e-6 * max(1.0, abs(o.objective))
    k = support.kkt_with(O, lp, g.x, g.y)
    assert k["gap_rel"] <= 1e-8 and k["primal_rel"] <= 1e-8
    for it in (1, 10, 30):
        cfg_it = SolverConfig(epsilon=1e-300, iteration_limit=it)
        gi, oi = solve(lp, cfg_it), support.solve_with(O, lp, cfg_it)
        assert max_rel(gi.x, oi.x) <= 1e-10 and max_rel(gi.y, oi.y) <= 1e-10
    g2 = solve(lp, cfg)
    assert g2.iterations == g.iterations and np.array_equal(g2.x, g.x)


def test_operator_budget_and_counters(gpu):
    lp = support.lp_from_json(RANDOM[1]["lp"])
    r = solve(lp, SolverConfig(epsilon=1e-6))
    assert r.spmv_loop == 2 * r.iterations
    assert r.spmv_checks == 2 * r.kkt_checks
    assert r.spmv_setup == 2 * r.power_iterations


def test_limits_and_edge_configs(gpu):
    scalar = LpProblem(1, 1, [0, 1], [0], [1.0], [1.0], [0.0], [INF], [1.0], [INF])
    r = solve(scalar, SolverConfig(time_limit_seconds=0.0))
    assert r.status == "time_limit" and r.iterations == 0
    assert r.residuals.primal_inf == pytest.approx(1.0)
    r = solve(scalar, SolverConfig(iteration_limit=3, epsilon=1e-300))
    assert r.status == "iteration_limit" and r.iterations == 3
    r = solve(scalar, SolverConfig(epsilon=1e-8))
    assert r.status == "optimal" and r.objective == pytest.approx(1.0, rel=1e-6)
    box = LpProblem(0, 3, [0], [], [], [2.0, -1.0, 0.5], [-1.0, -2.0, 0.25], [4.0, 3.0, 5.0],
                    [], [])
    r = solve(box, SolverConfig(epsilon=1e-8))
    assert r.status == "optimal" and r.iterations <= 200
    assert r.x == pytest.approx([-1.0, 3.0, 0.25], rel=1e-6)


def test_restarts_disabled_straight_line(gpu):
    """test_restart_engine.cpp:230-256 analog: without restarts and scaling,
    1000 reflected Halpern steps agree with the reference loop to 1e-10."""
    lp = support.lp_from_json(RANDOM[3]["lp"])
    for gamma in (0.0, 1.0):
        cfg = SolverConfig(scaling_enabled=False, restarts_enabled=False, reflection_gamma=gamma,
                           pid_kp=0.0, epsilon=1e-300, iteration_limit=1000,
                           check_interval=100000)
        g = solve(lp, cfg)
        o = support.solve_with(support.oracle(), lp, cfg)
        assert g.iterations == o.iterations == 1000
        assert max(np.max(np.abs(g.x - o.x)), np.max(np.abs(g.y - o.y))) <= 1e-10


def test_kkt_residuals_match_oracle(gpu):
    for inst in RANDOM:
        lp = support.lp_from_json(inst["lp"])
        sp = inst["spmv"]
        got = vars(kkt_residuals(lp, sp["x"], sp["y"]))
        want = inst["kkt_xy"]
        for k, v in want.items():
            assert got[k] == pytest.approx(v, rel=1e-12, abs=1e-300), k


def test_residual_history_matches_oracle_prefix(gpu):
    lp = support.lp_from_json(RANDOM[4]["lp"])
    cfg = SolverConfig(epsilon=1e-300, iteration_limit=100, record_residual_history=True)
    g = solve(lp, cfg)
    o = support.solve_with(support.oracle(), lp, cfg)
    assert len(g.fixed_point_residual_history) == len(o.fixed_point_residual_history) == 100
    assert max_rel(g.fixed_point_residual_history, o.fixed_point_residual_history) <= 1e-9


def test_invalid_inputs_raise_reference_errors(gpu):
    from paper_2507_14051_b200 import InvalidProblemError, UsageError

    bad = LpProblem(1, 1, [0, 1], [0], [1.0], [1.0], [2.0], [1.0], [0.0], [1.0])
    with pytest.raises(InvalidProblemError):
        solve(bad)
    ok = LpProblem(1, 1, [0, 1], [0], [1.0], [1.0], [0.0], [1.0], [0.0], [1.0])
    with pytest.raises(UsageError):
        solve(ok, SolverConfig(stepsize_multiplier=1.5))


@pytest.mark.parametrize("resident,graph", [(0, True), (0, False), (1, True)],
                         ids=["graph", "plain", "resident"])
def test_device_breakdown_branch(gpu, resident, graph):
    """The indefinite-norm branch of the device control (pdhg.cpp:101-115):
    a step that violates eta ||A|| <= 1 (a = 2, eta = 1, set directly on the
    device: solve() would reject it with UsageError) drives the fixed-point
    radicand below both roundoff floors in the second iteration, q = -18
    exactly (hand value of the reference formulas on this 1x1 LP); the block
    stops there with the breakdown flag, in every engine and launch mode."""
    from paper_2507_14051_b200 import LpProblem

    lp = LpProblem(1, 1, [0, 1], [0], [2.0], [1.0], [-10.0], [10.0], [1.0], [1.0])
    with DeviceContext(lp, use_graph=graph, resident=resident) as dev:
        dev.scale(enabled=False)
        eta = 1.0
        dev.set_step(eta=eta, omega=1.0, gamma=1.0, tau=eta, sigma=eta, sigma_inv=1.0 / eta,
                     primal_scale=1.0 / eta, dual_scale=1.0 / eta, beta_sufficient=0.2,
                     beta_necessary=0.8, beta_artificial=0.36, check_interval=64,
                     iteration_limit=1000, restarts_enabled=0, record_history=0)
        dev.reset_iterate()
        out = dev.run_block()
    assert out["breakdown"] == 1
    assert out["iterations_done"] == 2 and out["q_last"] == -18.0


def test_device_kkt_counts_nan_iterates(gpu):
    """A NaN iterate is counted by the device KKT sums (the host turns the
    count into NumericalBreakdownError, termination.cpp:58-118)."""
    from paper_2507_14051_b200 import LpProblem, NumericalBreakdownError

    lp = LpProblem(1, 1, [0, 1], [0], [2.0], [1.0], [-10.0], [10.0], [1.0], [1.0])
    with DeviceContext(lp, use_graph=False) as dev:
        dev.scale(enabled=False)
        dev.set_iterate([float("nan")], [0.0])
        s = dev.kkt(0)
    assert s["nan_x"] == 1


def const_bound_lps():
    t = c3_transport(S=40, T=70)  # x >= 0, no upper bounds: both variable bounds constant
    # every bound constant (and kept constant: scaling off below)
    r = random_rows_lp(3, 300, 400, np.random.default_rng(2).integers(1, 30, 300))
    r = LpProblem(r.num_cons, r.num_vars, r.row_ptr, r.col_index, r.values, r.objective,
                  [-1.0] * r.num_vars, [2.0] * r.num_vars, [-3.0] * r.num_cons,
                  [math.inf] * r.num_cons)
    return [("transport", t, True, ["var_lb", "var_ub"]),
            ("all_constant_unscaled", r, False, ["var_lb", "var_ub", "con_lb", "con_ub"])]


@pytest.mark.parametrize("rows", ["0", "1"], ids=["merge_path", "thread_rows"])
@pytest.mark.parametrize("case", const_bound_lps(), ids=lambda c: c[0])
def test_constant_bounds_are_parameters_and_change_nothing(gpu, case, rows, monkeypatch):
    """Bounds that are one value on every row / column after scaling are
    passed to the epilogues as kernel parameters instead of loaded
    (ConstInputs, rhp_cuda.cu detect_constant_inputs): detected as such, and
    the solve is bitwise the one that loads them (RHP_CONST_INPUTS=0), in
    graph and plain launches."""
    from paper_2507_14051_b200.lp import set_resident

    _, lp, scaling, want = case
    monkeypatch.setenv("RHP_THREAD_ROWS", rows)
    with DeviceContext(lp) as dev:
        dev.scale(enabled=scaling)
        assert dev.layout()["const_bounds"] == want
    cfg = SolverConfig(epsilon=1e-7, scaling_enabled=scaling)
    out = {}
    try:
        set_resident(0)  # the multi-CTA engines (the resident kernel stages whole vectors)
        for flag in ("1", "0"):
            monkeypatch.setenv("RHP_CONST_INPUTS", flag)
            for graph in (True, False):
                set_device_options(use_graph=graph)
                out[flag, graph] = solve(lp, cfg)
    finally:
        set_resident(-1)
        set_device_options()
    base = out["0", True]
    assert base.status == "optimal"
    for r in out.values():
        assert r.iterations == base.iterations
        assert np.array_equal(r.x, base.x) and np.array_equal(r.y, base.y)


@pytest.mark.parametrize("case", ["transport", "uniform_rows_A", "ragged_short_rows"])
def test_uniform_and_sliced_rows_are_bitwise_the_csr_path(gpu, case, monkeypatch):
    """Thread-per-row operators whose rows all have one length skip the
    row-pointer reads (row i starts at i * len; rhp_cuda.cu
    apply_engine_rule), and with RHP_SLICED=1 read a sliced copy (32-row
    slices, element-major; build_sliced): SpMVs and solves bitwise equal to
    the row-pointer path (RHP_UNIFORM=0) — same elements, same order — with a
    row count that is not a multiple of 32; ragged rows keep row pointers."""
    from paper_2507_14051_b200.lp import set_resident

    rng = np.random.default_rng(4)
    if case == "transport":
        lp, which = c3_transport(S=40, T=70), "At"
    elif case == "uniform_rows_A":  # 1001 rows of exactly 5 distinct columns, box bounds
        m, n = 1001, 777
        cols = np.sort((np.arange(m)[:, None] * 7 + np.arange(5)[None, :] * 131) % n, axis=1)
        lp = LpProblem(m, n, np.arange(0, 5 * m + 1, 5), cols.ravel(),
                       rng.uniform(0.5, 2.0, 5 * m) * rng.choice([-1.0, 1.0], 5 * m),
                       rng.uniform(-1, 1, n), [-1.0] * n, [1.0] * n, [-10.0] * m, [3.0] * m)
        which = "A"
    else:
        lp, which = random_rows_lp(7, 1001, 777, rng.integers(0, 9, 1001)), None
    x, y = rng.uniform(-1, 1, lp.num_vars), rng.uniform(-1, 1, lp.num_cons)
    got = {}
    for mode, env in (("csr", {"RHP_UNIFORM": "0"}), ("uniform", {}), ("sliced", {"RHP_SLICED": "1"})):
        monkeypatch.delenv("RHP_UNIFORM", raising=False)
        monkeypatch.delenv("RHP_SLICED", raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        with DeviceContext(lp) as dev:
            dev.scale()
            lay = dev.layout()
            got[mode, "spmv"] = (dev.spmv(x), dev.spmv(y, True))
        if which:
            assert lay["uniform_rows"][which] == (mode != "csr")
            assert lay["sliced"][which] == (mode == "sliced")
        else:
            assert not any(lay["uniform_rows"].values()) or not lay["thread_rows"]["A"]
        try:
            set_resident(0)
            got[mode, "solve"] = solve(lp, SolverConfig(epsilon=1e-7))
        finally:
            set_resident(-1)
    base = got["csr", "solve"]
    assert base.status == "optimal"
    for mode in ("uniform", "sliced"):
        for a, b in zip(got[mode, "spmv"], got["csr", "spmv"]):
            assert np.array_equal(a, b), mode
        r = got[mode, "solve"]
        assert r.iterations == base.iterations, mode
        assert np.array_equal(r.x, base.x) and np.array_equal(r.y, base.y), mode


def row_band_lp():
    """Rows [1000, 2500) of length 12 whose column advances with the row at
    every element position (row 1000 + r holds columns t * 1500 + r, the
    shape of C4's arc-capacity rows), between ragged random rows (1..20)."""
    rng = np.random.default_rng(11)
    m, n, B = 3000, 18000, 1500
    rows = []
    for i in range(m):
        if 1000 <= i < 2500:
            rows.append(np.arange(12) * B + (i - 1000))
        else:
            rows.append(np.sort(rng.choice(n, rng.integers(1, 21), replace=False)))
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
    ci = np.concatenate(rows)
    v = rng.uniform(0.5, 2.0, len(ci)) * rng.choice([-1.0, 1.0], len(ci))
    return LpProblem(m, n, rp, ci, v, rng.uniform(-1, 1, n), [-1.0] * n, [1.0] * n,
                     [-5.0] * m, [5.0] * m)


@pytest.mark.parametrize("colsegs", [False, True], ids=["plain", "with_column_segments"])
def test_row_band_matches_oracle(gpu, colsegs, monkeypatch):
    """A thread-per-row row band carved out of a merge-path operator
    (rhp_cuda.cu carve_row_band; forced here, the LP is below the size
    thresholds), alone and next to column segments of another row band:
    SpMVs within 1e-13 of the oracle, first iterates within 1e-10, the
    solve's objective within 1e-6 and the oracle's KKT check at eps."""
    lp = row_band_lp()
    monkeypatch.setenv("RHP_ROW_BAND", "force")
    if colsegs:  # 1 KB column segments over rows [0, 1000)
        monkeypatch.setenv("RHP_SEG_BYTES", "1024")
        monkeypatch.setenv("RHP_SEG_FORCE", "1")
        monkeypatch.setenv("RHP_SEG_BAND", "0,1000")
    rng = np.random.default_rng(9)
    x, y = rng.uniform(-1, 1, lp.num_vars), rng.uniform(-1, 1, lp.num_cons)
    O = support.oracle()
    with DeviceContext(lp) as dev:
        dev.scale(enabled=False)
        lay = dev.layout()
        ax, aty = dev.spmv(x), dev.spmv(y, True)
    assert lay["row_band"]["A"] and not lay["row_band"]["At"]
    col_segs = -(-lp.num_vars * 8 // 1024) if colsegs else 1
    assert lay["segments"]["A"] == col_segs + 1
    assert max_rel(ax, support.spmv_with(O, lp, x)) <= 1e-13
    assert max_rel(aty, support.spmv_with(O, lp, y, True)) <= 1e-13
    from paper_2507_14051_b200.lp import set_resident

    k = 100
    cfg = SolverConfig(epsilon=1e-7)
    try:
        set_resident(0)  # the segmented multi-CTA engines
        g = solve(lp, SolverConfig(epsilon=1e-300, iteration_limit=k))
        o = support.solve_with(O, lp, SolverConfig(epsilon=1e-300, iteration_limit=k))
        assert max_rel(g.x, o.x) <= 1e-10 and max_rel(g.y, o.y) <= 1e-10
        g = solve(lp, cfg)
    finally:
        set_resident(-1)
    o = support.solve_with(O, lp, cfg)
    assert g.status == o.status == "optimal"
    assert abs(g.objective - o.objective) <= 1e-6 * max(1.0, abs(o.objective))
    r = support.kkt_with(O, lp, g.x, g.y)
    assert r["gap_rel"] <= 1e-7 and r["primal_rel"] <= 1e-7
