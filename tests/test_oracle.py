"""CPU suite: pins the C oracle (oracle/rhpdhg_oracle.c) against the
reference — bit-for-bit against the reference library compiled from its own
sources (oracle/_ref, when present) and against the committed golden
fixtures generated from the reference (tests/golden, tools/make_golden.py)."""
import math

import numpy as np
import pytest

import support
from paper_2507_14051_b200.generators import c1_small, c3_transport, random_rows_lp
from paper_2507_14051_b200.lp import SolverConfig

ANALYTIC = support.load_golden("analytic_lps.json")["instances"]
RANDOM = support.load_golden("random_feasible.json")["instances"]
SUITE = support.load_golden("random_suite.json")["instances"]

needs_ref = pytest.mark.skipif(not support.ref_available(), reason="oracle/_ref not built")


def same_report(a, b):
    assert a["status"] == b["status"]
    for k in ("iterations", "restart_count", "kkt_checks", "power_iterations", "spmv_loop",
              "spmv_checks", "spmv_setup"):
        assert a[k] == b[k], k
    for k in ("objective", "final_primal_weight", "matrix_norm_estimate"):
        assert a[k] == b[k] or (math.isnan(a[k]) and math.isnan(b[k])), k
    assert a["x"] == b["x"] and a["y"] == b["y"]
    for k, v in a["residuals"].items():
        assert v == b["residuals"][k], k


@pytest.mark.parametrize("inst", ANALYTIC, ids=[i["name"] for i in ANALYTIC])
@pytest.mark.parametrize("eps", ["0.0001", "1e-08"])
def test_oracle_matches_golden_analytic(inst, eps):
    lp = support.lp_from_json(inst["lp"])
    got = support.report_summary(support.solve_with(support.oracle(), lp,
                                                    SolverConfig(epsilon=float(eps))))
    same_report(got, inst["results"][eps])


@pytest.mark.parametrize("inst", SUITE[::5], ids=[i["name"] for i in SUITE[::5]])
def test_oracle_matches_golden_random_suite(inst):
    lp = support.lp_from_json(inst["lp"])
    got = support.report_summary(support.solve_with(
        support.oracle(), lp, SolverConfig(epsilon=1e-8, iteration_limit=20000)))
    same_report(got, inst["result_1e-8_cap20k"])
    if got["status"] == "optimal":  # HiGHS objective of the fixture, 1e-5 relative
        h = inst["highs_objective"]
        assert abs(got["objective"] - h) <= 1e-5 * max(1.0, abs(h))


def test_golden_random_suite_meets_acceptance_criterion_2():
    """With the stock (no-FMA) reference build all 50 fixture LPs reach 1e-8
    and match HiGHS to 1e-5 (acceptance_main.cpp:153-215). SURVEY.md's 4
    '+inf gap' instances come from a -march=native (FMA-contracted) build:
    the defect is roundoff-triggered."""
    for i in SUITE:
        r = i["result_1e-8_cap20k"]
        assert r["status"] == "optimal", i["name"]
        h = i["highs_objective"]
        assert abs(r["objective"] - h) <= 1e-5 * max(1.0, abs(h)), i["name"]


@pytest.mark.parametrize("inst", RANDOM, ids=[i["name"] for i in RANDOM])
def test_oracle_matches_golden_pieces(inst):
    lp = support.lp_from_json(inst["lp"])
    O = support.oracle()
    same_report(support.report_summary(support.solve_with(O, lp, SolverConfig(epsilon=1e-8))),
                inst["solve_1e-8"])
    sc = support.scale_with(O, lp)
    for k, v in inst["scaling"].items():
        assert sc[k].tolist() == v, k
    assert support.power_with(O, lp) == (inst["power"]["value"], inst["power"]["iterations"],
                                         inst["power"]["converged"])
    sp = inst["spmv"]
    assert support.spmv_with(O, lp, sp["x"]).tolist() == sp["ax"]
    assert support.spmv_with(O, lp, sp["y"], True).tolist() == sp["aty"]
    assert support.kkt_with(O, lp, sp["x"], sp["y"]) == inst["kkt_xy"]
    for k, snap in inst["snapshots"].items():
        r = support.solve_with(O, lp, SolverConfig(epsilon=1e-300, iteration_limit=int(k)))
        assert r.x.tolist() == snap["x"] and r.y.tolist() == snap["y"], k


@needs_ref
@pytest.mark.parametrize("maker", [
    lambda: c1_small(m=300, n=600),
    lambda: random_rows_lp(7, 400, 500, np.random.default_rng(1).integers(1, 40, 400)),
    lambda: c3_transport(S=20, T=30),
], ids=["c1_like", "ragged", "transport"])
def test_oracle_bitwise_equals_reference(maker):
    lp = maker()
    for cfg in (SolverConfig(epsilon=1e-6), SolverConfig(epsilon=1e-4, scaling_enabled=False),
                SolverConfig(epsilon=1e-300, iteration_limit=300, restarts_enabled=False,
                             reflection_gamma=0.5, record_residual_history=True)):
        a = support.solve_with(support.oracle(), lp, cfg)
        b = support.solve_with(support.ref(), lp, cfg)
        same_report(support.report_summary(a), support.report_summary(b))
        assert a.fixed_point_residual_history.tolist() == b.fixed_point_residual_history.tolist()
    assert support.power_with(support.oracle(), lp) == support.power_with(support.ref(), lp)
    so, sr = support.scale_with(support.oracle(), lp), support.scale_with(support.ref(), lp)
    for k in so:
        assert np.array_equal(so[k], sr[k]), k


@needs_ref
def test_oracle_power_start_matches_mt19937_64():
    """v_j = 2*U53 - 1 from std::mt19937_64 (pdhg.cpp:127-128): the oracle's C
    generator agrees with the reference's power iteration end to end."""
    lp = c1_small(m=50, n=80, per_row=5)
    for seed in (0, 1, 12345):
        assert support.power_with(support.oracle(), lp, seed=seed) == \
            support.power_with(support.ref(), lp, seed=seed)
