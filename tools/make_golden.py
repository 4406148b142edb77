"""Generates the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs only where /root/reference exists (this container): it drives the
unmodified reference library compiled from its own sources
(oracle/_ref/librhpdhg_ref.so, `make ref`) through oracle/ref_adapter.cpp, and
reads the reference's own test fixtures:
  * tests/fixtures/lp/*.mps      -> parsed by the reference's parse_mps_file,
                                    solved by the reference at eps 1e-4 / 1e-8
                                    (SURVEY.md Appendix A golden counters)
  * tests/fixtures/random_lp.json -> the 50 HiGHS-referenced random LPs
                                    (objectives from the fixture), solved by the
                                    reference at 1e-8 with a 20k iteration cap
  * testutil::random_feasible_lp  -> the generator of the reference unit tests
                                    (tests/oracles.hpp:61-110) at the seeds used
                                    there, plus iterate snapshots after k
                                    iterations for the first-100-iterates test
  * scaling / power iteration / SpMV outputs of the reference on those LPs.
The fixtures are written as JSON (Python floats round-trip exactly).

Usage: python tools/make_golden.py   (after `make ref`)
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import support  # noqa: E402
from paper_2507_14051_b200.lp import LpProblem, SolverConfig  # noqa: E402

REF_TESTS = Path("/root/reference/proj/tests")
OUT = ROOT / "tests" / "golden"

ANALYTIC = ["scalar", "twovar", "equality", "boxonly", "freevar", "degenerate", "negbound",
            "maxsense", "range", "fixedvar", "offset", "eqrange"]
# (seed, m, n) of random_feasible_lp calls in the reference unit tests
# (test_solver.cpp:70,84,94; test_restart_engine.cpp:231,259; plus larger ones)
RANDOM_SEEDS = [(103, 10, 15), (107, 8, 12), (109, 8, 12), (79, 5, 5), (83, 12, 18),
                (5001, 30, 45), (5002, 60, 90)]
SNAP_K = [1, 2, 3, 5, 10, 20, 50, 64, 65, 100]


def dense_json_to_lp(inst) -> LpProblem:
    A = np.array(inst["A"], dtype=float)
    m, n = inst["m"], inst["n"]
    rows, cols = np.nonzero(A)
    # null encodes an infinite bound of the side's sign (acceptance_main.cpp:70)
    fix = lambda v, sign: [sign * float("inf") if x is None else float(x) for x in v]
    return LpProblem.from_triplets(m, n, rows, cols, A[rows, cols], objective=fix(inst["c"], 1),
                                   var_lb=fix(inst["var_lb"], -1), var_ub=fix(inst["var_ub"], 1),
                                   con_lb=fix(inst["con_lb"], -1), con_ub=fix(inst["con_ub"], 1),
                                   name=inst["name"])


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    R = support.ref()

    # 1. analytic fixtures
    items = []
    for name in ANALYTIC:
        lp = support.ref_lp_from_handle(
            R.ref_lp_from_mps(str(REF_TESTS / "fixtures" / "lp" / f"{name}.mps").encode()))
        lp.name = name
        res = {}
        for eps in (1e-4, 1e-8):
            r = support.solve_with(R, lp, SolverConfig(epsilon=eps))
            res[repr(eps)] = support.report_summary(r)
        items.append({"name": name, "lp": support.lp_to_json(lp), "results": res})
    (OUT / "analytic_lps.json").write_text(json.dumps(
        {"generator": "tools/make_golden.py", "source": "reference tests/fixtures/lp/*.mps",
         "instances": items}))

    # 2. random suite with HiGHS objectives
    suite = json.loads((REF_TESTS / "fixtures" / "random_lp.json").read_text())
    items = []
    for inst in suite["instances"]:
        lp = dense_json_to_lp(inst)
        r = support.solve_with(R, lp, SolverConfig(epsilon=1e-8, iteration_limit=20000))
        items.append({"name": inst["name"], "highs_objective": inst["reference_objective"],
                      "lp": support.lp_to_json(lp), "result_1e-8_cap20k": support.report_summary(r)})
    (OUT / "random_suite.json").write_text(json.dumps(
        {"generator": "tools/make_golden.py", "source": "reference tests/fixtures/random_lp.json",
         "master_seed": suite.get("master_seed"), "instances": items}))

    # 3. random_feasible_lp instances: full solves, iterate snapshots, setup pieces
    items = []
    for seed, m, n in RANDOM_SEEDS:
        lp = support.ref_lp_from_handle(R.ref_lp_random_feasible(seed, m, n, 0.35))
        lp.name = f"rfl_{seed}_{m}x{n}"
        entry = {"name": lp.name, "seed": seed, "lp": support.lp_to_json(lp)}
        entry["solve_1e-8"] = support.report_summary(
            support.solve_with(R, lp, SolverConfig(epsilon=1e-8)))
        snaps = {}
        for k in SNAP_K:
            r = support.solve_with(R, lp, SolverConfig(epsilon=1e-300, iteration_limit=k))
            snaps[str(k)] = {"x": r.x.tolist(), "y": r.y.tolist(), "restarts": r.restart_count,
                             "omega": r.final_primal_weight}
        entry["snapshots"] = snaps
        sc = support.scale_with(R, lp)
        entry["scaling"] = {k: v.tolist() for k, v in sc.items()}
        val, its, conv = support.power_with(R, lp)
        entry["power"] = {"value": val, "iterations": its, "converged": conv}
        rng = np.random.default_rng(seed)
        xv = rng.uniform(-1, 1, lp.num_vars)
        yv = rng.uniform(-1, 1, lp.num_cons)
        entry["spmv"] = {"x": xv.tolist(), "ax": support.spmv_with(R, lp, xv).tolist(),
                         "y": yv.tolist(), "aty": support.spmv_with(R, lp, yv, True).tolist()}
        entry["kkt_xy"] = support.kkt_with(R, lp, xv, yv)
        items.append(entry)
    (OUT / "random_feasible.json").write_text(json.dumps(
        {"generator": "tools/make_golden.py",
         "source": "reference testutil::random_feasible_lp (tests/oracles.hpp:61-110)",
         "instances": items}))
    print("wrote", sorted(p.name for p in OUT.glob("*.json")))


if __name__ == "__main__":
    main()
