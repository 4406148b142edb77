"""The reference's OWN unit tests (/root/reference/proj/tests/test_*.cpp,
compiled unmodified by `make -C oracle reftests` against this repo's
include/rhpdhg headers and librhpdhg.so, with the doctest stand-in
tests/refshim/doctest.h) run as a test of the drop-in boundary.

The binary is built where /root/reference exists (build()) and travels to
the GPU box as oracle/_ref/ref_unit_tests; it links the PRODUCT library, so
every product, step, norm and scaling it checks runs on the GPU.

Suites: test_lp_model, test_mps_io, test_scaling, test_pdhg_core,
test_restart_engine, test_termination, test_solver (86 test cases; the
acceptance suite needs Eigen and the CLI tests need CLI11, both absent).
"""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "oracle" / "_ref" / "ref_unit_tests"
TOTAL_CASES = 86

# cases that exercise no device code (parsers, config, scoring, scalar rules)
HOST_ONLY = ["project_box clamps", "project_box rejects", "project_box is idempotent",
             "p_support hand values", "p_support is positively", "project_dual_cone reflects",
             "sparse matrix construction validates", "LpProblem validation catches",
             "simple fixture parses", "bounds keys map", "negative UP with unset",
             "ranges follow the standard", "fixed and free format", "OBJSENSE MAX",
             "objective RHS becomes", "markers are ignored", "extra N rows",
             "parse errors carry", "parsing ignores trailing", "canonical text round-trips",
             "gzip input", "solution report document", "empty-problem report",
             "time-limit report flags", "is_optimal applies", "sgm10 formula",
             "size classes follow", "benchmark over an empty", "config files apply",
             "restart conditions fire", "initial weight is one", "default_stepsize arithmetic",
             "step config validation"]


def _need_binary():
    if not BIN.exists():
        pytest.fail(f"{BIN} missing: build() compiles it where /root/reference exists "
                    "(make -C oracle reftests)")


def _run(args, timeout):
    return subprocess.run([str(BIN), *args], capture_output=True, text=True, timeout=timeout,
                          cwd=str(ROOT))


def _summary(out):
    line = [l for l in out.splitlines() if l.startswith("test cases:")][-1]
    f = dict(part.strip().split(": ") for part in line.split("|"))
    return {k: int(v) for k, v in f.items()}


def test_reference_suite_host_cases():
    """The host-only reference cases pass without a GPU (no device code)."""
    _need_binary()
    r = _run(HOST_ONLY, 120)
    s = _summary(r.stdout)
    assert s["test cases"] == len(HOST_ONLY), r.stdout
    assert s["failed"] == 0, r.stderr[-4000:]


@pytest.mark.gpu
def test_reference_suite_all_cases_on_gpu(gpu):
    """All 86 reference unit-test cases, unmodified, against the GPU library."""
    _need_binary()
    r = _run([], 1200)
    s = _summary(r.stdout)
    assert s["test cases"] == TOTAL_CASES, r.stdout
    assert s["failed"] == 0 and r.returncode == 0, r.stderr[-6000:]
