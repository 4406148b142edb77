"""CPU suite: the MPS loader (host C++, rhpdhg::parse_mps_file) — LP load is
part of the drop-in boundary (mps.hpp:17-25). Runs without a GPU."""
import gzip
import math

import numpy as np
import pytest

import support
from paper_2507_14051_b200.lp import ParseError, read_mps, write_mps

ANALYTIC = support.load_golden("analytic_lps.json")["instances"]
REF_FIX = support.Path("/root/reference/proj/tests/fixtures")


def same_lp(a, b):
    assert (a.num_cons, a.num_vars) == (b.num_cons, b.num_vars)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_index, b.col_index)
    assert np.array_equal(a.values, b.values)
    for k in ("objective", "var_lb", "var_ub", "con_lb", "con_ub"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.objective_offset == b.objective_offset and a.maximization == b.maximization


@pytest.mark.parametrize("inst", ANALYTIC, ids=[i["name"] for i in ANALYTIC])
def test_roundtrip_of_golden_analytic_lps(tmp_path, inst):
    lp = support.lp_from_json(inst["lp"])
    if lp.maximization:  # written in min form; read back as min form
        lp.maximization = False
    p = tmp_path / f"{inst['name']}.mps"
    write_mps(lp, p)
    got, _ = read_mps(p)
    same_lp(got, lp)
    with open(p, "rb") as f, gzip.open(str(p) + ".gz", "wb") as g:
        g.write(f.read())
    got_gz, _ = read_mps(str(p) + ".gz")
    same_lp(got_gz, lp)


def test_sections_bounds_ranges_and_warnings(tmp_path):
    text = """NAME demo
OBJSENSE
    MAX
ROWS
 N  obj
 N  extra
 E  e1
 L  l1
 G  g1
COLUMNS
    MARKER   'MARKER'   'INTORG'
    x  obj 1.5D0  e1 1
    MARKER   'MARKER'   'INTEND'
    y  obj -2   l1 3   g1 1
    z  e1 4  extra 9
RHS
    rhs obj 10   e1 2   l1 5   g1 1
RANGES
    rng e1 -1  l1 2  g1 -3
BOUNDS
 UP bnd x -1
 BV bnd y
 FR bnd z
ENDATA
"""
    p = tmp_path / "demo.mps"
    p.write_text(text)
    lp, warnings = read_mps(p)
    assert lp.maximization and lp.objective.tolist() == [-1.5, 2.0, -0.0]
    assert lp.objective_offset == 10.0  # -(-10) after the max negation
    assert lp.con_lb.tolist() == [1.0, 3.0, 1.0] and lp.con_ub.tolist() == [2.0, 5.0, 4.0]
    assert lp.var_lb.tolist() == [-math.inf, 0.0, -math.inf]
    assert lp.var_ub.tolist() == [-1.0, 1.0, math.inf]
    assert any("extra free row" in w for w in warnings)
    assert any("integrality markers" in w for w in warnings)
    assert any("negative UP bound" in w for w in warnings)


@pytest.mark.parametrize("body,frag", [
    ("NAME x\nROWS\n N obj\nCOLUMNS\n x obj 1\n", "missing ENDATA"),
    ("NAME x\nROWS\n N obj\nCOLUMNS\n x obj 1\nROWS\nENDATA\n", "section out of order"),
    ("NAME x\nROWS\n N obj\nCOLUMNS\n x nope 1\nENDATA\n", "undeclared row"),
    ("NAME x\nROWS\n N obj\nCOLUMNS\n x obj 1x\nENDATA\n", "malformed number"),
    ("NAME x\nROWS\n Q r\nENDATA\n", "unknown row sense"),
])
def test_parse_errors_carry_line_numbers(tmp_path, body, frag):
    p = tmp_path / "bad.mps"
    p.write_text(body)
    with pytest.raises(ParseError, match=frag):
        read_mps(p)


@pytest.mark.skipif(not (REF_FIX.is_dir() and support.ref_available()),
                    reason="reference fixtures / oracle/_ref not available")
def test_loader_matches_reference_parser_on_its_fixtures():
    files = sorted(REF_FIX.glob("lp/*.mps")) + sorted(REF_FIX.glob("mps/*.mps"))
    assert files
    for f in files:
        try:
            want = support.ref_lp_from_handle(support.ref().ref_lp_from_mps(str(f).encode()))
        except RuntimeError:
            with pytest.raises(ParseError):
                read_mps(f)
            continue
        got, _ = read_mps(f)
        same_lp(got, want)


# ---------------------------------------------------------------- parallel --
def _mps_variants(tmp_path):
    """Texts that exercise the parallel COLUMNS path and its fallbacks."""
    from paper_2507_14051_b200.generators import c1_small, random_rows_lp

    out = []
    big = random_rows_lp(3, 3000, 5000, np.full(3000, 40))
    p = tmp_path / "big.mps"
    write_mps(big, p)
    out.append(p)
    with open(p, "rb") as f, gzip.open(str(tmp_path / "big.mps.gz"), "wb") as g:
        g.write(f.read())
    out.append(tmp_path / "big.mps.gz")
    # a column that reappears after others (rows must be re-sorted), markers,
    # CRLF line ends and comment lines inside COLUMNS
    lp = c1_small(m=300, n=400)
    p2 = tmp_path / "c1.mps"
    write_mps(lp, p2)
    lines = p2.read_text().splitlines()
    ci = lines.index("COLUMNS")
    body = lines[ci + 1:lines.index("RHS")]
    moved = [l for l in body if l.split()[0] == "X7" and "OBJ" not in l]
    keep = [l for l in body if l not in moved]
    new = (lines[:ci + 1] + ["    MARKER 'MARKER' 'INTORG'"] + keep[:50] +
           ["* a comment", "    MARKER 'MARKER' 'INTEND'"] + keep[50:] + moved +
           lines[lines.index("RHS"):])
    p3 = tmp_path / "reordered.mps"
    p3.write_bytes(("\r\n".join(new) + "\r\n").encode())
    out.append(p3)
    # a duplicate entry (fallback: the sequential reader's ParseError)
    dup = lines[:ci + 1] + body + [body[-1]] + lines[lines.index("RHS"):]
    p4 = tmp_path / "dup.mps"
    p4.write_text("\n".join(dup) + "\n")
    out.append(p4)
    return out


def test_parallel_reader_equals_sequential_reader(tmp_path, monkeypatch):
    for path in _mps_variants(tmp_path):
        monkeypatch.delenv("RHPDHG_MPS_SEQUENTIAL", raising=False)
        try:
            got, gw = read_mps(path)
            gerr = None
        except ParseError as e:
            got, gerr = None, str(e)
        monkeypatch.setenv("RHPDHG_MPS_SEQUENTIAL", "1")
        try:
            want, ww = read_mps(path)
            werr = None
        except ParseError as e:
            want, werr = None, str(e)
        assert gerr == werr, path
        if want is not None:
            same_lp(got, want)
            assert gw == ww, path
    assert werr is not None and "duplicate entry" in werr  # the last variant


@pytest.mark.gpu
def test_gpu_directory_benchmark_sgm10(gpu, tmp_path):
    """rhpdhg::run_benchmark on the GPU (bench.cpp:171-266): analytic LPs plus
    a broken file, the reference's JSON schema, SGM10 rows; 2 workers."""
    import json

    from paper_2507_14051_b200.lp import run_benchmark

    for inst in ANALYTIC[:4]:
        lp = support.lp_from_json(inst["lp"])
        lp.maximization = False
        write_mps(lp, tmp_path / f"{inst['name']}.mps")
    (tmp_path / "broken.mps").write_text("NAME broken\nROWS\nGARBAGE\n")
    out = tmp_path / "report.json"
    for workers in (1, 2):
        table = run_benchmark(str(tmp_path), workers=workers, small_limit_seconds=30.0,
                              json_path=str(out))
        d = json.loads(out.read_text())
        assert d["schema_version"] == 1 and len(d["records"]) == 5
        assert d["records"][0]["instance"] == "boxonly" or d["records"][0]["status"] in (
            "optimal", "error")
        st = {r["instance"]: r["status"] for r in d["records"]}
        assert st["broken"] == "error" and sum(v == "optimal" for v in st.values()) == 4
        assert [s["group"] for s in d["summary"]] == ["small", "medium", "large", "total"]
        assert d["summary"][3]["count"] == 5 and d["summary"][3]["solved"] == 4
        assert "SGM10" in table
