"""CPU suite: the native libraries load and export every symbol that
include/*.h declares (no compute calls: there is no GPU here)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2507_14051_b200 import capi

ROOT = Path(__file__).resolve().parent.parent


def declared(header):
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b((?:rhp|rhpdhg)_[a-z_0-9]+)\s*\(", text)))


def exported(so):
    out = subprocess.run(["nm", "-D", "--defined-only", str(so)], capture_output=True, text=True,
                         check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


@pytest.mark.parametrize("header,so", [("rhpdhg_cuda.h", "librhp_cuda.so"),
                                       ("rhpdhg_c.h", "librhpdhg.so")])
def test_library_exports_every_declared_symbol(header, so):
    path = capi.LIB_DIR / so
    assert path.exists(), f"{path} not built"
    missing = [s for s in declared(header) if s not in exported(path)]
    assert not missing, missing


def test_python_binding_lists_match_headers():
    assert sorted(capi.CUDA_SYMBOLS) == declared("rhpdhg_cuda.h")
    assert sorted(capi.HOST_SYMBOLS) == declared("rhpdhg_c.h")


def test_libraries_load_and_bind():
    cuda = capi.load_cuda()
    host = capi.load_host()
    for s in capi.CUDA_SYMBOLS:
        assert hasattr(cuda, s)
    for s in capi.HOST_SYMBOLS:
        assert hasattr(host, s)


def test_device_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(capi.LIB_DIR / "librhp_cuda.so")],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out
    for other in ("sm_80", "sm_90"):
        assert other not in out


def test_struct_layouts_match_c():
    """Sizes of the ctypes mirrors equal sizeof() of the C structs (compiled probe)."""
    probe = ROOT / "tests" / "_layout_probe.c"
    exe = Path("/tmp") / "rhpdhg_layout_probe"
    probe.write_text(
        '#include <stdio.h>\n#include "rhpdhg_cuda.h"\n'
        'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(rhpdhg_lp_view),'
        ' sizeof(rhpdhg_config_c), sizeof(rhpdhg_kkt_c), sizeof(rhpdhg_report_c),'
        ' sizeof(rhp_options), sizeof(rhp_step), sizeof(rhp_block_out), sizeof(rhp_kkt_sums),'
        ' sizeof(rhp_layout_info)); return 0;}\n')
    try:
        subprocess.run(["gcc", "-I", str(ROOT / "include"), str(probe), "-o", str(exe)], check=True)
        sizes = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True,
                                             check=True).stdout.split()))
    finally:
        probe.unlink(missing_ok=True)
    mine = [C.sizeof(t) for t in (capi.LpView, capi.ConfigC, capi.KktC, capi.ReportC,
                                  capi.RhpOptions, capi.RhpStep, capi.RhpBlockOut,
                                  capi.RhpKktSums, capi.RhpLayoutInfo)]
    assert mine == sizes


def test_solve_without_gpu_fails_loudly():
    """No CPU fallback: a solve without a device raises DeviceError."""
    from paper_2507_14051_b200 import LpProblem, solve, DeviceError
    import support

    if support.have_gpu():
        pytest.skip("a GPU is visible")
    lp = LpProblem(1, 1, [0, 1], [0], [1.0], [1.0], [0.0], [float("inf")], [1.0], [float("inf")])
    with pytest.raises(DeviceError):
        solve(lp)
