"""CPU checks of bench.py's contract that need no GPU: the reference arm
prints one JSON line with the contract keys (it runs the reference compiled
from its sources on the host), and a WORLD_SIZE that differs from --gpus is
refused instead of silently measuring another world size."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _bench(args, env=None, timeout=600):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                          text=True, timeout=timeout, cwd=str(ROOT), env=e)


def test_reference_arm_contract_line():
    import support

    if not support.ref_available():
        pytest.skip("oracle/_ref not built here")
    r = _bench(["--impl", "reference", "--config", "c1", "--steps", "3", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "PDHG iter/s"
    assert line["unit"] == "iter/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["steps"] == 3 and line["warmup"] == 1
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] == 1 and cb["value"] == line["value"]
    assert cb["host_cores"] >= 1 and cb["cpu_model"]
    assert line["e2e"] == {"value": line["value"], "unit": "iter/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_world_size_mismatch_is_refused():
    r = _bench(["--gpus", "2", "--config", "c1"], env={"WORLD_SIZE": "1"}, timeout=120)
    assert r.returncode != 0
    assert "WORLD_SIZE=1" in (r.stderr + r.stdout)
