"""One small device workload for tests/test_sanitizer.py, run as its own
process under compute-sanitizer (memcheck / racecheck / synccheck).

    python tools/sanitize_case.py resident|multicta_segments|peer_one_rank|per_op

No torch import: only the product's ctypes bindings, so the sanitizer sees
the product's kernels (and NCCL's for peer_one_rank) and nothing else.
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2507_14051_b200 import SolverConfig, solve  # noqa: E402
from paper_2507_14051_b200.generators import c1_small, random_rows_lp  # noqa: E402
from paper_2507_14051_b200.lp import nccl_unique_id, set_distributed, set_resident  # noqa: E402


def ragged():
    L = np.random.default_rng(5).integers(0, 60, 700)
    L[::97] = 3000  # split rows across warps (ticketed partials)
    return random_rows_lp(17, 700, 900, L)


def main(case):
    cfg = SolverConfig(epsilon=1e-6, iteration_limit=300)
    if case == "resident":  # cluster-resident block kernel (DSMEM reductions)
        rep = solve(c1_small(m=400, n=700), cfg)
    elif case == "multicta_segments":  # merge-path + thread-per-row engines, split rows, segments
        os.environ["RHP_SEG_BYTES"] = "1024"
        os.environ["RHP_SEG_FORCE"] = "1"
        set_resident(0)
        rep = solve(ragged(), cfg)
    elif case == "peer_one_rank":  # NVLink peer exchange protocol, rank = its own peer
        os.environ["RHP_PEER_EXCHANGE"] = "1"
        set_resident(0)
        set_distributed(0, 1, nccl_unique_id())
        rep = solve(ragged(), cfg)
    else:
        raise SystemExit(f"unknown case {case}")
    print(f"{case}: {rep.status} after {rep.iterations} iterations")


if __name__ == "__main__":
    main(sys.argv[1])
