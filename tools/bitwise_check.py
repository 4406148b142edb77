"""Solve a config for a fixed iteration count with the library found via
RHPDHG_LIB_DIR (or the in-tree build) and save x, y: for bitwise A/B of
builds that must not change results.
  python tools/bitwise_check.py c2 400 out.npz"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_14051_b200 import SolverConfig, generators, solve  # noqa: E402

cfg, iters, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
lp = generators.CONFIGS[cfg]()
rep = solve(lp, SolverConfig(epsilon=1e-300, iteration_limit=iters))
np.savez(out, x=np.asarray(rep.x), y=np.asarray(rep.y), it=rep.iterations)
print(cfg, rep.iterations, rep.objective)
