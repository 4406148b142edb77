"""Time/iterations to 1e-4, 1e-6, 1e-8 relative KKT for one config through
the resumable session (run on the GPU box).

    python tools/convergence_probe.py c2 [cap]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2507_14051_b200 import generators  # noqa: E402
from paper_2507_14051_b200.lp import Session, SolverConfig  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 500_000
lp = generators.CONFIGS[name]()
t0 = time.perf_counter()
s = Session(lp, SolverConfig(epsilon=1e-8, iteration_limit=cap))
marks = {}
running = True
while running:
    running = s.advance(64 * 16)
    info = s.info()
    r = info["residuals"]
    worst = max(r.gap_rel, r.primal_rel, r.dual_eq / r.dual_denom)
    for eps in (1e-4, 1e-6, 1e-8):
        if eps not in marks and worst <= eps:
            marks[eps] = (info["total"], time.perf_counter() - t0)
            print(json.dumps({"eps": eps, "iterations": info["total"],
                              "seconds": time.perf_counter() - t0}), flush=True)
rep = s.finish()
print(json.dumps({"config": name, "status": rep.status, "iterations": rep.iterations,
                  "restarts": rep.restart_count, "seconds": time.perf_counter() - t0,
                  "setup_s": rep.setup_seconds, "residuals": vars(rep.residuals),
                  "objective": rep.objective}), flush=True)
