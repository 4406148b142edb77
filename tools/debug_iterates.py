"""Debug helper: compare product vs oracle iterates of one golden LP for a
range of iteration limits (run on the GPU box)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import support  # noqa: E402
from paper_2507_14051_b200 import SolverConfig, solve  # noqa: E402
from paper_2507_14051_b200.device import DeviceContext  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rfl_107_8x12"
inst = next(i for i in support.load_golden("random_feasible.json")["instances"] if i["name"] == name)
lp = support.lp_from_json(inst["lp"])
with DeviceContext(lp) as dev:
    print("layout", dev.layout())
for k in list(range(1, 12)) + [20, 30, 40, 45, 50]:
    cfg = SolverConfig(epsilon=1e-300, iteration_limit=k, record_residual_history=True)
    g = solve(lp, cfg)
    o = support.solve_with(support.oracle(), lp, cfg)
    dx = np.max(np.abs(g.x - o.x)) if lp.num_vars else 0
    dy = np.max(np.abs(g.y - o.y)) if lp.num_cons else 0
    print(f"k={k:3d} rs g/o={g.restart_count}/{o.restart_count} omega g/o={g.final_primal_weight:.6g}/"
          f"{o.final_primal_weight:.6g} |dx|={dx:.3e} |dy|={dy:.3e} xg0={g.x[:3]} xo0={o.x[:3]}")
    if dx > 1e-6:
        print("  hist g", g.fixed_point_residual_history[-8:])
        print("  hist o", o.fixed_point_residual_history[-8:])
        break
