#!/bin/bash
# Per-phase setup times of a session on a bench config: tools/setup_trace.sh c4
cd "$(dirname "$0")/.."
RHPDHG_SETUP_TRACE=1 python - "$@" <<'PY'
import sys, time
sys.path.insert(0, '.')
from paper_2507_14051_b200 import generators
from paper_2507_14051_b200.lp import Session, SolverConfig
for cfg in sys.argv[1:] or ['c4']:
    t = time.perf_counter(); lp = generators.CONFIGS[cfg](); print(cfg, 'generate', round(time.perf_counter() - t, 3), file=sys.stderr)
    for rep in range(2):
        t = time.perf_counter(); s = Session(lp, SolverConfig(epsilon=1e-8)); info = s.info(); s.close()
        print(cfg, 'session', rep, round(time.perf_counter() - t, 3), 'setup_seconds', info['setup_seconds'], 'power_its', info.get('power_iterations'), file=sys.stderr)
PY
