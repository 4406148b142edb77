import sys, time, json
sys.path.insert(0, '.')
import numpy as np
from paper_2507_14051_b200 import generators
from paper_2507_14051_b200.device import DeviceContext
from paper_2507_14051_b200.lp import Session, SolverConfig
for cfg in sys.argv[1].split(','):
    t=time.perf_counter(); lp = generators.CONFIGS[cfg](); tg=time.perf_counter()-t
    with DeviceContext(lp) as d: pass  # warm context
    t=time.perf_counter()
    with DeviceContext(lp) as d:
        tc=time.perf_counter()-t
    t=time.perf_counter(); s=Session(lp, SolverConfig(epsilon=1e-8)); ts=time.perf_counter()-t
    info=s.info(); s.close()
    print(json.dumps({"cfg":cfg,"gen_s":tg,"create_s":tc,"session_s":ts,"setup_seconds":info["setup_seconds"], "power_its": info.get("power_iterations")}))
