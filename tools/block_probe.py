"""Per-block timing probe (run on the GPU box): device time of one block of
PDHG iterations (rhp_last_block_ms) vs the wall time of the host loop around
it, for the resident and multi-CTA engines.

    python tools/block_probe.py [c1|c3|c2]
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2507_14051_b200 import generators  # noqa: E402
from paper_2507_14051_b200.device import DeviceContext  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c1"
lp = generators.CONFIGS[cfgname]()
for resident in (1, 0):
    for graph in (True, False):
        with DeviceContext(lp, use_graph=graph) as dev:
            dev.lib.rhp_destroy(dev.h)  # re-create with the resident option
            from paper_2507_14051_b200 import capi
            import ctypes as C

            opt = capi.RhpOptions(device=0, rank=0, world_size=1, use_graph=int(graph),
                                  block_limit=64, nccl_id=None, resident=resident)
            h = C.c_void_p()
            dev._ok(dev.lib.rhp_create(C.byref(dev._view), C.byref(opt), C.byref(h)))
            dev.h = h
            dev.scale()
            eta = 0.5
            dev.set_step(eta=eta, omega=1.0, gamma=1.0, tau=eta, sigma=eta, sigma_inv=1 / eta,
                         primal_scale=1 / eta, dual_scale=1 / eta, beta_sufficient=0.2,
                         beta_necessary=0.8, beta_artificial=0.36, check_interval=64,
                         iteration_limit=2**62, restarts_enabled=0, record_history=0)
            dev.reset_iterate()
            for _ in range(3):
                dev.run_block()
            dms, wall, its = [], [], 0
            for _ in range(20):
                t = time.perf_counter()
                out = dev.run_block()
                wall.append(time.perf_counter() - t)
                dms.append(dev.last_block_ms())
                its += out["iterations_done"]
            t = time.perf_counter()
            for _ in range(5):
                dev.kkt(0)
            kkt = (time.perf_counter() - t) / 5
            print(f"{cfgname} resident={resident} graph={graph}: iters/block={its / 20:.0f} "
                  f"device {np.mean(dms) * 1e3 / (its / 20):.2f} us/iter, wall "
                  f"{np.mean(wall) * 1e6 / (its / 20):.2f} us/iter, kkt check {kkt * 1e6:.0f} us",
                  flush=True)
