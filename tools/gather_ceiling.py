"""Random-gather ceiling probe (run on the GPU box).

Times a kernel that does nothing but the SpMV's irreducible work on C2's own
column indices: stream the int32 index array (and optionally the fp64 values)
coalesced, gather x[idx] (8-B random loads from an L2-resident vector), sum
per thread, write one double per thread. The SpMV kernels cannot beat this
kernel's time for the same index array, so K1/K2 are reported against it.

    python tools/gather_ceiling.py [--out gpurun_out/gather_ceiling.json]

Compiled at run time with torch.utils.cpp_extension.load_inline (probe only;
not part of the product).
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch
from torch.utils.cpp_extension import load_inline

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2507_14051_b200.generators import c2_powerlaw  # noqa: E402

CUDA_SRC = r"""
#include <torch/extension.h>
#include <cuda_runtime.h>
template <int U, bool VALS>
__global__ void __launch_bounds__(256) gather_kernel(const int* __restrict__ idx, const double* __restrict__ v,
                                                     const double* __restrict__ x, long n, double* out) {
  double s = 0.0;
  const long stride = (long)gridDim.x * blockDim.x * U;
  for (long b = (long)blockIdx.x * blockDim.x * U + threadIdx.x; b < n; b += stride) {
    int c[U]; double w[U];
#pragma unroll
    for (int k = 0; k < U; ++k) { long i = b + (long)k * blockDim.x; c[k] = i < n ? __ldcs(idx + i) : 0; w[k] = (VALS && i < n) ? __ldcs(v + i) : 1.0; }
    double g[U];
#pragma unroll
    for (int k = 0; k < U; ++k) g[k] = __ldg(x + c[k]);
#pragma unroll
    for (int k = 0; k < U; ++k) s = fma(w[k], g[k], s);
  }
  out[(long)blockIdx.x * blockDim.x + threadIdx.x] = s;
}
double run(torch::Tensor idx, torch::Tensor v, torch::Tensor x, torch::Tensor out, int blocks, int unroll,
           bool vals, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto launch = [&]() {
    const int* ip = idx.data_ptr<int>(); const double* vp = v.data_ptr<double>();
    const double* xp = x.data_ptr<double>(); double* op = out.data_ptr<double>(); long n = idx.numel();
    if (unroll == 4) { if (vals) gather_kernel<4, true><<<blocks, 256>>>(ip, vp, xp, n, op); else gather_kernel<4, false><<<blocks, 256>>>(ip, vp, xp, n, op); }
    else if (unroll == 8) { if (vals) gather_kernel<8, true><<<blocks, 256>>>(ip, vp, xp, n, op); else gather_kernel<8, false><<<blocks, 256>>>(ip, vp, xp, n, op); }
    else { if (vals) gather_kernel<16, true><<<blocks, 256>>>(ip, vp, xp, n, op); else gather_kernel<16, false><<<blocks, 256>>>(ip, vp, xp, n, op); }
  };
  for (int i = 0; i < 3; ++i) launch();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a); cudaEventDestroy(b);
  return ms / reps;
}
"""
CPP_SRC = ("double run(torch::Tensor idx, torch::Tensor v, torch::Tensor x, torch::Tensor out, "
           "int blocks, int unroll, bool vals, int reps);")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/gather_ceiling.json")
    args = ap.parse_args()
    mod = load_inline("gather_ceiling", CPP_SRC, cuda_sources=CUDA_SRC, functions=["run"],
                      extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"],
                      verbose=False)
    lp = c2_powerlaw()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    res = []
    # A (K1's gather of x over n) and A^T (K2's gather of y over m)
    rp, ci = lp.row_ptr, lp.col_index
    row_of = np.repeat(np.arange(lp.num_cons, dtype=np.int64), np.diff(rp))
    order = np.lexsort((row_of, ci))
    cases = {"A_gather_x": (ci.astype(np.int32), lp.values, lp.num_vars),
             "At_gather_y": (row_of[order].astype(np.int32), lp.values[order], lp.num_cons)}
    for name, (idx_np, v_np, nx) in cases.items():
        idx = torch.from_numpy(idx_np).cuda()
        v = torch.from_numpy(np.ascontiguousarray(v_np)).cuda()
        x = torch.randn(nx, dtype=torch.float64, device="cuda")
        for per_sm in (3, 4, 6, 8):
            for unroll in (4, 8, 16):
                for vals in (False, True):
                    blocks = sms * per_sm
                    out = torch.empty(blocks * 256, dtype=torch.float64, device="cuda")
                    ms = mod.run(idx, v, x, out, blocks, unroll, vals, 20)
                    nnz = idx.numel()
                    res.append({"case": name, "ctas_per_sm": per_sm, "unroll": unroll, "vals": vals,
                                "us": ms * 1e3, "gathers_per_ns": nnz / (ms * 1e6),
                                "stream_gbs": (4 + 8 * vals) * nnz / (ms * 1e-3) / 1e9})
                    print(json.dumps(res[-1]), flush=True)
    best = {}
    for r in res:
        k = (r["case"], r["vals"])
        if k not in best or r["us"] < best[k]["us"]:
            best[k] = r
    print("BEST", json.dumps([best[k] for k in sorted(best)]), flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps({"runs": res, "best": [best[k] for k in sorted(best)]}, indent=1))


if __name__ == "__main__":
    main()
