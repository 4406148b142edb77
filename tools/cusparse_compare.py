"""cuSPARSE fp64 CSR SpMV next to the product's SpMV engine (SURVEY.md §8(f)
rank 4: evidence that the hand-written kernels beat the library call).

For each operator (A and A^T of the named configs) it times, with CUDA events
after warm-up:
  * cusparseSpMV (CUSPARSE_SPMV_CSR_ALG1 and ALG2, int32 indices, fp64),
    y = A x, buffers and descriptors created outside the timed loop;
  * the product's plain SpMV (spmv_fused<EpiStore>, the K1/K2 engine without
    the PDHG epilogue) through DeviceContext.time_spmv;
and checks that both results agree.

    python tools/cusparse_compare.py [--configs c2,c3] [--out gpurun_out/cusparse.json]

Bytes per SpMV (the roofline numerator used everywhere in this repo):
12 nnz + 8 (rows + 1) + 8 cols + 8 rows. Library-call probe only; not part
of the product path.
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

from paper_2507_14051_b200 import generators  # noqa: E402
from paper_2507_14051_b200.device import DeviceContext  # noqa: E402

SRC = r"""
#include <torch/extension.h>
#include <cusparse.h>
#include <cuda_runtime.h>

#define CS(x) do { cusparseStatus_t s_ = (x); TORCH_CHECK(s_ == CUSPARSE_STATUS_SUCCESS, "cusparse ", (int)s_, " at ", __LINE__); } while (0)

// Returns {ms per SpMV, result}
std::vector<torch::Tensor> spmv(torch::Tensor rp, torch::Tensor ci, torch::Tensor v, torch::Tensor x,
                                int64_t rows, int64_t cols, int alg, int reps) {
  cusparseHandle_t h; CS(cusparseCreate(&h));
  cusparseSpMatDescr_t A; cusparseDnVecDescr_t X, Y;
  auto y = torch::zeros({rows}, x.options());
  CS(cusparseCreateCsr(&A, rows, cols, v.numel(), rp.data_ptr<int>(), ci.data_ptr<int>(), v.data_ptr<double>(),
                       CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO, CUDA_R_64F));
  CS(cusparseCreateDnVec(&X, cols, x.data_ptr<double>(), CUDA_R_64F));
  CS(cusparseCreateDnVec(&Y, rows, y.data_ptr<double>(), CUDA_R_64F));
  double one = 1.0, zero = 0.0;
  cusparseSpMVAlg_t a = alg == 2 ? CUSPARSE_SPMV_CSR_ALG2 : CUSPARSE_SPMV_CSR_ALG1;
  size_t bytes = 0;
  CS(cusparseSpMV_bufferSize(h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, X, &zero, Y, CUDA_R_64F, a, &bytes));
  auto buf = torch::empty({(long)bytes + 16}, x.options().dtype(torch::kUInt8));
#if CUSPARSE_VERSION >= 12400
  CS(cusparseSpMV_preprocess(h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, X, &zero, Y, CUDA_R_64F, a, buf.data_ptr()));
#endif
  for (int i = 0; i < 3; ++i)
    CS(cusparseSpMV(h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, X, &zero, Y, CUDA_R_64F, a, buf.data_ptr()));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i)
    CS(cusparseSpMV(h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, A, X, &zero, Y, CUDA_R_64F, a, buf.data_ptr()));
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  cusparseDestroySpMat(A); cusparseDestroyDnVec(X); cusparseDestroyDnVec(Y); cusparseDestroy(h);
  return {torch::full({1}, (double)ms / reps, x.options()), y};
}
"""
CPP = ("std::vector<torch::Tensor> spmv(torch::Tensor rp, torch::Tensor ci, torch::Tensor v, torch::Tensor x, "
       "int64_t rows, int64_t cols, int alg, int reps);")


def transpose(m, n, rp, ci, v):
    row = np.repeat(np.arange(m, dtype=np.int64), np.diff(rp))
    order = np.lexsort((row, ci))
    trp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(trp, ci + 1, 1)
    return np.cumsum(trp), row[order], v[order]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c3")
    ap.add_argument("--out", default="gpurun_out/cusparse.json")
    args = ap.parse_args()
    mod = load_inline("cusparse_compare", CPP, cuda_sources=SRC, functions=["spmv"],
                      extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"],
                      extra_ldflags=["-lcusparse"], verbose=False)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    res = []
    for cfg in args.configs.split(","):
        lp = generators.CONFIGS[cfg]()
        m, n = lp.num_cons, lp.num_vars
        ops = {"A": (m, n, lp.row_ptr, lp.col_index, lp.values),
               "At": (n, m) + transpose(m, n, lp.row_ptr, lp.col_index, lp.values)}
        with DeviceContext(lp) as dev:
            ours = {"A": dev.time_spmv(False, 20), "At": dev.time_spmv(True, 20)}
            rng = np.random.default_rng(1)
            for name, (rows, cols, rp, ci, v) in ops.items():
                xh = rng.uniform(-1, 1, cols)
                mine = dev.spmv(xh, transpose=(name == "At"))
                x = torch.from_numpy(xh).cuda()
                t_rp = torch.from_numpy(rp.astype(np.int32)).cuda()
                t_ci = torch.from_numpy(ci.astype(np.int32)).cuda()
                t_v = torch.from_numpy(np.ascontiguousarray(v)).cuda()
                nb = 12 * ci.size + 8 * (rows + 1) + 8 * cols + 8 * rows
                r = {"config": cfg, "op": name, "rows": rows, "cols": cols, "nnz": int(ci.size),
                     "bytes": nb, "ours_us": ours[name] * 1e3,
                     "ours_gbs": nb / (ours[name] * 1e-3) / 1e9}
                for alg in (1, 2):
                    ms, y = mod.spmv(t_rp, t_ci, t_v, x, rows, cols, alg, 20)
                    ms = float(ms[0])
                    yc = y.cpu().numpy()
                    r[f"cusparse_alg{alg}_us"] = ms * 1e3
                    r[f"cusparse_alg{alg}_gbs"] = nb / (ms * 1e-3) / 1e9
                    r[f"max_rel_diff_alg{alg}"] = float(np.max(np.abs(yc - mine)) /
                                                        max(1e-300, np.max(np.abs(yc))))
                r["speedup_vs_best_cusparse"] = min(r["cusparse_alg1_us"], r["cusparse_alg2_us"]) / r["ours_us"]
                r["ours_frac_of_hbm"] = r["ours_gbs"] / peak
                print(json.dumps(r), flush=True)
                res.append(r)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
