"""Random-gather engine probe (run on the GPU box): is the L1TEX wavefront
limit of LDG gathers (~2 cycles per 8-B random gather per SM, see
profiles/r1_ncu_c2_kernels.md) beaten by the tensor-memory accelerator?

Every variant computes sum(v[i] * x[idx[i]]) over C2's own column indices
(10M random gathers into an 8 MB, L2-resident x) and is timed with CUDA
events:

  ldg      — LDG gathers, U per thread in flight (the SpMV engine's path)
  ldgsts   — cp.async 8-B gathers straight into shared memory (no registers
             held while in flight), 2-stage ring per warp
  g4w4     — TMA tile::gather4 over x viewed as [n/4, 4] (32-B rows = one L2
             sector per gather), each lane issues one gather4 per 128-nnz chunk
  g4w2     — the same over x viewed as [n/2, 2] (16-B rows)
  bulk16   — one 16-B cp.async.bulk per gather

    python tools/tma_gather_probe.py [--out gpurun_out/tma_gather.json]

Probe only (torch.utils.cpp_extension.load_inline); not part of the product.
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
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
               :: "r"(su32(b)), "r"(par) : "memory"); }
__device__ __forceinline__ void g4(void* dst, const CUtensorMap* tm, int r0, int r1, int r2, int r3, uint64_t* b) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               :: "r"(su32(dst)), "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(b)) : "memory"); }
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(b)) : "memory"); }

template <int U>
__global__ void __launch_bounds__(256) k_ldg(const int* __restrict__ idx, const double* __restrict__ v,
                                             const double* __restrict__ x, long n, double* out) {
  double s = 0.0;
  const long stride = (long)gridDim.x * blockDim.x * U;
  for (long b = (long)blockIdx.x * blockDim.x * U + threadIdx.x; b < n; b += stride) {
    int c[U]; double w[U], g[U];
#pragma unroll
    for (int k = 0; k < U; ++k) { long i = b + (long)k * blockDim.x; c[k] = i < n ? __ldcs(idx + i) : 0; w[k] = i < n ? __ldcs(v + i) : 0.0; }
#pragma unroll
    for (int k = 0; k < U; ++k) g[k] = __ldg(x + c[k]);
#pragma unroll
    for (int k = 0; k < U; ++k) s = fma(w[k], g[k], s);
  }
  out[(long)blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// MODE 0: gather4 W=4 (128 B per lane per chunk), 1: gather4 W=2 (64 B used of
// a 128-B lane slot), 2: 4 x 16-B bulk copies per lane (64 B).
template <int MODE, int NB>
__global__ void __launch_bounds__(128) k_tma(const int* __restrict__ idx, const double* __restrict__ v,
                                             const __grid_constant__ CUtensorMap tm, const double* __restrict__ x,
                                             long nchunks, double* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bars[4][NB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* buf = reinterpret_cast<double*>(sm) + (size_t)warp * NB * 512;  // NB slots of 4 KB
  if (lane == 0) for (int s = 0; s < NB; ++s) bar_init(&bars[warp][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long wg = (long)blockIdx.x * 4 + warp, nw = (long)gridDim.x * 4;
  constexpr uint32_t BYTES = MODE == 0 ? 4096u : 2048u;
  auto issue = [&](long ch, int s) {
    if (ch >= nchunks) return;
    const int4 c = __ldcs(reinterpret_cast<const int4*>(idx + ch * 128) + lane);
    if (lane == 0) bar_expect(&bars[warp][s], BYTES);
    __syncwarp();
    double* d = buf + s * 512 + lane * 16;
    if (MODE == 0) g4(d, &tm, c.x >> 2, c.y >> 2, c.z >> 2, c.w >> 2, &bars[warp][s]);
    else if (MODE == 1) g4(d, &tm, c.x >> 1, c.y >> 1, c.z >> 1, c.w >> 1, &bars[warp][s]);
    else {
      bulk(d + 0, x + (c.x & ~1), 16, &bars[warp][s]);
      bulk(d + 2, x + (c.y & ~1), 16, &bars[warp][s]);
      bulk(d + 4, x + (c.z & ~1), 16, &bars[warp][s]);
      bulk(d + 6, x + (c.w & ~1), 16, &bars[warp][s]);
    }
  };
  double acc = 0.0;
  long k = 0;
  for (int s = 0; s < NB; ++s) issue(wg + (long)s * nw, s);
  for (long ch = wg; ch < nchunks; ch += NB * nw) {
#pragma unroll
    for (int s = 0; s < NB; ++s) {
      const long c0 = ch + (long)s * nw;
      if (c0 < nchunks) {
        bar_wait(&bars[warp][s], (uint32_t)(k & 1));
        const int4 c = __ldcs(reinterpret_cast<const int4*>(idx + c0 * 128) + lane);
        const double2 w0 = __ldcs(reinterpret_cast<const double2*>(v + c0 * 128) + 2 * lane);
        const double2 w1 = __ldcs(reinterpret_cast<const double2*>(v + c0 * 128) + 2 * lane + 1);
        const double* d = buf + s * 512 + lane * 16;
        double g0, g1, g2, g3;
        if (MODE == 0) { g0 = d[c.x & 3]; g1 = d[4 + (c.y & 3)]; g2 = d[8 + (c.z & 3)]; g3 = d[12 + (c.w & 3)]; }
        else { g0 = d[c.x & 1]; g1 = d[2 + (c.y & 1)]; g2 = d[4 + (c.z & 1)]; g3 = d[6 + (c.w & 1)]; }
        acc = fma(w0.x, g0, acc); acc = fma(w0.y, g1, acc); acc = fma(w1.x, g2, acc); acc = fma(w1.y, g3, acc);
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(c0 + (long)NB * nw, s);
      }
    }
    ++k;
  }
  out[(long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// cp.async (LDGSTS) gathers: each warp owns a 2-stage ring of 2 x 256
// doubles; lane L gathers elements L + 32 t of a 256-element chunk.
template <int NS>
__global__ void __launch_bounds__(256) k_ldgsts(const int* __restrict__ idx, const double* __restrict__ v,
                                                const double* __restrict__ x, long nchunks, double* out) {
  __shared__ __align__(16) double ring[8][NS][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long wg = (long)blockIdx.x * 8 + warp, nw = (long)gridDim.x * 8;
  auto issue = [&](long ch, int s) {
    if (ch < nchunks) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int c = __ldcs(idx + ch * 256 + t * 32 + lane);
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(&ring[warp][s][t * 32 + lane]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(d), "l"(x + c) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc = 0.0;
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) issue(wg + s * nw, s);
  int s = 0;
  for (long ch = wg; ch < nchunks; ch += nw) {
    issue(ch + (long)(NS - 1) * nw, (s + NS - 1) % NS);
    asm volatile("cp.async.wait_group %0;" :: "n"(NS - 1) : "memory");
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 8; ++t) acc = fma(__ldcs(v + ch * 256 + t * 32 + lane), ring[warp][s][t * 32 + lane], acc);
    __syncwarp();
    s = (s + 1) % NS;
  }
  out[(long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap make_map(const double* x, long n, int w) {
  static EncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    TORCH_CHECK(fn != nullptr, "no cuTensorMapEncodeTiled");
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)(n / w)};
  cuuint64_t strides[1] = {(cuuint64_t)w * 8};
  cuuint32_t box[2] = {(cuuint32_t)w, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)x, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TORCH_CHECK(r == CUDA_SUCCESS, "tensor map encode failed ", (int)r);
  return m;
}

double run(torch::Tensor idx, torch::Tensor v, torch::Tensor x, torch::Tensor out, int variant, int blocks,
           int nb, int reps) {
  const int* ip = idx.data_ptr<int>(); const double* vp = v.data_ptr<double>();
  const double* xp = x.data_ptr<double>(); double* op = out.data_ptr<double>();
  const long n = idx.numel();
  const long nchunks = n / 128;
  CUtensorMap m4 = make_map(xp, x.numel(), 4), m2 = make_map(xp, x.numel(), 2);
  auto launch = [&]() {
    const size_t shm = (size_t)4 * nb * 4096;
    if (variant == 0) {
      if (nb == 16) k_ldg<16><<<blocks, 256>>>(ip, vp, xp, nchunks * 128, op);
      else if (nb == 4) k_ldg<4><<<blocks, 256>>>(ip, vp, xp, nchunks * 128, op);
      else k_ldg<8><<<blocks, 256>>>(ip, vp, xp, nchunks * 128, op);
      return;
    }
    if (variant == 4) {
      if (nb == 2) k_ldgsts<2><<<blocks, 256>>>(ip, vp, xp, nchunks / 2, op);
      else k_ldgsts<3><<<blocks, 256>>>(ip, vp, xp, nchunks / 2, op);
      return;
    }
#define L(MODE, NB) { auto k = k_tma<MODE, NB>; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm); \
      k<<<blocks, 128, shm>>>(ip, vp, MODE == 1 ? m2 : m4, xp, nchunks, op); }
    if (nb == 2) { if (variant == 1) L(0, 2) else if (variant == 2) L(1, 2) else L(2, 2) }
    else if (nb == 4) { if (variant == 1) L(0, 4) else if (variant == 2) L(1, 4) else L(2, 4) }
    else { if (variant == 1) L(0, 8) else if (variant == 2) L(1, 8) else L(2, 8) }
#undef L
  };
  for (int i = 0; i < 3; ++i) launch();
  cudaError_t e = cudaDeviceSynchronize();
  TORCH_CHECK(e == cudaSuccess, cudaGetErrorString(e));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  e = cudaGetLastError();
  TORCH_CHECK(e == cudaSuccess, cudaGetErrorString(e));
  cudaEventDestroy(a); cudaEventDestroy(b);
  return ms / reps;
}
"""
CPP_SRC = ("double run(torch::Tensor idx, torch::Tensor v, torch::Tensor x, torch::Tensor out, int variant, "
           "int blocks, int nb, int reps);")
NAMES = {0: "ldg", 1: "g4w4", 2: "g4w2", 3: "bulk16", 4: "ldgsts"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/tma_gather.json")
    ap.add_argument("--variants", default="0,1,2,3")
    args = ap.parse_args()
    mod = load_inline("tma_gather_probe", CPP_SRC, cuda_sources=CUDA_SRC, functions=["run"],
                      extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo"],
                      extra_ldflags=["-lcuda"], verbose=False)
    lp = c2_powerlaw()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    nnz = (lp.col_index.size // 128) * 128
    idx = torch.from_numpy(lp.col_index[:nnz].astype(np.int32)).cuda()
    v = torch.from_numpy(np.ascontiguousarray(lp.values[:nnz])).cuda()
    x = torch.randn(lp.num_vars + 8, dtype=torch.float64, device="cuda")
    ref = float((v.cpu() * x.cpu()[idx.cpu().long()]).sum())
    res = []
    grid = {0: ((2, 3, 4, 6), (4, 8, 16)), 1: ((2, 3, 4, 6), (2, 4, 8)), 2: ((2, 3, 4, 6), (2, 4, 8)),
            3: ((2, 3, 4, 6), (2, 4, 8)), 4: ((1, 2, 3, 4), (2, 3))}
    for variant in [int(v) for v in args.variants.split(",")]:
        for per_sm in grid[variant][0]:
            for nb in grid[variant][1]:
                if variant in (1, 2, 3) and per_sm * 4 * nb * 4096 > 220 * 1024:
                    continue
                if variant == 4 and per_sm * 8 * nb * 2048 > 220 * 1024:
                    continue
                blocks = sms * per_sm
                out = torch.zeros(blocks * 256, dtype=torch.float64, device="cuda")
                try:
                    ms = mod.run(idx, v, x, out, variant, blocks, nb, 20)
                    got = float(out.sum())
                    err = abs(got - ref) / max(1.0, abs(ref))
                except Exception as e:  # noqa: BLE001
                    print(json.dumps({"variant": NAMES[variant], "error": str(e)}), flush=True)
                    continue
                r = {"variant": NAMES[variant], "ctas_per_sm": per_sm, "nb": nb, "us": ms * 1e3,
                     "gathers_per_ns": nnz / (ms * 1e6),
                     "cycles_per_gather_per_sm": (ms * 1e-3) * 1.965e9 * sms / nnz, "rel_err": err}
                res.append(r)
                print(json.dumps(r), flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
