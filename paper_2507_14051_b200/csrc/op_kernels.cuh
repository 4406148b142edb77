// op_kernels.cuh — kernels of the per-operation API (the reference's
// pdhg.hpp / restart.hpp / scaling.hpp functions called one at a time by
// callers and unit tests, include/rhpdhg_cuda.h rhp_op_*). These are device
// round trips of single operations, not the fused solve path: each
// elementwise formula is written with non-contracted ops in the reference's
// evaluation order, so every elementwise output is bit-identical to the
// reference's on identical inputs.
#pragma once
// (kernels are `static`: the header is included by rhp_cuda.cu and ops.cu)

#include "device_common.cuh"

namespace rhp {

// pdhg.cpp:41-45: x+ = min(max(x - tau (c - aty), l), u)
static __global__ void k_op_primal(int64_t n, double tau, const double* __restrict__ x,
                            const double* __restrict__ aty, const double* __restrict__ c,
                            const double* __restrict__ lb, const double* __restrict__ ub,
                            double* __restrict__ xp) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double t = sub(x[j], mul(tau, sub(c[j], aty[j])));
    xp[j] = smin(smax(t, lb[j]), ub[j]);
  }
}

// pdhg.cpp:49-56: amid = 2 ax+ - ax; v = y/sigma - amid;
// proj = min(max(v, -u_c), -l_c); y+ = y - sigma amid - sigma proj
static __global__ void k_op_dual(int64_t m, double sigma, double sigma_inv, const double* __restrict__ y,
                          const double* __restrict__ ax, const double* __restrict__ axp,
                          const double* __restrict__ cl, const double* __restrict__ cu,
                          double* __restrict__ yp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double amid = sub(mul(2.0, axp[i]), ax[i]);
    const double v = sub(mul(sigma_inv, y[i]), amid);
    const double proj = smin(smax(v, -cu[i]), -cl[i]);
    yp[i] = sub(sub(y[i], mul(sigma, amid)), mul(sigma, proj));
  }
}

// out = a - b (pdhg.cpp:60-63 displacements)
static __global__ void k_op_sub(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                         double* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = sub(a[j], b[j]);
}

// restart.cpp:25-30: out = a ((1+g) next - g cur) + b anchor
static __global__ void k_op_affine(int64_t n, double a, double g, double b,
                            const double* __restrict__ next, const double* __restrict__ cur,
                            const double* __restrict__ anchor, double* __restrict__ out) {
  const double opg = 1.0 + g;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = affine(a, opg, g, b, next[j], cur[j], anchor[j]);
}

// out = s * v (scaling.cpp:83-94 unscale_iterate)
static __global__ void k_op_mul(int64_t n, const double* __restrict__ s, const double* __restrict__ v,
                         double* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = mul(s[j], v[j]);
}

// Deterministic sums for the quadratic form and the PID movement norms:
// part[blk*4 + t] = per-block sums of
//   t=0: sum (p[j] - pm[j])^2 (pm may be null), t=1: sum q[i]^2,
//   t=2: sum q[i] (r[i] - rs[i]) (r null: 0; rs null: sum q[i] r[i]),
//   t=3: sum p[j]^2
// (quadratic_form pdhg.cpp:68-75; distance2 / norm2 restart.cpp:8-21)
// Fixed thread->element map and fixed shuffle/warp tree: run-to-run identical.
constexpr int kOpBlock = 256;
constexpr int kOpGrid = 120;

__device__ __forceinline__ void op_block_sum4(double (&acc)[4], double* out) {
  __shared__ double sh[4][kOpBlock / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    double v = acc[t];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) sh[t][w] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      double s = 0.0;
      for (int k = 0; k < kOpBlock / 32; ++k) s += sh[t][k];
      out[t] = s;
    }
  }
}

static __global__ void __launch_bounds__(kOpBlock) k_op_sums4(int64_t n, const double* __restrict__ p,
                                                       const double* __restrict__ pm, int64_t m,
                                                       const double* __restrict__ q,
                                                       const double* __restrict__ r,
                                                       const double* __restrict__ rs,
                                                       double* __restrict__ part) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += stride) {
    const double pj = p[j];
    const double d = pm ? sub(pj, pm[j]) : pj;
    acc[0] = fma(d, d, acc[0]);
    acc[3] = fma(pj, pj, acc[3]);
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += stride) {
    const double qi = q[i];
    acc[1] = fma(qi, qi, acc[1]);
    if (r) acc[2] = fma(qi, rs ? sub(r[i], rs[i]) : r[i], acc[2]);
  }
  op_block_sum4(acc, part + 4 * blockIdx.x);
}

static __global__ void k_op_sums4_final(const double* __restrict__ part, int blocks, double* out) {
  if (threadIdx.x < 4) {
    double s = 0.0;
    for (int b = 0; b < blocks; ++b) s += part[4 * b + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

}  // namespace rhp
