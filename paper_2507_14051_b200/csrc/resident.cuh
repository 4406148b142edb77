// resident.cuh — the cluster-resident PDHG block kernel for small LPs.
//
// For LPs whose whole iteration is a few hundred KB, launch latency and the
// dependent global round trips of the K1/K2 path dominate (~10 us per
// kernel). Here ONE thread-block cluster (up to 16 CTAs of 1024 threads, one
// per SM) runs a whole device block of iterations in a single launch. Each
// CTA owns a contiguous slice of the rows of A and of A^T (balanced by
// nonzeros); at launch it copies its two CSR slices into shared memory (they
// are constant), so every row sum reads the matrix from shared memory and
// only the x+/y+ gather goes to L2. Per iteration:
//
//   publish x-side partial sums (smem, buffer t&1)
//   cluster barrier 1            (x+ complete everywhere)
//   A x+ for this CTA's rows + dual/Halpern epilogue (EpiDual::row);
//   publish y-side partial sums
//   cluster barrier 2            (y+ complete everywhere)
//   every CTA sums all CTAs' partials in rank order through DSMEM and runs
//   the same control (pdhg_control on a shared-memory copy of Ctl)
//   A^T y+ for this CTA's columns + aty Halpern + next primal step
//   (EpiAty::row), unless the control stopped the block
//
// Same per-element formulas as K1/K2 (the Epi*::row functions); only
// summation orders differ from the multi-CTA path. Vectors written by other
// CTAs inside the kernel (x+, y+) are gathered with coherent L2 loads; the
// cluster barrier's release/acquire orders them.
#pragma once

#include <cooperative_groups.h>

#include "pdhg_kernels.cuh"

namespace rhp {

#ifndef RHP_RES_THREADS
#define RHP_RES_THREADS 512  // C1: 122k (256) -> 125k iter/s; 1024 exceeds shared memory
#endif
constexpr int kResThreads = RHP_RES_THREADS;
constexpr int kResWarps = kResThreads / 32;
constexpr int kResMaxCtas = 16;
constexpr size_t kResSmemMax = 200 * 1024;  // per-CTA matrix slices must fit

struct ResParams {
  Csr A, At;
  const double* xp;         // x+ (gathered by A x+; written by other CTAs in-kernel)
  const double* yp;         // y+ (gathered by A^T y+)
  const int32_t* a_split;   // [C+1] rows of A per CTA
  const int32_t* at_split;  // [C+1] rows of A^T per CTA
  int wa, wat;              // lanes per row for A and A^T
  EpiDual dual;             // pointers set; scalars refreshed per iteration
  EpiAty aty;
  EpiPrimal primal;
  Ctl* ctl;
};

// A CSR slice staged in shared memory: rows [r0, r1), row pointers relative
// to the slice's first nonzero.
struct Slice {
  int64_t r0, r1;
  const int32_t* rp;
  const int32_t* ci;
  const double* v;
};

__device__ __forceinline__ unsigned char* align16p(unsigned char* p) {
  return reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
}

__device__ __forceinline__ Slice stage_slice(const Csr& M, int64_t r0, int64_t r1,
                                             unsigned char*& cursor) {
  const int64_t b = M.rp[r0], nz = M.rp[r1] - b, rows = r1 - r0;
  int32_t* rp = reinterpret_cast<int32_t*>(cursor);
  cursor = align16p(cursor + 4 * (rows + 1));
  double* v = reinterpret_cast<double*>(cursor);
  cursor = align16p(cursor + 8 * nz);
  int32_t* ci = reinterpret_cast<int32_t*>(cursor);
  cursor = align16p(cursor + 4 * nz);
  for (int64_t i = threadIdx.x; i <= rows; i += blockDim.x)
    rp[i] = static_cast<int32_t>(M.rp[r0 + i] - b);
  for (int64_t e = threadIdx.x; e < nz; e += blockDim.x) {
    v[e] = M.v[b + e];
    ci[e] = M.ci[b + e];
  }
  return Slice{r0, r1, rp, ci, v};
}

// Row-group walk shared by the block-start primal step and the A^T pass, so
// a column's partial sums land in the same thread in both (block-length
// invariance of the residual).
template <int W, class F>
__device__ __forceinline__ void rows_by_groups(const Slice& S, const double* xg, bool sum,
                                               F&& on_row) {
  const int g = threadIdx.x / W, lane = threadIdx.x % W;
  constexpr int G = kResThreads / W;
  for (int64_t rr = S.r0; rr < S.r1; rr += G) {  // uniform trip count across the CTA
    const int64_t r = rr + g;
    double s = 0.0;
    if (sum && r < S.r1) {
      const int lo = S.rp[r - S.r0], hi = S.rp[r - S.r0 + 1];
      for (int e = lo + lane; e < hi; e += 4 * W) {  // 4 predicated gathers in flight
        double xv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) xv[k] = e + k * W < hi ? __ldcg(xg + S.ci[e + k * W]) : 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k)  // sequential sum in element order
          if (e + k * W < hi) s = fma(S.v[e + k * W], xv[k], s);
      }
    }
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0 && r < S.r1) on_row(r, s);
  }
}

template <class F>
__device__ __forceinline__ void rows_dispatch(int w, const Slice& S, const double* xg, bool sum,
                                              F&& on_row) {
  switch (w) {
    case 1: rows_by_groups<1>(S, xg, sum, on_row); break;
    case 2: rows_by_groups<2>(S, xg, sum, on_row); break;
    case 4: rows_by_groups<4>(S, xg, sum, on_row); break;
    case 8: rows_by_groups<8>(S, xg, sum, on_row); break;
    case 16: rows_by_groups<16>(S, xg, sum, on_row); break;
    default: rows_by_groups<32>(S, xg, sum, on_row); break;
  }
}

// Warp-level butterfly of N partials; lane 0 publishes them (no CTA barrier).
template <int N>
__device__ __forceinline__ void warp_publish(const double* acc, double* out) {
#pragma unroll
  for (int q = 0; q < N; ++q) {
    double v = acc[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0) out[q] = v;
  }
}

__global__ void __launch_bounds__(kResThreads) k_resident(ResParams p) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int cta = static_cast<int>(cl.block_rank());
  extern __shared__ __align__(16) unsigned char rsm[];
  __shared__ Ctl lc;  // this CTA's copy of the loop control
  // per-warp partials of iteration parity t&1: [0..4] y-side, [5..8] x-side
  __shared__ double wpub[2][kResWarps][9];
  __shared__ double gath[9][kResMaxCtas * kResWarps];
  if (threadIdx.x == 0) {
    lc = *p.ctl;
    lc.graph_mode = 0;
    if (cta != 0) lc.record_history = 0;  // CTA 0 writes the history
    lc.stop = 0;
    lc.block_iters = 0;
  }
  unsigned char* cursor = rsm;
  const Slice SA = stage_slice(p.A, p.a_split[cta], p.a_split[cta + 1], cursor);
  const Slice ST = stage_slice(p.At, p.at_split[cta], p.at_split[cta + 1], cursor);
  // this CTA's rows of the iterate live in shared memory for the whole block:
  //   A side  [y, ax, con_lb, con_ub, y0, ax0]        (EpiDual input order)
  //   A^T side [aty, aty0, x, c, var_lb, var_ub, x0]  (EpiAty input order)
  const int ra = static_cast<int>(SA.r1 - SA.r0), rt = static_cast<int>(ST.r1 - ST.r0);
  double* sa = reinterpret_cast<double*>(cursor);
  double* st = sa + 6 * ra;
  EpiDual dual = p.dual;
  EpiAty aty = p.aty;
  EpiPrimal pr = p.primal;
  for (int k = 0; k < 6; ++k)
    for (int i = threadIdx.x; i < ra; i += kResThreads) sa[k * ra + i] = dual.in[k][SA.r0 + i];
  for (int k = 0; k < 7; ++k)
    for (int j = threadIdx.x; j < rt; j += kResThreads) st[k * rt + j] = aty.in[k][ST.r0 + j];
  __syncthreads();
  // outputs of the epilogues: state in shared memory, x+/y+ to global
  double* const y_g = dual.y;
  double* const ax_g = dual.ax;
  double* const aty_g = aty.aty;
  double* const x_g = aty.o.x;
  dual.y = sa - SA.r0;
  dual.ax = sa + ra - SA.r0;
  aty.aty = st - ST.r0;
  aty.o.x = st + 2 * rt - ST.r0;
  pr.o.x = aty.o.x;

  // block start: primal step for this CTA's columns (same row->thread walk as
  // the A^T pass, no row sums)
  double acc3[4] = {0.0, 0.0, 0.0, 0.0};
  pr.a = halpern_a(lc.k);
  pr.b = halpern_b(lc.k);
  pr.g = lc.gamma;
  pr.opg = 1.0 + lc.gamma;
  pr.tau = lc.tau;
  rows_dispatch(p.wat, ST, p.yp, false, [&](int64_t j, double) {
    const int l = static_cast<int>(j - ST.r0);
    const double e[6] = {st[l], st[2 * rt + l], st[3 * rt + l], st[4 * rt + l], st[5 * rt + l],
                         st[6 * rt + l]};
    pr.row(j, 0.0, e, 1, acc3);
  });
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned nb = cl.num_blocks();
  const int nw = static_cast<int>(nb) * kResWarps;  // partials per quantity in the cluster
  for (int it = 0;; ++it) {
    double(*mine)[9] = wpub[it & 1];
    warp_publish<4>(acc3, &mine[warp][5]);
    cl.sync();  // (1) x+ and the x-side partials are complete in every CTA
    dual.sigma = lc.sigma;
    dual.sigma_inv = lc.sigma_inv;
    dual.a = halpern_a(lc.k);
    dual.b = halpern_b(lc.k);
    dual.g = lc.gamma;
    dual.opg = 1.0 + lc.gamma;
    double acc1[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    rows_dispatch(p.wa, SA, p.xp, true, [&](int64_t i, double s) {
      dual.row(i, s, sa + (i - SA.r0), ra, acc1);
    });
    warp_publish<5>(acc1, &mine[warp][0]);
    cl.sync();  // (2) y+ and the y-side partials are complete in every CTA
    // warp q reduces quantity q over all warps of the cluster straight from
    // DSMEM (lane-strided loads issued together, fixed butterfly order) ...
    for (int q = warp; q < 9; q += kResWarps) {
      double vals[kResMaxCtas * kResWarps / 32];
#pragma unroll
      for (int k = 0; k < kResMaxCtas * kResWarps / 32; ++k) {
        const int src = lane + 32 * k;
        vals[k] = src < nw ? cl.map_shared_rank(&mine[0][0], src / kResWarps)[(src % kResWarps) * 9 + q]
                           : 0.0;
      }
      double v = 0.0;
#pragma unroll
      for (int k = 0; k < kResMaxCtas * kResWarps / 32; ++k) v += vals[k];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) gath[q][0] = v;
    }
    __syncthreads();
    // ... then one thread runs the control on the cluster totals
    if (threadIdx.x == 0) {
      double sums[9];
      for (int q = 0; q < 9; ++q) sums[q] = gath[q][0];
      pdhg_control(&lc, sums, sums + 5, 0);
    }
    __syncthreads();
    const bool stop = lc.stop != 0;
    aty.a = halpern_a(lc.k - 1);
    aty.b = halpern_b(lc.k - 1);
    aty.a2 = halpern_a(lc.k);
    aty.b2 = halpern_b(lc.k);
    aty.g = lc.gamma;
    aty.opg = 1.0 + lc.gamma;
    aty.tau = lc.tau;
    aty.stop = stop;
    acc3[0] = acc3[1] = acc3[2] = acc3[3] = 0.0;
    rows_dispatch(p.wat, ST, p.yp, true, [&](int64_t j, double s) {
      aty.row(j, s, st + (j - ST.r0), rt, acc3);
    });
    if (stop) break;
  }
  __syncthreads();
  // write the iterate back for the host-side check / restart
  for (int i = threadIdx.x; i < ra; i += kResThreads) {
    y_g[SA.r0 + i] = sa[i];
    ax_g[SA.r0 + i] = sa[ra + i];
  }
  for (int j = threadIdx.x; j < rt; j += kResThreads) {
    aty_g[ST.r0 + j] = st[j];
    x_g[ST.r0 + j] = st[2 * rt + j];
  }
  cl.sync();  // every CTA's last stores and DSMEM reads are done
  if (cta == 0 && threadIdx.x == 0) {
    lc.graph_mode = p.ctl->graph_mode;
    lc.record_history = p.ctl->record_history;
    *p.ctl = lc;
  }
}

}  // namespace rhp
