// spmv.cuh — row-length-binned fp64 CSR SpMV with a fused per-row epilogue.
//
// Replaces SparseMatrix::multiply / multiply_transpose
// (/root/reference/proj/src/sparse_matrix.cpp:67-87). Both A and A^T are
// stored explicitly as CSR (A^T = the reference's CSC copy), so neither
// product needs atomics and every output row is produced by exactly one
// thread group in a fixed order (deterministic).
//
// Rows are permuted at ctx creation so that each bin of similar row length
// is contiguous. One launch covers all bins: the flat tile
// index space is split into segments, one per bin, and a persistent grid
// (multiple of the SM count) walks the tiles with a static stride, so block
// partials of the fused reductions have a fixed assignment.
//   kind k in 0..5 : 2^k lanes per row, kBlock/2^k rows per tile. Lane-strided
//                    coalesced loads of values/indices (evict-first), x gather
//                    through the read-only path, xor-butterfly row sum.
//   kind 6         : one CTA per chunk (<= chunk nnz) of a long row; rows of
//                    several chunks are completed by the last chunk to land.
// The epilogue runs once per row with the finished row sum. Rows of a tile
// are staged through shared memory so the epilogue's vector traffic is
// coalesced (thread t handles row row0+t).
#pragma once

#include "device_common.cuh"

namespace rhp {

template <int W>
__device__ __forceinline__ double row_dot(const Csr& A, const double* __restrict__ xg, int64_t row,
                                          int lane) {
  double s0 = 0.0, s1 = 0.0;
  int64_t e = A.rp[row] + lane;
  const int64_t end = A.rp[row + 1];
  // two independent accumulators, four loads in flight per lane
  for (; e + 3 * W < end; e += 4 * W) {
    const int c0 = ld_stream(A.ci + e), c1 = ld_stream(A.ci + e + W);
    const int c2 = ld_stream(A.ci + e + 2 * W), c3 = ld_stream(A.ci + e + 3 * W);
    const double v0 = ld_stream(A.v + e), v1 = ld_stream(A.v + e + W);
    const double v2 = ld_stream(A.v + e + 2 * W), v3 = ld_stream(A.v + e + 3 * W);
    const double x0 = __ldg(xg + c0), x1 = __ldg(xg + c1);
    const double x2 = __ldg(xg + c2), x3 = __ldg(xg + c3);
    s0 = fma(v0, x0, s0);
    s1 = fma(v1, x1, s1);
    s0 = fma(v2, x2, s0);
    s1 = fma(v3, x3, s1);
  }
  for (; e < end; e += W) s0 = fma(ld_stream(A.v + e), __ldg(xg + ld_stream(A.ci + e)), s0);
  return s0 + s1;
}

template <int W, class Epi>
__device__ __forceinline__ void tile_sub(const Csr& A, const double* __restrict__ xg,
                                         const Seg& sg, int64_t tile, Epi& epi,
                                         double (&acc)[Epi::NRED], double* ssum) {
  constexpr int RPT = kBlock / W;
  const int64_t row0 = sg.row_begin + (tile - sg.tile_begin) * RPT;
  const int g = threadIdx.x / W, lane = threadIdx.x % W;
  const int64_t row = row0 + g;
  const bool valid = row < sg.row_end;
  double s = 0.0;
  if constexpr (W == 1) {
    if (valid) {
      int64_t e = A.rp[row];
      const int64_t end = A.rp[row + 1];
      double s1 = 0.0;
      for (; e + 1 < end; e += 2) {
        s = fma(ld_stream(A.v + e), __ldg(xg + ld_stream(A.ci + e)), s);
        s1 = fma(ld_stream(A.v + e + 1), __ldg(xg + ld_stream(A.ci + e + 1)), s1);
      }
      if (e < end) s = fma(ld_stream(A.v + e), __ldg(xg + ld_stream(A.ci + e)), s);
      s += s1;
      epi.row(row, s, acc);
    }
  } else {
    if (valid) s = row_dot<W>(A, xg, row, lane);
    // converged: every lane of the warp takes part in the butterfly
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) ssum[g] = s;
    __syncthreads();
    if (threadIdx.x < RPT && row0 + threadIdx.x < sg.row_end)
      epi.row(row0 + threadIdx.x, ssum[threadIdx.x], acc);
    __syncthreads();
  }
}

template <class Epi>
__device__ __forceinline__ void tile_long(const Csr& A, const double* __restrict__ xg,
                                          const Sched& s, const Seg& sg, int64_t tile, Epi& epi,
                                          double (&acc)[Epi::NRED]) {
  __shared__ double red[kWarps];
  __shared__ double total_s;
  const int64_t chunk = tile - sg.tile_begin;
  const int64_t row = s.chunk_row[chunk];
  const int64_t beg = s.chunk_beg[chunk], end = s.chunk_end[chunk];
  double s0 = 0.0, s1 = 0.0;
  int64_t e = beg + threadIdx.x;
  for (; e + 3 * kBlock < end; e += 4 * kBlock) {
    const int c0 = ld_stream(A.ci + e), c1 = ld_stream(A.ci + e + kBlock);
    const int c2 = ld_stream(A.ci + e + 2 * kBlock), c3 = ld_stream(A.ci + e + 3 * kBlock);
    const double v0 = ld_stream(A.v + e), v1 = ld_stream(A.v + e + kBlock);
    const double v2 = ld_stream(A.v + e + 2 * kBlock), v3 = ld_stream(A.v + e + 3 * kBlock);
    s0 = fma(v0, __ldg(xg + c0), s0);
    s1 = fma(v1, __ldg(xg + c1), s1);
    s0 = fma(v2, __ldg(xg + c2), s0);
    s1 = fma(v3, __ldg(xg + c3), s1);
  }
  for (; e < end; e += kBlock) s0 = fma(ld_stream(A.v + e), __ldg(xg + ld_stream(A.ci + e)), s0);
  double v = s0 + s1;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) t += red[w];
    total_s = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int slot = s.chunk_slot[chunk];
    if (slot < 0) {
      epi.row(row, total_s, acc);
    } else {
      s.chunk_part[chunk] = total_s;
      __threadfence();
      const unsigned int cnt = (unsigned int)s.chunk_count[chunk];
      if (atomicAdd(s.slot_ticket + slot, 1u) == cnt - 1) {
        __threadfence();
        const int first = s.chunk_first[chunk];
        double t = 0.0;
        for (unsigned int c = 0; c < cnt; ++c) t += __ldcg(s.chunk_part + first + c);
        double la[Epi::NRED];
#pragma unroll
        for (int q = 0; q < Epi::NRED; ++q) la[q] = 0.0;
        epi.row(row, t, la);
#pragma unroll
        for (int q = 0; q < Epi::NRED; ++q) s.long_red[(size_t)slot * 16 + q] = la[q];
        s.slot_ticket[slot] = 0u;
      }
    }
  }
  __syncthreads();
}

// Epi must provide: static constexpr int NRED (>= 1); bool REDUCE; bool enter() (block-uniform
// early exit); void row(int64_t, double, double(&)[NRED]); and, when
// Epi::FINAL, void finalize(const Sched&, int grid) run by the last block.
template <class Epi>
__global__ void __launch_bounds__(kBlock) spmv_fused(Csr A, const double* __restrict__ xg,
                                                     Sched s, Epi epi, double* part,
                                                     unsigned int* ticket) {
  if (!epi.enter()) return;
  __shared__ double ssum[kBlock];
  double acc[Epi::NRED];
#pragma unroll
  for (int q = 0; q < Epi::NRED; ++q) acc[q] = 0.0;
  for (int64_t tile = blockIdx.x; tile < s.total_tiles; tile += gridDim.x) {
    int sgi = 0;
    while (tile >= s.seg[sgi].tile_end) ++sgi;
    const Seg sg = s.seg[sgi];
    switch (sg.kind) {
      case 0: tile_sub<1>(A, xg, sg, tile, epi, acc, ssum); break;
      case 1: tile_sub<2>(A, xg, sg, tile, epi, acc, ssum); break;
      case 2: tile_sub<4>(A, xg, sg, tile, epi, acc, ssum); break;
      case 3: tile_sub<8>(A, xg, sg, tile, epi, acc, ssum); break;
      case 4: tile_sub<16>(A, xg, sg, tile, epi, acc, ssum); break;
      case 5: tile_sub<32>(A, xg, sg, tile, epi, acc, ssum); break;
      default: tile_long(A, xg, s, sg, tile, epi, acc); break;
    }
  }
  if constexpr (Epi::REDUCE) {
    block_reduce_store<Epi::NRED>(acc, part, gridDim.x, blockIdx.x);
    if constexpr (Epi::FINAL) {
      if (elect_last_block(ticket)) {
        epi.finalize(s, part, (int)gridDim.x);
        if (threadIdx.x == 0) *ticket = 0u;
      }
    }
  }
}

}  // namespace rhp
