// spmv.cuh — nnz-balanced fp64 CSR SpMV with TMA-staged tiles and a fused
// per-row epilogue.
//
// Replaces SparseMatrix::multiply / multiply_transpose
// (/root/reference/proj/src/sparse_matrix.cpp:67-87). Both A and A^T are
// stored explicitly as CSR (A^T = the reference's CSC copy), so neither
// product needs atomics and every output row is produced in a fixed order
// (deterministic).
//
// Tiles (built on the host, layout.cu):
//   stream tile: a run of consecutive rows holding <= kTileNnz nonzeros and
//     <= kTileRows rows.
//   chunk tile: one CTA per <= kChunkNnz slice of a row longer than
//     kTileNnz; a row of several chunks is completed by the last chunk to
//     land (fixed-order sum of the chunk partials).
// A persistent grid walks the tiles with a static stride, so each CTA's
// reduction partials have a fixed composition.
//
// Stream tiles are double-buffered through shared memory by the bulk-copy
// engine: while the CTA computes tile i from stage i&1, one thread has
// already issued cp.async.bulk copies of tile i+1's values, column indices,
// row pointers and the epilogue's per-row input vectors (y, ax, bounds,
// anchor, ...) into stage (i+1)&1, completing on an mbarrier. Tile
// descriptors are loaded two tiles ahead, so issuing never waits on memory.
// Compute per tile, all from shared memory except the x gather:
//   (1) products v*x[c] in place (x through the read-only path, L2 resident),
//   (2) row sums by groups of W lanes (W from the tile's mean row length;
//       fixed per tile, so the order is deterministic; W = 1 is the
//       reference's sequential order),
//   (3) the epilogue, one thread per row, inputs from the stage, outputs
//       stored straight to global memory (coalesced).
#pragma once

#include "device_common.cuh"
#include "tma.cuh"

namespace rhp {

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Epilogue per-row inputs: staged by TMA with the tile (1) or loaded by the
// row's thread into registers at tile start, overlapping the gather (0).
#ifndef RHP_EPI_TMA
#define RHP_EPI_TMA 1
#endif
constexpr bool kEpiTma = RHP_EPI_TMA != 0;

// Shared-memory layout of one pipeline stage for an epilogue with NIN
// per-row input vectors. Offsets keep every TMA destination 16-B aligned;
// the +2/+8/+4 slack absorbs the 16-B alignment of the copied source ranges.
template <int NIN>
struct Stage {
  static constexpr int kVals = kTileNnz + 2;  // doubles
  static constexpr int kRp = kTileRows + 4;   // int64
  static constexpr int kIn = kTileRows + 4;   // doubles per input vector
  static constexpr int kIdx = kTileNnz + 8;   // int32
  static constexpr size_t off_vals = 0;
  static constexpr size_t off_rp = align16(off_vals + 8 * kVals);
  static constexpr size_t off_in = align16(off_rp + 8 * kRp);
  static constexpr size_t off_idx = align16(off_in + 8 * size_t(kIn) * NIN);
  static constexpr size_t bytes = align16(off_idx + 4 * kIdx);
};

// Dynamic shared memory of spmv_fused<Epi>: two stages, row sums, barriers.
template <int NIN>
__host__ __device__ constexpr size_t spmv_smem_bytes() {
  return 2 * Stage<NIN>::bytes + 8 * kTileRows + 16;
}

struct TileDesc {
  int64_t r0, r1, b, e;
};

__device__ __forceinline__ TileDesc load_desc(const Sched& s, int64_t t) {
  return TileDesc{s.tile_row[t], s.tile_row_end[t], s.tile_nz[2 * t], s.tile_nz[2 * t + 1]};
}

// Thread 0: issue the bulk copies of one stream tile into a stage.
template <class Epi>
__device__ __forceinline__ void issue_tile(const Csr& A, const Epi& epi, const TileDesc& d,
                                           unsigned char* stage, uint64_t* bar) {
  using L = Stage<Epi::NIN>;
  const int64_t vb = d.b & ~int64_t(1), ve = (d.e + 1) & ~int64_t(1);
  const int64_t ib = d.b & ~int64_t(3), ie = (d.e + 3) & ~int64_t(3);
  const int64_t rb = d.r0 & ~int64_t(1), re = (d.r1 + 2) & ~int64_t(1);  // rp needs r1 inclusive
  const int64_t xb = d.r0 & ~int64_t(1), xe = (d.r1 + 1) & ~int64_t(1);
  const uint32_t bv = static_cast<uint32_t>(8 * (ve - vb));
  const uint32_t bi = static_cast<uint32_t>(4 * (ie - ib));
  const uint32_t br = static_cast<uint32_t>(8 * (re - rb));
  const uint32_t bx = kEpiTma ? static_cast<uint32_t>(8 * (xe - xb)) : 0u;
  mbar_arrive_expect_tx(bar, bv + bi + br + bx * Epi::NIN);
  if (bv) tma_load_1d(stage + L::off_vals, A.v + vb, bv, bar);
  if (bi) tma_load_1d(stage + L::off_idx, A.ci + ib, bi, bar);
  tma_load_1d(stage + L::off_rp, A.rp + rb, br, bar);
  if constexpr (kEpiTma) {
#pragma unroll
    for (int k = 0; k < Epi::NIN; ++k)
      tma_load_1d(stage + L::off_in + 8 * size_t(L::kIn) * k, epi.in[k] + xb, bx, bar);
  }
}

template <int W>
__device__ __forceinline__ void stage_row_sums(const int64_t* rps, int rows, int64_t b,
                                               const double* prod, double* rowsum) {
  const int g = threadIdx.x / W, lane = threadIdx.x % W;
  constexpr int G = kBlock / W;
  for (int rr = 0; rr < rows; rr += G) {  // uniform trip count: all lanes shuffle
    const int r = rr + g;
    double s = 0.0;
    if (r < rows) {
      const int lo = static_cast<int>(rps[r] - b), hi = static_cast<int>(rps[r + 1] - b);
      for (int k = lo + lane; k < hi; k += W) s += prod[k];
    }
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0 && r < rows) rowsum[r] = s;
  }
}

// Lanes per row group for the shared-memory row sums of a stream tile.
__device__ __forceinline__ int group_width(int nnz, int rows) {
  const int mean = rows > 0 ? (nnz + rows - 1) / rows : 1;
  if (mean <= 4) return 1;
  if (mean <= 8) return 2;
  if (mean <= 16) return 4;
  if (mean <= 32) return 8;
  if (mean <= 64) return 16;
  return 32;
}

template <class Epi>
__device__ __forceinline__ void compute_tile(const double* __restrict__ xg, const TileDesc& d,
                                             unsigned char* stage, Epi& epi,
                                             double (&acc)[Epi::NRED], double* rowsum) {
  using L = Stage<Epi::NIN>;
  const int rows = static_cast<int>(d.r1 - d.r0);
  const int nnz = static_cast<int>(d.e - d.b);
  double* vals = reinterpret_cast<double*>(stage + L::off_vals) + (d.b & 1);
  const int* idx = reinterpret_cast<const int*>(stage + L::off_idx) + (d.b & 3);
  const int64_t* rps = reinterpret_cast<const int64_t*>(stage + L::off_rp) + (d.r0 & 1);
  const double* ein = reinterpret_cast<const double*>(stage + L::off_in) + (d.r0 & 1);
  // register path: the row's epilogue inputs, loaded now, used in (3)
  constexpr int NI = Epi::NIN > 0 ? Epi::NIN : 1;
  double ereg[NI];
  if constexpr (!kEpiTma) {
    if (threadIdx.x < rows) {
#pragma unroll
      for (int k = 0; k < Epi::NIN; ++k) ereg[k] = epi.in[k][d.r0 + threadIdx.x];
    }
  }
  // (1) products in place. All indices and all x gathers of a thread are
  // loaded into registers before the first shared-memory store, so the
  // kTileNnz/kBlock gathers are in flight together (an interleaved
  // load/store loop would serialise them on possible aliasing).
  {
    constexpr int P = kTileNnz / kBlock;
    int c[P];
    double xv[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int i = k * kBlock + threadIdx.x;
      c[k] = i < nnz ? idx[i] : 0;
    }
#pragma unroll
    for (int k = 0; k < P; ++k) xv[k] = ld_gather(xg + c[k]);
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int i = k * kBlock + threadIdx.x;
      if (i < nnz) vals[i] = vals[i] * xv[k];
    }
  }
  __syncthreads();
  // (2) deterministic row sums
  switch (group_width(nnz, rows)) {
    case 1: stage_row_sums<1>(rps, rows, d.b, vals, rowsum); break;
    case 2: stage_row_sums<2>(rps, rows, d.b, vals, rowsum); break;
    case 4: stage_row_sums<4>(rps, rows, d.b, vals, rowsum); break;
    case 8: stage_row_sums<8>(rps, rows, d.b, vals, rowsum); break;
    case 16: stage_row_sums<16>(rps, rows, d.b, vals, rowsum); break;
    default: stage_row_sums<32>(rps, rows, d.b, vals, rowsum); break;
  }
  __syncthreads();
  // (3) epilogue, thread per row
  if (threadIdx.x < rows) {
    if constexpr (kEpiTma)
      epi.row(d.r0 + threadIdx.x, rowsum[threadIdx.x], ein + threadIdx.x, L::kIn, acc);
    else
      epi.row(d.r0 + threadIdx.x, rowsum[threadIdx.x], ereg, 1, acc);
  }
}

template <class Epi>
__device__ __forceinline__ void tile_chunk(const Csr& A, const double* __restrict__ xg,
                                           const Sched& s, int64_t chunk, Epi& epi,
                                           double (&acc)[Epi::NRED]) {
  __shared__ double red[kWarps];
  __shared__ double total_s;
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
    double ein[Epi::NIN > 0 ? Epi::NIN : 1];
#pragma unroll
    for (int k = 0; k < Epi::NIN; ++k) ein[k] = epi.in[k][row];
    const int slot = s.chunk_slot[chunk];
    if (slot < 0) {
      epi.row(row, total_s, ein, 1, acc);
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
        epi.row(row, t, ein, 1, la);
#pragma unroll
        for (int q = 0; q < Epi::NRED; ++q) s.long_red[(size_t)slot * 16 + q] = la[q];
        s.slot_ticket[slot] = 0u;
      }
    }
  }
  __syncthreads();
}

// Epi provides: NRED (>= 1) reductions, NIN per-row input vectors `in[NIN]`
// (TMA-staged), REDUCE, FINAL; bool enter() (block-uniform early exit);
// void row(int64_t i, double rowsum, const double* e, int stride,
// double(&acc)[NRED]) with input k of row i at e[k*stride]; and, when FINAL,
// void finalize(const Sched&, const double* part, int grid) (last block).
template <class Epi>
__global__ void __launch_bounds__(kBlock, kMinBlocks) spmv_fused(Csr A, const double* __restrict__ xg,
                                                                 Sched s, Epi epi, double* part,
                                                                 unsigned int* ticket) {
  if (!epi.enter()) return;
  extern __shared__ __align__(128) unsigned char smem[];
  using L = Stage<Epi::NIN>;
  double* rowsum = reinterpret_cast<double*>(smem + 2 * L::bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * L::bytes + 8 * kTileRows);
  double acc[Epi::NRED];
#pragma unroll
  for (int q = 0; q < Epi::NRED; ++q) acc[q] = 0.0;
  __shared__ TileDesc sdesc[2];  // descriptor of the tile in each stage
  const int64_t grid = gridDim.x;
  // Tile order: the chunk tiles of long rows first (longest work first, so
  // they do not form a tail), then the stream tiles. CTA b takes tiles
  // b, b+grid, ...; t below indexes stream tiles only.
  const int64_t n_chunks = s.total_tiles - s.n_stream;
  int64_t tc = blockIdx.x;
  int64_t t = tc;
  if (t < n_chunks) t += ((n_chunks - t + grid - 1) / grid) * grid;
  t -= n_chunks;
  TileDesc next{}, after{};
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    if (t < s.n_stream) {  // the first stream tile streams in while chunks run
      sdesc[0] = load_desc(s, t);
      issue_tile(A, epi, sdesc[0], smem, &bars[0]);
    }
    if (t + grid < s.n_stream) next = load_desc(s, t + grid);
    if (t + 2 * grid < s.n_stream) after = load_desc(s, t + 2 * grid);
  }
  __syncthreads();
  for (; tc < n_chunks; tc += grid) tile_chunk(A, xg, s, tc, epi, acc);
  for (int it = 0; t < s.n_stream; t += grid, ++it) {
    const int st = it & 1;
    if (threadIdx.x == 0) {
      if (t + grid < s.n_stream) {
        fence_proxy_async();  // this stage's previous generic accesses precede the copy
        sdesc[st ^ 1] = next;
        issue_tile(A, epi, next, smem + (st ^ 1) * L::bytes, &bars[st ^ 1]);
      }
      next = after;
      if (t + 3 * grid < s.n_stream) after = load_desc(s, t + 3 * grid);
    }
    const TileDesc d = sdesc[st];  // written before the barrier ending the previous tile
    mbar_wait(&bars[st], (it >> 1) & 1);
    compute_tile(xg, d, smem + st * L::bytes, epi, acc, rowsum);
    __syncthreads();  // stage st is free for the copy issued next iteration
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

// Runs only the epilogue of spmv_fused<Epi>, with exactly its tile -> block
// and row -> thread assignment (row sum argument 0, inputs read from global
// memory). A kernel whose reductions must be bit-identical to the epilogue
// fused into an SpMV (the block-start primal step vs the primal step fused
// into the A^T pass) uses this walker so the per-thread accumulation
// sequences are the same.
template <class Epi>
__global__ void __launch_bounds__(kBlock) epilogue_walk(Sched s, Epi epi, double* part) {
  if (!epi.enter()) return;
  double acc[Epi::NRED];
#pragma unroll
  for (int q = 0; q < Epi::NRED; ++q) acc[q] = 0.0;
  double ein[Epi::NIN > 0 ? Epi::NIN : 1];
  const int64_t n_chunks = s.total_tiles - s.n_stream;  // same order as spmv_fused
  for (int64_t tile = blockIdx.x; tile < s.total_tiles; tile += gridDim.x) {
    int64_t row = -1;
    int slot = -1;
    if (tile >= n_chunks) {
      const int64_t ts = tile - n_chunks;
      const int64_t r0 = s.tile_row[ts], r1 = s.tile_row_end[ts];
      if (r0 + threadIdx.x < r1) row = r0 + threadIdx.x;
    } else if (threadIdx.x == 0) {
      const int64_t chunk = tile;
      slot = s.chunk_slot[chunk];
      if (slot < 0 || chunk == s.chunk_first[chunk]) row = s.chunk_row[chunk];
    }
    if (row < 0) continue;
#pragma unroll
    for (int k = 0; k < Epi::NIN; ++k) ein[k] = epi.in[k][row];
    if (slot < 0) {
      epi.row(row, 0.0, ein, 1, acc);
    } else {
      double la[Epi::NRED];
#pragma unroll
      for (int q = 0; q < Epi::NRED; ++q) la[q] = 0.0;
      epi.row(row, 0.0, ein, 1, la);
#pragma unroll
      for (int q = 0; q < Epi::NRED; ++q) s.long_red[(size_t)slot * 16 + q] = la[q];
    }
  }
  block_reduce_store<Epi::NRED>(acc, part, gridDim.x, blockIdx.x);
  epi.walk_done();
}

}  // namespace rhp
