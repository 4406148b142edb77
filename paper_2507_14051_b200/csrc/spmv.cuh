// spmv.cuh — warp-autonomous merge-path fp64 CSR SpMV with a fused per-row
// epilogue.
//
// Replaces SparseMatrix::multiply / multiply_transpose
// (/root/reference/proj/src/sparse_matrix.cpp:67-87). Both A and A^T are
// stored explicitly as CSR (A^T = the reference's CSC copy), so neither
// product needs atomics and every output row is produced in a fixed order
// (deterministic).
//
// Work split (layout.cu, build_schedule): warp w of the persistent grid owns
// one contiguous merge-path range of the operator — rows + nonzeros balanced
// across all warps, boundaries at row starts except inside long rows. A warp
// never synchronises with the other warps of its CTA while it walks its
// range; the only CTA barriers are in the final reduction of the epilogue
// sums.
//
// Per window of kWin = 32 * kPer consecutive nonzeros (lane L holds the kPer
// contiguous elements kPer*L ...):
//   (0) column indices and values arrive by 16-B vector loads (evict-first);
//       the next window's are issued as soon as this window's gathers are;
//   (1) products v * x[c] (x through the read-only path, L2 resident);
//   (2) row-start flags from the row pointers (one byte per element, shared);
//   (3) a segmented inclusive scan of the products: sequential inside a lane,
//       then a 5-step shuffle scan across lanes; the partial sum of a row that
//       continues from the previous window ("carry") is added to the first
//       element. A row's sum is the scan value at its last element;
//   (4) rows ending in the window run the epilogue, lane j <-> the j-th row
//       still open (groups of 32), inputs loaded by that lane.
// Rows cut by range boundaries ("split rows") are finished by the last warp
// to contribute (Sched comment in device_common.cuh).
//
// epilogue_walk<Epi> runs the same walk without the products, so a kernel
// whose reductions must be bit-identical to an epilogue fused into the SpMV
// (the block-start primal step K3 vs the primal step fused into K2) sees the
// same row -> lane sequences.
#pragma once

#include <type_traits>
#include <utility>

#include "device_common.cuh"

namespace rhp {

// Slot of window element e in WarpSmem::val: element t of lane L at
// t * 32 + L, so the scan-value stores of a warp (one per t) hit 32
// consecutive doubles (2 wavefronts, no bank conflicts).
__device__ __forceinline__ int sv(int64_t e) {
  const unsigned u = static_cast<unsigned>(e);  // 0 <= e < kWin
  return static_cast<int>((u % kPer) * 32u + u / kPer);
}

// Position type of the warp walk (RHP_IDX32: 32-bit, see warp_range).
#if RHP_IDX32
using ix = int32_t;
constexpr ix kIxMax = INT32_MAX;
#else
using ix = int64_t;
constexpr ix kIxMax = INT64_MAX;
#endif

struct WarpSmem {
  double val[kWin];          // products, then segmented-scan values
  unsigned char flag[kWin];  // 1 where a row starts
};

// Column indices / values of the kPer nonzeros of one lane starting at
// element i (a multiple of 4). Reads at most 3 elements past the operator's
// end (inside the 64-B padding of every device array).
__device__ __forceinline__ void ld_idx(const int32_t* ci, int64_t i, int (&c)[kPer]) {
#pragma unroll
  for (int h = 0; h < kPer / 4; ++h) {
    const int4 q = __ldcs(reinterpret_cast<const int4*>(ci + i) + h);
    c[4 * h + 0] = q.x;
    c[4 * h + 1] = q.y;
    c[4 * h + 2] = q.z;
    c[4 * h + 3] = q.w;
  }
}

__device__ __forceinline__ void ld_vals(const double* v, int64_t i, double (&x)[kPer]) {
#pragma unroll
  for (int h = 0; h < kPer / 2; ++h) {
    const double2 d = __ldcs(reinterpret_cast<const double2*>(v + i) + h);
    x[2 * h + 0] = d.x;
    x[2 * h + 1] = d.y;
  }
}

// Epilogues with a `cin` member (ConstInputs) may declare inputs constant:
// bit k of cin.mask set -> input k is cin.val[k] for every row and is not
// loaded (bounds such as x >= 0 after scaling: 16 of K2's ~136 B per column
// on C4). in[k] stays valid for the kernels that stage whole vectors.
template <class E, class = void>
struct HasConstInputs : std::false_type {};
template <class E>
struct HasConstInputs<E, std::void_t<decltype(std::declval<E>().cin)>> : std::true_type {};

template <class Epi>
__device__ __forceinline__ void load_inputs(const Epi& epi, int64_t row,
                                            double (&ein)[Epi::NIN > 0 ? Epi::NIN : 1]) {
#pragma unroll
  for (int k = 0; k < Epi::NIN; ++k) {
    if constexpr (RHP_CONST_INPUTS_KERNEL && HasConstInputs<Epi>::value) {
      ein[k] = (epi.cin.mask >> k) & 1u ? epi.cin.val[k] : epi.in[k][row];
    } else {
      ein[k] = epi.in[k][row];
    }
  }
}

// Last-arriver completion of a split row: store this warp's partial, and if
// every contributor has stored, sum them in warp order and run the epilogue
// (its reductions go to long_red[slot]).
template <class Epi>
__device__ __forceinline__ void contribute(const Sched& s, Epi& epi, int slot, int64_t entry,
                                        double partial) {
  s.slot_part[entry] = partial;
  __threadfence();
  const unsigned int cnt = static_cast<unsigned int>(s.slot_count[slot]);
  if (atomicAdd(s.slot_ticket + slot, 1u) != cnt - 1) return;
  __threadfence();
  const int64_t first = s.slot_first[slot];
  double t = __ldcg(s.slot_part + 2 * first + 1);  // the first contributor's tail partial
  for (unsigned int k = 1; k < cnt; ++k) t += __ldcg(s.slot_part + 2 * (first + k));
  const int64_t row = s.slot_row[slot];
  if (s.seg_in) t = add(__ldcg(s.seg_in + row), t);
  double ein[Epi::NIN > 0 ? Epi::NIN : 1];
  load_inputs(epi, row, ein);
  double la[Epi::NRED];
#pragma unroll
  for (int q = 0; q < Epi::NRED; ++q) la[q] = 0.0;
  epi.row(row, t, ein, 1, la);
#pragma unroll
  for (int q = 0; q < Epi::NRED; ++q) s.long_red[(size_t)slot * 16 + q] = la[q];
  s.slot_ticket[slot] = 0u;
}

// One merge-path chunk w, walked by one warp. WALK: epilogue only (row sums
// 0), same row -> lane map.
template <class Epi, bool WALK, bool L1G = false>
__device__ __forceinline__ void chunk_range(const int w, const int32_t* ci, const double* vals,
                                            const double* __restrict__ xg, const Sched& s,
                                            Epi& epi, double (&acc)[Epi::NRED], WarpSmem& sm) {
  const int lane = threadIdx.x & 31;
  // row and nonzero positions fit 32 bits (ingest.cu caps an operator at
  // 2^31 - 2^16 nonzeros): 32-bit locals halve their registers and shuffles
  const int64_t* rp = s.rp;
  const ix row_head = static_cast<ix>(s.warp_row[w]), r_end = static_cast<ix>(s.warp_row[w + 1]);
  const ix e0 = static_cast<ix>(s.warp_nz[w]), e_end = static_cast<ix>(s.warp_nz[w + 1]);
  const int hslot = s.head_slot[w];
  const ix rows = static_cast<ix>(s.rows);
  const ix r_lim = r_end < rows ? r_end + 1 : rows;  // rows whose end may be read
  ix r = row_head;
  ix rstart = static_cast<ix>(rp[r]);  // start of row r (warp-uniform)
  double carry = 0.0;
  // windows are aligned to 4 nonzeros (16-B vector loads); elements outside
  // [e0, e_end) are masked to zero
  ix wb = e0 & ~ix(3);
  int cn[kPer];  // column indices of this lane's elements of the current window
  if constexpr (!WALK) {
    if (wb + kPer * lane < e_end) ld_idx(ci, wb + kPer * lane, cn);
  }
  for (;; wb += kWin) {
    const ix we = wb + kWin < e_end ? wb + kWin : e_end;  // valid end of the window
    // ends of the next 32 rows: group 0 of the flags and of the completion pass
    ix re0 = r + lane < r_lim ? static_cast<ix>(rp[r + lane + 1]) : kIxMax;
    // epilogue inputs of row r + lane, loaded at the top of the window: the
    // first completion group below finishes exactly these rows (lane j <->
    // row r + j), so their loads leave the window's critical path. Used by
    // the walkers (K3: 21 -> 15 us on C2); in the SpMV proper the extra live
    // registers cost more than they hide (C2 K1 68.8 -> 71.9 us, C4 K1
    // 674 -> 698 us), so there only with RHP_EPI_PREFETCH=1.
    constexpr bool kPre = WALK || RHP_EPI_PREFETCH;
    double epre[Epi::NIN > 0 ? Epi::NIN : 1];
    const ix pre_row = r + lane;
    if constexpr (kPre) {
      if (pre_row < r_end) load_inputs(epi, pre_row, epre);
    }
    if constexpr (!WALK) {
      const ix mine = wb + kPer * lane;  // first element of this lane
      // (1) values and gathers of this window, then the next window's indices
      double p[kPer], vc[kPer];
      if (mine < we) ld_vals(vals, mine, vc);
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        const bool ok = mine + t >= e0 && mine + t < we;
        p[t] = ok ? ld_gather<L1G>(xg + cn[t]) : 0.0;
        if (!ok) vc[t] = 0.0;
      }
      if (mine + kWin < e_end) ld_idx(ci, mine + kWin, cn);
      // (2) row-start flags
#pragma unroll
      for (int h = 0; h < kPer / 4; ++h) reinterpret_cast<uint32_t*>(sm.flag)[lane * (kPer / 4) + h] = 0u;
      __syncwarp();
      if (lane == 0 && rstart >= wb && rstart < we) sm.flag[rstart - wb] = 1;
      for (ix g = r, re = re0;;) {
        if (re >= wb && re < we) sm.flag[re - wb] = 1;
        if (__shfl_sync(0xffffffffu, re, 31) >= we) break;
        g += 32;
        re = g + lane < r_lim ? static_cast<ix>(rp[g + lane + 1]) : kIxMax;
      }
#pragma unroll
      for (int t = 0; t < kPer; ++t) p[t] = mul(vc[t], p[t]);
      __syncwarp();
      // (3) segmented scan
      uint32_t fl[kPer / 4];
#pragma unroll
      for (int h = 0; h < kPer / 4; ++h)
        fl[h] = reinterpret_cast<const uint32_t*>(sm.flag)[lane * (kPer / 4) + h];
      auto flag_at = [&](int t) { return (fl[t >> 2] >> (8 * (t & 3))) & 1u; };
      if (lane == 0 && !flag_at(0)) p[0] = add(carry, p[0]);
      int hs = 0;
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        if (flag_at(t)) hs = 1;
        else if (t > 0) p[t] = add(p[t - 1], p[t]);
      }
      double agg = p[kPer - 1];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_up_sync(0xffffffffu, agg, d);
        const int oh = __shfl_up_sync(0xffffffffu, hs, d);
        if (lane >= d) {
          if (!hs) agg = add(o, agg);
          hs |= oh;
        }
      }
      const double excl = __shfl_up_sync(0xffffffffu, agg, 1);
      if (lane > 0) {
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
          if (flag_at(t)) break;
          p[t] = add(excl, p[t]);
        }
      }
      // every value is stored, though only the row ends are read back:
      // storing just those (predicated stores, a shuffle for the next lane's
      // first flag) cut the shared-store wavefronts but cost more issue
      // slots (C4 K1 688 -> 699 us, C2 K1 70.2 -> 70.8 us)
#pragma unroll
      for (int t = 0; t < kPer; ++t) sm.val[sv(kPer * lane + t)] = p[t];
      __syncwarp();
    }
    // (4) rows ending in this window
    for (ix re = re0;;) {
      const ix row = r + lane;
      const bool inr = row < r_end;
      if (!inr) re = kIxMax;
      ix rs = __shfl_up_sync(0xffffffffu, re, 1);
      if (lane == 0) rs = rstart;
      const bool done = inr && re <= we;
      if (done) {
        double sum = 0.0;
        if constexpr (!WALK) sum = re > rs ? sm.val[sv(re - 1 - wb)] : 0.0;
        double ein[Epi::NIN > 0 ? Epi::NIN : 1];
        if (row == row_head && hslot >= 0) {
          if constexpr (WALK) {
            load_inputs(epi, row, ein);
            double la[Epi::NRED];
#pragma unroll
            for (int q = 0; q < Epi::NRED; ++q) la[q] = 0.0;
            epi.row(row, 0.0, ein, 1, la);
#pragma unroll
            for (int q = 0; q < Epi::NRED; ++q) s.long_red[(size_t)hslot * 16 + q] = la[q];
          } else {
            contribute(s, epi, hslot, 2 * static_cast<int64_t>(w), sum);
          }
        } else {
          if constexpr (!WALK) {
            if (s.seg_in) sum = add(__ldcg(s.seg_in + row), sum);
          }
          if (kPre && row == pre_row) {
            epi.row(row, sum, epre, 1, acc);
          } else {
            load_inputs(epi, row, ein);
            epi.row(row, sum, ein, 1, acc);
          }
        }
      }
      const int nc = __popc(__ballot_sync(0xffffffffu, done));
      if (nc > 0) rstart = __shfl_sync(0xffffffffu, re, nc - 1);  // end of the last finished row
      r += nc;
      if (nc < 32) break;
      re = r + lane < r_end ? static_cast<ix>(rp[r + lane + 1]) : kIxMax;
    }
    if constexpr (!WALK) {
      // partial sum of the row left open at the window's end
      if (we > wb) carry = rstart < we ? sm.val[sv(we - 1 - wb)] : 0.0;
      __syncwarp();  // the next window overwrites the shared arrays
    }
    if (wb + kWin >= e_end) break;
  }
  if constexpr (!WALK) {
    // the range ends inside row r_end: contribute its partial
    if (lane == 0 && r_end < s.rows && e_end > rstart) {
      if (r_end == row_head && hslot >= 0) contribute(s, epi, hslot, 2 * static_cast<int64_t>(w), carry);
      else contribute(s, epi, s.tail_slot[w], 2 * static_cast<int64_t>(w) + 1, carry);
    }
  }
}

// A warp walks the chunks w, w + W, w + 2W, ... (W = warps of the grid): at
// any moment the whole grid works on one band of consecutive chunks, so the
// columns those rows gather from form a narrow working set in L2 whenever
// the matrix has row locality (C4: one commodity's 8 MB slice of x instead of
// all 160 MB). The epilogue reductions accumulate over the warp's chunks.
template <class Epi, bool WALK, bool L1G = false>
__device__ __forceinline__ void warp_range(const int32_t* ci, const double* vals,
                                           const double* __restrict__ xg, const Sched& s,
                                           Epi& epi, double (&acc)[Epi::NRED], WarpSmem& sm) {
  const int w = static_cast<int>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  for (int c = w; c < s.n_chunks; c += s.n_warps)
    chunk_range<Epi, WALK, L1G>(c, ci, vals, xg, s, epi, acc, sm);
}

// Thread-per-row engine, for operators whose rows are all short
// (Sched::thread_rows: max row length <= kThreadRowMax, chosen at setup —
// C3's A^T rows have 2 nonzeros, C4's 3). Thread g of the grid owns rows g,
// g + G, g + 2G, ... (G = threads of the grid), RHP_ROWS_IN_FLIGHT (2) rows in flight per
// thread. No scan, no shared memory and no split rows: a row's products are
// summed sequentially in element order — the reference's own order
// (sparse_matrix.cpp:67-87), so these row sums are bit-identical to its — and
// the epilogue inputs, independent of the sum, are loaded first, so a row
// costs one dependent chain (row pointers -> indices -> gathers) with its
// epilogue loads in its shadow. WALK: epilogue only, same row -> thread map.
// RF rows in flight per thread: RHP_ROWS_IN_FLIGHT (2), RHP_UNIFORM_RF (1)
// for uniform rows (no row-pointer round: one row's loads already fill the
// memory pipe; C4 K2 612 -> 564 us, C3 22.9 -> 20.9 us; the walkers keep 2).
template <class Epi, bool WALK, bool L1G = false, int RF = RHP_ROWS_IN_FLIGHT>
__device__ __forceinline__ void thread_rows(const int32_t* ci, const double* vals,
                                            const double* __restrict__ xg, const Sched& s,
                                            Epi& epi, double (&acc)[Epi::NRED]) {
  constexpr int NI = Epi::NIN > 0 ? Epi::NIN : 1;
  constexpr int EC = RF >= 4 ? 2 : 4;     // elements per row per step
  const int64_t G = static_cast<int64_t>(gridDim.x) * kBlock;
  const int64_t R = s.rows;
  // thread g owns rows g, g + G, g + 2G, ... and finishes them in that order
  // whatever RF is, so the reductions do not depend on RF
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x; i0 < R; i0 += RF * G) {
    double e[RF][NI], sm[RF];
    int64_t lo[RF];
    int len[RF];
#pragma unroll
    for (int f = 0; f < RF; ++f) {
      const int64_t i = i0 + f * G;
      if (i < R) load_inputs(epi, i, e[f]);
      sm[f] = 0.0;
    }
    if constexpr (!WALK) {
      // sliced copy (coalesced element loads, 1-B lengths instead of row
      // pointers) when built, else CSR; same elements in the same order
#if RHP_UNIFORM_ROWS
      const int w = s.uniform_len;
      const bool sliced = s.sell_ci != nullptr;
#else  // A/B variant: the row-pointer path only
      constexpr int w = 0;
      constexpr bool sliced = false;
#endif
      const int32_t* cix = sliced ? s.sell_ci : ci;
      const double* vx = sliced ? s.sell_v : vals;
      const int64_t es = sliced ? 32 : 1;  // element stride of a row
      int lmax = 0;
#pragma unroll
      for (int f = 0; f < RF; ++f) {
        const int64_t i = i0 + f * G;
        if (w > 0) {  // no row-pointer round before the index loads
          lo[f] = sliced ? (i >> 5) * (32 * static_cast<int64_t>(w)) + (i & 31) : i * w;
          len[f] = i < R ? w : 0;
        } else {
          lo[f] = i < R ? s.rp[i] : 0;
          len[f] = i < R ? static_cast<int>(s.rp[i + 1] - lo[f]) : 0;
        }
        lmax = max(lmax, len[f]);
      }
      // uniform rows of a multiple of 4 in CSR order: a row's 4 elements of
      // one step are 16-B aligned (i * w), one int4 + two double2 loads
      const bool vec = RHP_ROWS_VEC && EC == 4 && w > 0 && (w & 3) == 0 && !sliced;
      for (int t = 0; t < lmax; t += EC) {
        int c[RF][EC];
        double v[RF][EC], g[RF][EC];
#pragma unroll
        for (int f = 0; f < RF; ++f) {
          if (vec) {
            const bool ok = t < len[f];
            const int4 q = ok ? __ldcs(reinterpret_cast<const int4*>(cix + lo[f] + t)) : make_int4(0, 0, 0, 0);
            const double2 a = ok ? __ldcs(reinterpret_cast<const double2*>(vx + lo[f] + t)) : make_double2(0.0, 0.0);
            const double2 b = ok ? __ldcs(reinterpret_cast<const double2*>(vx + lo[f] + t) + 1) : make_double2(0.0, 0.0);
            c[f][0] = q.x; c[f][1] = q.y; c[f][2] = q.z; c[f][3] = q.w;
            v[f][0] = a.x; v[f][1] = a.y; v[f][2] = b.x; v[f][3] = b.y;
            continue;
          }
#pragma unroll
          for (int u = 0; u < EC; ++u) {
            const bool ok = t + u < len[f];
            c[f][u] = ok ? __ldcs(cix + lo[f] + (t + u) * es) : 0;
            v[f][u] = ok ? __ldcs(vx + lo[f] + (t + u) * es) : 0.0;
          }
        }
#pragma unroll
        for (int f = 0; f < RF; ++f)
#pragma unroll
          for (int u = 0; u < EC; ++u)
            g[f][u] = t + u < len[f] ? ld_gather<L1G>(xg + c[f][u]) : 0.0;
#pragma unroll
        for (int f = 0; f < RF; ++f)
#pragma unroll
          for (int u = 0; u < EC; ++u)
            if (t + u < len[f]) sm[f] = add(sm[f], mul(v[f][u], g[f][u]));
      }
      if (s.seg_in) {
#pragma unroll
        for (int f = 0; f < RF; ++f)
          if (i0 + f * G < R) sm[f] = add(__ldcg(s.seg_in + i0 + f * G), sm[f]);
      }
    }
#pragma unroll
    for (int f = 0; f < RF; ++f)
      if (i0 + f * G < R) epi.row(i0 + f * G, sm[f], e[f], 1, acc);
  }
}

// The epilogue's block reductions and the last block's finalize.
template <class Epi>
__device__ __forceinline__ void spmv_tail(const Sched& s, Epi& epi, const double (&acc)[Epi::NRED],
                                          double* part, unsigned int* ticket) {
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

// L1G: L1-allocating gathers (ld_gather).
// Epi provides: NRED (>= 1) reductions, NIN per-row input vectors `in[NIN]`,
// REDUCE, FINAL; bool enter() (block-uniform early exit); void row(int64_t
// i, double rowsum, const double* e, int stride, double(&acc)[NRED]) with
// input k of row i at e[k*stride]; and, when FINAL, void finalize(const
// Sched&, const double* part, int grid) (last block).
// Merge-path operators launch this kernel, which holds only the merge path:
// sharing one kernel with the thread-per-row variants cost C2's K2 4 us
// (70.4 vs 66.4 us, A/B on one box).
template <class Epi, bool L1G = false>
__global__ void __launch_bounds__(kBlock, kMinBlocks) spmv_fused(Csr A, const double* __restrict__ xg,
                                                                 Sched s, Epi epi, double* part,
                                                                 unsigned int* ticket) {
  pdl_wait();
  pdl_trigger();
  if (!epi.enter()) return;
  __shared__ __align__(16) WarpSmem wsm[kWarps];
  double acc[Epi::NRED];
#pragma unroll
  for (int q = 0; q < Epi::NRED; ++q) acc[q] = 0.0;
  warp_range<Epi, false, L1G>(A.ci, A.v, xg, s, epi, acc, wsm[threadIdx.x >> 5]);
  spmv_tail(s, epi, acc, part, ticket);
}

// Thread-per-row operators (Sched::thread_rows) launch this one; same
// epilogue contract as spmv_fused, built for kRowsMinBlocks (4) CTAs per SM
// with the operator's grid sized for it (rhp_cuda.cu thread_rows_rule; C4
// K2 602 -> 450 us). It still carries the merge path
// (RHP_ROWS_KERNEL_COMBINED, never taken at run time): the thread-per-row
// code nvcc emits without it is slower (C4 K2 537 vs 450 us at 4 CTAs/SM,
// 619 vs 565 us at 2), and so is the rows-only kernel under a shared-memory
// carveout preference (25-100 %: C4 K2 1.29 ms) — kept for the measured
// speed.
template <class Epi, bool L1G = false>
__global__ void __launch_bounds__(kBlock, kRowsMinBlocks) spmv_rows(Csr A, const double* __restrict__ xg,
                                                                Sched s, Epi epi, double* part,
                                                                unsigned int* ticket) {
  pdl_wait();
  pdl_trigger();
  if (!epi.enter()) return;
  double acc[Epi::NRED];
#pragma unroll
  for (int q = 0; q < Epi::NRED; ++q) acc[q] = 0.0;
#if RHP_ROWS_KERNEL_COMBINED
  __shared__ __align__(16) WarpSmem wsm[kWarps];
  if (!s.thread_rows) {
    warp_range<Epi, false, L1G>(A.ci, A.v, xg, s, epi, acc, wsm[threadIdx.x >> 5]);
  } else
#endif
  if (RHP_UNIFORM_ROWS && s.uniform_len > 0)
    thread_rows<Epi, false, L1G, RHP_UNIFORM_RF>(A.ci, A.v, xg, s, epi, acc);
  else
    thread_rows<Epi, false, L1G>(A.ci, A.v, xg, s, epi, acc);
  spmv_tail(s, epi, acc, part, ticket);
}

// Long-row engine (an operator made of few very long rows, e.g. C3's A:
// 2000 rows of 1000 nonzeros; rhp_cuda.cu apply_cta_rule, every row >=
// kCtaRowMin nonzeros). CTA b owns the contiguous rows [cta_row[b],
// cta_row[b+1]) (balanced by nonzeros on the host) and walks them
// kCtaRowsBatch at a time: thread t takes elements t, t + kBlock, ... of
// every row of the batch, kCtaRowUnroll of them per row at once (coalesced
// index / value loads, then all the batch's gathers in flight), then each
// row's partials are reduced by a fixed shuffle tree per warp and a fixed
// warp order in shared memory, and lane q of warp 0 runs row q's epilogue.
// Built for kCtaRowBlocks CTAs per SM (register budget 64 at 256 threads) on
// its own grid (DevOp::cta_grid): latency is hidden by resident warps rather
// than by the long windows of the merge-path engine. No split rows, no
// tickets, no slots (n_multi 0). Deterministic: fixed element -> thread map
// and reduction order.
template <class Epi, bool L1G = false>
__global__ void __launch_bounds__(kBlock, kCtaRowBlocks) spmv_cta_rows(Csr A, const double* __restrict__ xg,
                                                                       Sched s, const int32_t* cta_row,
                                                                       Epi epi, double* part,
                                                                       unsigned int* ticket) {
  pdl_wait();
  pdl_trigger();
  if (!epi.enter()) return;
  constexpr int RB = kCtaRowsBatch, K = kCtaRowUnroll;
  __shared__ double red[RB][kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[Epi::NRED];
#pragma unroll
  for (int q = 0; q < Epi::NRED; ++q) acc[q] = 0.0;
  const int64_t r0 = cta_row[blockIdx.x], r1 = cta_row[blockIdx.x + 1];
  for (int64_t base = r0; base < r1; base += RB) {
    int64_t lo[RB], hi[RB];
    double p[RB];
    int64_t len = 0;
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const int64_t row = base + q;
      lo[q] = row < r1 ? s.rp[row] : 0;
      hi[q] = row < r1 ? s.rp[row + 1] : 0;
      len = max(len, hi[q] - lo[q]);
      p[q] = 0.0;
    }
    for (int64_t t0 = threadIdx.x; t0 < len; t0 += static_cast<int64_t>(K) * kBlock) {
      int c[RB][K];
      double v[RB][K];
#pragma unroll
      for (int q = 0; q < RB; ++q)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int64_t e = lo[q] + t0 + static_cast<int64_t>(k) * kBlock;
          const bool ok = e < hi[q];
          c[q][k] = ok ? __ldcs(A.ci + e) : 0;
          v[q][k] = ok ? __ldcs(A.v + e) : 0.0;
        }
#pragma unroll
      for (int q = 0; q < RB; ++q)
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (lo[q] + t0 + static_cast<int64_t>(k) * kBlock < hi[q])
            p[q] = fma(v[q][k], ld_gather<L1G>(xg + c[q][k]), p[q]);
    }
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      double x = p[q];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
      if (lane == 0) red[q][warp] = x;
    }
    __syncthreads();
    if (warp == 0 && lane < RB && base + lane < r1) {
      const int64_t row = base + lane;
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) sum += red[lane][w];
      if (s.seg_in) sum = add(__ldcg(s.seg_in + row), sum);
      double ein[Epi::NIN > 0 ? Epi::NIN : 1];
      load_inputs(epi, row, ein);
      epi.row(row, sum, ein, 1, acc);
    }
    __syncthreads();  // red is rewritten by the next batch
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

// Runs only the epilogue of spmv_fused<Epi>, with exactly its row -> lane
// assignment (row sum argument 0, inputs read from global memory).
template <class Epi>
__global__ void __launch_bounds__(kBlock) epilogue_walk(Sched s, Epi epi, double* part) {
  pdl_wait();
  pdl_trigger();
  if (!epi.enter()) return;
  __shared__ __align__(16) WarpSmem wsm[kWarps];
  double acc[Epi::NRED];
#pragma unroll
  for (int q = 0; q < Epi::NRED; ++q) acc[q] = 0.0;
  if (s.thread_rows) thread_rows<Epi, true>(nullptr, nullptr, nullptr, s, epi, acc);
  else warp_range<Epi, true>(nullptr, nullptr, nullptr, s, epi, acc, wsm[threadIdx.x >> 5]);
  block_reduce_store<Epi::NRED>(acc, part, gridDim.x, blockIdx.x);
  epi.walk_done();
}

}  // namespace rhp
