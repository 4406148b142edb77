// device_common.cuh — shared device-side definitions of the rhpdhg CUDA library.
//
// Conventions
//  * fp64 everywhere. Elementwise formulas that the reference evaluates in a
//    fixed order (pdhg.cpp:41-63, restart.cpp:23-30, scaling.cpp:10-34) are
//    written with explicit __dmul_rn/__dadd_rn/__dsub_rn so nvcc cannot
//    contract them into FMAs: each such value is then bit-identical to the
//    reference's on the same inputs. SpMV row sums and reductions use FMA
//    and tree orders (documented drift).
//  * All reductions are deterministic: a fixed lane/warp tree per block, then
//    a fixed-order sum of per-block partials by the last block to finish.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

namespace rhp {

// Per-epilogue constant inputs (spmv.cuh load_inputs): bit k of mask set ->
// input k equals val[k] on every row.
struct ConstInputs {
  unsigned mask;
  double val[8];
};

#ifndef RHP_BLOCK
#define RHP_BLOCK 256
#endif
constexpr int kBlock = RHP_BLOCK;    // threads per CTA for every hot kernel
constexpr int kWarps = kBlock / 32;
// SpMV engine (spmv.cuh): every warp owns one contiguous merge-path range of
// its operator and walks it in windows of kWin = 32 * kPer nonzeros.
#ifndef RHP_WIN_PER
#define RHP_WIN_PER 8
#endif
#ifndef RHP_MIN_BLOCKS
#define RHP_MIN_BLOCKS 2
#endif
constexpr int kMinBlocks = RHP_MIN_BLOCKS;  // resident CTAs per SM the SpMV is built for
// The thread-per-row kernel is built for 4 resident CTAs per SM (64
// registers; its never-taken merge-path copy spills, its row loop does not
// need more): one row in flight per thread is hidden by occupancy. C4 K2
// 602 -> 450 us (0.97 of the HBM roofline), C3 K2 21.5 -> 18.9 us; 3 CTAs:
// 520 us; the rows-only kernel at 4 CTAs: 537 us (A/B on one box).
#ifndef RHP_ROWS_MIN_BLOCKS
#define RHP_ROWS_MIN_BLOCKS 4
#endif
constexpr int kRowsMinBlocks = RHP_ROWS_MIN_BLOCKS;  // ... and the thread-per-row kernel
constexpr int kPer = RHP_WIN_PER;           // nonzeros per lane per window
constexpr int kWin = 32 * kPer;             // nonzeros per warp window
static_assert(kPer == 4 || kPer == 8 || kPer == 16, "window of 4, 8 or 16 nonzeros per lane");
// Cost of a row in nonzeros when balancing warp ranges (row pointer, flags,
// epilogue inputs and outputs vs index, value and gather per nonzero).
#ifndef RHP_ROW_WEIGHT
#define RHP_ROW_WEIGHT 3.0
#endif
constexpr double kRowWeight = RHP_ROW_WEIGHT;

// std::max / std::min semantics (first argument wins on ties and NaN), which
// the reference's projections rely on (lp_problem.cpp:62, pdhg.cpp:44,54).
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// a*((1+g)*next - g*cur) + b*anchor, restart.cpp:29 evaluation order.
__device__ __forceinline__ double affine(double a, double opg, double g, double b, double next,
                                         double cur, double anchor) {
  return add(mul(a, sub(mul(opg, next), mul(g, cur))), mul(b, anchor));
}

// Streaming loads for matrix data: evict-first so the gathered vectors stay
// resident in L2 while the (larger than L2) matrix streams through.
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ int ld_stream(const int* p) { return __ldcs(p); }
__device__ __forceinline__ int64_t ld_stream(const int64_t* p) { return __ldcs((const long long*)p); }

// Gather of the SpMV input vector: L1::no_allocate (a random gather over a
// vector much larger than L1 almost never hits, and allocating evicts useful
// lines) with an evict_last L2 policy (createpolicy + L2::cache_hint), so the
// streamed matrix (evict_first) and the epilogue vectors never push the
// gathered vector out of L2: C4 (x = 160 MB > L2) 1117 -> 1170 iter/s, C2
// +0.7 %, C3 and C5 neutral. L1G (RHP_L1_GATHER=1, rhp_cuda.cu
// choose_gather_policy): the L1-allocating variant of the same load.
template <bool L1G = false>
__device__ __forceinline__ double ld_gather(const double* p) {
  double e;
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  if constexpr (L1G) asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(e) : "l"(p), "l"(pol));
  else asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(e) : "l"(p), "l"(pol));
  return e;
}

// Programmatic dependent launch (launch_spmv sets the attribute): wait until
// the preceding kernel has completed and its writes are visible (a no-op when
// launched without the attribute), then let the next kernel's CTAs be
// scheduled as this grid's CTAs retire, so its launch latency overlaps this
// kernel's tail.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Merge-path engine: load a window's epilogue inputs (rows r .. r+31) before
// its gathers (spmv.cuh chunk_range). Off by default (A/B variant).
#ifndef RHP_UNIFORM_ROWS
#define RHP_UNIFORM_ROWS 1  // thread-per-row: arithmetic row starts for uniform rows (spmv.cuh)
#endif
#ifndef RHP_EPI_PREFETCH
#define RHP_EPI_PREFETCH 0
#endif

// 32-bit row / nonzero positions inside the SpMV warp walk.
#ifndef RHP_IDX32
#define RHP_IDX32 1
#endif

// Target cost (nonzeros + 3 rows) of one merge-path chunk when the gathered
// vector exceeds kGatherL2Bytes: max(1, cost / (warps * kChunkCost)) chunks
// per warp (layout.cu build_schedule).
#ifndef RHP_CHUNK_COST
#define RHP_CHUNK_COST 2048
#endif
constexpr int kChunkCost = RHP_CHUNK_COST;
constexpr double kGatherL2Bytes = 32.0 * 1024 * 1024;

// Operators whose longest row has at most kThreadRowMax nonzeros use the
// thread-per-row engine (spmv.cuh thread_rows; rhp_cuda.cu choose_engines).
constexpr int64_t kThreadRowMax = 8;
// Operators whose every row has at least kCtaRowMin nonzeros use the long-row
// engine (spmv.cuh spmv_cta_rows), kCtaRowsBatch rows per CTA pass.
constexpr int64_t kCtaRowMin = 256;
#ifndef RHP_CTA_BATCH
#define RHP_CTA_BATCH 4
#endif
#ifndef RHP_CTA_UNROLL
#define RHP_CTA_UNROLL 4
#endif
#ifndef RHP_CTA_BLOCKS
#define RHP_CTA_BLOCKS 4
#endif
constexpr int kCtaRowsBatch = RHP_CTA_BATCH;   // rows walked at once per CTA
constexpr int kCtaRowUnroll = RHP_CTA_UNROLL;  // elements per row per thread in flight
constexpr int kCtaRowBlocks = RHP_CTA_BLOCKS;  // resident CTAs per SM the kernel is built for
#ifndef RHP_ROWS_IN_FLIGHT
#define RHP_ROWS_IN_FLIGHT 2
#endif
#ifndef RHP_CONST_INPUTS_KERNEL
#define RHP_CONST_INPUTS_KERNEL 1  // epilogue inputs may be kernel parameters (ConstInputs)
#endif
#ifndef RHP_ROWS_KERNEL_COMBINED
#define RHP_ROWS_KERNEL_COMBINED 1  // spmv_rows also carries the merge path (spmv.cuh)
#endif
#ifndef RHP_ROWS_VEC
#define RHP_ROWS_VEC 1  // thread-per-row, uniform rows of a multiple of 4: 16-B index/value loads
#endif
#ifndef RHP_UNIFORM_RF
#define RHP_UNIFORM_RF 1  // rows in flight of the thread-per-row engine on uniform rows
#endif

// K1/K2 pairs per body of the block graph's WHILE node (one conditional
// evaluation per body; copies after a stop exit at entry). C2: 2 -> 6893,
// 4 -> 6967, 8 -> 6971 iter/s; C3: 22.4k -> 22.9k -> 23.1k.
#ifndef RHP_GRAPH_UNROLL
#define RHP_GRAPH_UNROLL 8
#endif
constexpr int kGraphUnroll = RHP_GRAPH_UNROLL;

// Loop control shared by host and device (one per ctx, device resident).
struct Ctl {
  // -- parameters written by the host (rhp_set_step)
  double eta, omega, gamma;
  double tau, sigma, sigma_inv, primal_scale, dual_scale;
  double beta_s, beta_n, beta_a;
  int64_t check_interval, iteration_limit, block_limit;
  int32_t restarts_enabled, record_history;
  // -- loop state
  int64_t k, total, block_iters;
  double r_anchor, r_prev, r_last, q_last;
  int32_t stop, verdict, check_due, breakdown;
  int32_t k1_token, bench;         // bench: kernels ignore the block-stop guards (rhp_time_kernels)
  // PID inputs of the current Halpern iterate
  double x_dist2, y_dist2, x_norm2, y_norm2;
  // -- KKT sums
  double kkt_cx, kkt_py, kkt_pr, kkt_viol2, kkt_eq2, kkt_cone2;
  double kkt_py_inf, kkt_pr_inf, kkt_nan_x, kkt_nan_y;
  // -- power iteration
  double pw_vw, pw_ww;
  // -- last-block tickets (one per finalizing kernel family)
  unsigned int ticket_dual, ticket_kkt, ticket_pow, ticket_spare;
  unsigned long long cond_handle;  // cudaGraphConditionalHandle of the block WHILE node
  int32_t graph_mode;
  int32_t k1_token_pending;        // row-partitioned path: K1 ran, control not yet
  double* hist;                    // [block_limit] residual history of the current block
  int* stop_mirror;                // partitioned plain mode: mapped host flags [block_limit]
  unsigned long long peer_epoch;   // peer exchange sequence (peer.cuh): only grows
};

// Operator schedule (built by layout.cu for a given warp count): chunk c is
// the merge-path range that starts at row warp_row[c], nonzero warp_nz[c]
// and ends where chunk c+1 starts (rows + nonzeros balanced, boundaries
// snapped to row starts except inside long rows); warp w walks chunks w,
// w + n_warps, ... A row cut by one or more chunk boundaries is a "split row"
// with a slot: every chunk that touches it stores its partial sum, and the
// last one to arrive adds them in chunk order and runs the row's epilogue
// (reductions into long_red[slot]).
struct Sched {
  int32_t thread_rows;        // 1: thread-per-row engine (spmv.cuh thread_rows), no chunks or slots
  int32_t n_multi;            // split rows (slots)
  int32_t n_warps;            // warps of the grid the schedule was built for (grid * kWarps)
  int32_t n_chunks;           // merge-path chunks (a multiple of n_warps); warp w walks w, w+W, ...
  int64_t rows;
  const int64_t* rp;          // the operator's row pointers
  const int64_t* warp_row;    // [n_chunks + 1] first row of chunk c
  const int64_t* warp_nz;     // [n_chunks + 1] first nonzero of chunk c
  const int32_t* head_slot;   // [n_chunks] slot of warp_row[c] when the chunk starts inside it, else -1
  const int32_t* tail_slot;   // [n_chunks] slot of the row the chunk ends inside, else -1
  const int64_t* slot_row;    // [n_multi]
  const int32_t* slot_first;  // [n_multi] first contributing chunk (it holds the row's start)
  const int32_t* slot_count;  // [n_multi] contributing warps (consecutive)
  double* slot_part;          // [2 * n_chunks] per chunk: head partial, tail partial
  unsigned int* slot_ticket;  // [n_multi]
  double* long_red;           // [n_multi * 16] epilogue reductions of split rows
  const double* seg_in;       // column-segmented operators (segments.cuh): running row sums of the
                              // previous segments, added to every row sum before its epilogue; else null
  // thread-per-row operators whose rows all have the same length (C3's and
  // C4's A^T): row i starts at i * uniform_len, no row pointers are read
  // (rhp_cuda.cu apply_engine_rule); 0 -> row pointers
  int32_t uniform_len;
  // with uniform_len: the same nonzeros in 32-row slices stored
  // element-major (element t of row i at (i / 32) * 32 * uniform_len + 32 t
  // + i % 32: one coalesced load per element position of a warp's 32 rows);
  // null -> CSR order (rhp_cuda.cu build_sliced, RHP_SLICED=1)
  const int32_t* sell_ci;
  const double* sell_v;
};

struct Csr {
  const int64_t* rp;
  const int32_t* ci;
  const double* v;
  int64_t rows;
};

// ------------------------------------------------------------ reductions --
// Block-reduce N per-thread values (fixed xor-butterfly + fixed warp order)
// and store thread 0's totals into part[q*stride + slot].
template <int N>
__device__ __forceinline__ void block_reduce_store(const double (&acc)[N], double* part,
                                                   int stride, int slot) {
  __shared__ double sm[N][kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < N; ++q) {
    double v = acc[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) sm[q][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < N) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += sm[threadIdx.x][w];
    part[(size_t)threadIdx.x * stride + slot] = s;
  }
  __syncthreads();
}

// Thread-strided sums of `count` partials per quantity (SoA, `stride`),
// added into v in index order. The loads of a batch (B per quantity) are all
// issued before any add, so the finalizing block pays one L2 round trip per
// batch rather than one per partial — this sum sits on the serial tail of
// every finalizing kernel.
template <int N, int B = 2>
__device__ __forceinline__ void thread_partials(const double* part, int count, int stride,
                                                double (&v)[N]) {
  for (int base = 0; base < count; base += B * kBlock) {
    double t[N][B];
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int i = base + b * kBlock + threadIdx.x;
        t[q][b] = i < count ? __ldcg(part + (size_t)q * stride + i) : 0.0;
      }
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
      for (int b = 0; b < B; ++b) v[q] += t[q][b];
  }
}

// The same for the epilogue reductions of split rows (slot-major, 16 apart).
template <int N, int B = 4>
__device__ __forceinline__ void thread_slots(const double* long_red, int n_multi, double (&v)[N]) {
  for (int base = 0; base < n_multi; base += B * kBlock) {
    double t[N][B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int i = base + b * kBlock + threadIdx.x;
#pragma unroll
      for (int q = 0; q < N; ++q) t[q][b] = i < n_multi ? __ldcg(long_red + (size_t)i * 16 + q) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
      for (int b = 0; b < B; ++b) v[q] += t[q][b];
  }
}

// Fixed block tree (xor butterfly, then warps in order) of N per-thread
// values; every thread receives the totals.
template <int N>
__device__ __forceinline__ void block_tree(const double (&v)[N], double (&out)[N]) {
  __shared__ double sm[N][kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < N; ++q) {
    double t = v[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (lane == 0) sm[q][warp] = t;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < N; ++q) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += sm[q][w];
    out[q] = s;
  }
  __syncthreads();
}

// Block-wide fixed-order sum of `count` partials per quantity (SoA, stride);
// every thread receives the totals.
template <int N>
__device__ __forceinline__ void block_sum_partials(const double* part, int count, int stride,
                                                   double (&out)[N]) {
  double v[N];
#pragma unroll
  for (int q = 0; q < N; ++q) v[q] = 0.0;
  thread_partials<N>(part, count, stride, v);
  block_tree<N>(v, out);
}

// Adds the epilogue reductions of split rows: block-parallel, fixed order
// (thread-strided sums, then the fixed block tree).
template <int N>
__device__ __forceinline__ void add_slots(const double* long_red, int n_multi, double (&out)[N]) {
  if (n_multi == 0) return;
  double v[N], t[N];
#pragma unroll
  for (int q = 0; q < N; ++q) v[q] = 0.0;
  thread_slots<N>(long_red, n_multi, v);
  block_tree<N>(v, t);
#pragma unroll
  for (int q = 0; q < N; ++q) out[q] += t[q];
}

template <int N>
__device__ __forceinline__ void add_long_slots(const Sched& s, double (&out)[N]) {
  add_slots<N>(s.long_red, s.n_multi, out);
}

// The end-of-iteration sums of K1's finalize in one pass: y-side sums t1
// (K1's partials + A's split-row slots) and x-side sums t3 (the previous
// primal walker's partials + A^T's split-row slots). All loads are issued
// before the single block tree. Same values as block_sum_partials followed
// by add_slots for each side.
template <int N1, int N3>
__device__ __forceinline__ void iteration_sums(const double* part1, int grid1, const double* red1,
                                               int multi1, const double* part3, int grid3,
                                               const double* red3, int multi3, double (&t1)[N1],
                                               double (&t3)[N3]) {
  constexpr int N = 2 * (N1 + N3);
  double v[N];
#pragma unroll
  for (int q = 0; q < N; ++q) v[q] = 0.0;
  double* a1 = v;
  double* s1 = v + N1;
  double* a3 = v + 2 * N1;
  double* s3 = v + 2 * N1 + N3;
  thread_partials<N1>(part1, grid1, grid1, *reinterpret_cast<double(*)[N1]>(a1));
  thread_partials<N3>(part3, grid3, grid3, *reinterpret_cast<double(*)[N3]>(a3));
  thread_slots<N1>(red1, multi1, *reinterpret_cast<double(*)[N1]>(s1));
  thread_slots<N3>(red3, multi3, *reinterpret_cast<double(*)[N3]>(s3));
  double o[N];
  block_tree<N>(v, o);
#pragma unroll
  for (int q = 0; q < N1; ++q) t1[q] = multi1 ? o[q] + o[N1 + q] : o[q];
#pragma unroll
  for (int q = 0; q < N3; ++q) t3[q] = multi3 ? o[2 * N1 + q] + o[2 * N1 + N3 + q] : o[2 * N1 + q];
}

// Last-block-done election. Returns true in exactly one block, after every
// block's partial stores are visible to it. The verdict travels through
// __syncthreads_or (a register result), not a shared variable, so the
// finalize's shared-memory trees that follow cannot race with its readers
// (compute-sanitizer racecheck, tests/test_sanitizer.py).
__device__ __forceinline__ bool elect_last_block(unsigned int* ticket) {
  __threadfence();
  __syncthreads();
  int mine = 0;
  if (threadIdx.x == 0) mine = atomicAdd(ticket, 1u) == gridDim.x - 1;
  const bool last = __syncthreads_or(mine) != 0;
  if (last) __threadfence();
  return last;
}

}  // namespace rhp
