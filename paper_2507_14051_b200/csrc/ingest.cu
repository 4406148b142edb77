// ingest.cu — device-side LP ingest.
//
// Replaces the host O(nnz) work of building the device layout: the borrowed
// CSR of rows [row_begin, row_end) is uploaded as is, then on the GPU
//   * validated exactly like SparseMatrix (sparse_matrix.cpp:23-31,
//     model.cpp from_csr): column in range, value finite, columns strictly
//     increasing in a row — the FIRST offending element in row-major order is
//     found (atomicMin over element positions) and reported with the host's
//     message;
//   * explicit zeros dropped (stable compaction by an exclusive scan of the
//     keep flags; row pointers re-derived from the scan);
//   * column indices narrowed to int32;
//   * CSR(A^T) = the reference's CSC (rows ascending inside every column,
//     sparse_matrix.cpp:53-64) built by a STABLE radix sort of the element
//     positions keyed by column (cub::DeviceRadixSort, LSD → rows stay in
//     ascending order within a column), row pointers by a column histogram +
//     exclusive scan, then a gather of row ids and values.
// Only the row pointers (O(m + n)) come back to the host, for the warp
// schedules. C4 (60M nonzeros): host layout 2.6 s -> device ingest ≈ 0.2 s.
#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "ingest.cuh"

namespace rhp {
namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw DeviceFailure(std::string("device ingest: ") + what + ": " + cudaGetErrorString(e));
}
#define ICK(call) ck((call), #call)

// Scratch device buffer freed at scope exit.
template <class T>
struct Scratch {
  T* p = nullptr;
  explicit Scratch(size_t count) { ICK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T) + 64)); }
  ~Scratch() {
    if (p) cudaFree(p);
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
};

constexpr int kThreads = 256;
inline unsigned blocks_for(int64_t n) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads, 1 << 20)));
}

// first[e] = 1 when element e starts a (non-empty) row
__global__ void k_mark_row_starts(const int64_t* rp, int64_t rows, unsigned char* first) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    if (rp[r + 1] > rp[r]) first[rp[r]] = 1;
}

// err[0]: first element with a bad column / non-finite value / unsorted column
// (min over positions); nzero: explicit zeros; ci32: narrowed columns.
__global__ void k_validate(const int64_t* ci, const double* v, const unsigned char* first, int64_t nz,
                           int64_t cols, unsigned long long* err, unsigned long long* nzero,
                           int32_t* ci32) {
  unsigned long long zeros = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = ci[e];
    const double x = v[e];
    const bool bad = j < 0 || j >= cols || !isfinite(x) || (!first[e] && j <= ci[e - 1]);
    if (bad) atomicMin(err, static_cast<unsigned long long>(e));
    ci32[e] = static_cast<int32_t>(j);
    zeros += x == 0.0;
  }
  if (zeros) atomicAdd(nzero, zeros);
}

__global__ void k_keep_flags(const double* v, int64_t nz, int32_t* keep) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nz;
       e += (int64_t)gridDim.x * blockDim.x)
    keep[e] = v[e] != 0.0;
}

// compaction of the kept elements to their scanned positions
__global__ void k_compact(const int32_t* ci32, const double* v, const int32_t* keep, const int64_t* pos,
                          int64_t nz, int32_t* ci_out, double* v_out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nz;
       e += (int64_t)gridDim.x * blockDim.x)
    if (keep[e]) {
      ci_out[pos[e]] = ci32[e];
      v_out[pos[e]] = v[e];
    }
}

__global__ void k_remap_rp(const int64_t* rp_raw, const int64_t* pos, int64_t rows, int64_t* rp) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= rows;
       r += (int64_t)gridDim.x * blockDim.x)
    rp[r] = pos[rp_raw[r]];
}

__global__ void k_iota(int32_t* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = static_cast<int32_t>(i);
}

__global__ void k_col_hist(const int32_t* ci, int64_t nz, int64_t* cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nz;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + ci[e]), 1ull);
}

// A^T element s <- A element src[s]: its row (binary search in A's row
// pointers) and value
__global__ void k_gather_t(const int32_t* src, const int64_t* rp, int64_t rows, const double* v,
                           int64_t nz, int32_t* t_ci, double* t_v) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nz;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = src[s];
    int64_t lo = 0, hi = rows - 1;  // last row r with rp[r] <= e
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (rp[mid] <= e) lo = mid;
      else hi = mid - 1;
    }
    t_ci[s] = static_cast<int32_t>(lo);
    t_v[s] = v[e];
  }
}

int end_bit_for(int64_t n) {
  int b = 1;
  while (b < 31 && (int64_t{1} << b) < n) ++b;
  return b;
}


// A^T (arrays allocated, rows = n) from A: stable radix sort of the element
// positions keyed by column, so rows stay ascending inside every column.
void build_transpose(const DeviceCsr& A, int64_t n, DeviceCsr& At, cudaStream_t s) {
  const int64_t nnz = A.nnz, m = A.rows;
  ICK(cudaMemsetAsync(At.rp, 0, (n + 1) * sizeof(int64_t), s));
  if (!nnz) return;
  Scratch<int32_t> keys_out(nnz), idx_in(nnz), idx_out(nnz);
  k_iota<<<blocks_for(nnz), kThreads, 0, s>>>(idx_in.p, nnz);
  size_t tb = 0;
  const int eb = end_bit_for(n);
  ICK(cub::DeviceRadixSort::SortPairs(nullptr, tb, A.ci, keys_out.p, idx_in.p, idx_out.p, nnz, 0, eb, s));
  Scratch<unsigned char> tmp(tb);
  ICK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, A.ci, keys_out.p, idx_in.p, idx_out.p, nnz, 0, eb, s));
  Scratch<int64_t> cnt(n + 1);
  ICK(cudaMemsetAsync(cnt.p, 0, (n + 1) * sizeof(int64_t), s));
  k_col_hist<<<blocks_for(nnz), kThreads, 0, s>>>(A.ci, nnz, cnt.p);
  size_t tb2 = 0;
  ICK(cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt.p, At.rp, n + 1, s));
  Scratch<unsigned char> tmp2(tb2);
  ICK(cub::DeviceScan::ExclusiveSum(tmp2.p, tb2, cnt.p, At.rp, n + 1, s));
  k_gather_t<<<blocks_for(nnz), kThreads, 0, s>>>(idx_out.p, A.rp, m, A.v, nnz, At.ci, At.v);
  ICK(cudaGetLastError());
  ICK(cudaStreamSynchronize(s));
}

// ---- locality relabelling ------------------------------------------------
//
// The SpMV gathers x[c] (A) and y[r] (A^T) one 8-B element per nonzero; what
// the gathers cost is the number of distinct 32-B sectors a warp's window
// touches (L1TEX / L2 sector throughput, not HBM bytes). When
// the gathered vectors are larger than L2's comfortable share, rows and
// columns are renumbered in first-touch order — columns by the first row that
// uses them, then rows by the first (renumbered) column they use, twice —
// so the columns of neighbouring rows sit in neighbouring sectors (C4's
// arcs of one node, its commodity rows next to its capacity rows). The
// relabelling is kept only if the measured sectors per window drop by
// kRelabelGain; the device order maps (HostLayout::prow / pcol) carry it to
// every host<->device copy, so nothing outside the device sees it. The
// arithmetic is unchanged; only summation orders move (tolerance-level, like
// any reduction order).

constexpr double kRelabelGain = 0.8;  // keep when sectors(new) <= 0.8 * sectors(old)
constexpr int kRelabelPasses = 2;
constexpr double kRelabelSkip = 0.95;  // sectors per nonzero of an already scattered operator

// key[j] = first row touching column j (A^T rows ascend), empty: UINT32_MAX
__global__ void k_col_first(const int64_t* trp, const int32_t* tci, int64_t n, uint32_t* key) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    key[j] = trp[j + 1] > trp[j] ? static_cast<uint32_t>(tci[trp[j]]) : 0xFFFFFFFFu;
}

// key[i] = smallest new label among row i's columns, empty: UINT32_MAX
__global__ void k_row_first(const int64_t* rp, const int32_t* ci, int64_t m, const int32_t* clab,
                            uint32_t* key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t k = 0xFFFFFFFFu;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) k = min(k, static_cast<uint32_t>(clab[ci[e]]));
    key[i] = k;
  }
}

// lab[order[i]] = i
__global__ void k_invert(const int32_t* order, int64_t n, int32_t* lab) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    lab[order[i]] = static_cast<int32_t>(i);
}

// out[i] = in[order[i]] (composition of order maps)
__global__ void k_compose(const int32_t* in, const int32_t* order, int64_t n, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[order[i]];
}

// element keys (new row << 32 | new column) of A, one thread per row
__global__ void k_elem_keys(const int64_t* rp, const int32_t* ci, int64_t m, const int32_t* rlab,
                            const int32_t* clab, uint64_t* key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t hi = static_cast<uint64_t>(static_cast<uint32_t>(rlab[i])) << 32;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e)
      key[e] = hi | static_cast<uint32_t>(clab[ci[e]]);
  }
}

__global__ void k_split_keys(const uint64_t* key, int64_t nz, int32_t* ci, int64_t* cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nz;
       e += (int64_t)gridDim.x * blockDim.x) {
    ci[e] = static_cast<int32_t>(key[e] & 0xFFFFFFFFull);
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + (key[e] >> 32)), 1ull);
  }
}

// distinct 32-B sectors of the gathered vector per window of 256 consecutive
// nonzeros (one window per CTA pass: block radix sort + adjacent difference)
__global__ void __launch_bounds__(256) k_window_sectors(const int32_t* ci, int64_t nz,
                                                        unsigned long long* total) {
  using Sort = cub::BlockRadixSort<uint32_t, 256, 1>;
  __shared__ typename Sort::TempStorage ts;
  __shared__ uint32_t sorted[256];
  unsigned long long mine = 0;
  for (int64_t w = blockIdx.x; w * 256 < nz; w += gridDim.x) {
    const int64_t e = w * 256 + threadIdx.x;
    uint32_t k[1] = {e < nz ? static_cast<uint32_t>(ci[e]) >> 2 : 0xFFFFFFFFu};
    Sort(ts).Sort(k);
    sorted[threadIdx.x] = k[0];
    __syncthreads();
    const bool fresh = k[0] != 0xFFFFFFFFu && (threadIdx.x == 0 || sorted[threadIdx.x - 1] != k[0]);
    const int cnt = __syncthreads_count(fresh);
    if (threadIdx.x == 0) mine += static_cast<unsigned long long>(cnt);
    __syncthreads();
  }
  if (threadIdx.x == 0 && mine) atomicAdd(total, mine);
}

unsigned long long window_sectors(const DeviceCsr& op, cudaStream_t s) {
  if (!op.nnz) return 0;
  Scratch<unsigned long long> t(1);
  ICK(cudaMemsetAsync(t.p, 0, sizeof(unsigned long long), s));
  const int64_t wins = (op.nnz + 255) / 256;
  k_window_sectors<<<static_cast<unsigned>(std::min<int64_t>(wins, 148 * 16)), 256, 0, s>>>(op.ci, op.nnz, t.p);
  ICK(cudaGetLastError());
  unsigned long long h = 0;
  ICK(cudaMemcpyAsync(&h, t.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  ICK(cudaStreamSynchronize(s));
  return h;
}

// order[i] = the index with the i-th smallest key (ties by index: stable)
void order_by_key(const uint32_t* key, int64_t n, int32_t* order, cudaStream_t s) {
  Scratch<uint32_t> kout(n);
  Scratch<int32_t> idx(n);
  k_iota<<<blocks_for(n), kThreads, 0, s>>>(idx.p, n);
  size_t tb = 0;
  ICK(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, kout.p, idx.p, order, n, 0, 32, s));
  Scratch<unsigned char> tmp(tb);
  ICK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key, kout.p, idx.p, order, n, 0, 32, s));
}

// One first-touch pass: new column order from A^T, new row order from the
// renumbered columns, then A rebuilt (rows by new label, columns ascending
// by new label) and A^T from it. order_r / order_c (device) compose: entry
// i = the ORIGINAL index now at position i.
void relabel_pass(DeviceCsr& A, DeviceCsr& At, int64_t m, int64_t n, int32_t* order_r, int32_t* order_c,
                  cudaStream_t s) {
  const int64_t nnz = A.nnz;
  Scratch<uint32_t> ckey(n), rkey(m);
  Scratch<int32_t> cord(n), clab(n), rord(m), rlab(m), tmp_r(m), tmp_c(n);
  k_col_first<<<blocks_for(n), kThreads, 0, s>>>(At.rp, At.ci, n, ckey.p);
  order_by_key(ckey.p, n, cord.p, s);
  k_invert<<<blocks_for(n), kThreads, 0, s>>>(cord.p, n, clab.p);
  k_row_first<<<blocks_for(m), kThreads, 0, s>>>(A.rp, A.ci, m, clab.p, rkey.p);
  order_by_key(rkey.p, m, rord.p, s);
  k_invert<<<blocks_for(m), kThreads, 0, s>>>(rord.p, m, rlab.p);
  {
    Scratch<uint64_t> kin(nnz), kout(nnz);
    Scratch<double> vout(nnz);
    k_elem_keys<<<blocks_for(m), kThreads, 0, s>>>(A.rp, A.ci, m, rlab.p, clab.p, kin.p);
    size_t tb = 0;
    const int eb = 32 + end_bit_for(m);
    ICK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin.p, kout.p, A.v, vout.p, nnz, 0, eb, s));
    Scratch<unsigned char> tmp(tb);
    ICK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, kin.p, kout.p, A.v, vout.p, nnz, 0, eb, s));
    Scratch<int64_t> cnt(m + 1);
    ICK(cudaMemsetAsync(cnt.p, 0, (m + 1) * sizeof(int64_t), s));
    k_split_keys<<<blocks_for(nnz), kThreads, 0, s>>>(kout.p, nnz, A.ci, cnt.p);
    size_t tb2 = 0;
    ICK(cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt.p, A.rp, m + 1, s));
    Scratch<unsigned char> tmp2(tb2);
    ICK(cub::DeviceScan::ExclusiveSum(tmp2.p, tb2, cnt.p, A.rp, m + 1, s));
    ICK(cudaMemcpyAsync(A.v, vout.p, nnz * sizeof(double), cudaMemcpyDeviceToDevice, s));
    ICK(cudaGetLastError());
    ICK(cudaStreamSynchronize(s));
  }
  build_transpose(A, n, At, s);
  k_compose<<<blocks_for(m), kThreads, 0, s>>>(order_r, rord.p, m, tmp_r.p);
  k_compose<<<blocks_for(n), kThreads, 0, s>>>(order_c, cord.p, n, tmp_c.p);
  ICK(cudaMemcpyAsync(order_r, tmp_r.p, m * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  ICK(cudaMemcpyAsync(order_c, tmp_c.p, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  ICK(cudaGetLastError());
  ICK(cudaStreamSynchronize(s));
}

// locality: 0 auto (gathered vector > kGatherL2Bytes / 4 and fewer sectors),
// < 0 off, > 0 forced (tests). Returns whether the layout was relabelled;
// order_r / order_c (host) then hold the original index at each position.
bool maybe_relabel(DeviceCsr& A, DeviceCsr& At, int64_t m, int64_t n, int locality,
                   std::vector<int32_t>& order_r, std::vector<int32_t>& order_c, double (&sectors)[4],
                   cudaStream_t s) {
  for (double& x : sectors) x = 0.0;
  if (locality < 0 || A.nnz == 0 || m == 0 || n == 0) return false;
  const double big = kGatherL2Bytes / 4.0;
  if (locality == 0 && !(8.0 * static_cast<double>(n) > big || 8.0 * static_cast<double>(m) > big))
    return false;
  const double sa0 = static_cast<double>(window_sectors(A, s)), st0 = static_cast<double>(window_sectors(At, s));
  const double before = sa0 + st0;
  sectors[0] = sa0 / static_cast<double>(A.nnz);
  sectors[1] = st0 / static_cast<double>(A.nnz);
  // every gather already on a sector of its own (uniformly scattered
  // columns, C5): first touch has nothing to regroup (C2-like LPs gain ~10 %
  // at best, below kRelabelGain) — skip the passes (C5: ~10 s of setup)
  if (locality == 0 && sectors[0] > kRelabelSkip && sectors[1] > kRelabelSkip) return false;
  // keep A's original arrays until the verdict (A^T is rebuilt from them on
  // a revert); skipped in auto mode when the device cannot hold the copies
  // and the sort buffers (~60 B per nonzero)
  const int64_t nnz = A.nnz;
  if (locality == 0) {
    size_t free_b = 0, total_b = 0;
    ICK(cudaMemGetInfo(&free_b, &total_b));
    if (static_cast<double>(free_b) < 1.25 * 60.0 * static_cast<double>(nnz) + 1e9) return false;
  }
  Scratch<int64_t> a_rp(m + 1);
  Scratch<int32_t> a_ci(nnz);
  Scratch<double> a_v(nnz);
  ICK(cudaMemcpyAsync(a_rp.p, A.rp, (m + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  ICK(cudaMemcpyAsync(a_ci.p, A.ci, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  ICK(cudaMemcpyAsync(a_v.p, A.v, nnz * sizeof(double), cudaMemcpyDeviceToDevice, s));
  Scratch<int32_t> ordr(m), ordc(n);
  k_iota<<<blocks_for(m), kThreads, 0, s>>>(ordr.p, m);
  k_iota<<<blocks_for(n), kThreads, 0, s>>>(ordc.p, n);
  ICK(cudaGetLastError());
  int passes = kRelabelPasses;
  if (const char* e = std::getenv("RHP_RELABEL_PASSES")) passes = std::max(1, std::atoi(e));
  const bool trace = std::getenv("RHPDHG_SETUP_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  for (int p = 0; p < passes; ++p) relabel_pass(A, At, m, n, ordr.p, ordc.p, s);
  if (trace) {
    ICK(cudaStreamSynchronize(s));
    std::fprintf(stderr, "    relabel %d passes %9.3f s\n", passes,
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  const double sa = static_cast<double>(window_sectors(A, s)), st = static_cast<double>(window_sectors(At, s));
  sectors[2] = sa / static_cast<double>(nnz);
  sectors[3] = st / static_cast<double>(nnz);
  if (locality == 0 && sa + st > kRelabelGain * before) {  // not worth it: restore
    ICK(cudaMemcpyAsync(A.rp, a_rp.p, (m + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    ICK(cudaMemcpyAsync(A.ci, a_ci.p, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    ICK(cudaMemcpyAsync(A.v, a_v.p, nnz * sizeof(double), cudaMemcpyDeviceToDevice, s));
    build_transpose(A, n, At, s);
    return false;
  }
  order_r.resize(static_cast<size_t>(m));
  order_c.resize(static_cast<size_t>(n));
  ICK(cudaMemcpyAsync(order_r.data(), ordr.p, m * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  ICK(cudaMemcpyAsync(order_c.data(), ordc.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  ICK(cudaStreamSynchronize(s));
  return true;
}

}  // namespace

void ingest_device(const rhpdhg_lp_view& lp, int64_t row_begin, int64_t row_end, HostLayout& L,
                   DeviceCsr& A, DeviceCsr& At, int locality, cudaStream_t s) {
  const int64_t n = lp.num_vars;
  if (n > INT32_MAX || lp.num_cons > INT32_MAX)
    throw std::invalid_argument("device layout supports at most 2^31-1 rows and columns");
  const int64_t m = row_end - row_begin;
  L.m_global = lp.num_cons;
  L.n = n;
  L.row_begin = row_begin;
  L.row_end = row_end;
  L.m = m;
  const int64_t base = m > 0 ? lp.row_ptr[row_begin] : 0;
  const int64_t z0 = m > 0 ? lp.row_ptr[row_end] - base : 0;
  if (z0 >= INT32_MAX - (1 << 16))  // 32-bit positions in the SpMV walk (spmv.cuh)
    throw std::invalid_argument("device layout supports at most 2^31 - 2^16 nonzeros per GPU");
  for (int64_t i = row_begin; i < row_end; ++i)
    if (lp.row_ptr[i + 1] < lp.row_ptr[i]) throw std::invalid_argument("row_ptr not monotone");

  // (1) raw upload (row pointers rebased on the host: O(m))
  std::vector<int64_t> rp_raw(static_cast<size_t>(m) + 1);
  for (int64_t i = 0; i <= m; ++i) rp_raw[i] = lp.row_ptr[row_begin + i] - base;
  Scratch<int64_t> d_rp_raw(m + 1), d_ci64(z0);
  Scratch<double> d_v_raw(z0);
  ICK(cudaMemcpyAsync(d_rp_raw.p, rp_raw.data(), (m + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  if (z0) {
    ICK(cudaMemcpyAsync(d_ci64.p, lp.col_index + base, z0 * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    ICK(cudaMemcpyAsync(d_v_raw.p, lp.values + base, z0 * sizeof(double), cudaMemcpyHostToDevice, s));
  }

  // (2) validation + narrowing
  Scratch<unsigned char> d_first(z0);
  Scratch<unsigned long long> d_flags(2);
  Scratch<int32_t> d_ci32(z0);
  const unsigned long long none = ~0ull;
  ICK(cudaMemsetAsync(d_first.p, 0, std::max<int64_t>(z0, 1), s));
  ICK(cudaMemcpyAsync(d_flags.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));
  ICK(cudaMemsetAsync(d_flags.p + 1, 0, sizeof(unsigned long long), s));
  if (m) k_mark_row_starts<<<blocks_for(m), kThreads, 0, s>>>(d_rp_raw.p, m, d_first.p);
  if (z0)
    k_validate<<<blocks_for(z0), kThreads, 0, s>>>(d_ci64.p, d_v_raw.p, d_first.p, z0, n, d_flags.p,
                                                   d_flags.p + 1, d_ci32.p);
  ICK(cudaGetLastError());
  unsigned long long flags[2];
  ICK(cudaMemcpyAsync(flags, d_flags.p, sizeof(flags), cudaMemcpyDeviceToHost, s));
  ICK(cudaStreamSynchronize(s));
  if (flags[0] != none) {
    // the first offending element in row-major order, checked in the host's order
    const int64_t e = static_cast<int64_t>(flags[0]) + base;
    const int64_t i = static_cast<int64_t>(std::upper_bound(lp.row_ptr + row_begin, lp.row_ptr + row_end + 1, e) -
                                           lp.row_ptr) - 1;
    const int64_t j = lp.col_index[e];
    const std::string at = "(" + std::to_string(i) + "," + std::to_string(j) + ")";
    if (j < 0 || j >= n) throw std::out_of_range("matrix entry " + at + " out of bounds");
    if (!std::isfinite(lp.values[e])) throw std::domain_error("matrix entry " + at + " is not finite");
    throw std::domain_error("duplicate or unsorted matrix entry " + at);
  }

  // (3) explicit zeros dropped (rare: a stable compaction)
  const int64_t nnz = z0 - static_cast<int64_t>(flags[1]);
  L.nnz = nnz;
  A.rows = m;
  A.nnz = nnz;
  A.rp = dev_alloc_zero<int64_t>(m + 1);
  A.ci = dev_alloc_zero<int32_t>(nnz);
  A.v = dev_alloc_zero<double>(nnz);
  if (flags[1] == 0) {
    ICK(cudaMemcpyAsync(A.rp, d_rp_raw.p, (m + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    if (nnz) {
      ICK(cudaMemcpyAsync(A.ci, d_ci32.p, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
      ICK(cudaMemcpyAsync(A.v, d_v_raw.p, nnz * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
  } else {
    Scratch<int32_t> keep(z0);
    Scratch<int64_t> pos(z0 + 1);
    k_keep_flags<<<blocks_for(z0), kThreads, 0, s>>>(d_v_raw.p, z0, keep.p);
    ICK(cudaMemsetAsync(keep.p + z0, 0, sizeof(int32_t), s));  // scan to z0 + 1: pos[z0] = nnz
    size_t tb = 0;
    ICK(cub::DeviceScan::ExclusiveSum(nullptr, tb, keep.p, pos.p, z0 + 1, s));
    Scratch<unsigned char> tmp(tb);
    ICK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, keep.p, pos.p, z0 + 1, s));
    k_compact<<<blocks_for(z0), kThreads, 0, s>>>(d_ci32.p, d_v_raw.p, keep.p, pos.p, z0, A.ci, A.v);
    k_remap_rp<<<blocks_for(m + 1), kThreads, 0, s>>>(d_rp_raw.p, pos.p, m, A.rp);
    ICK(cudaGetLastError());
    ICK(cudaStreamSynchronize(s));
  }

  // (4) CSR(A^T): stable radix sort of element positions by column
  At.rows = n;
  At.nnz = nnz;
  At.rp = dev_alloc_zero<int64_t>(n + 1);
  At.ci = dev_alloc_zero<int32_t>(nnz);
  At.v = dev_alloc_zero<double>(nnz);
  build_transpose(A, n, At, s);

  // (4b) locality relabelling of rows and columns (large gathered vectors)
  std::vector<int32_t> order_r, order_c;
  L.relabel = maybe_relabel(A, At, m, n, locality, order_r, order_c, L.sectors, s);

  A.v_orig = dev_alloc_zero<double>(nnz);
  At.v_orig = dev_alloc_zero<double>(nnz);
  if (nnz) {
    ICK(cudaMemcpyAsync(A.v_orig, A.v, nnz * sizeof(double), cudaMemcpyDeviceToDevice, s));
    ICK(cudaMemcpyAsync(At.v_orig, At.v, nnz * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }

  // (5) host copies of the row pointers (warp schedules, resident split)
  HostOperator& ha = L.A;
  ha.rows = m;
  ha.cols = n;
  ha.nnz = nnz;
  ha.rp.resize(static_cast<size_t>(m) + 1);
  HostOperator& ht = L.At;
  ht.rows = n;
  ht.cols = m;
  ht.nnz = nnz;
  ht.rp.resize(static_cast<size_t>(n) + 1);
  ICK(cudaMemcpyAsync(ha.rp.data(), A.rp, (m + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  ICK(cudaMemcpyAsync(ht.rp.data(), At.rp, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  ICK(cudaStreamSynchronize(s));

  // (6) order maps: device row / column -> original (identity unless relabelled)
  L.prow.resize(static_cast<size_t>(m));
  for (int64_t r = 0; r < m; ++r)
    L.prow[r] = static_cast<int32_t>(row_begin + (L.relabel ? order_r[r] : r));
  L.pcol.resize(static_cast<size_t>(n));
  for (int64_t j = 0; j < n; ++j) L.pcol[j] = L.relabel ? order_c[j] : static_cast<int32_t>(j);
}

}  // namespace rhp
