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
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
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

}  // namespace

void ingest_device(const rhpdhg_lp_view& lp, int64_t row_begin, int64_t row_end, HostLayout& L,
                   DeviceCsr& A, DeviceCsr& At, cudaStream_t s) {
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
  if (nnz) {
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

  // (6) identity order maps (rows and columns keep the original order)
  L.prow.resize(static_cast<size_t>(m));
  for (int64_t r = 0; r < m; ++r) L.prow[r] = static_cast<int32_t>(row_begin + r);
  L.pcol.resize(static_cast<size_t>(n));
  for (int64_t j = 0; j < n; ++j) L.pcol[j] = static_cast<int32_t>(j);
}

}  // namespace rhp
