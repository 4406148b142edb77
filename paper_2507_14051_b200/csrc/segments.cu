// segments.cu — column segmentation of a device operator (segments.cuh).
//
// Two passes over the operator, one thread per row (a row's columns are
// ascending, so its elements of segment k form one contiguous run): count
// the run lengths per (segment, row), exclusive-scan them into each
// segment's row pointers (cub), then scatter indices and values. O(nnz),
// done once after scaling; the row pointers come back to the host for the
// segments' warp schedules.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <string>

#include "segments.cuh"

namespace rhp {
namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw DeviceFailure(std::string("column segments: ") + what + ": " + cudaGetErrorString(e));
}
#define SCK(call) ck((call), #call)

constexpr int kThreads = 256;
inline unsigned blocks_for(int64_t n) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads, 1 << 20)));
}

// first segment whose end is past column c
__device__ __forceinline__ int seg_of(const int32_t* cb, int S, int32_t c) {
  int lo = 0, hi = S - 1;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (cb[mid + 1] > c) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// cnt[k * (rows + 1) + r] = elements of row r in segment k (zeroed before);
// rows outside the band [rb, re) count everything in the last segment
__global__ void k_seg_count(const int64_t* rp, const int32_t* ci, int64_t rows, const int32_t* cb,
                            int S, int64_t rb, int64_t re, int64_t* cnt) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const int64_t lo = rp[r], hi = rp[r + 1];
    if (lo == hi) continue;
    if (r < rb || r >= re) {
      cnt[static_cast<int64_t>(S - 1) * (rows + 1) + r] = hi - lo;
      continue;
    }
    int k = seg_of(cb, S, ci[lo]);
    int64_t run = 0;
    for (int64_t e = lo; e < hi; ++e) {
      const int32_t c = ci[e];
      if (c >= cb[k + 1]) {
        cnt[static_cast<int64_t>(k) * (rows + 1) + r] = run;
        run = 0;
        k = seg_of(cb, S, c);
      }
      ++run;
    }
    cnt[static_cast<int64_t>(k) * (rows + 1) + r] = run;
  }
}

__global__ void k_seg_scatter(const int64_t* rp, const int32_t* ci, const double* v, int64_t rows,
                              const int32_t* cb, int S, int64_t rb, int64_t re,
                              int64_t* const* srp, int32_t* const* sci, double* const* sv) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const int64_t lo = rp[r], hi = rp[r + 1];
    if (lo == hi) continue;
    const bool band = r >= rb && r < re;
    // intermediate segments index the band's rows locally
    auto start = [&](int k) { return k < S - 1 ? srp[k][r - rb] : srp[S - 1][r]; };
    int k = band ? seg_of(cb, S, ci[lo]) : S - 1;
    int64_t out = start(k);
    for (int64_t e = lo; e < hi; ++e) {
      const int32_t c = ci[e];
      if (band && c >= cb[k + 1]) {
        k = seg_of(cb, S, c);
        out = start(k);
      }
      sci[k][out] = c;
      sv[k][out] = v[e];
      ++out;
    }
  }
}

}  // namespace

void split_columns(const DeviceCsr& op, const std::vector<int32_t>& cb, int64_t rb, int64_t re,
                   std::vector<DeviceCsr>& out, std::vector<std::vector<int64_t>>& host_rp,
                   cudaStream_t s) {
  const int S = static_cast<int>(cb.size()) - 1;
  const int64_t rows = op.rows;
  out.assign(static_cast<size_t>(S), DeviceCsr{});
  host_rp.assign(static_cast<size_t>(S), {});
  int32_t* d_cb = dev_alloc_zero<int32_t>(cb.size());
  int64_t* cnt = dev_alloc_zero<int64_t>(static_cast<size_t>(S) * (rows + 1));
  SCK(cudaMemcpyAsync(d_cb, cb.data(), cb.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  k_seg_count<<<blocks_for(rows), kThreads, 0, s>>>(op.rp, op.ci, rows, d_cb, S, rb, re, cnt);
  SCK(cudaGetLastError());
  size_t tb = 0;
  SCK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, op.rp, rows + 1, s));
  void* tmp = nullptr;
  SCK(cudaMalloc(&tmp, std::max<size_t>(tb, 1)));
  std::vector<int64_t*> prp(S);
  std::vector<int32_t*> pci(S);
  std::vector<double*> pv(S);
  for (int k = 0; k < S; ++k) {
    DeviceCsr& d = out[k];
    // intermediate segments: the band's rows only; the last one: all rows
    const int64_t r0 = k < S - 1 ? rb : 0, nr = k < S - 1 ? re - rb : rows;
    d.rows = nr;
    d.rp = dev_alloc_zero<int64_t>(nr + 1);
    SCK(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt + static_cast<int64_t>(k) * (rows + 1) + r0, d.rp,
                                      nr + 1, s));
    host_rp[k].resize(static_cast<size_t>(nr) + 1);
    SCK(cudaMemcpyAsync(host_rp[k].data(), d.rp, (nr + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SCK(cudaStreamSynchronize(s));
    d.nnz = host_rp[k][nr];
    d.ci = dev_alloc_zero<int32_t>(d.nnz);
    d.v = dev_alloc_zero<double>(d.nnz);
    prp[k] = d.rp;
    pci[k] = d.ci;
    pv[k] = d.v;
  }
  int64_t** d_prp = dev_alloc_zero<int64_t*>(S);
  int32_t** d_pci = dev_alloc_zero<int32_t*>(S);
  double** d_pv = dev_alloc_zero<double*>(S);
  SCK(cudaMemcpyAsync(d_prp, prp.data(), S * sizeof(int64_t*), cudaMemcpyHostToDevice, s));
  SCK(cudaMemcpyAsync(d_pci, pci.data(), S * sizeof(int32_t*), cudaMemcpyHostToDevice, s));
  SCK(cudaMemcpyAsync(d_pv, pv.data(), S * sizeof(double*), cudaMemcpyHostToDevice, s));
  k_seg_scatter<<<blocks_for(rows), kThreads, 0, s>>>(op.rp, op.ci, op.v, rows, d_cb, S, rb, re, d_prp,
                                                      d_pci, d_pv);
  SCK(cudaGetLastError());
  SCK(cudaStreamSynchronize(s));
  for (void* p : {(void*)d_prp, (void*)d_pci, (void*)d_pv, (void*)d_cb, (void*)cnt, tmp}) cudaFree(p);
}

}  // namespace rhp
