// ops.cu — matrix-free per-operation entry points of include/rhpdhg_cuda.h
// (rhp_op_sums, rhp_op_mul): the reductions behind the reference's p_norm /
// fixed_point_residual (pdhg.cpp:68-115) and pid_update (restart.cpp:85-91),
// and unscale_iterate's products (scaling.cpp:83-94), run on the device from
// host vectors. One lazily grown workspace (stream + buffers) per device,
// serialised by a mutex; every call is synchronous.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "op_kernels.cuh"
#include "rhpdhg_cuda.h"

using namespace rhp;

void rhp_internal_set_error(const std::string& msg);  // rhp_cuda.cu

namespace {

struct OpError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw OpError(std::string(what) + ": " + cudaGetErrorString(e));
}

struct Workspace {
  int device = 0;
  cudaStream_t s = nullptr;
  double* buf = nullptr;  // [cap] device scratch
  size_t cap = 0;
  double* part = nullptr;  // [4 * kOpGrid] block partials + 4 results
  double* host = nullptr;  // pinned [4]
};

std::mutex g_mu;

Workspace& workspace(int device, size_t need) {
  static std::map<int, Workspace> all;
  Workspace& w = all[device];
  ck(cudaSetDevice(device), "cudaSetDevice");
  if (!w.s) {
    w.device = device;
    ck(cudaStreamCreateWithFlags(&w.s, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaMalloc(&w.part, (4 * kOpGrid + 8) * sizeof(double)), "cudaMalloc");
    ck(cudaMallocHost(&w.host, 8 * sizeof(double)), "cudaMallocHost");
  }
  if (need > w.cap) {
    if (w.buf) ck(cudaFree(w.buf), "cudaFree");
    w.buf = nullptr;
    w.cap = 0;
    const size_t cap = std::max<size_t>(need, 1 << 16);
    ck(cudaMalloc(&w.buf, cap * sizeof(double)), "cudaMalloc");
    w.cap = cap;
  }
  return w;
}

template <class F>
int op_guarded(F&& f) {
  try {
    std::lock_guard<std::mutex> lock(g_mu);
    f();
    return RHPDHG_OK;
  } catch (const std::invalid_argument& e) {
    rhp_internal_set_error(e.what());
    return RHPDHG_E_USAGE;
  } catch (const std::exception& e) {
    rhp_internal_set_error(e.what());
    return RHPDHG_E_DEVICE;
  }
}

int grid_for(int64_t len) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kOpGrid, (len + kOpBlock - 1) / kOpBlock)));
}

void put(double* dst, const double* src, int64_t len, cudaStream_t s) {
  if (len > 0) ck(cudaMemcpyAsync(dst, src, len * sizeof(double), cudaMemcpyHostToDevice, s), "upload");
}

}  // namespace

extern "C" {

int rhp_op_sums(int device, int64_t n, const double* p, const double* pm, int64_t m,
                const double* q, const double* r, const double* rs, double* out4) {
  return op_guarded([&] {
    if (n < 0 || m < 0) throw std::invalid_argument("rhp_op_sums: negative length");
    const size_t nn = static_cast<size_t>(n), mm = static_cast<size_t>(m);
    Workspace& w = workspace(device, 2 * nn + 3 * mm + 8);
    double* dp = w.buf;
    double* dpm = pm ? dp + nn : nullptr;
    double* dq = w.buf + 2 * nn;
    double* dr = r ? dq + mm : nullptr;
    double* drs = (r && rs) ? dq + 2 * mm : nullptr;
    put(dp, p, n, w.s);
    if (pm) put(dpm, pm, n, w.s);
    put(dq, q, m, w.s);
    if (dr) put(dr, r, m, w.s);
    if (drs) put(drs, rs, m, w.s);
    const int g = grid_for(std::max(n, m));
    k_op_sums4<<<g, kOpBlock, 0, w.s>>>(n, dp, dpm, m, dq, dr, drs, w.part);
    k_op_sums4_final<<<1, 32, 0, w.s>>>(w.part, g, w.part + 4 * kOpGrid);
    ck(cudaGetLastError(), "k_op_sums4");
    ck(cudaMemcpyAsync(w.host, w.part + 4 * kOpGrid, 4 * sizeof(double), cudaMemcpyDeviceToHost, w.s),
       "download");
    ck(cudaStreamSynchronize(w.s), "rhp_op_sums");
    for (int t = 0; t < 4; ++t) out4[t] = w.host[t];
  });
}

int rhp_op_mul(int device, int64_t n, const double* s, const double* v, double* out) {
  return op_guarded([&] {
    if (n < 0) throw std::invalid_argument("rhp_op_mul: negative length");
    if (n == 0) return;
    const size_t nn = static_cast<size_t>(n);
    Workspace& w = workspace(device, 3 * nn);
    put(w.buf, s, n, w.s);
    put(w.buf + nn, v, n, w.s);
    k_op_mul<<<grid_for(n), kOpBlock, 0, w.s>>>(n, w.buf, w.buf + nn, w.buf + 2 * nn);
    ck(cudaGetLastError(), "k_op_mul");
    ck(cudaMemcpyAsync(out, w.buf + 2 * nn, nn * sizeof(double), cudaMemcpyDeviceToHost, w.s),
       "download");
    ck(cudaStreamSynchronize(w.s), "rhp_op_mul");
  });
}

}  // extern "C"
