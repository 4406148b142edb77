// ingest.cuh — device-side LP ingest (ingest.cu): validation, zero dropping,
// int32 columns and CSR(A^T) built on the GPU from the borrowed host CSR.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "layout.cuh"
#include "rhpdhg_c.h"

namespace rhp {

// A CUDA runtime failure (mapped to RHPDHG_E_DEVICE by the C ABI).
struct DeviceFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// One CSR operator in device memory (12 B per nonzero + row pointers).
struct DeviceCsr {
  int64_t rows = 0, nnz = 0;
  int64_t* rp = nullptr;
  int32_t* ci = nullptr;
  double* v = nullptr;       // current values (original, then scaled)
  double* v_orig = nullptr;  // original values, kept until scaling is done
};

// Zeroed device array with 64 B of tail padding (the SpMV's vector loads may
// read past the last element; never used).
template <class T>
T* dev_alloc_zero(size_t count) {
  void* p = nullptr;
  const size_t bytes = std::max<size_t>(count, 1) * sizeof(T) + 64;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
  // synchronous: the ctx stream is non-blocking, so an asynchronous memset on
  // the legacy stream could land after later work on the ctx stream
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess)
    throw DeviceFailure(std::string("device allocation of ") + std::to_string(bytes) +
                        " bytes: " + cudaGetErrorString(e));
  return static_cast<T*>(p);
}

// Uploads rows [row_begin, row_end) of lp's CSR and builds both device
// operators (A: local rows x n, A^T: n x local rows) and the host row
// pointers / order maps of L. Throws std::out_of_range (column out of
// range), std::domain_error (non-finite value, duplicate/unsorted entry),
// std::invalid_argument (too large), DeviceFailure. locality (rhp_options):
// 0 auto / < 0 off / > 0 forced first-touch relabelling of rows and columns
// (ingest.cu maybe_relabel; L.prow / L.pcol carry it).
void ingest_device(const rhpdhg_lp_view& lp, int64_t row_begin, int64_t row_end, HostLayout& L,
                   DeviceCsr& A, DeviceCsr& At, int locality, cudaStream_t s);

}  // namespace rhp
