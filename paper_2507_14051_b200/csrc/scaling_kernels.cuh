// scaling_kernels.cuh — device Ruiz + Pock-Chambolle preconditioning
// (reference scaling.cpp:10-81, sparse_matrix.cpp:101-136) and the power
// iteration's normalisation. Setup-time kernels: one thread per row, each
// row summed sequentially in the reference's element order with
// non-contracted arithmetic, so every scaled value and scale factor is
// bit-identical to the reference's.
#pragma once

#include "device_common.cuh"

namespace rhp {

// Per-row max |a| -> sqrt or 1 (scaling.cpp:56-61). Max is order-free.
__global__ void k_row_absmax_sqrt(const int64_t* rp, const double* w, int64_t rows, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * kBlock) {
    double mx = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const double a = fabs(w[e]);
      if (a > mx) mx = a;
    }
    out[i] = mx > 0.0 ? sqrt(mx) : 1.0;
  }
}

// w /= row_fac[row] * col_fac[col] (scaling.cpp:62: value /= rmax*cmax;
// multiplication is commutative, so A and A^T copies agree bit-for-bit).
__global__ void k_ruiz_divide(const int64_t* rp, const int32_t* ci, double* w, int64_t rows,
                              const double* row_fac, const double* col_fac) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * kBlock) {
    const double fr = row_fac[i];
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) w[e] = __ddiv_rn(w[e], mul(fr, col_fac[ci[e]]));
  }
}

__global__ void k_vec_div(double* s, const double* by, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kBlock)
    s[i] = __ddiv_rn(s[i], by[i]);
}

// Sliced copy of a uniform-length (w) CSR operator (rhp_cuda.cu
// build_sliced): element t of row i to (i / 32) * 32 w + 32 t + i % 32.
__global__ void k_build_sliced(const int32_t* ci, const double* v, int64_t rows, int w,
                               int32_t* sci, double* sv) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * kBlock) {
    const int64_t o = (i >> 5) * 32 * w + (i & 31);
    for (int t = 0; t < w; ++t) {
      sci[o + 32 * t] = ci[i * w + t];
      sv[o + 32 * t] = v[i * w + t];
    }
  }
}

// flag[0] |= 1 unless every v[i] equals v[0] bitwise (constant-input
// detection for the epilogues, rhp_cuda.cu detect_constant_inputs)
__global__ void k_not_constant(const double* v, int64_t n, unsigned* flag) {
  const unsigned long long v0 = __double_as_longlong(v[0]);
  bool diff = false;
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kBlock)
    diff |= static_cast<unsigned long long>(__double_as_longlong(v[i])) != v0;
  if (__syncthreads_or(diff) && threadIdx.x == 0) atomicOr(flag, 1u);
}

__global__ void k_vec_mul(double* s, const double* by, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kBlock)
    s[i] = mul(s[i], by[i]);
}

// out_e = (f_row * a_e) * f_col (sparse_matrix.cpp:109 for CSR with
// f_row = r, f_col = c; :112 for CSC with f_row = c, f_col = r).
__global__ void k_scale_values(const int64_t* rp, const int32_t* ci, const double* src,
                               double* dst, int64_t rows, const double* f_row,
                               const double* f_col) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * kBlock) {
    const double fr = f_row[i];
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) dst[e] = mul(mul(fr, src[e]), f_col[ci[e]]);
  }
}

// Row 1-norms of the CSR values, sequential per row (sparse_matrix.cpp:130-133):
// out = 1/sqrt(norm) or 1 (scaling.cpp:73).
__global__ void k_pc_rows(const int64_t* rp, const double* v, int64_t rows, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * kBlock) {
    double acc = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) acc = add(acc, fabs(v[e]));
    out[i] = acc > 0.0 ? __ddiv_rn(1.0, sqrt(acc)) : 1.0;
  }
}

// Column 1-norms as the reference accumulates them: for column j, the CSR
// values (r_i a_ij) c_j added in ascending row order (sparse_matrix.cpp:134).
// Walks row j of A^T (ascending rows) recomputing the CSR value from a_ij.
__global__ void k_pc_cols(const int64_t* rp, const int32_t* ci, const double* a_orig,
                          int64_t rows, const double* rs, const double* cs, double* out) {
  for (int64_t j = blockIdx.x * (int64_t)kBlock + threadIdx.x; j < rows;
       j += (int64_t)gridDim.x * kBlock) {
    const double cj = cs[j];
    double acc = 0.0;
    for (int64_t e = rp[j]; e < rp[j + 1]; ++e)
      acc = add(acc, fabs(mul(mul(rs[ci[e]], a_orig[e]), cj)));
    out[j] = acc > 0.0 ? __ddiv_rn(1.0, sqrt(acc)) : 1.0;
  }
}

// apply_scales on the vectors (scaling.cpp:21-32):
//   c <- cs*c, lb <- lb/cs, ub <- ub/cs ; con bounds <- rs*bound
__global__ void k_apply_col_scales(double* c, double* lb, double* ub, const double* cs, int64_t n) {
  for (int64_t j = blockIdx.x * (int64_t)kBlock + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kBlock) {
    const double s = cs[j];
    c[j] = mul(s, c[j]);
    lb[j] = __ddiv_rn(lb[j], s);
    ub[j] = __ddiv_rn(ub[j], s);
  }
}

__global__ void k_apply_row_scales(double* lb, double* ub, const double* rs, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * kBlock) {
    const double s = rs[i];
    lb[i] = mul(s, lb[i]);
    ub[i] = mul(s, ub[i]);
  }
}

// Row-partitioned scaling: per-rank raw column maxima / 1-norm partials are
// combined with an NCCL allreduce (max / sum) before the sqrt step.
__global__ void k_row_absmax_raw(const int64_t* rp, const double* w, int64_t rows, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * kBlock) {
    double mx = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const double a = fabs(w[e]);
      if (a > mx) mx = a;
    }
    out[i] = mx;
  }
}

__global__ void k_sqrt_or_one(double* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kBlock)
    v[i] = v[i] > 0.0 ? sqrt(v[i]) : 1.0;
}

__global__ void k_pc_cols_raw(const int64_t* rp, const int32_t* ci, const double* a_orig,
                              int64_t rows, const double* rs, const double* cs, double* out) {
  for (int64_t j = blockIdx.x * (int64_t)kBlock + threadIdx.x; j < rows;
       j += (int64_t)gridDim.x * kBlock) {
    const double cj = cs[j];
    double acc = 0.0;
    for (int64_t e = rp[j]; e < rp[j + 1]; ++e)
      acc = add(acc, fabs(mul(mul(rs[ci[e]], a_orig[e]), cj)));
    out[j] = acc;
  }
}

__global__ void k_inv_sqrt_or_one(double* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kBlock)
    v[i] = v[i] > 0.0 ? __ddiv_rn(1.0, sqrt(v[i])) : 1.0;
}

// v = w / ||w|| (pdhg.cpp:149)
__global__ void k_normalize(double* v, const double* w, double wn, int64_t n) {
  for (int64_t j = blockIdx.x * (int64_t)kBlock + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kBlock)
    v[j] = __ddiv_rn(w[j], wn);
}

}  // namespace rhp
