// layout.cuh — host-side construction of the device data layout.
//
// The reference keeps A as CSR + CSC with int64 indices in the original row
// and column order (sparse_matrix.cpp:20-65). The device keeps two CSR
// operators, A (m_local x n) and A^T (n x m_local), with
//   * int32 column indices and int64 row pointers (12 B per nonzero),
//   * rows permuted so rows of similar length are contiguous (one bin per
//     SpMV vector width), columns permuted the same way by column length,
//   * the elements of every row kept in the reference's order (ascending
//     original column for A, ascending original row for A^T), so sequential
//     per-row sums in the scaling kernels match the reference bit-for-bit.
// All m- and n-vectors on the device are stored in the permuted order.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "rhpdhg_c.h"

namespace rhp {

constexpr int kKinds = 7;            // 6 sub-warp widths + CTA chunks
constexpr int64_t kChunkNnz = 8192;  // max nonzeros per CTA chunk of a long row

// kind of a row with L nonzeros: 2^kind lanes per row, or 6 = CTA chunks
inline int row_kind(int64_t L) {
  if (L <= 4) return 0;
  if (L <= 8) return 1;
  if (L <= 16) return 2;
  if (L <= 32) return 3;
  if (L <= 64) return 4;
  if (L <= 512) return 5;
  return 6;
}

struct HostOperator {
  int64_t rows = 0, cols = 0, nnz = 0;
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> v;
  Sched sched{};                          // host copy; device pointers filled later
  std::vector<int32_t> chunk_row, chunk_first, chunk_count, chunk_slot;
  std::vector<int64_t> chunk_beg, chunk_end;
  int64_t bin_rows[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

struct HostLayout {
  int64_t m_global = 0, n = 0;
  int64_t row_begin = 0, row_end = 0;  // this rank's original rows
  int64_t m = 0;                       // local rows
  int64_t nnz = 0;                     // local nonzeros (explicit zeros dropped)
  std::vector<int32_t> prow;           // device row -> original row (global index)
  std::vector<int32_t> pcol;           // device col -> original col
  std::vector<int32_t> icol;           // original col -> device col
  // element maps for returning device values in the reference's orders
  std::vector<int64_t> a_dev_to_csr;   // device A element -> reference CSR position (local)
  std::vector<int64_t> at_dev_to_csc;  // device A^T element -> reference CSC position (local)
  HostOperator A, At;
};

// Builds the layout of rows [row_begin, row_end) of the LP (throws
// std::invalid_argument / std::domain_error with the reference's messages
// on malformed input).
void build_layout(const rhpdhg_lp_view& lp, int64_t row_begin, int64_t row_end, HostLayout& out);

// Balanced contiguous row partition by nonzeros: returns
// world_size+1 row offsets.
std::vector<int64_t> partition_rows(const rhpdhg_lp_view& lp, int world_size);

}  // namespace rhp
