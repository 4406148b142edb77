// layout.cuh — host-side construction of the device data layout.
//
// The reference keeps A as CSR + CSC with int64 indices (sparse_matrix.cpp:
// 20-65). The device keeps two CSR operators, A (m_local x n) and A^T
// (n x m_local = the reference's CSC), with int32 column indices and int64
// row pointers (12 B per nonzero), rows in the ORIGINAL order and the
// elements of every row in the reference's order (ascending column for A,
// ascending row for A^T), so sequential per-row sums match the reference
// bit-for-bit where the kernels sum sequentially (scaling, short rows).
// Each operator gets a merge-path warp schedule (spmv.cuh) once the grid is
// known (build_schedule).
//
// The operators are built on the device (ingest.cu); the host keeps the row
// pointers for the schedules. The permutation maps (prow/pcol) are kept in
// the interface for layouts that reorder rows; the current layout is the
// identity.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "rhpdhg_c.h"

namespace rhp {

// length class of a row, for diagnostics (rhp_layout_info)
inline int row_kind(int64_t L) {
  if (L <= 4) return 0;
  if (L <= 8) return 1;
  if (L <= 16) return 2;
  if (L <= 32) return 3;
  if (L <= 64) return 4;
  if (L <= 512) return 5;
  if (L <= 1024) return 6;
  return 7;
}

// Host side of a device operator: its row pointers (the column indices and
// values live on the device only, ingest.cu) and its warp schedule.
struct HostOperator {
  int64_t rows = 0, cols = 0, nnz = 0;
  std::vector<int64_t> rp;
  Sched sched{};  // host copy; device pointers filled at upload
  // warp schedule (Sched in device_common.cuh)
  std::vector<int64_t> warp_row, warp_nz, slot_row;
  std::vector<int32_t> head_slot, tail_slot, slot_first, slot_count;
  int64_t bin_rows[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // rows per length class
};

struct HostLayout {
  int64_t m_global = 0, n = 0;
  int64_t row_begin = 0, row_end = 0;  // this rank's original rows
  int64_t m = 0;                       // local rows
  int64_t nnz = 0;                     // local nonzeros (explicit zeros dropped)
  std::vector<int32_t> prow;           // device row -> original row (global index)
  std::vector<int32_t> pcol;           // device col -> original col
  bool relabel = false;                // first-touch locality order (ingest.cu)
  double sectors[4] = {0, 0, 0, 0};    // gather sectors / nnz: A, A^T before, after
  HostOperator A, At;
};

// Merge-path warp schedule of one operator for n_warps warps: ranges
// balanced by nonzeros + row_weight * rows, boundaries snapped to row starts
// except inside rows longer than the snap length.
void build_schedule(HostOperator& op, int64_t n_warps, double row_weight);

// Balanced contiguous row partition by nonzeros: returns
// world_size+1 row offsets.
std::vector<int64_t> partition_rows(const rhpdhg_lp_view& lp, int world_size);

}  // namespace rhp
