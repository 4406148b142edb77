// layout.cu — host-side build of the device layout and tile schedules
// (see layout.cuh). Host code only; compiled by nvcc with the device library.
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

#include "layout.cuh"

namespace rhp {

// Greedy nnz-balanced tiling in row order: a stream tile grows while it has
// <= kTileNnz nonzeros and <= kTileRows rows; a row longer than kTileNnz
// closes the current tile and is cut into chunk tiles of <= kChunkNnz.
void build_schedule(HostOperator& op) {
  op.tile_row.clear();
  op.tile_row_end.clear();
  op.tile_nz.clear();
  op.chunk_row.clear();
  op.chunk_beg.clear();
  op.chunk_end.clear();
  op.chunk_first.clear();
  op.chunk_count.clear();
  op.chunk_slot.clear();
  for (int k = 0; k < 8; ++k) op.bin_rows[k] = 0;
  int32_t n_multi = 0;
  int64_t r = 0;
  while (r < op.rows) {
    const int64_t L = op.rp[r + 1] - op.rp[r];
    op.bin_rows[row_kind(L)]++;
    if (L > kTileNnz) {
      const int64_t b = op.rp[r], e = op.rp[r + 1];
      const int64_t nch = (e - b + kChunkNnz - 1) / kChunkNnz;
      const int32_t first = static_cast<int32_t>(op.chunk_row.size());
      const int32_t slot = nch > 1 ? n_multi++ : -1;
      for (int64_t c = 0; c < nch; ++c) {
        op.chunk_row.push_back(static_cast<int32_t>(r));
        op.chunk_beg.push_back(b + c * kChunkNnz);
        op.chunk_end.push_back(std::min(e, b + (c + 1) * kChunkNnz));
        op.chunk_first.push_back(first);
        op.chunk_count.push_back(static_cast<int32_t>(nch));
        op.chunk_slot.push_back(slot);
      }
      ++r;
      continue;
    }
    const int64_t r0 = r;
    int64_t nz = 0;
    while (r < op.rows && r - r0 < kTileRows) {
      const int64_t len = op.rp[r + 1] - op.rp[r];
      if (len > kTileNnz || nz + len > kTileNnz) break;
      if (r > r0) op.bin_rows[row_kind(len)]++;
      nz += len;
      ++r;
    }
    op.tile_row.push_back(static_cast<int32_t>(r0));
    op.tile_row_end.push_back(static_cast<int32_t>(r));
    op.tile_nz.push_back(op.rp[r0]);
    op.tile_nz.push_back(op.rp[r]);
  }
  Sched& s = op.sched;
  s = Sched{};
  s.n_multi = n_multi;
  s.n_stream = static_cast<int64_t>(op.tile_row.size());
  s.total_tiles = s.n_stream + static_cast<int64_t>(op.chunk_row.size());
}

std::vector<int64_t> partition_rows(const rhpdhg_lp_view& lp, int world_size) {
  std::vector<int64_t> off(static_cast<size_t>(world_size) + 1, lp.num_cons);
  off[0] = 0;
  const int64_t m = lp.num_cons;
  const int64_t total = m > 0 ? lp.row_ptr[m] - lp.row_ptr[0] : 0;
  // contiguous blocks with ~(nnz + rows)/P weight each, so empty rows spread
  const double weight_total = static_cast<double>(total + m);
  int p = 1;
  for (int64_t i = 0; i < m && p < world_size; ++i) {
    const double w = static_cast<double>(lp.row_ptr[i + 1] - lp.row_ptr[0] + (i + 1));
    if (w >= weight_total * p / world_size) off[p++] = i + 1;
  }
  for (; p < world_size; ++p) off[p] = m;
  return off;
}

void build_layout(const rhpdhg_lp_view& lp, int64_t row_begin, int64_t row_end, HostLayout& L) {
  const int64_t n = lp.num_vars;
  if (n > INT32_MAX || lp.num_cons > INT32_MAX)
    throw std::invalid_argument("device layout supports at most 2^31-1 rows and columns");
  L.m_global = lp.num_cons;
  L.n = n;
  L.row_begin = row_begin;
  L.row_end = row_end;
  const int64_t m = row_end - row_begin;
  L.m = m;

  // (1) local CSR in the original order with explicit zeros dropped
  //     (sparse_matrix.cpp:23-31 validation and zero removal)
  HostOperator& A = L.A;
  A.rows = m;
  A.cols = n;
  A.rp.assign(static_cast<size_t>(m) + 1, 0);
  for (int64_t i = 0; i < m; ++i) {
    const int64_t gi = row_begin + i;
    int64_t cnt = 0, prev = -1;
    for (int64_t e = lp.row_ptr[gi]; e < lp.row_ptr[gi + 1]; ++e) {
      const int64_t j = lp.col_index[e];
      const double v = lp.values[e];
      if (j < 0 || j >= n)
        throw std::out_of_range("matrix entry (" + std::to_string(gi) + "," + std::to_string(j) +
                                ") out of bounds");
      if (!std::isfinite(v))
        throw std::domain_error("matrix entry (" + std::to_string(gi) + "," + std::to_string(j) +
                                ") is not finite");
      if (j <= prev)
        throw std::domain_error("duplicate or unsorted matrix entry (" + std::to_string(gi) +
                                "," + std::to_string(j) + ")");
      prev = j;
      if (v != 0.0) ++cnt;
    }
    A.rp[i + 1] = A.rp[i] + cnt;
  }
  const int64_t nnz = A.rp[m];
  L.nnz = A.nnz = nnz;
  A.ci.resize(static_cast<size_t>(nnz));
  A.v.resize(static_cast<size_t>(nnz));
  L.a_dev_to_csr.resize(static_cast<size_t>(nnz));
  for (int64_t i = 0, k = 0; i < m; ++i) {
    const int64_t gi = row_begin + i;
    for (int64_t e = lp.row_ptr[gi]; e < lp.row_ptr[gi + 1]; ++e) {
      if (lp.values[e] == 0.0) continue;
      A.ci[k] = static_cast<int32_t>(lp.col_index[e]);
      A.v[k] = lp.values[e];
      L.a_dev_to_csr[k] = k;
      ++k;
    }
  }

  // (2) A^T = CSC of the local block in the reference's order (rows
  //     ascending per column, sparse_matrix.cpp:53-64)
  HostOperator& T = L.At;
  T.rows = n;
  T.cols = m;
  T.nnz = nnz;
  T.rp.assign(static_cast<size_t>(n) + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) T.rp[A.ci[e] + 1]++;
  for (int64_t j = 0; j < n; ++j) T.rp[j + 1] += T.rp[j];
  T.ci.resize(static_cast<size_t>(nnz));
  T.v.resize(static_cast<size_t>(nnz));
  L.at_dev_to_csc.resize(static_cast<size_t>(nnz));
  {
    std::vector<int64_t> next(T.rp.begin(), T.rp.end() - 1);
    for (int64_t i = 0; i < m; ++i)
      for (int64_t e = A.rp[i]; e < A.rp[i + 1]; ++e) {
        const int64_t s = next[A.ci[e]]++;
        T.ci[s] = static_cast<int32_t>(i);
        T.v[s] = A.v[e];
      }
    for (int64_t s = 0; s < nnz; ++s) L.at_dev_to_csc[s] = s;
  }

  // (3) identity order maps
  L.prow.resize(static_cast<size_t>(m));
  for (int64_t r = 0; r < m; ++r) L.prow[r] = static_cast<int32_t>(row_begin + r);
  L.pcol.resize(static_cast<size_t>(n));
  L.icol.resize(static_cast<size_t>(n));
  for (int64_t c = 0; c < n; ++c) L.pcol[c] = L.icol[c] = static_cast<int32_t>(c);

  // (4) tile schedules
  build_schedule(A);
  build_schedule(T);
}

}  // namespace rhp
