// layout.cu — host-side build of the permuted, binned device layout
// (see layout.cuh). Host code only; compiled by nvcc with the rest of the
// device library.
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

#include "layout.cuh"

namespace rhp {

namespace {

// Stable counting sort of items by kind: returns order[new] = old.
std::vector<int32_t> order_by_kind(const std::vector<int8_t>& kind, int64_t count,
                                   int64_t* bin_counts) {
  for (int k = 0; k < 8; ++k) bin_counts[k] = 0;
  for (int64_t i = 0; i < count; ++i) bin_counts[kind[i]]++;
  int64_t start[8];
  int64_t acc = 0;
  for (int k = 0; k < 8; ++k) {
    start[k] = acc;
    acc += bin_counts[k];
  }
  std::vector<int32_t> order(static_cast<size_t>(count));
  for (int64_t i = 0; i < count; ++i) order[start[kind[i]]++] = static_cast<int32_t>(i);
  return order;
}

// Schedule segments for an operator whose rows are already sorted by kind.
void build_schedule(HostOperator& op, const std::vector<int8_t>& kind_sorted) {
  Sched& s = op.sched;
  s = Sched{};
  int64_t row = 0, tile = 0;
  int nseg = 0;
  for (int k = 0; k < kKinds; ++k) {
    const int64_t rb = row;
    while (row < op.rows && kind_sorted[row] == k) ++row;
    if (row == rb) continue;
    Seg& sg = s.seg[nseg++];
    sg.kind = k;
    sg.row_begin = rb;
    sg.row_end = row;
    sg.tile_begin = tile;
    if (k < 6) {
      const int64_t rpt = kBlock >> k;
      tile += (row - rb + rpt - 1) / rpt;
    } else {
      int32_t n_multi = 0;
      for (int64_t r = rb; r < row; ++r) {
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
      }
      s.n_multi = n_multi;
      tile += static_cast<int64_t>(op.chunk_row.size());
    }
    sg.tile_end = tile;
  }
  // sentinel segment so the device segment search always terminates
  for (int i = nseg; i < kMaxSeg; ++i) {
    s.seg[i].kind = 0;
    s.seg[i].row_begin = s.seg[i].row_end = op.rows;
    s.seg[i].tile_begin = s.seg[i].tile_end = INT64_MAX;
  }
  s.nseg = nseg;
  s.total_tiles = tile;
}

}  // namespace

std::vector<int64_t> partition_rows(const rhpdhg_lp_view& lp, int world_size) {
  std::vector<int64_t> off(static_cast<size_t>(world_size) + 1, lp.num_cons);
  off[0] = 0;
  const int64_t m = lp.num_cons;
  const int64_t total = m > 0 ? lp.row_ptr[m] - lp.row_ptr[0] : 0;
  // contiguous blocks with ~total/P nonzeros each (rows weighted by nnz + 1
  // so empty rows still spread)
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
  std::vector<int64_t> rp(static_cast<size_t>(m) + 1, 0);
  for (int64_t i = 0; i < m; ++i) {
    const int64_t gi = row_begin + i;
    int64_t cnt = 0;
    int64_t prev = -1;
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
    rp[i + 1] = rp[i] + cnt;
  }
  const int64_t nnz = rp[m];
  L.nnz = nnz;
  std::vector<int32_t> ci(static_cast<size_t>(nnz));
  std::vector<double> v(static_cast<size_t>(nnz));
  for (int64_t i = 0, k = 0; i < m; ++i) {
    const int64_t gi = row_begin + i;
    for (int64_t e = lp.row_ptr[gi]; e < lp.row_ptr[gi + 1]; ++e) {
      if (lp.values[e] == 0.0) continue;
      ci[k] = static_cast<int32_t>(lp.col_index[e]);
      v[k] = lp.values[e];
      ++k;
    }
  }

  // (2) CSC of the local block in the reference's order (rows ascending per
  //     column, sparse_matrix.cpp:53-64)
  std::vector<int64_t> cp(static_cast<size_t>(n) + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) cp[ci[e] + 1]++;
  for (int64_t j = 0; j < n; ++j) cp[j + 1] += cp[j];
  std::vector<int32_t> ri(static_cast<size_t>(nnz));
  std::vector<int64_t> csc_of_csr(static_cast<size_t>(nnz));
  {
    std::vector<int64_t> next(cp.begin(), cp.end() - 1);
    for (int64_t i = 0; i < m; ++i)
      for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
        const int64_t s = next[ci[e]]++;
        ri[s] = static_cast<int32_t>(i);
        csc_of_csr[e] = s;
      }
  }

  // (3) bin rows and columns by length (stable)
  std::vector<int8_t> rk(static_cast<size_t>(m)), ck(static_cast<size_t>(n));
  for (int64_t i = 0; i < m; ++i) rk[i] = static_cast<int8_t>(row_kind(rp[i + 1] - rp[i]));
  for (int64_t j = 0; j < n; ++j) ck[j] = static_cast<int8_t>(row_kind(cp[j + 1] - cp[j]));
  const std::vector<int32_t> prow_local = order_by_kind(rk, m, L.A.bin_rows);
  const std::vector<int32_t> pcol = order_by_kind(ck, n, L.At.bin_rows);
  std::vector<int32_t> irow(static_cast<size_t>(m));
  for (int64_t r = 0; r < m; ++r) irow[prow_local[r]] = static_cast<int32_t>(r);
  L.icol.assign(static_cast<size_t>(n), 0);
  for (int64_t c = 0; c < n; ++c) L.icol[pcol[c]] = static_cast<int32_t>(c);
  L.pcol = pcol;
  L.prow.resize(static_cast<size_t>(m));
  for (int64_t r = 0; r < m; ++r) L.prow[r] = static_cast<int32_t>(row_begin + prow_local[r]);

  // (4) device A: permuted rows, relabelled columns, original element order
  HostOperator& A = L.A;
  A.rows = m;
  A.cols = n;
  A.nnz = nnz;
  A.rp.assign(static_cast<size_t>(m) + 1, 0);
  A.ci.resize(static_cast<size_t>(nnz));
  A.v.resize(static_cast<size_t>(nnz));
  L.a_dev_to_csr.resize(static_cast<size_t>(nnz));
  std::vector<int8_t> rk_sorted(static_cast<size_t>(m));
  for (int64_t r = 0, k = 0; r < m; ++r) {
    const int64_t i = prow_local[r];
    rk_sorted[r] = rk[i];
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e, ++k) {
      A.ci[k] = L.icol[ci[e]];
      A.v[k] = v[e];
      L.a_dev_to_csr[k] = e;
    }
    A.rp[r + 1] = A.rp[r] + (rp[i + 1] - rp[i]);
  }
  build_schedule(A, rk_sorted);

  // (5) device A^T: permuted columns as rows, relabelled row indices,
  //     elements in ascending original row (the reference CSC order)
  HostOperator& T = L.At;
  T.rows = n;
  T.cols = m;
  T.nnz = nnz;
  T.rp.assign(static_cast<size_t>(n) + 1, 0);
  T.ci.resize(static_cast<size_t>(nnz));
  T.v.resize(static_cast<size_t>(nnz));
  L.at_dev_to_csc.resize(static_cast<size_t>(nnz));
  std::vector<double> vt(static_cast<size_t>(nnz));
  for (int64_t e = 0; e < nnz; ++e) vt[csc_of_csr[e]] = v[e];
  std::vector<int8_t> ck_sorted(static_cast<size_t>(n));
  for (int64_t c = 0, k = 0; c < n; ++c) {
    const int64_t j = pcol[c];
    ck_sorted[c] = ck[j];
    for (int64_t s = cp[j]; s < cp[j + 1]; ++s, ++k) {
      T.ci[k] = irow[ri[s]];
      T.v[k] = vt[s];
      L.at_dev_to_csc[k] = s;
    }
    T.rp[c + 1] = T.rp[c] + (cp[j + 1] - cp[j]);
  }
  build_schedule(T, ck_sorted);
}

}  // namespace rhp
