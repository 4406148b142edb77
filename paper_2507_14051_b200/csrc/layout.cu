// layout.cu — host-side build of the device layout and warp schedules
// (see layout.cuh). Host code only; compiled by nvcc with the device library.
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

#include "layout.cuh"

#ifndef RHP_SNAP_WINS
#define RHP_SNAP_WINS 8
#endif
#ifndef RHP_SNAP_FRAC
#define RHP_SNAP_FRAC 1.25
#endif

namespace rhp {

// Merge-path warp ranges (Sched in device_common.cuh). Boundary k sits at
// cost k * total / W, cost(r, e) = e + row_weight * r; it snaps to the nearer
// row start unless the row is longer than the snap length (min(8 windows,
// 1.25 ranges): a warp may take up to 1.25x its share rather than split a row
// — split rows cost a fence, a ticket and a serial sum at the range end; C3's
// 1000-nonzero rows: K1 33 -> 23 us), in which case the row is split there.
// Consecutive boundaries inside one row share its slot.
void build_schedule(HostOperator& op, int64_t n_warps, double row_weight) {
  const int64_t NW = std::max<int64_t>(1, n_warps);
  const int64_t R = op.rows, Z = op.nnz;
  // chunks per warp (warp w walks chunks w, w+NW, ...): one when the gathered
  // vector is L2-resident anyway (interleaving only adds chunk starts: C2
  // -3% at 2 chunks/warp); else ~kChunkCost of work each, so the grid sweeps
  // the rows in narrow bands (C4: 521 -> 718 iter/s)
  const double work = static_cast<double>(Z) + row_weight * static_cast<double>(R);
  const bool resident = static_cast<double>(op.cols) * 8.0 <= kGatherL2Bytes;
  const int64_t cpw =
      resident ? 1
               : std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(
                                                            work / (static_cast<double>(NW) * kChunkCost)),
                                                        (INT32_MAX / 2) / NW));
  const int64_t W = NW * cpw;  // chunks
  const std::vector<int64_t>& rp = op.rp;
  for (int k = 0; k < 8; ++k) op.bin_rows[k] = 0;
  for (int64_t r = 0; r < R; ++r) op.bin_rows[row_kind(rp[r + 1] - rp[r])]++;
  op.warp_row.assign(static_cast<size_t>(W) + 1, R);
  op.warp_nz.assign(static_cast<size_t>(W) + 1, Z);
  op.warp_row[0] = 0;
  op.warp_nz[0] = 0;
  const double total = static_cast<double>(Z) + row_weight * static_cast<double>(R);
  const double per = total / static_cast<double>(W);
  const int64_t snap = std::max<int64_t>(
      1, std::min<int64_t>(RHP_SNAP_WINS * kWin, static_cast<int64_t>(per * RHP_SNAP_FRAC)));
  auto cost = [&](int64_t r) { return static_cast<double>(rp[r]) + row_weight * static_cast<double>(r); };
  int64_t pr = 0, pe = 0;
  for (int64_t k = 1; k < W; ++k) {
    const double T = per * static_cast<double>(k);
    // last row r with cost(r) <= T
    int64_t lo = 0, hi = R;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (cost(mid) <= T) lo = mid;
      else hi = mid - 1;
    }
    int64_t r = lo, e = R > 0 ? rp[lo] : 0;
    if (r < R) {
      const int64_t len = rp[r + 1] - rp[r];
      if (len <= snap) {
        if (T - cost(r) > cost(r + 1) - T) ++r;
        e = rp[r];
      } else {
        const double off = T - cost(r) - row_weight;
        const int64_t j = off <= 0 ? 0 : std::min<int64_t>(len, static_cast<int64_t>(off));
        e = rp[r] + j;
        if (j == len) {
          ++r;
          e = rp[r];
        }
      }
    }
    if (e < pe || (e == pe && r < pr)) {  // keep boundaries monotone
      r = pr;
      e = pe;
    }
    op.warp_row[k] = r;
    op.warp_nz[k] = e;
    pr = r;
    pe = e;
  }
  op.head_slot.assign(static_cast<size_t>(W), -1);
  op.tail_slot.assign(static_cast<size_t>(W), -1);
  op.slot_row.clear();
  op.slot_first.clear();
  op.slot_count.clear();
  for (int64_t k = 1; k < W; ++k) {
    const int64_t r = op.warp_row[k], e = op.warp_nz[k];
    if (r >= R || e <= rp[r]) continue;  // boundary at a row start
    if (op.slot_row.empty() || op.slot_row.back() != r) {
      op.slot_row.push_back(r);
      op.slot_first.push_back(static_cast<int32_t>(k - 1));
      op.slot_count.push_back(0);
    }
    const int32_t sl = static_cast<int32_t>(op.slot_row.size()) - 1;
    op.slot_count[sl] = static_cast<int32_t>(k - op.slot_first[sl] + 1);
    op.head_slot[k] = sl;
    op.tail_slot[k - 1] = sl;
  }
  Sched& s = op.sched;
  s = Sched{};
  s.n_multi = static_cast<int32_t>(op.slot_row.size());
  s.n_warps = static_cast<int32_t>(NW);
  s.n_chunks = static_cast<int32_t>(W);
  s.rows = R;
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

}  // namespace rhp
