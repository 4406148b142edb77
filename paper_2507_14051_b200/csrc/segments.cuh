// segments.cuh — column-segmented copies of a device operator (segments.cu).
//
// When the vector an operator gathers from is larger than L2 (C5: x is
// 160 MB, y 400 MB; B200's L2 is 126 MB), a random gather is a random 32-B
// DRAM sector read and the SpMV runs at the DRAM sector rate, not the
// streaming rate. The operator is then split by column ranges into S
// segments of at most RHP_SEG_BYTES of gathered vector each, every segment
// a CSR over all rows with only its columns (each row's elements keep their
// order, so a segment's part of a row is a contiguous run of the row). The
// SpMV walks the segments one after another — segment k adds its row sums
// to the running partial (Sched::seg_in) — so while one segment runs, the
// grid gathers from one L2-resident slice of the vector.
#pragma once

#include <cstdint>
#include <vector>

#include "ingest.cuh"

namespace rhp {

// Splits `op` (rows x cols, columns ascending inside every row) into
// S = cb.size()-1 column segments [cb[k], cb[k+1]); out[k] gets its own row
// pointers, int32 columns and (current) values, host_rp[k] its row pointers.
// Only the rows of the band [rb, re) are split: the intermediate segments
// k < S-1 are CSRs over those rows alone (local row r - rb), and every row
// outside the band keeps all its elements in the last segment (which spans
// all rows). Rows whose gathers are already L2-local (C4's commodity-blocked
// conservation and capacity rows) then cost one pass, not S.
void split_columns(const DeviceCsr& op, const std::vector<int32_t>& cb, int64_t rb, int64_t re,
                   std::vector<DeviceCsr>& out, std::vector<std::vector<int64_t>>& host_rp,
                   cudaStream_t s);

}  // namespace rhp
