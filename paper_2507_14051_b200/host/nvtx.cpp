// nvtx.cpp — NVTX ranges around the host phases of a solve (SURVEY.md §5
// tracing): setup and its stages, each device block, KKT checks, restarts
// and the final fetch show up as named ranges on the timeline of a profiler.
#include <nvtx3/nvToolsExt.h>

#include "session.hpp"

namespace rhpdhg::detail {

NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

}  // namespace rhpdhg::detail
