// trace.h -- NVTX ranges (tracing): every C-ABI call, each
// lf_advance batch and each enqueued Heun step carry a named range, visible to
// nsys / ncu's NVTX filters.  NVTX v3 is header-only: without a tool attached a
// range costs a null-pointer test.
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace lfb {

struct TraceRange {
  explicit TraceRange(const char* name) { nvtxRangePushA(name); }
  ~TraceRange() { nvtxRangePop(); }
  TraceRange(const TraceRange&) = delete;
  TraceRange& operator=(const TraceRange&) = delete;
};

}  // namespace lfb

#define LF_TRACE_CAT2(a, b) a##b
#define LF_TRACE_CAT(a, b) LF_TRACE_CAT2(a, b)
#define LF_TRACE(name) ::lfb::TraceRange LF_TRACE_CAT(lf_trace_, __LINE__)(name)
