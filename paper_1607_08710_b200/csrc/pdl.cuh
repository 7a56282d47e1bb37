// pdl.cuh -- programmatic dependent launch for the per-step kernel chain
// (ghost fill -> predictor -> ghost fill -> corrector -> finalize).
//
// A chain kernel is launched with programmatic stream serialization, so the
// front end pre-launches it while its predecessor drains, and it executes
// griddepcontrol.wait before its first access to the predecessor's results
// (the wait returns once the predecessor grid has completed and its writes are
// visible; after a normal launch it returns at once).  Every chain kernel waits
// before touching global memory, so completion is transitive along the chain.
// LF_PDL=0 in the environment launches them normally (A/B).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace lfb {

#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LF_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline void launch_chain(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                         cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace lfb
