// fused_step.cu -- placeholder until the fused kernel lands.
#include "fused.h"

namespace lfb {
bool fused_supported(lf_handle*) { return false; }
int fused_heun(lf_handle*, double, double, double, int64_t, double*, lf_step_out*) { return LF_ERR_ARGUMENT; }
int fused_advance(lf_handle*, int, double, double, double*, int64_t*, double*, lf_step_out*, int*) { return LF_ERR_ARGUMENT; }
int fused_time_steps(lf_handle*, int, double, double*, double*, int*) { return LF_ERR_ARGUMENT; }
void fused_release(lf_handle*) {}
int64_t fused_bytes(lf_handle*) { return 0; }
}  // namespace lfb
