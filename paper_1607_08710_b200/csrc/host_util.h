// host_util.h -- host-side helpers of the C ABI (not on the device hot path).
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/lagflux_b200.h"

namespace lfb {

// apply_boundary (grid.cpp:116-121) on host arrays in the reference layout
// (gx = 2, gy = 2 in 2D / 0 in 1D, leading dimension ld); used by
// lf_download(fill_ghosts = 1) for dumps.
void host_apply_boundary(const lf_desc& d, double* const field[4], int64_t ld);

// 1D tables of the seeded smooth-perturbation generator (cases.py):
// tx = [k][m][sin|cos][nx], ty = [k][m][sin|cos][ny], amp = [k][m].
void fourier_tables(uint64_t seed, const lf_desc& d, std::vector<double>& tx,
                    std::vector<double>& ty, std::vector<double>& amp);

}  // namespace lfb
