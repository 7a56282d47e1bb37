// dropin_swap_run.hpp -- test infrastructure (never the product): dropin_swap.hpp plus
// the driver swap.  Force-included ahead of the reference's tests/acceptance.cpp, it
// also rewrites that program's `run_hydro_case(c, ...)` calls (acceptance.cpp:83, 104,
// 141, 158, 192, 230, 245, 385, 442) to lagflux::b200::run_hydro_case
// (include/lagflux_b200_run.hpp): the device-resident driver loop with dumps written
// from the device.  run.cpp itself is compiled without this header (it defines the
// reference's run_hydro_case, which the GPU driver falls back to for lagremap1d cases).
#pragma once

#include "lagflux_b200_run.hpp"   // (before the class macro: it names b200::LagfluxSolver itself)
#include "dropin_swap.hpp"

#define run_hydro_case b200::run_hydro_case
