// dropin_check.cpp -- the reference's own LagfluxSolver next to the drop-in
// lagflux::b200::LagfluxSolver (include/lagflux_b200.hpp), through the
// reference's C++ types only.
//
// Built by oracle/Makefile together with the reference sources (so the binary
// lands in oracle/_ref/, git-ignored) and run by tests/test_gpu_dropin.py on
// the GPU box.  Exit status 0 iff every field value (==), dt, diagnostic,
// boundary outflow and error text agrees.
#include <cmath>
#include <cstdio>
#include <utility>
#include <limits>
#include <string>
#include <vector>

#include "lagflux/error.hpp"
#include "lagflux/multimat.hpp"
#include "lagflux/solver.hpp"
#include "lagflux_b200.hpp"

using namespace lagflux;

namespace {

int failures = 0;

void expect(bool ok, const std::string& what) {
  if (!ok) {
    ++failures;
    std::printf("MISMATCH: %s\n", what.c_str());
  }
}

bool same_interior(const CartesianGrid& g, const CellField& a, const CellField& b) {
  for (int c = 0; c < 4; ++c)
    for (int j = g.gy; j < g.gy + g.ny; ++j)
      for (int i = g.gx; i < g.gx + g.nx; ++i)
        if (!(a.comp[c][g.idx(i, j)] == b.comp[c][g.idx(i, j)])) return false;
  return true;
}

CellField smooth_field(const CartesianGrid& g, PerfectGasEos eos) {
  constexpr double two_pi = 6.283185307179586476925286766559;
  CellField f(g);
  for (int j = g.gy; j < g.gy + g.ny; ++j)
    for (int i = g.gx; i < g.gx + g.nx; ++i) {
      const double x = g.xc(i), y = g.yc(j);
      PrimitiveState w;
      w.rho = 1.0 + 0.3 * std::sin(two_pi * x) * std::sin(two_pi * y);
      w.u = 0.2 * std::cos(two_pi * x);
      w.v = -0.3 * std::sin(two_pi * y);
      w.p = 1.0 + 0.2 * std::cos(two_pi * x) * std::cos(two_pi * y);
      f.set_state(g, i, j, conserved_from_primitive(w, eos));
    }
  return f;
}

CellField sod_field(const CartesianGrid& g, PerfectGasEos eos) {
  CellField f(g);
  for (int j = g.gy; j < g.gy + g.ny; ++j)
    for (int i = g.gx; i < g.gx + g.nx; ++i) {
      const PrimitiveState w = g.xc(i) < 0.5 ? PrimitiveState{1.0, 0.0, 0.0, 1.0}
                                             : PrimitiveState{0.125, 0.0, 0.0, 0.1};
      f.set_state(g, i, j, conserved_from_primitive(w, eos));
    }
  return f;
}

void run_pair(const char* name, const CartesianGrid& g, const BoundaryCondition& bc,
              CellField f0, int steps, double cfl, double limit, bool auto_sync) {
  const PerfectGasEos eos{1.4};
  const SchemeParams params{};
  const TimeControls controls{cfl, limit, 1 << 30};
  LagfluxSolver ref(g, bc, eos, params, 1);
  b200::LagfluxSolver gpu(g, bc, eos, params, 1);
  gpu.set_auto_sync(auto_sync);
  SolverState a, b;
  a.field = f0;
  b.field = f0;
  for (int s = 0; s < steps && a.time < limit; ++s) {
    if (s == steps / 2) {
      // a diagnostic compute_dt of another field between steps must not disturb
      // the resident state (with or without auto_sync)
      expect(ref.compute_dt(f0, controls, 0.0, 1e30) == gpu.compute_dt(f0, controls, 0.0, 1e30),
             std::string(name) + ": compute_dt between steps");
      if (auto_sync) {
        // state.field is authoritative with auto_sync: a host edit between steps
        // (one cell scaled by 1.5: same velocity, 1.5x pressure) must be seen
        const std::size_t k = std::size_t(g.gy + g.ny / 2) * std::size_t(g.nxt()) + std::size_t(g.gx + g.nx / 3);
        for (int c = 0; c < 4; ++c) {
          a.field.comp[size_t(c)][k] *= 1.5;
          b.field.comp[size_t(c)][k] *= 1.5;
        }
      }
    }
    const double da = ref.heun_step(a, controls, limit);
    const double db = gpu.heun_step(b, controls, limit);
    if (da != db) {
      expect(false, std::string(name) + ": dt of step " + std::to_string(s));
      return;
    }
  }
  if (!auto_sync) gpu.sync_to_host(b);
  expect(same_interior(g, a.field, b.field), std::string(name) + ": final field");
  expect(a.time == b.time && a.step == b.step, std::string(name) + ": time / step");
  expect(a.diagnostics.size() == b.diagnostics.size(), std::string(name) + ": diagnostics count");
  for (size_t k = 0; k < a.diagnostics.size() && k < b.diagnostics.size(); ++k) {
    const StepDiagnostics &x = a.diagnostics[k], &y = b.diagnostics[k];
    if (!(x.dt == y.dt && x.time == y.time && x.min_rho == y.min_rho && x.min_p == y.min_p &&
          x.step == y.step)) {
      expect(false, std::string(name) + ": diagnostics " + std::to_string(k));
      break;
    }
  }
  for (int c = 0; c < 4; ++c)
    expect(a.boundary_outflow[size_t(c)] == b.boundary_outflow[size_t(c)],
           std::string(name) + ": boundary outflow");
  // the conservation audit (grid.cpp:122-133), resident state summed on the device
  const std::array<double, 4> ta = interior_totals(g, a.field), tb = gpu.interior_totals(b);
  for (int c = 0; c < 4; ++c) expect(ta[size_t(c)] == tb[size_t(c)], std::string(name) + ": interior totals");
  std::printf("%s: %zu steps compared\n", name, a.diagnostics.size());
}

// The triple-point regions (cases/triple_point.case) on a small mesh: three
// materials, each cell's energy from its own material's gamma (run.cpp:29-78).
void run_multimaterial(int nx, int ny, int steps, bool auto_sync) {
  const CartesianGrid g = make_grid_2d(nx, ny, 0.0, 7.0, 0.0, 3.0);
  const BoundaryCondition bc{BcKind::reflective, BcKind::reflective, BcKind::reflective,
                             BcKind::reflective};
  const MaterialSet set = make_material_set({1.5, 1.4, 1.5});
  CellField f(g);
  MaterialCells m(g, 3);
  for (int j = g.gy; j < g.gy + g.ny; ++j)
    for (int i = g.gx; i < g.gx + g.nx; ++i) {
      const double x = g.xc(i), y = g.yc(j);
      const int mat = x < 1.0 ? 0 : (y >= 1.5 ? 1 : 2);
      const PrimitiveState w = mat == 0 ? PrimitiveState{1.0, 0.0, 0.0, 1.0}
                               : mat == 1 ? PrimitiveState{0.125, 0.0, 0.0, 0.1}
                                          : PrimitiveState{1.0, 0.0, 0.0, 0.1};
      f.set_state(g, i, j, conserved_from_primitive(w, PerfectGasEos{set.gammas[size_t(mat)]}));
      m.partial[size_t(mat)][size_t(g.idx(i, j))] = w.rho;
    }
  const SchemeParams params{};
  const TimeControls controls{0.25, 1e30, 1 << 30};
  LagfluxSolver ref(g, bc, PerfectGasEos{1.4}, params, 1, &set);
  b200::LagfluxSolver gpu(g, bc, PerfectGasEos{1.4}, params, 1, &set);
  gpu.set_auto_sync(auto_sync);
  SolverState a, b;
  a.field = f;
  b.field = f;
  MaterialCells ma = m, mb = m;
  for (int s = 0; s < steps; ++s) {
    const double da = ref.heun_step(a, controls, 1e30, &ma);
    const double db = gpu.heun_step(b, controls, 1e30, &mb);
    if (da != db) {
      expect(false, "multimaterial: dt of step " + std::to_string(s));
      return;
    }
  }
  if (!auto_sync) gpu.sync_to_host(b, &mb);
  expect(same_interior(g, a.field, b.field), "multimaterial: final field");
  bool parts = true;
  for (int k = 0; k < 3; ++k)
    for (int j = g.gy; j < g.gy + g.ny; ++j)
      for (int i = g.gx; i < g.gx + g.nx; ++i)
        parts = parts && ma.partial[size_t(k)][size_t(g.idx(i, j))] ==
                             mb.partial[size_t(k)][size_t(g.idx(i, j))];
  expect(parts, "multimaterial: partial densities");
  for (size_t k = 0; k < a.diagnostics.size(); ++k)
    if (!(a.diagnostics[k].min_p == b.diagnostics[k].min_p &&
          a.diagnostics[k].min_rho == b.diagnostics[k].min_rho)) {
      expect(false, "multimaterial: diagnostics " + std::to_string(k));
      break;
    }
  std::printf("multimaterial%s: %zu steps compared\n", auto_sync ? "" : "-resident",
              a.diagnostics.size());
}

}  // namespace

// The free edge_flux (solver.cpp:45-53): general normals, two EOS, the u* == 0
// mean branch, and sound_speed's throw.
void edge_flux_pair() {
  const PrimitiveState a{1.0, 0.3, -0.2, 1.0}, b{0.125, -0.1, 0.4, 0.1}, c{1.0, 0.0, 0.0, 1.0};
  const Vec2 normals[3] = {{1.0, 0.0}, {0.0, 1.0}, {0.6, 0.8}};
  for (const Vec2& n : normals)
    for (const auto& pr : {std::make_pair(a, b), std::make_pair(b, a), std::make_pair(c, c)}) {
      const EdgeFlux x = edge_flux(pr.first, pr.second, n, PerfectGasEos{1.4}, PerfectGasEos{1.6});
      const EdgeFlux y = b200::edge_flux(pr.first, pr.second, n, PerfectGasEos{1.4}, PerfectGasEos{1.6});
      expect(x.mass == y.mass && x.mom_x == y.mom_x && x.mom_y == y.mom_y && x.energy == y.energy &&
                 std::signbit(x.mom_x) == std::signbit(y.mom_x) &&
                 std::signbit(x.mom_y) == std::signbit(y.mom_y),
             "edge_flux");
    }
  std::string ref_what, gpu_what;
  const PrimitiveState bad{1.0, 0.0, 0.0, -2.5};
  try {
    edge_flux(a, bad, Vec2{1.0, 0.0}, PerfectGasEos{1.4});
  } catch (const InvalidStateError& e) {
    ref_what = e.what();
  }
  try {
    b200::edge_flux(a, bad, Vec2{1.0, 0.0}, PerfectGasEos{1.4});
  } catch (const InvalidStateError& e) {
    gpu_what = e.what();
  }
  expect(!ref_what.empty() && ref_what == gpu_what, "edge_flux error: " + ref_what + " | " + gpu_what);
  std::printf("edge_flux: compared\n");
  // the free compute_dt (solver.cpp:55-59)
  const CartesianGrid g = make_grid_2d(40, 30, 0.0, 1.0, 0.0, 0.75);
  const CellField f = smooth_field(g, PerfectGasEos{1.4});
  const TimeControls tc{0.45, 1e30, 1 << 30};
  expect(compute_dt(g, f, PerfectGasEos{1.4}, tc, 0.0, 1e30) ==
             b200::compute_dt(g, f, PerfectGasEos{1.4}, tc, 0.0, 1e30),
         "free compute_dt");
}

int main() {
  const PerfectGasEos eos{1.4};
  edge_flux_pair();
  {
    const CartesianGrid g = make_grid_2d(64, 48, 0.0, 1.0, 0.0, 0.75);
    run_pair("smooth-periodic", g, {BcKind::periodic, BcKind::periodic, BcKind::periodic, BcKind::periodic},
             smooth_field(g, eos), 40, 0.5, 1e30, true);
    run_pair("smooth-periodic-resident", g,
             {BcKind::periodic, BcKind::periodic, BcKind::periodic, BcKind::periodic},
             smooth_field(g, eos), 40, 0.5, 1e30, false);
  }
  {
    const CartesianGrid g = make_grid_2d(400, 4, 0.0, 1.0, 0.0, 1.0);
    run_pair("sod-reflective", g, {BcKind::reflective, BcKind::reflective, BcKind::reflective, BcKind::reflective},
             sod_field(g, eos), 1000, 0.5, 0.2, true);
  }
  {
    const CartesianGrid g = make_grid_2d(50, 30, 0.0, 1.0, 0.0, 0.6);
    run_pair("mixed-bc", g, {BcKind::reflective, BcKind::transmissive, BcKind::periodic, BcKind::periodic},
             smooth_field(g, eos), 30, 0.45, 1e30, true);
  }
  {
    // compute_dt, euler_stage and the PositivityError text (test_solver.cpp:161-180, 371-384)
    const CartesianGrid g = make_grid_1d(50, 0.0, 1.0);
    LagfluxSolver ref(g, BoundaryCondition{}, eos, SchemeParams{}, 1);
    b200::LagfluxSolver gpu(g, BoundaryCondition{}, eos, SchemeParams{}, 1);
    CellField f = sod_field(g, eos);
    const TimeControls controls{0.25, 10.0, 1000};
    expect(ref.compute_dt(f, controls, 0.0, 10.0) == gpu.compute_dt(f, controls, 0.0, 10.0), "compute_dt");
    CellField oa(g), ob(g), fa = f, fb = f;
    ref.euler_stage(fa, 8e-4, oa);
    gpu.euler_stage(fb, 8e-4, ob);
    expect(same_interior(g, oa, ob), "euler_stage");
    std::string ea, eb;
    try {
      CellField x = f;
      ref.euler_stage(x, 10.0, oa, 7);
    } catch (const PositivityError& e) {
      ea = e.what();
    }
    try {
      CellField x = f;
      gpu.euler_stage(x, 10.0, ob, 7);
    } catch (const PositivityError& e) {
      eb = e.what();
    }
    expect(!ea.empty() && ea == eb, "PositivityError text: '" + ea + "' vs '" + eb + "'");
  }
  {
    // advance() (the run.cpp:180-210 loop on the device) against heun_step calls of the
    // reference: dump-style limit times hit exactly, then a CFL far past stability so
    // that a step fails -- same exception text, same completed steps and diagnostics
    const CartesianGrid g = make_grid_2d(96, 40, 0.0, 1.0, 0.0, 0.5);
    const BoundaryCondition bc{BcKind::transmissive, BcKind::reflective, BcKind::reflective,
                               BcKind::transmissive};
    for (int auto_sync = 0; auto_sync < 2; ++auto_sync) {
      LagfluxSolver ref(g, bc, eos, SchemeParams{}, 2);
      b200::LagfluxSolver gpu(g, bc, eos, SchemeParams{}, 2);
      gpu.set_auto_sync(auto_sync != 0);
      SolverState a, b;
      a.field = sod_field(g, eos);
      b.field = a.field;
      const TimeControls controls{0.45, 0.05, 1 << 30};
      const double limits[3] = {0.0125, 0.03, 0.05};
      for (double limit : limits) {
        while (a.time < limit) ref.heun_step(a, controls, limit);
        gpu.advance(b, controls, limit, std::numeric_limits<std::int64_t>::max());
        expect(a.time == b.time && a.step == b.step, "advance: time / step at a limit");
      }
      if (!auto_sync) gpu.sync_to_host(b);
      expect(same_interior(g, a.field, b.field), "advance: field");
      expect(a.diagnostics.size() == b.diagnostics.size(), "advance: diagnostics count");
      for (std::size_t k = 0; k < a.diagnostics.size() && k < b.diagnostics.size(); ++k)
        if (a.diagnostics[k].dt != b.diagnostics[k].dt || a.diagnostics[k].min_p != b.diagnostics[k].min_p)
          expect(false, "advance: diagnostics " + std::to_string(k));
      expect(a.boundary_outflow == b.boundary_outflow, "advance: boundary outflow");
      const TimeControls wild{40.0, 1e30, 1 << 30};
      std::string ea, eb;
      try {
        for (int k = 0; k < 50; ++k) ref.heun_step(a, wild, 1e30);
      } catch (const Error& e) {
        ea = e.what();
      }
      try {
        gpu.advance(b, wild, 1e30, 50);
      } catch (const Error& e) {
        eb = e.what();
      }
      expect(!ea.empty() && ea == eb, "advance: error text '" + ea + "' vs '" + eb + "'");
      expect(a.step == b.step && a.time == b.time && a.diagnostics.size() == b.diagnostics.size(),
             "advance: completed steps before the failure");
      std::printf("advance (auto_sync %d): %lld steps, three limit times and a failing batch compared\n",
                  auto_sync, static_cast<long long>(a.step));
    }
  }
  run_multimaterial(70, 30, 40, true);
  run_multimaterial(70, 30, 40, false);
  std::printf("%s (%d mismatches)\n", failures ? "FAIL" : "OK", failures);
  return failures ? 1 : 0;
}
