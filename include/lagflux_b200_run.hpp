// lagflux_b200_run.hpp -- the reference's driver loop on the device.
//
// lagflux::b200::run_hydro_case(config, write_outputs) replaces
// lagflux::run_hydro_case (src/run.cpp:132-227, declared in include/lagflux/run.hpp:63)
// for SolverKind::lagflux cases: same arguments, same HydroRun (grid, state with
// time / step / diagnostics / boundary_outflow / final field, materials, summary),
// same output files (dumps "<prefix>_%04zu.csv" at the scheduled times and at a
// max_steps truncation, "<prefix>_diag.csv"), the diagnostics flushed before an error
// propagates.  What changes is where the work runs: the state is uploaded once, the
// steps between two dump events are one device-resident batch (lf_advance: dt, time
// and the diagnostics stay on the device), every dump is derived and formatted from the
// device copy (lf_write_field_csv_async: a host thread writes the file while the run
// keeps stepping) and the field comes back once, at the end.  Compiled inside the
// reference's build like lagflux_b200.hpp; a caller swaps
//
//     const HydroRun run = run_hydro_case(c, true);          // tools/main.cpp, acceptance.cpp
// for
//     const HydroRun run = b200::run_hydro_case(c, true);
//
// Other solver kinds (lagremap1d, advect2d) are not on the GPU path: they go to the
// reference's own run_hydro_case unchanged.
#pragma once

#include <algorithm>
#include <cstdio>
#include <limits>
#include <string>
#include <vector>

#include "lagflux/config.hpp"
#include "lagflux/csv.hpp"
#include "lagflux/run.hpp"
#include "lagflux_b200.hpp"

namespace lagflux::b200 {

inline HydroRun run_hydro_case(const CaseConfig& c, bool write_outputs, int device = 0) {
  if (c.solver != SolverKind::lagflux) return lagflux::run_hydro_case(c, write_outputs);

  HydroRun run;
  run.grid = build_grid(c);
  const CartesianGrid& g = run.grid;
  run.state.field = CellField(g);
  const bool multimat = !c.material_gammas.empty();
  if (multimat) {
    run.materials = make_material_set(c.material_gammas);
    run.material_cells = MaterialCells(g, run.materials->count());
  }
  MaterialCells* cells = multimat ? &*run.material_cells : nullptr;
  initialize_hydro(c, g, run.state.field, cells);

  const PerfectGasEos eos{c.gamma};
  const SchemeParams params{make_limiter(c.beta), c.spatial_order, c.time_order};
  const TimeControls controls{c.cfl, c.t_final, c.max_steps};
  LagfluxSolver solver(g, c.boundary(), eos, params, c.threads,
                       multimat ? &*run.materials : nullptr, device);
  solver.set_auto_sync(false);   // the device copy is the state until the run ends

  // dump events: the scheduled times and t_final, sorted and unique; times <= 0 (and
  // t_final == 0) ask for a dump of the initial state (run.cpp make_schedule)
  std::vector<double> events = c.dump_times;
  events.push_back(c.t_final);
  std::sort(events.begin(), events.end());
  events.erase(std::unique(events.begin(), events.end()), events.end());
  bool at_start = c.t_final == 0.0;
  std::vector<double> times;
  for (double v : events) {
    if (v <= 0.0) at_start = true;
    else times.push_back(v);
  }

  const std::uint64_t digest = config_digest(c);
  std::size_t dump_index = 0;
  const auto dump = [&](double time) {
    if (!write_outputs) return;
    char tail[16];
    std::snprintf(tail, sizeof tail, "_%04zu.csv", dump_index++);
    const std::string path = c.output_prefix + tail;
    solver.write_field_csv(path, digest, time, false);   // snapshot now, file in the background
    run.summary.dump_paths.push_back(path);
  };
  const auto flush_diagnostics = [&]() {
    if (!write_outputs) return;
    run.summary.diagnostics_path = c.output_prefix + "_diag.csv";
    write_text_file(run.summary.diagnostics_path, diagnostics_csv(run.state.diagnostics));
  };

  try {
    solver.advance(run.state, controls, 0.0, 0, cells);   // uploads the state, takes no step
    if (at_start) dump(0.0);   // the initial state is dumped from the device like every other
    std::size_t next_event = 0;
    while (run.state.time < c.t_final && run.state.step < c.max_steps) {
      const double limit = next_event < times.size() ? times[next_event] : c.t_final;
      solver.advance(run.state, controls, limit, std::numeric_limits<std::int64_t>::max(), cells);
      while (next_event < times.size() && run.state.time >= times[next_event]) {
        dump(run.state.time);
        ++next_event;
      }
    }
  } catch (const Error&) {
    // advance() has copied the failing step's field back; pending dumps finish first
    try { solver.wait_dumps(); } catch (const Error&) {}
    flush_diagnostics();
    throw;
  }

  // RunSummary (run.hpp:14-25): counts, whether max_steps cut the run short, and the
  // minima over every step's diagnostics (0 when no step ran)
  RunSummary& sum = run.summary;
  const std::vector<StepDiagnostics>& diag = run.state.diagnostics;
  sum.steps = run.state.step;
  sum.final_time = run.state.time;
  sum.truncated_by_max_steps = sum.final_time < c.t_final;
  if (diag.empty()) {
    sum.min_rho = sum.min_p = 0.0;
  } else {
    double lo_rho = std::numeric_limits<double>::infinity(), lo_p = lo_rho;
    for (const StepDiagnostics& d : diag) {
      if (d.min_rho < lo_rho) lo_rho = d.min_rho;
      if (d.min_p < lo_p) lo_p = d.min_p;
    }
    sum.min_rho = lo_rho;
    sum.min_p = lo_p;
  }

  if (run.summary.truncated_by_max_steps) dump(run.state.time);
  solver.wait_dumps();
  solver.sync_to_host(run.state, cells);   // HydroRun carries the final field
  flush_diagnostics();
  return run;
}

}  // namespace lagflux::b200
