// driver_check.cpp -- test infrastructure: lagflux::run_hydro_case (the reference's
// driver loop, run.cpp:132-227, on the CPU solver) and lagflux::b200::run_hydro_case
// (include/lagflux_b200_run.hpp, device-resident) side by side on the same CaseConfig:
// the same HydroRun (time, step, every diagnostics record, boundary outflow, final
// field and partial densities, summary) and byte-identical output files, for a
// scheduled-dump run, a max_steps truncation, a multimaterial run and a run that fails
// (same exception type and text, diagnostics flushed, dumps so far on disk).
// Built with the reference sources by oracle/Makefile (`make -C oracle driver`).
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>

#include "lagflux/config.hpp"
#include "lagflux/run.hpp"
#include "lagflux_b200_run.hpp"

using namespace lagflux;

static int failures = 0;
static void expect(bool ok, const std::string& what) {
  if (!ok) {
    ++failures;
    std::printf("MISMATCH %s\n", what.c_str());
  }
}

static std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

static bool same_field(const CartesianGrid& g, const CellField& a, const CellField& b) {
  for (int c = 0; c < 4; ++c)
    for (int j = g.gy; j < g.gy + g.ny; ++j)
      if (std::memcmp(&a.comp[std::size_t(c)][g.idx(g.gx, j)], &b.comp[std::size_t(c)][g.idx(g.gx, j)],
                      sizeof(double) * std::size_t(g.nx)) != 0)
        return false;
  return true;
}

struct Outcome {
  bool threw = false;
  std::string error;   // typeid name + what()
  HydroRun run;
};

template <class F>
static Outcome drive(F&& f, CaseConfig c, const std::string& dir) {
  // the same relative prefix in a directory of its own (config_digest covers the prefix,
  // and the dumps' header line carries the digest)
  std::filesystem::create_directories(dir);
  const std::filesystem::path home = std::filesystem::current_path();
  std::filesystem::current_path(dir);
  Outcome o;
  try {
    o.run = f(c, true);
  } catch (const Error& e) {
    o.threw = true;
    o.error = std::string(typeid(e).name()) + ": " + e.what();
  }
  std::filesystem::current_path(home);
  return o;
}

static void compare(const char* name, const CaseConfig& c) {
  const std::string base = std::string("driver_check_out/") + name;
  std::filesystem::remove_all(base);
  const Outcome a = drive([](const CaseConfig& k, bool w) { return run_hydro_case(k, w); }, c, base + "/ref");
  const Outcome b = drive([](const CaseConfig& k, bool w) { return b200::run_hydro_case(k, w); }, c, base + "/b200");
  expect(a.threw == b.threw && a.error == b.error,
         std::string(name) + ": outcome '" + a.error + "' vs '" + b.error + "'");
  if (!a.threw && !b.threw) {
    const HydroRun &ra = a.run, &rb = b.run;
    expect(ra.state.time == rb.state.time && ra.state.step == rb.state.step, std::string(name) + ": time / step");
    expect(ra.state.boundary_outflow == rb.state.boundary_outflow, std::string(name) + ": boundary outflow");
    expect(same_field(ra.grid, ra.state.field, rb.state.field), std::string(name) + ": final field");
    expect(ra.state.diagnostics.size() == rb.state.diagnostics.size(), std::string(name) + ": diagnostics count");
    expect(ra.summary.steps == rb.summary.steps && ra.summary.final_time == rb.summary.final_time &&
               ra.summary.truncated_by_max_steps == rb.summary.truncated_by_max_steps &&
               ra.summary.min_rho == rb.summary.min_rho && ra.summary.min_p == rb.summary.min_p &&
               ra.summary.dump_paths.size() == rb.summary.dump_paths.size(),
           std::string(name) + ": summary");
    if (ra.material_cells && rb.material_cells)
      for (int k = 0; k < ra.material_cells->count(); ++k)
        for (int j = ra.grid.gy; j < ra.grid.gy + ra.grid.ny; ++j)
          if (std::memcmp(&ra.material_cells->partial[std::size_t(k)][ra.grid.idx(ra.grid.gx, j)],
                          &rb.material_cells->partial[std::size_t(k)][ra.grid.idx(ra.grid.gx, j)],
                          sizeof(double) * std::size_t(ra.grid.nx)) != 0) {
            expect(false, std::string(name) + ": partial densities");
            k = ra.material_cells->count();
            break;
          }
  }
  // every file either driver wrote: the same names, the same bytes
  std::size_t files = 0;
  for (const auto& e : std::filesystem::directory_iterator(base + "/ref")) {
    const std::string fn = e.path().filename().string();
    const std::string other = base + "/b200/" + fn;
    expect(std::filesystem::exists(other) && slurp(e.path().string()) == slurp(other),
           std::string(name) + ": file " + fn);
    ++files;
  }
  for (const auto& e : std::filesystem::directory_iterator(base + "/b200"))
    expect(std::filesystem::exists(base + "/ref/" + e.path().filename().string()),
           std::string(name) + ": extra file " + e.path().filename().string());
  std::printf("%s: %s, %zu files compared\n", name, a.threw ? a.error.c_str() : "completed", files);
}

int main() {
  {
    // Sod to t = 0.2 with an initial dump and three scheduled ones (limit times hit exactly)
    CaseConfig c = parse_case("sod");
    c.nx = 200;
    c.dump_times = {0.0, 0.05, 0.1, 0.2};
    compare("sod-dumps", c);
  }
  {
    // 2D, truncated by max_steps: the extra dump of the last state
    CaseConfig c = parse_case("sod2d");
    c.nx = 96;
    c.ny = 64;
    c.max_steps = 37;
    c.dump_times = {0.004};
    compare("sod2d-truncated", c);
  }
  {
    // three materials, coarse triple point, two dumps
    CaseConfig c = parse_case("triple_point");
    c.nx = 70;
    c.ny = 30;
    c.t_final = 0.2;
    c.dump_times = {0.1};
    compare("triple-point", c);
  }
  {
    // a run that fails after some steps: CFL far past stability
    CaseConfig c = parse_case("sod2d");
    c.nx = 80;
    c.ny = 48;
    c.cfl = 30.0;
    c.dump_times = {0.0};
    compare("sod2d-failing", c);
  }
  {
    // and one that fails only after a number of completed steps (their diagnostics are
    // flushed, the scheduled dump before the failure is on disk)
    CaseConfig c = parse_case("sod2d");
    c.nx = 80;
    c.ny = 48;
    c.cfl = 2.5;   // stable only while the dump times clip dt
    c.dump_times = {0.001, 0.002, 0.003, 0.004};
    compare("sod2d-failing-late", c);
  }
  std::printf("%s (%d mismatches)\n", failures ? "FAIL" : "OK", failures);
  return failures ? 1 : 0;
}
