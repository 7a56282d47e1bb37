// lagflux_b200.hpp -- C++ drop-in for lagflux::LagfluxSolver over the C ABI.
//
// Header-only adapter compiled inside the reference's C++ build: it takes and
// returns the reference's own types (include/lagflux/solver.hpp:39-131) and
// throws the reference's exception types with the reference's what() texts
// (include/lagflux/error.hpp:9-64), so a caller swaps
//
//     lagflux::LagfluxSolver solver(g, bc, eos, params, threads);        // run.cpp:154
// for
//     lagflux::b200::LagfluxSolver solver(g, bc, eos, params, threads);
//
// and links liblagflux_b200.so.  Residency: the GPU keeps SolverState::field
// between steps.  With auto_sync (the default) state.field is authoritative,
// exactly like the reference: every heun_step uploads it and copies the
// interior back, so host edits between steps are seen.  A driver that only
// reads the field at dumps calls set_auto_sync(false) and sync_to_host(state)
// before each dump (one line in run.cpp's dump lambda) to avoid the copies;
// then the device copy is authoritative for the resident state (identified by
// address and by the time / step the last heun_step left in it -- a different
// SolverState, or one whose time or step was reset, is uploaded afresh), and
// compute_dt / euler_stage / interior_totals on another field first save the
// resident state into its host field.  MaterialCells follow the same rules.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "lagflux/error.hpp"
#include "lagflux/multimat.hpp"
#include "lagflux/solver.hpp"
#include "lagflux_b200.h"

namespace lagflux::b200 {

// edge_flux (solver.cpp:45-53) evaluated on the device; throws InvalidStateError
// like sound_speed for a non-physical trace.  One face per call: a device round
// trip, for API parity -- batch faces through lf_edge_flux.
inline EdgeFlux edge_flux(const PrimitiveState& w_minus, const PrimitiveState& w_plus, Vec2 n,
                          PerfectGasEos eos_minus, PerfectGasEos eos_plus, int device = 0) {
  const double wm[4] = {w_minus.rho, w_minus.u, w_minus.v, w_minus.p};
  const double wp[4] = {w_plus.rho, w_plus.u, w_plus.v, w_plus.p};
  const double nr[2] = {n.x, n.y};
  double f[4];
  lf_error e{};
  const int rc = lf_edge_flux(1, wm, wp, nr, &eos_minus.gamma, &eos_plus.gamma, f, nullptr, device, &e);
  if (rc == LF_ERR_PRIMITIVE) throw InvalidStateError(e.message);
  if (rc) throw Error(e.message);
  return EdgeFlux{f[0], f[1], f[2], f[3]};
}
inline EdgeFlux edge_flux(const PrimitiveState& w_minus, const PrimitiveState& w_plus, Vec2 n,
                          PerfectGasEos eos) {
  return b200::edge_flux(w_minus, w_plus, n, eos, eos, 0);
}

class LagfluxSolver {
 public:
  LagfluxSolver(const CartesianGrid& g, const BoundaryCondition& bc, PerfectGasEos eos,
                SchemeParams params, int threads = 1, const MaterialSet* materials = nullptr,
                int device = 0)
      : grid_(g), threads_(threads < 1 ? 1 : threads) {
    // constructor checks of solver.cpp:66-69
    if (g.nx < 1 || g.ny < 1) throw ConfigError("grid has no interior cells");
    if (g.gx < 2 || (g.dim == 2 && g.gy < 2))
      throw ConfigError("MUSCL stencils need at least two ghost layers");
    validate_boundary(bc, g.dim);
    if (g.gx != 2 || g.gy != (g.dim == 2 ? 2 : 0))
      throw ConfigError("the B200 path uses the reference's ghost width 2");
    lf_desc d{};
    d.dim = g.dim;
    d.nx = g.nx;
    d.ny = g.ny;
    d.dx = g.dx;
    d.dy = g.dy;
    d.x0 = g.x0;
    d.y0 = g.y0;
    d.gamma = eos.gamma;
    d.beta = params.limiter.beta;
    d.spatial_order = params.spatial_order;
    d.time_order = params.time_order;
    d.bc[0] = kind(bc.x_low);
    d.bc[1] = kind(bc.x_high);
    d.bc[2] = kind(bc.y_low);
    d.bc[3] = kind(bc.y_high);
    int rc = lf_create(&d, &device, 1, &h_);
    if (rc == 0 && materials != nullptr) {
      rc = lf_set_materials(h_, materials->count(), materials->gammas.data());
      n_mat_ = materials->count();
    }
    if (rc) {
      const std::string msg = error_text();
      lf_destroy(h_);
      h_ = nullptr;
      throw ConfigError(msg);
    }
  }
  ~LagfluxSolver() { lf_destroy(h_); }
  LagfluxSolver(const LagfluxSolver&) = delete;
  LagfluxSolver& operator=(const LagfluxSolver&) = delete;

  // solver.cpp:482-487 -- `in`'s ghosts are not refilled on the host (the
  // device fills its own copy); `out`'s interior receives the stage.
  void euler_stage(CellField& in, double dt, CellField& out, std::int64_t step = -1) {
    evict();
    upload(in);
    check(lf_euler_stage(h_, dt, step));
    download(out);
  }

  // solver.cpp:489-546
  double heun_step(SolverState& state, const TimeControls& controls, double limit_time,
                   MaterialCells* materials = nullptr) {
    if (n_mat_ == 0) materials = nullptr;  // solver.cpp:490
    if (n_mat_ > 0 && materials == nullptr)
      throw ConfigError("multimaterial step needs material storage");
    if (auto_sync_ || !is_resident(state)) {
      evict();
      upload(state.field);
      resident_ = &state;
      resident_time_ = state.time;
      resident_step_ = state.step;
    }
    if (materials != nullptr && (auto_sync_ || resident_mat_ != materials)) {
      check(lf_upload_partials(h_, partial_ptrs(*materials).p, grid_.nxt()));
      resident_mat_ = materials;
    }
    lf_step_out o{};
    const int rc = lf_heun_step(h_, controls.cfl, state.time, limit_time, state.step,
                                state.boundary_outflow.data(), &o);
    if (rc) {
      if (auto_sync_) download(state.field);  // a corrector failure leaves its output, as in the reference
      check(rc);
    }
    state.time = o.time;
    state.step = o.step;
    resident_time_ = o.time;
    resident_step_ = o.step;
    state.diagnostics.push_back({o.step, o.time, o.dt, o.min_rho, o.min_p});
    if (auto_sync_) {
      download(state.field);
      if (materials != nullptr) check(lf_download_partials(h_, partial_ptrs(*materials).p, grid_.nxt()));
    }
    return o.dt;
  }

  // The run.cpp:180-210 loop between two dump events, on the device (lf_advance): up
  // to max_count heun_steps while state.time < limit_time, each with the reference's
  // dt clipping against limit_time; dt, time and the diagnostics stay on the device
  // and come back once per batch.  state.time / step / diagnostics / boundary_outflow
  // are updated as by that many heun_step calls; state.field follows the residency
  // rules above (auto_sync: uploaded before and copied back after the batch).
  // Returns the steps taken; a failing step throws the reference's exception after
  // the completed steps were recorded.
  std::int64_t advance(SolverState& state, const TimeControls& controls, double limit_time,
                       std::int64_t max_count, MaterialCells* materials = nullptr) {
    if (n_mat_ == 0) materials = nullptr;
    if (n_mat_ > 0 && materials == nullptr)
      throw ConfigError("multimaterial step needs material storage");
    if (auto_sync_ || !is_resident(state)) {
      evict();
      upload(state.field);
      resident_ = &state;
      resident_time_ = state.time;
      resident_step_ = state.step;
    }
    if (materials != nullptr && (auto_sync_ || resident_mat_ != materials)) {
      check(lf_upload_partials(h_, partial_ptrs(*materials).p, grid_.nxt()));
      resident_mat_ = materials;
    }
    const double t_end = limit_time < controls.t_final ? limit_time : controls.t_final;
    std::int64_t done = 0;
    std::vector<lf_step_out> rec;
    int rc = 0;
    while (rc == 0 && done < max_count && state.time < t_end && state.step < controls.max_steps) {
      std::int64_t chunk = max_count - done;
      if (chunk > controls.max_steps - state.step) chunk = controls.max_steps - state.step;
      if (chunk > 4096) chunk = 4096;
      rec.resize(std::size_t(chunk));
      int taken = 0;
      double time = state.time;
      std::int64_t step = state.step;
      rc = lf_advance(h_, int(chunk), controls.cfl, t_end, &time, &step,
                      state.boundary_outflow.data(), rec.data(), &taken);
      for (int k = 0; k < taken; ++k)
        state.diagnostics.push_back(
            {rec[std::size_t(k)].step, rec[std::size_t(k)].time, rec[std::size_t(k)].dt,
             rec[std::size_t(k)].min_rho, rec[std::size_t(k)].min_p});
      state.time = time;
      state.step = step;
      resident_time_ = time;
      resident_step_ = step;
      done += taken;
      if (taken < chunk) break;  // reached t_end (or failed: rc)
    }
    if (auto_sync_ || rc) {
      download(state.field);  // a corrector failure leaves its output, as in the reference
      if (materials != nullptr) {
        const int rp = lf_download_partials(h_, partial_ptrs(*materials).p, grid_.nxt());
        if (rc == 0) check(rp);   // (after a failing step its error is the one reported)
      }
    }
    check(rc);
    return done;
  }

  // field_csv + write_text_file of the resident state (csv.cpp:26-83, run.cpp:162-168),
  // derived and formatted from the device copy, byte-identical; with wait = false a
  // host thread writes the file while the caller keeps stepping (wait_dumps joins)
  void write_field_csv(const std::string& path, std::uint64_t digest, double time,
                       bool wait = true) {
    check(wait ? lf_write_field_csv(h_, path.c_str(), digest, time, threads_)
               : lf_write_field_csv_async(h_, path.c_str(), digest, time, threads_));
  }
  void wait_dumps() { check(lf_wait_dumps(h_)); }

  // solver.cpp:434-480
  double compute_dt(const CellField& field, const TimeControls& controls, double time,
                    double limit_time) const {
    evict();
    upload(field);
    double dt = 0.0;
    check(lf_compute_dt(h_, controls.cfl, time, limit_time, &dt));
    return dt;
  }

  // interior_totals(grid, state.field) (grid.cpp:122-133), summed on the device in
  // the reference's order: the resident copy of `state`, else its host field
  std::array<double, 4> interior_totals(const SolverState& state) const {
    if (auto_sync_ || !is_resident(state)) {
      evict();
      upload(state.field);
    }
    std::array<double, 4> t{};
    check(lf_interior_totals(h_, t.data()));
    return t;
  }

  const CartesianGrid& grid() const { return grid_; }
  int threads() const { return threads_; }

  // residency control (see the header comment)
  void set_auto_sync(bool on) { auto_sync_ = on; }
  // opt-in tolerance arithmetic (lf_set_math): contract = true trades bit equality
  // with the reference for the north star's tolerance (relative L1 <= 1e-10, dt to 1e-12)
  void set_contract_math(bool contract) {
    check(lf_set_math(h_, contract ? LF_MATH_CONTRACT : LF_MATH_EXACT));
  }
  void sync_to_host(SolverState& state, MaterialCells* materials = nullptr) const {
    if (!is_resident(state)) throw Error("state is not resident on this solver");
    download(state.field);
    if (materials != nullptr) {
      if (resident_mat_ != materials) throw Error("material cells are not resident on this solver");
      check(lf_download_partials(h_, partial_ptrs(*materials).p, grid_.nxt()));
    }
  }
  lf_handle* handle() const { return h_; }

 private:
  static int kind(BcKind k) {
    return k == BcKind::reflective ? LF_REFLECTIVE
                                   : (k == BcKind::periodic ? LF_PERIODIC : LF_TRANSMISSIVE);
  }
  std::string error_text() const {
    lf_error e{};
    lf_last_error(h_, &e);
    return e.message;
  }
  void check(int rc) const {
    if (!rc) return;
    lf_error e{};
    lf_last_error(h_, &e);
    switch (e.kind) {
      case LF_ERR_POSITIVITY: throw PositivityError(e.message, e.i, e.j, e.step, e.dt);
      case LF_ERR_CONFIG: throw ConfigError(e.message);
      case LF_ERR_DT_STATE:
      case LF_ERR_PRIMITIVE:
      case LF_ERR_TRACE:
      case LF_ERR_FRACTION: throw InvalidStateError(e.message);
      default: throw Error(e.message);
    }
  }
  void upload(const CellField& f) const {
    double* p[4] = {const_cast<double*>(f.comp[0].data()), const_cast<double*>(f.comp[1].data()),
                    const_cast<double*>(f.comp[2].data()), const_cast<double*>(f.comp[3].data())};
    check(lf_upload(h_, p, grid_.nxt()));
  }
  struct PartialPtrs {
    double* p[16];
  };
  static PartialPtrs partial_ptrs(MaterialCells& m) {
    PartialPtrs r{};
    for (int k = 0; k < m.count() && k < 16; ++k) r.p[k] = m.partial[std::size_t(k)].data();
    return r;
  }
  void download(CellField& f) const {
    double* p[4] = {f.comp[0].data(), f.comp[1].data(), f.comp[2].data(), f.comp[3].data()};
    check(lf_download(h_, p, grid_.nxt(), 0));
  }
  bool is_resident(const SolverState& s) const {
    return resident_ == &s && s.time == resident_time_ && s.step == resident_step_;
  }
  // the device copy is about to be replaced: without auto_sync it is the only
  // current copy of the resident state, so save it (and its partials) first
  void evict() const {
    if (resident_ != nullptr && !auto_sync_ && is_resident(*resident_)) {
      download(resident_->field);
      if (resident_mat_ != nullptr)
        check(lf_download_partials(h_, partial_ptrs(*resident_mat_).p, grid_.nxt()));
    }
    resident_ = nullptr;
    resident_mat_ = nullptr;
  }

  CartesianGrid grid_;
  int threads_;
  lf_handle* h_ = nullptr;
  mutable SolverState* resident_ = nullptr;
  mutable MaterialCells* resident_mat_ = nullptr;
  double resident_time_ = 0.0;
  std::int64_t resident_step_ = 0;
  int n_mat_ = 0;
  bool auto_sync_ = true;
};

// The free compute_dt (solver.cpp:55-59): a solver with default boundaries and
// scheme parameters evaluates compute_dt of `field` on the device.
inline double compute_dt(const CartesianGrid& g, const CellField& field, PerfectGasEos eos,
                         const TimeControls& controls, double time, double limit_time,
                         int device = 0) {
  LagfluxSolver solver(g, BoundaryCondition{}, eos, SchemeParams{}, 1, nullptr, device);
  return solver.compute_dt(field, controls, time, limit_time);
}

}  // namespace lagflux::b200
