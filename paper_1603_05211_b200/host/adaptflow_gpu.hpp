// adaptflow_gpu.hpp — the drop-in C++ shim a maintainer adds to the reference
// tree (/root/reference/proj/core) so its solver entry points run on the B200
// through libafgpu's C ABI (include/af_gpu.h). Header-only; it uses the
// reference's own types (UniformGrid, BlockData, CaseSpec, SchemeConfig,
// RunReport, MROptions) and rethrows the reference's exceptions with the
// reference's messages. See INTEGRATION.md for how the bodies of
// run_uniform / step_block / run_mr forward here.
//
// Reference seams mirrored:
//   gpu::step_block   step.hpp:77-79 (RK2 branch, step.cpp:237-251); the
//                     ghost refill callback becomes the BoundaryCondition the
//                     device folds into its stencil mapping (grid.cpp:9-62)
//   gpu::run_uniform  unigrid.hpp:24-26 / unigrid.cpp:7-50
//   gpu::run_mr       mr_solver.hpp:78-79 / mr_solver.cpp:318-400 (returns the
//                     final to_uniform(L) grid instead of the host MRTree)
#pragma once

#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "adaptflow/cases.hpp"
#include "adaptflow/errors.hpp"
#include "adaptflow/grid.hpp"
#include "adaptflow/metrics.hpp"
#include "adaptflow/mr_solver.hpp"
#include "adaptflow/scheme.hpp"
#include "adaptflow/step.hpp"
#include "adaptflow/unigrid.hpp"
#include "af_gpu.h"

namespace adaptflow {
namespace gpu {

// af_status + af_error -> the reference's exception hierarchy (errors.hpp).
[[noreturn]] inline void rethrow(af_status st, const af_error& e) {
  const std::string msg = e.message;
  switch (st) {
    case AF_E_NONPHYSICAL: throw NonPhysicalState(msg);
    case AF_E_REGISTER_MISMATCH: throw RegisterMismatch(msg);
    case AF_E_CONFIG:
    case AF_E_UNSUPPORTED: throw ConfigError(msg);
    case AF_E_LEVEL_MISMATCH: throw LevelMismatch(msg);
    default: throw Error("libafgpu: " + msg);
  }
}

inline af_config make_config(int dim, int level, double origin, double extent,
                             const GasModel& gas, const BoundaryCondition& bc,
                             const SchemeConfig& s, int device = 0) {
  af_config c{};
  c.dim = dim;
  c.level = level;
  c.origin = origin;
  c.extent = extent;
  c.gamma = gas.gamma;
  for (int f = 0; f < 6; ++f)
    c.bc[f] = bc.faces[f] == BcKind::Periodic     ? AF_BC_PERIODIC
              : bc.faces[f] == BcKind::Reflective ? AF_BC_REFLECTIVE
                                                  : AF_BC_OUTFLOW;
  c.flux = s.flux == FluxKind::AusmPlus ? AF_FLUX_AUSM_PLUS : AF_FLUX_AUSMDV;
  c.limiter = s.limiter == LimiterKind::Minmod ? AF_LIMITER_MINMOD : AF_LIMITER_VAN_ALBADA;
  c.integrator = s.integrator == IntegratorKind::RK2 ? AF_INTEGRATOR_RK2
                                                     : AF_INTEGRATOR_MUSCL_HANCOCK;
  c.device = device;
  return c;
}

// Interior cells of a block as the ABI's AoS (ConservedState is 5 doubles).
inline std::vector<double> to_aos(const BlockData& b) {
  std::vector<double> out(static_cast<size_t>(b.interior_cells()) * 5);
  size_t c = 0;
  b.for_interior([&](int i, int j, int k) {
    std::memcpy(&out[5 * c++], &b.at(i, j, k), sizeof(ConservedState));
  });
  return out;
}

inline void from_aos(const std::vector<double>& aos, BlockData& b) {
  size_t c = 0;
  b.for_interior([&](int i, int j, int k) {
    std::memcpy(&b.at(i, j, k), &aos[5 * c++], sizeof(ConservedState));
  });
}

// A uniform mesh resident on one GPU.
class UniformDevice {
 public:
  UniformDevice(const UniformGrid& g, const GasModel& gas, const BoundaryCondition& bc,
                const SchemeConfig& s, int device = 0) {
    const af_config c = make_config(g.dim(), g.level(), g.origin(), g.extent(), gas, bc, s, device);
    check(af_uniform_create(&c, nullptr, &h_));
  }
  ~UniformDevice() { af_uniform_destroy(h_); }
  UniformDevice(const UniformDevice&) = delete;
  UniformDevice& operator=(const UniformDevice&) = delete;

  void upload(const BlockData& b) { check(af_uniform_upload(h_, to_aos(b).data())); }
  void download(BlockData& b) {
    std::vector<double> aos(static_cast<size_t>(b.interior_cells()) * 5);
    check(af_uniform_download(h_, aos.data()));
    from_aos(aos, b);
  }
  StepDiag step(double dt) {
    af_step_diag d{};
    check(af_uniform_step(h_, dt, &d));
    StepDiag out;
    out.max_wave_speed = d.max_wave_speed;
    out.fallbacks = d.fallbacks;
    return out;
  }

 private:
  void check(af_status st) {
    if (st == AF_OK) return;
    af_error e{};
    af_uniform_last_error(h_, &e);
    rethrow(st, e);
  }
  af_uniform* h_ = nullptr;
};

// step_block (step.hpp:77-79) for one block whose ghosts follow `bc`.
inline StepDiag step_block(BlockData& u, const UniformGrid& geometry, double dt,
                           const SchemeConfig& cfg, const GasModel& gas,
                           const BoundaryCondition& bc) {
  UniformDevice dev(geometry, gas, bc, cfg);
  dev.upload(u);
  const StepDiag d = dev.step(dt);
  dev.download(u);
  return d;
}

// run_uniform (unigrid.cpp:7-50): same data, same fixed dt, same report.
inline UniformRunResult run_uniform(const CaseSpec& spec, int level, long n_steps,
                                    const SchemeConfig& scheme,
                                    const StepCallback& on_step = nullptr) {
  UniformRunResult out;
  out.grid = UniformGrid(spec.dim, level, spec.origin, spec.extent);
  init_case(spec, out.grid);
  RunReport& rep = out.report;
  rep.method = Method::FV;
  rep.case_name = spec.name;
  rep.level = level;
  rep.n_steps = n_steps;
  rep.preset_scheme = scheme.is_preset();
  const double dt = spec.t_end / static_cast<double>(n_steps);
  const double dx = out.grid.dx();
  const long n_c = out.grid.block().interior_cells();
  rep.cells_per_step.assign(static_cast<size_t>(n_steps), n_c);
  rep.leaves_per_step.assign(static_cast<size_t>(n_steps), n_c);
  UniformDevice dev(out.grid, spec.gas, spec.bc, scheme);
  dev.upload(out.grid.block());
  using clock = std::chrono::steady_clock;
  double wall = 0.0;
  for (long step = 0; step < n_steps; ++step) {
    const auto t0 = clock::now();
    StepDiag diag;
    try {
      diag = dev.step(dt);
    } catch (const NonPhysicalState& e) {
      throw NonPhysicalState("step " + std::to_string(step) + ": " + e.what());
    }
    rep.max_cfl = std::max(rep.max_cfl, diag.max_wave_speed * dt / dx);
    rep.fallbacks += diag.fallbacks;
    wall += std::chrono::duration<double>(clock::now() - t0).count();
    if (on_step) {
      dev.download(out.grid.block());
      on_step(step, out.grid);
    }
  }
  rep.wall_seconds = wall;
  dev.download(out.grid.block());
  return out;
}

struct MRDeviceResult {
  UniformGrid grid;  // MRTree::to_uniform(level) of the final tree
  RunReport report;
  std::vector<NodeKey> leaves;  // MRTree::leaves() of the final tree
};

// run_mr (mr_solver.cpp:318-400): fixed dt_fine = t_end / n_steps.
inline MRDeviceResult run_mr(const CaseSpec& spec, int level, long n_steps,
                             const SchemeConfig& scheme, const MROptions& options,
                             const std::vector<double>* eps_level = nullptr) {
  UniformGrid init(spec.dim, level, spec.origin, spec.extent);
  init_case(spec, init);
  const af_config c = make_config(spec.dim, level, spec.origin, spec.extent, spec.gas, spec.bc,
                                  scheme);
  af_mr_options o{};
  o.eps = options.epsilon;
  o.eps_level = eps_level ? eps_level->data() : nullptr;
  o.min_leaf_level = 0;
  o.local_time = options.local_time ? 1 : 0;
  o.lt_gap = options.local_time_level_gap;
  af_mr* m = nullptr;
  auto check = [&](af_status st) {
    if (st == AF_OK) return;
    af_error e{};
    af_mr_last_error(m, &e);
    if (m) af_mr_destroy(m);
    rethrow(st, e);
  };
  check(af_mr_create(&c, &o, &m));
  check(af_mr_build(m, to_aos(init.block()).data()));
  std::vector<af_mr_cycle> cyc(static_cast<size_t>(n_steps));
  af_run_diag d{};
  const double dt_fine = spec.t_end / static_cast<double>(n_steps);
  const auto t0 = std::chrono::steady_clock::now();
  check(af_mr_run(m, n_steps, 0.0, dt_fine, cyc.data(), n_steps, &d));
  MRDeviceResult out{UniformGrid(spec.dim, level, spec.origin, spec.extent), RunReport{}, {}};
  RunReport& rep = out.report;
  rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  rep.method = options.local_time ? Method::MRLT : Method::MR;
  rep.case_name = spec.name;
  rep.level = level;
  rep.n_steps = n_steps;
  rep.preset_scheme = scheme.is_preset();
  rep.max_cfl = d.max_cfl;
  rep.fallbacks = d.fallbacks;
  for (const af_mr_cycle& k : cyc) {
    if (k.sub <= 0) break;
    for (long s = 0; s < k.sub; ++s) {
      rep.cells_per_step.push_back(k.nodes);
      rep.leaves_per_step.push_back(k.leaves);
    }
  }
  std::vector<double> aos(static_cast<size_t>(init.block().interior_cells()) * 5);
  check(af_mr_to_uniform(m, level, aos.data()));
  from_aos(aos, out.grid.block());
  size_t n = 0;
  check(af_mr_leaf_keys(m, nullptr, &n));
  out.leaves.resize(n);
  check(af_mr_leaf_keys(m, reinterpret_cast<uint64_t*>(out.leaves.data()), &n));
  af_mr_destroy(m);
  return out;
}

}  // namespace gpu
}  // namespace adaptflow
