// adaptflow_gpu.hpp — the drop-in C++ shim a maintainer adds to the reference
// tree (/root/reference/proj/core) so its solver entry points run on the B200
// through libafgpu's C ABI (include/af_gpu.h). Header-only; it uses the
// reference's own types (UniformGrid, BlockData, CaseSpec, SchemeConfig,
// RunReport, MROptions) and rethrows the reference's exceptions with the
// reference's messages. See INTEGRATION.md for how the bodies of
// run_uniform / step_block / run_mr forward here.
//
// Reference seams mirrored:
//   gpu::rk2_stage    step.hpp:62-64 with FluxField capture (step.hpp:16-50)
//   gpu::step_block   step.hpp:77-79 (RK2 branch, step.cpp:237-251); the
//                     ghost refill callback becomes the BoundaryCondition the
//                     device folds into its stencil mapping (grid.cpp:9-62)
//   gpu::run_uniform  unigrid.hpp:24-26 / unigrid.cpp:7-50
//   gpu::run_mr       mr_solver.hpp:78-79 / mr_solver.cpp:318-400 (returns the
//                     final to_uniform(L) grid instead of the host MRTree)
//   gpu::reference_solution  cases.hpp:58-59 / cases.cpp:181-210: the cached uniform
//                     reference, computed by gpu::run_uniform on a cache miss; same
//                     cache files, same key text, same CacheCorrupt conditions
//   gpu::AmrDevice    PatchHierarchy (amr.hpp:123-242) on the device
//   gpu::run_amr      amr_solver.hpp:34-35 / amr_solver.cpp:62-133 (returns the
//                     device hierarchy instead of the host PatchHierarchy)
#pragma once

#include <algorithm>
#include <chrono>
#include <cstring>
#include <filesystem>
#include <functional>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "adaptflow/amr.hpp"
#include "adaptflow/amr_solver.hpp"
#include "adaptflow/cases.hpp"
#include "adaptflow/errors.hpp"
#include "adaptflow/grid.hpp"
#include "adaptflow/metrics.hpp"
#include "adaptflow/mr_solver.hpp"
#include "adaptflow/scheme.hpp"
#include "adaptflow/snapshot.hpp"
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
  // rk2_stage on host AoS states; capture (nullable): FluxField-layout buffer
  StepDiag stage(const std::vector<double>& base, const std::vector<double>& eval,
                 std::vector<double>& out, double stage_dt, double* capture) {
    af_step_diag d{};
    check(af_uniform_rk2_stage(h_, base.data(), eval.data(), out.data(), stage_dt, capture, &d));
    StepDiag r;
    r.max_wave_speed = d.max_wave_speed;
    r.fallbacks = d.fallbacks;
    return r;
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

// The device context step_block reuses across calls: one per host thread,
// rebuilt only when the geometry, gas, boundary condition or scheme changes.
struct StepBlockCache {
  std::unique_ptr<UniformDevice> dev;
  int dim = 0, level = -1, bc[6] = {0, 0, 0, 0, 0, 0}, flux = -1, limiter = -1, integ = -1;
  double origin = 0.0, extent = 0.0, gamma = 0.0;
  long creations = 0;  // contexts built so far (tests/cpp/shim_parity.cpp)

  UniformDevice& get(const UniformGrid& g, const GasModel& gas, const BoundaryCondition& b,
                     const SchemeConfig& s) {
    const af_config c = make_config(g.dim(), g.level(), g.origin(), g.extent(), gas, b, s);
    bool same = dev && dim == c.dim && level == c.level && origin == c.origin &&
                extent == c.extent && gamma == c.gamma && flux == c.flux &&
                limiter == c.limiter && integ == c.integrator;
    for (int f = 0; f < 6 && same; ++f) same = bc[f] == c.bc[f];
    if (!same) {
      dev.reset();
      dev = std::make_unique<UniformDevice>(g, gas, b, s);
      dim = c.dim;
      level = c.level;
      origin = c.origin;
      extent = c.extent;
      gamma = c.gamma;
      flux = c.flux;
      limiter = c.limiter;
      integ = c.integrator;
      for (int f = 0; f < 6; ++f) bc[f] = c.bc[f];
      ++creations;
    }
    return *dev;
  }
};

inline StepBlockCache& step_block_cache() {
  static thread_local StepBlockCache cache;
  return cache;
}

// step_block (step.hpp:77-79) for one block whose ghosts follow `bc`. The
// block lives in host memory, so each call uploads it and downloads the
// result; the device context is cached per thread (step_block_cache).
inline StepDiag step_block(BlockData& u, const UniformGrid& geometry, double dt,
                           const SchemeConfig& cfg, const GasModel& gas,
                           const BoundaryCondition& bc) {
  UniformDevice& dev = step_block_cache().get(geometry, gas, bc, cfg);
  dev.upload(u);
  const StepDiag d = dev.step(dt);
  dev.download(u);
  return d;
}

// rk2_stage (step.hpp:62-64): out = base + stage_dt * rhs(eval) for host
// blocks on `geometry`, eval's ghosts following `bc` (the reference expects
// them filled; the device maps them from bc). capture: the stage's fluxes
// into the caller's FluxField (step.hpp:16-50), as the AMR hierarchy's
// refluxing reads them (amr_hierarchy.cpp:476,488). out may alias base or
// eval. The device context is the step_block cache's.
inline StepDiag rk2_stage(const BlockData& base, const BlockData& eval, BlockData& out,
                          const UniformGrid& geometry, double stage_dt, const SchemeConfig& cfg,
                          const GasModel& gas, const BoundaryCondition& bc,
                          FluxField* capture = nullptr) {
  UniformDevice& dev = step_block_cache().get(geometry, gas, bc, cfg);
  const int dim = geometry.dim(), n = 1 << geometry.level();
  std::vector<double> o(static_cast<size_t>(out.interior_cells()) * 5), cap;
  if (capture) {
    cap.resize(static_cast<size_t>(dim) * (n + 1) * (dim == 3 ? (long)n * n : (long)n) * 5);
    if (capture->dim() != dim || capture->cells()[0] != n)
      *capture = FluxField(dim, {n, n, dim == 3 ? n : 1});
  }
  const StepDiag d = dev.stage(to_aos(base), to_aos(eval), o, stage_dt,
                               capture ? cap.data() : nullptr);
  from_aos(o, out);
  if (capture) {
    size_t f = 0;
    for (int a = 0; a < dim; ++a) {
      int fn[3] = {n, n, dim == 3 ? n : 1};
      fn[a] += 1;
      for (int k = 0; k < fn[2]; ++k)
        for (int j = 0; j < fn[1]; ++j)
          for (int i = 0; i < fn[0]; ++i, ++f)
            std::memcpy(&capture->face(a, i, j, k), &cap[5 * f], sizeof(FluxVector));
    }
  }
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

// A device-resident MR tree: the MRTree calls of the hot path (mr_tree.hpp)
// on libafgpu, with host views of the leaf set and the uniform projection.
class MRDevice {
 public:
  MRDevice(int dim, int level, double origin, double extent, const GasModel& gas,
           const BoundaryCondition& bc, const SchemeConfig& s, const af_mr_options& o,
           int device = 0)
      : dim_(dim), level_(level), origin_(origin), extent_(extent) {
    const af_config c = make_config(dim, level, origin, extent, gas, bc, s, device);
    check(af_mr_create(&c, &o, &m_));
  }
  ~MRDevice() { af_mr_destroy(m_); }
  MRDevice(const MRDevice&) = delete;
  MRDevice& operator=(const MRDevice&) = delete;

  // MRTree::from_uniform + set_min_leaf_level + coarsen (mr_solver.cpp:323-328)
  void build(const UniformGrid& g) { check(af_mr_build(m_, to_aos(g.block()).data())); }
  // MRTree::refine(eps, buffer_radius_per_level) (mr_tree.hpp:141)
  void refine(double eps, const std::vector<int>& buffer = {}) {
    check(af_mr_refine_buffer(m_, eps, buffer.data(), static_cast<int>(buffer.size())));
  }
  void refine_lt(int top) { check(af_mr_refine(m_, top)); }  // run_mr's LT form
  void add_virtual_leaves() { check(af_mr_add_virtual_leaves(m_)); }
  void remove_virtual_leaves() { check(af_mr_remove_virtual_leaves(m_)); }
  void coarsen() { check(af_mr_coarsen(m_)); }
  double evolve_global(double dt) {
    af_step_diag d{};
    check(af_mr_evolve_global(m_, dt, &d));
    return d.max_wave_speed;
  }
  double advance_local(int top, double t, double dt) {
    af_step_diag d{};
    check(af_mr_advance_local(m_, top, t, dt, &d));
    return d.max_wave_speed;
  }
  long leaf_count() {
    long lv = 0, nd = 0, in = 0;
    check(af_mr_counts(m_, &lv, &nd, &in));
    return lv;
  }
  long node_count() {
    long lv = 0, nd = 0, in = 0;
    check(af_mr_counts(m_, &lv, &nd, &in));
    return nd;
  }
  int coarsest_leaf_level() {
    int l = 0;
    check(af_mr_coarsest_leaf_level(m_, &l));
    return l;
  }
  // MRTree::leaves() (sorted pack_key)
  std::vector<NodeKey> leaves() {
    size_t n = 0;
    check(af_mr_leaf_keys(m_, nullptr, &n));
    std::vector<NodeKey> out(n);
    check(af_mr_leaf_keys(m_, reinterpret_cast<uint64_t*>(out.data()), &n));
    return out;
  }
  // MRTree::to_uniform(level) (mr_tree.cpp:608-621)
  UniformGrid to_uniform(int level) {
    UniformGrid g(dim_, level, origin_, extent_);
    std::vector<double> aos(static_cast<size_t>(g.block().interior_cells()) * 5);
    check(af_mr_to_uniform(m_, level, aos.data()));
    from_aos(aos, g.block());
    return g;
  }
  int dim() const { return dim_; }
  int max_level() const { return level_; }
  double origin() const { return origin_; }
  double extent() const { return extent_; }
  double dx(int level) const { return extent_ / static_cast<double>(1 << level); }
  af_mr* handle() { return m_; }
  void check(af_status st) {
    if (st == AF_OK) return;
    af_error e{};
    af_mr_last_error(m_, &e);
    rethrow(st, e);
  }

 private:
  af_mr* m_ = nullptr;
  int dim_, level_;
  double origin_, extent_;
};

// The tree as MROptions::on_sample observers use it (driver.cpp:47-60 reads
// leaves(), dx(), origin() and dim()), served from the device tree.
using SampleFn = std::function<void(long fine_steps_done, MRDevice& tree)>;

// dump_tree_mesh (driver.cpp:47-60) of a device tree: the same text.
inline std::string tree_mesh_text(MRDevice& tree) {
  std::ostringstream os;
  os.precision(12);
  for (NodeKey k : tree.leaves()) {
    const NodeId id = unpack_key(k);
    const double h = tree.dx(id.level);
    os << id.level;
    for (int a = 0; a < tree.dim(); ++a) os << ' ' << tree.origin() + id.idx[a] * h;
    for (int a = 0; a < tree.dim(); ++a) os << ' ' << tree.origin() + (id.idx[a] + 1) * h;
    os << '\n';
  }
  return os.str();
}

// run_mr (mr_solver.cpp:318-400): fixed dt_fine = t_end / n_steps.
// MROptions::on_sample observes a host MRTree, which the device run does not
// build; a caller that sets it gets ConfigError instead of a silent skip, and
// passes `sample` (called at the same point, mr_solver.cpp:394, with the
// device tree) instead. Without `sample` the whole run is one af_mr_run call
// (CUDA-graph cycles); with it the cycle loop runs here, one cycle at a time.
inline MRDeviceResult run_mr(const CaseSpec& spec, int level, long n_steps,
                             const SchemeConfig& scheme, const MROptions& options,
                             const std::vector<double>* eps_level = nullptr,
                             const SampleFn& sample = nullptr) {
  if (options.on_sample)
    throw ConfigError(
        "gpu::run_mr: MROptions::on_sample observes a host MRTree, which the device run does "
        "not build; pass a gpu::SampleFn (leaf keys, to_uniform and the mesh geometry of the "
        "device tree) instead");
  UniformGrid init(spec.dim, level, spec.origin, spec.extent);
  init_case(spec, init);
  af_mr_options o{};
  o.eps = options.epsilon;
  o.eps_level = eps_level ? eps_level->data() : nullptr;
  o.min_leaf_level = 0;
  o.local_time = options.local_time ? 1 : 0;
  o.lt_gap = options.local_time_level_gap;
  MRDevice tree(spec.dim, level, spec.origin, spec.extent, spec.gas, spec.bc, scheme, o);
  tree.build(init);
  MRDeviceResult out{UniformGrid(spec.dim, level, spec.origin, spec.extent), RunReport{}, {}};
  RunReport& rep = out.report;
  rep.method = options.local_time ? Method::MRLT : Method::MR;
  rep.case_name = spec.name;
  rep.level = level;
  rep.n_steps = n_steps;
  rep.preset_scheme = scheme.is_preset();
  const double dt_fine = spec.t_end / static_cast<double>(n_steps);
  if (!sample) {
    std::vector<af_mr_cycle> cyc(static_cast<size_t>(n_steps));
    af_run_diag d{};
    const auto t0 = std::chrono::steady_clock::now();
    tree.check(af_mr_run(tree.handle(), n_steps, 0.0, dt_fine, cyc.data(), n_steps, &d));
    rep.wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rep.max_cfl = d.max_cfl;
    rep.fallbacks = d.fallbacks;
    for (const af_mr_cycle& k : cyc) {
      if (k.sub <= 0) break;
      for (long s = 0; s < k.sub; ++s) {
        rep.cells_per_step.push_back(k.nodes);
        rep.leaves_per_step.push_back(k.leaves);
      }
    }
  } else {
    // the cycle loop of mr_solver.cpp:339-395 on the device calls
    using clock = std::chrono::steady_clock;
    double wall = 0.0, max_speed = 0.0;
    long done = 0;
    while (done < n_steps) {
      const auto t0 = clock::now();
      long sub = 1;
      int top = level;
      if (options.local_time) {
        top = std::max(tree.coarsest_leaf_level(), std::max(0, level - options.local_time_level_gap));
        long span = 1l << (level - top);
        while (span > n_steps - done) {
          span >>= 1;
          ++top;
        }
        sub = span;
        tree.refine_lt(top);
      } else {
        tree.refine_lt(-1);
      }
      tree.add_virtual_leaves();
      const long cells = tree.node_count(), leaves = tree.leaf_count();
      for (long s = 0; s < sub; ++s) {
        rep.cells_per_step.push_back(cells);
        rep.leaves_per_step.push_back(leaves);
      }
      try {
        if (options.local_time)
          tree.advance_local(top, static_cast<double>(done) * dt_fine,
                             static_cast<double>(sub) * dt_fine);
        else
          tree.evolve_global(dt_fine);
      } catch (const NonPhysicalState& e) {
        throw NonPhysicalState("step " + std::to_string(done) + ": " + e.what());
      }
      tree.remove_virtual_leaves();
      tree.coarsen();
      done += sub;
      wall += std::chrono::duration<double>(clock::now() - t0).count();
      sample(done, tree);
    }
    (void)max_speed;
    rep.wall_seconds = wall;
    tree.check(af_mr_solver_stats(tree.handle(), &rep.max_cfl, &rep.fallbacks));
  }
  out.grid = tree.to_uniform(level);
  out.leaves = tree.leaves();
  return out;
}

// reference_solution (cases.cpp:181-210): the uniform reference solution of a
// case at ref_level, from the cache directory when a valid snapshot is there,
// otherwise computed on the device and cached. The key text (the FNV-1a hash
// of reference_config_string and the string itself) and the file names are the
// reference's, so either implementation accepts the other's cache.
inline UniformGrid reference_solution(const CaseSpec& spec, int ref_level,
                                      const SchemeConfig& scheme, const std::string& cache_dir) {
  const std::string config = reference_config_string(spec, ref_level, scheme);
  unsigned long long h = 1469598103934665603ull;  // FNV-1a, 64 bit
  for (unsigned char c : config) {
    h ^= c;
    h *= 1099511628211ull;
  }
  const std::string key = "hash=" + std::to_string(h) + "\n" + config + "\n";
  std::string path, meta_path;
  if (!cache_dir.empty()) {
    std::filesystem::create_directories(cache_dir);
    path = reference_cache_path(spec, ref_level, scheme, cache_dir);
    meta_path = path + ".meta";
    if (std::filesystem::exists(path)) {
      if (!std::filesystem::exists(meta_path) || read_text_file(meta_path) != key)
        throw CacheCorrupt("cached reference " + path +
                           " does not match the requested configuration");
      Snapshot snap = read_snapshot(path);
      if (snap.grid.level() != ref_level || snap.grid.dim() != spec.dim)
        throw CacheCorrupt("cached reference " + path + " has wrong geometry");
      return std::move(snap.grid);
    }
  }
  UniformRunResult res = gpu::run_uniform(spec, ref_level, spec.steps_for_level(ref_level), scheme);
  if (!cache_dir.empty()) {
    write_snapshot(path, res.grid, spec.gas.gamma, spec.t_end);
    write_text_file(meta_path, key);
  }
  return std::move(res.grid);
}

// ---------------------------------------------------------------- AMR ----
// PatchHierarchy (amr.hpp:123-242) whose patch data live on the device.
class AmrDevice {
 public:
  AmrDevice(int dim, int base_exp, double origin, double extent, const BoundaryCondition& bc,
            const GasModel& gas, const AmrOptions& opts, const SchemeConfig& scheme)
      : dim_(dim), base_exp_(base_exp) {
    const af_config c = make_config(dim, base_exp, origin, extent, gas, bc, scheme);
    af_amr_options o{};
    o.eps_rho = opts.eps_rho;
    o.eps_p = opts.eps_p;
    o.cluster_efficiency = opts.cluster_efficiency;
    o.time_refine = opts.time_refine ? 1 : 0;
    o.flux_correction = opts.flux_correction ? 1 : 0;
    o.max_levels = opts.max_levels;
    const af_status st = af_amr_create(&c, &o, &h_);
    if (st != AF_OK) throw ConfigError("af_amr_create failed");
  }
  ~AmrDevice() { af_amr_destroy(h_); }
  AmrDevice(const AmrDevice&) = delete;
  AmrDevice& operator=(const AmrDevice&) = delete;

  void check(af_status st) const {
    if (st == AF_OK) return;
    af_error e{};
    af_amr_last_error(h_, &e);
    rethrow(st, e);
  }
  af_amr* handle() const { return h_; }
  int dim() const { return dim_; }
  int base_exp() const { return base_exp_; }

  void initialize(const std::function<ConservedState(double, double, double)>& ic) {
    auto thunk = [](double x, double y, double z, double* q, void* user) {
      const auto& f = *static_cast<const std::function<ConservedState(double, double, double)>*>(user);
      const ConservedState s = f(x, y, z);
      q[0] = s.rho;
      q[1] = s.mom[0];
      q[2] = s.mom[1];
      q[3] = s.mom[2];
      q[4] = s.rhoE;
    };
    check(af_amr_initialize(h_, thunk, const_cast<void*>(static_cast<const void*>(&ic))));
  }
  void sync_ghosts(int l, double tau) { check(af_amr_sync_ghosts(h_, l, tau)); }
  void remesh(int l) { check(af_amr_remesh(h_, l)); }
  StepDiag update_level(int l, double dt) {
    af_step_diag d{};
    check(af_amr_update_level(h_, l, dt, &d));
    StepDiag out;
    out.max_wave_speed = d.max_wave_speed;
    out.fallbacks = d.fallbacks;
    return out;
  }
  void average_down(int l) { check(af_amr_average_down(h_, l)); }
  void flux_correct(int l) { check(af_amr_flux_correct(h_, l)); }
  int n_levels() const {
    int n = 0;
    check(af_amr_n_levels(h_, &n));
    return n;
  }
  std::vector<Box> boxes(int l) const {
    int np = 0;
    check(af_amr_level_info(h_, l, &np, nullptr, nullptr, nullptr));
    std::vector<int> b(static_cast<size_t>(6) * std::max(np, 1));
    check(af_amr_boxes(h_, l, b.data(), np));
    std::vector<Box> out(static_cast<size_t>(np));
    for (int i = 0; i < np; ++i)
      for (int a = 0; a < 3; ++a) {
        out[i].lo[a] = b[6 * i + a];
        out[i].hi[a] = b[6 * i + 3 + a];
      }
    return out;
  }
  // Patch payloads of a level, patch after patch (ghost 0: interiors, 2: the
  // blocks with their ghost layers), 5 doubles per cell, x fastest.
  std::vector<double> patch_data(int l, int ghost = 0, bool old = false) const {
    long cells = 0;
    check(af_amr_patch_data_cells(h_, l, ghost, &cells));
    std::vector<double> out(static_cast<size_t>(5 * cells));
    check(af_amr_patch_data(h_, l, ghost, old ? 1 : 0, out.data()));
    return out;
  }
  UniformGrid assemble_level(int l, double origin, double extent) const {
    UniformGrid g(dim_, base_exp_ + l, origin, extent);
    std::vector<double> aos(static_cast<size_t>(5) * g.block().interior_cells());
    check(af_amr_assemble_level(h_, l, aos.data()));
    from_aos(aos, g.block());
    return g;
  }
  ConservedState total_conserved() const {
    double t[5];
    check(af_amr_total_conserved(h_, t));
    ConservedState s;
    s.rho = t[0];
    s.mom = {t[1], t[2], t[3]};
    s.rhoE = t[4];
    return s;
  }
  long total_cells() const {
    long a = 0, b = 0;
    check(af_amr_counts(h_, &a, &b));
    return a;
  }
  long composite_cells() const {
    long a = 0, b = 0;
    check(af_amr_counts(h_, &a, &b));
    return b;
  }
  bool properly_nested() const {
    int n = 0;
    check(af_amr_properly_nested(h_, &n));
    return n != 0;
  }
  std::string dump_boxes() const {
    const char* t = nullptr;
    check(af_amr_dump_boxes(h_, &t));
    return t ? std::string(t) : std::string();
  }

 private:
  af_amr* h_ = nullptr;
  int dim_, base_exp_;
};

struct AmrDeviceResult {
  std::unique_ptr<AmrDevice> hierarchy;
  RunReport report;
};

// run_amr (amr_solver.cpp:62-133) on the device. AmrRunOptions::on_sample
// observes a host PatchHierarchy, which this run does not build: the device
// form of the callback takes the AmrDevice instead.
using AmrSampleFn = std::function<void(long fine_steps_done, AmrDevice&)>;

inline AmrDeviceResult run_amr(const CaseSpec& spec, int level, long n_steps,
                               const SchemeConfig& scheme, const AmrRunOptions& options,
                               const AmrSampleFn& sample = nullptr) {
  if (options.on_sample)
    throw ConfigError(
        "gpu::run_amr: AmrRunOptions::on_sample observes a host PatchHierarchy, which the "
        "device run does not build; pass a gpu::AmrSampleFn instead");
  const int base_exp = amr_base_exp(spec.dim, level);
  if (base_exp < 0) throw ConfigError("amr needs level >= 1, got " + std::to_string(level));
  AmrOptions opts;
  opts.max_levels = level - base_exp;
  opts.time_refine = options.time_refine;
  opts.flux_correction = options.flux_correction;
  opts.eps_rho = options.eps_rho >= 0.0 ? options.eps_rho : spec.amr_eps_rho;
  opts.eps_p = options.eps_p >= 0.0 ? options.eps_p : spec.amr_eps_p;
  opts.cluster_efficiency = options.eta_tol >= 0.0 ? options.eta_tol : spec.cluster_efficiency;

  AmrDeviceResult out;
  out.hierarchy = std::make_unique<AmrDevice>(spec.dim, base_exp, spec.origin, spec.extent,
                                              spec.bc, spec.gas, opts, scheme);
  AmrDevice& h = *out.hierarchy;
  RunReport& rep = out.report;
  rep.method = options.time_refine ? Method::AMRLT : Method::AMR;
  rep.case_name = spec.name;
  rep.level = level;
  rep.n_steps = n_steps;
  rep.preset_scheme = scheme.is_preset();
  const double dt_finest = spec.t_end / static_cast<double>(n_steps);
  const long per_cycle = options.time_refine ? (1l << opts.max_levels) : 1;
  if (n_steps % per_cycle != 0)
    throw ConfigError("n_steps=" + std::to_string(n_steps) + " is not a multiple of the " +
                      std::to_string(per_cycle) + " substeps of one time-refined cycle");
  h.initialize([&spec](double x, double y, double z) { return spec.initial_state(x, y, z); });
  rep.cells_per_step.assign(static_cast<size_t>(n_steps), 0);
  rep.leaves_per_step.assign(static_cast<size_t>(n_steps), 0);
  const auto t0 = std::chrono::steady_clock::now();
  if (!sample) {
    af_run_diag d{};
    h.check(af_amr_run(h.handle(), n_steps, dt_finest, rep.cells_per_step.data(),
                       rep.leaves_per_step.data(), &d));
    rep.max_cfl = d.max_cfl;
    rep.fallbacks = d.fallbacks;
  } else {  // cycle by cycle, the observer after each (amr_solver.cpp:118-129)
    for (long done = 0; done < n_steps; done += per_cycle) {
      af_run_diag d{};
      try {
        h.check(af_amr_run(h.handle(), per_cycle, dt_finest, rep.cells_per_step.data() + done,
                           rep.leaves_per_step.data() + done, &d));
      } catch (const NonPhysicalState& e) {
        // the device numbers its cycles per call: restore the run's cycle index
        const std::string w = e.what();
        const std::string pre = "cycle 0: ";
        throw NonPhysicalState("cycle " + std::to_string(done / per_cycle) + ": " +
                               (w.rfind(pre, 0) == 0 ? w.substr(pre.size()) : w));
      }
      rep.max_cfl = std::max(rep.max_cfl, d.max_cfl);
      rep.fallbacks += d.fallbacks;
      sample(done + per_cycle, h);
    }
  }
  rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

}  // namespace gpu
}  // namespace adaptflow
