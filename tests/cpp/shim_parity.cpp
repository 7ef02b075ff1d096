// shim_parity.cpp — drop-in check: the reference's own entry points
// (run_uniform, run_mr on its built-in cases lax_liu_6 / ellipsoid3d, fixed
// dt = t_end / n_steps) against the same calls through the C++ shim
// (paper_1603_05211_b200/host/adaptflow_gpu.hpp -> libafgpu.so). Built by
// `make -C oracle shim` (needs the reference headers; the binary travels to
// the GPU box) and run by tests/test_shim_gpu.py. Exit 0 iff every check is
// bit-identical.
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <sstream>
#include <utility>
#include <string>
#include <vector>

#include "adaptflow/snapshot.hpp"
#include "adaptflow_gpu.hpp"

using namespace adaptflow;

static int failures = 0;

static bool same_grid(const UniformGrid& a, const UniformGrid& b) {
  bool ok = true;
  a.block().for_interior([&](int i, int j, int k) {
    const ConservedState& x = a.block().at(i, j, k);
    const ConservedState& y = b.block().at(i, j, k);
    const double xa[5] = {x.rho, x.mom[0], x.mom[1], x.mom[2], x.rhoE};
    const double ya[5] = {y.rho, y.mom[0], y.mom[1], y.mom[2], y.rhoE};
    for (int m = 0; m < 5; ++m)
      if (!(xa[m] == ya[m])) ok = false;  // +0 == -0
  });
  return ok;
}

static void report(const std::string& what, bool ok) {
  std::printf("%s %s\n", ok ? "OK  " : "FAIL", what.c_str());
  if (!ok) ++failures;
}

// run_amr (amr_solver.hpp:34-35) on a built-in case with its own step
// schedule: the per-cycle box lists through the sample observers, every patch
// block with its ghost layers, the report.
static void amr_case(const char* name, int L, bool time_refine, bool rk2) {
  const CaseSpec& s = find_case(name);
  const SchemeConfig sc = rk2 ? SchemeConfig::mr_preset() : SchemeConfig::amr_preset();
  const long n = s.steps_for_level(L);
  AmrRunOptions o;
  o.time_refine = time_refine;
  std::vector<long> ref_samples, dev_samples;
  std::vector<std::string> ref_boxes, dev_boxes;
  AmrRunOptions oref = o;
  oref.on_sample = [&](long steps, const PatchHierarchy& h) {
    ref_samples.push_back(steps);
    ref_boxes.push_back(h.dump_boxes());
  };
  AmrRunResult r = run_amr(s, L, n, sc, oref);
  gpu::AmrDeviceResult g = gpu::run_amr(s, L, n, sc, o, [&](long steps, gpu::AmrDevice& h) {
    dev_samples.push_back(steps);
    dev_boxes.push_back(h.dump_boxes());
  });
  const std::string tag = std::string("run_amr ") + s.name + " L=" + std::to_string(L) + " x " +
                          std::to_string(n) + " steps" + (o.time_refine ? " AMRLT" : " AMR") +
                          (rk2 ? " RK2" : "");
  report(tag + ": samples and box lists per cycle", ref_samples == dev_samples && ref_boxes == dev_boxes);
  report(tag + ": final dump_boxes", r.hierarchy->dump_boxes() == g.hierarchy->dump_boxes());
  bool same = r.hierarchy->n_levels() == g.hierarchy->n_levels();
  long patches = 0;
  for (int l = 0; same && l < r.hierarchy->n_levels(); ++l) {
    const std::vector<double> blocks = g.hierarchy->patch_data(l, 2);
    size_t c = 0;
    for (const Patch& p : r.hierarchy->level(l).patches) {
      ++patches;
      const BlockData& b = p.data;
      const int gz = b.ghost_along(2);
      for (int k = -gz; k < b.n(2) + gz && same; ++k)
        for (int j = -2; j < b.n(1) + 2 && same; ++j)
          for (int i = -2; i < b.n(0) + 2; ++i, ++c) {
            const ConservedState& q = b.at(i, j, k);
            const double v[5] = {q.rho, q.mom[0], q.mom[1], q.mom[2], q.rhoE};
            if (5 * c + 4 >= blocks.size() || std::memcmp(v, &blocks[5 * c], sizeof v) != 0) {
              same = false;
              break;
            }
          }
    }
    same = same && 5 * c == blocks.size();
  }
  report(tag + ": every patch block with ghosts (" + std::to_string(patches) + " patches)", same);
  report(tag + ": cells_per_step", r.report.cells_per_step == g.report.cells_per_step);
  report(tag + ": leaves_per_step", r.report.leaves_per_step == g.report.leaves_per_step);
  report(tag + ": max_cfl", r.report.max_cfl == g.report.max_cfl);
  report(tag + ": fallbacks", r.report.fallbacks == g.report.fallbacks);
  report(tag + ": levels above the base", g.hierarchy->n_levels() >= 2);
  std::printf("     reference %.2f s, device %.3f s\n", r.report.wall_seconds, g.report.wall_seconds);
}

int main(int argc, char** argv) {
  std::setvbuf(stdout, nullptr, _IONBF, 0);
  if (argc > 1 && std::string(argv[1]) == "amr-full") {
    // the paper's configuration sizes (base 64^2 / 8^3) with the cases' own
    // step schedules: lax_liu_6 up to 1024^2, ellipsoid3d up to 128^3
    amr_case("lax_liu_6", 9, true, false);
    amr_case("lax_liu_6", 10, true, false);
    amr_case("ellipsoid3d", 6, true, false);
    amr_case("ellipsoid3d", 7, true, false);
    std::printf("%s (%d failures)\n", failures ? "SHIM PARITY FAILED" : "SHIM PARITY OK", failures);
    return failures ? 1 : 0;
  }
  // Uniform FV: lax_liu_6 (MR preset AUSM+/van Albada/RK2), ellipsoid3d.
  {
    const CaseSpec& s = find_case("lax_liu_6");
    const SchemeConfig sc = SchemeConfig::mr_preset();
    const int L = 7;
    const long n = s.steps_for_level(L);
    UniformRunResult r = run_uniform(s, L, n, sc);
    UniformRunResult g = gpu::run_uniform(s, L, n, sc);
    report("run_uniform lax_liu_6 L=7 state", same_grid(r.grid, g.grid));
    report("run_uniform lax_liu_6 L=7 max_cfl", r.report.max_cfl == g.report.max_cfl);
  }
  {
    const CaseSpec& s = find_case("ellipsoid3d");
    const SchemeConfig sc = SchemeConfig::mr_preset();
    const int L = 4;
    const long n = s.steps_for_level(L);
    UniformRunResult r = run_uniform(s, L, n, sc);
    UniformRunResult g = gpu::run_uniform(s, L, n, sc);
    report("run_uniform ellipsoid3d L=4 state", same_grid(r.grid, g.grid));
    report("run_uniform ellipsoid3d L=4 max_cfl", r.report.max_cfl == g.report.max_cfl);
  }
  // step_block with the reference's refill = fill_ghosts(bc)
  {
    const CaseSpec& s = find_case("lax_liu_6");
    UniformGrid a(2, 6, s.origin, s.extent);
    init_case(s, a);
    UniformGrid b = a;
    const SchemeConfig sc = SchemeConfig::mr_preset();
    fill_ghosts(a.block(), s.bc);
    const StepDiag d1 = step_block(a.block(), a.dx(), 1e-3, sc, s.gas,
                                   [&](BlockData& blk) { fill_ghosts(blk, s.bc); });
    const StepDiag d2 = gpu::step_block(b.block(), b, 1e-3, sc, s.gas, s.bc);
    report("step_block lax_liu_6 L=6 state", same_grid(a, b));
    report("step_block StepDiag", d1.max_wave_speed == d2.max_wave_speed &&
                                      d1.fallbacks == d2.fallbacks);
  }
  // MR and MRLT on lax_liu_6 with its own epsilon and step schedule
  for (int lt = 0; lt <= 1; ++lt) {
    const CaseSpec& s = find_case("lax_liu_6");
    const SchemeConfig sc = SchemeConfig::mr_preset();
    const int L = 6;
    const long n = s.steps_for_level(L);
    MROptions o;
    o.epsilon = s.mr_epsilon;
    o.local_time = lt == 1;
    MRRunResult r = run_mr(s, L, n, sc, o);
    gpu::MRDeviceResult g = gpu::run_mr(s, L, n, sc, o);
    const std::string tag = lt ? "run_mr (MRLT) lax_liu_6 L=6" : "run_mr lax_liu_6 L=6";
    report(tag + " leaves", r.tree.leaves() == g.leaves);
    report(tag + " to_uniform state", same_grid(r.tree.to_uniform(L), g.grid));
    report(tag + " leaves_per_step", r.report.leaves_per_step == g.report.leaves_per_step);
    report(tag + " cells_per_step", r.report.cells_per_step == g.report.cells_per_step);
    report(tag + " max_cfl", r.report.max_cfl == g.report.max_cfl);
  }
  {
    const CaseSpec& s = find_case("ellipsoid3d");
    const SchemeConfig sc = SchemeConfig::mr_preset();
    const int L = 4;
    const long n = s.steps_for_level(L);
    MROptions o;
    o.epsilon = s.mr_epsilon;
    MRRunResult r = run_mr(s, L, n, sc, o);
    gpu::MRDeviceResult g = gpu::run_mr(s, L, n, sc, o);
    report("run_mr ellipsoid3d L=4 leaves", r.tree.leaves() == g.leaves);
    report("run_mr ellipsoid3d L=4 state", same_grid(r.tree.to_uniform(L), g.grid));
  }
  // step_block twice on one geometry: one cached device context, each call
  // bit-identical to the reference's step_block
  {
    const CaseSpec& s = find_case("lax_liu_6");
    UniformGrid a(2, 6, s.origin, s.extent);
    init_case(s, a);
    UniformGrid b = a;
    const SchemeConfig sc = SchemeConfig::mr_preset();
    const long c0 = gpu::step_block_cache().creations;
    for (int it = 0; it < 2; ++it) {
      fill_ghosts(a.block(), s.bc);
      step_block(a.block(), a.dx(), 1e-3, sc, s.gas,
                 [&](BlockData& blk) { fill_ghosts(blk, s.bc); });
      gpu::step_block(b.block(), b, 1e-3, sc, s.gas, s.bc);
    }
    report("step_block x2 state", same_grid(a, b));
    report("step_block x2 reuses one device context",
           gpu::step_block_cache().creations - c0 <= 1);
  }
  // rk2_stage with FluxField capture (the AMR refluxing seam), 2D and 3D:
  // the explicit midpoint's two stages through the shim against the
  // reference's rk2_stage, states and every captured face flux
  for (const char* name : {"lax_liu_6", "ellipsoid3d"}) {
    const CaseSpec& s = find_case(name);
    const int L = s.dim == 3 ? 4 : 6;
    UniformGrid u(s.dim, L, s.origin, s.extent);
    init_case(s, u);
    UniformGrid m_ref = u, o_ref = u, m_gpu = u, o_gpu = u;
    const SchemeConfig sc = SchemeConfig::mr_preset();
    const int n = 1 << L;
    const std::array<int, 3> cells = {n, n, s.dim == 3 ? n : 1};
    FluxField fr1(s.dim, cells), fr2(s.dim, cells), fg1, fg2;
    fill_ghosts(u.block(), s.bc);
    rk2_stage(u.block(), u.block(), m_ref.block(), u.dx(), 5e-4, sc, s.gas, &fr1);
    fill_ghosts(m_ref.block(), s.bc);
    rk2_stage(u.block(), m_ref.block(), o_ref.block(), u.dx(), 1e-3, sc, s.gas, &fr2);
    gpu::rk2_stage(u.block(), u.block(), m_gpu.block(), u, 5e-4, sc, s.gas, s.bc, &fg1);
    gpu::rk2_stage(u.block(), m_gpu.block(), o_gpu.block(), u, 1e-3, sc, s.gas, s.bc, &fg2);
    bool same_flux = fg1.dim() == s.dim && fg2.dim() == s.dim;
    for (int a = 0; a < s.dim && same_flux; ++a) {
      std::array<int, 3> fn = cells;
      fn[a] += 1;
      for (int k = 0; k < fn[2]; ++k)
        for (int j = 0; j < fn[1]; ++j)
          for (int i = 0; i < fn[0]; ++i)
            for (const auto* pr : {&fr1, &fr2}) {
              const FluxField& g = pr == &fr1 ? fg1 : fg2;
              const FluxVector& x = pr->face(a, i, j, k);
              const FluxVector& y = g.face(a, i, j, k);
              same_flux = same_flux && x.rho == y.rho && x.mom[0] == y.mom[0] &&
                          x.mom[1] == y.mom[1] && x.mom[2] == y.mom[2] && x.rhoE == y.rhoE;
            }
    }
    report(std::string("rk2_stage ") + name + " states", same_grid(m_ref, m_gpu) && same_grid(o_ref, o_gpu));
    report(std::string("rk2_stage ") + name + " FluxField capture", same_flux);
  }
  // MROptions::on_sample (mr_solver.cpp:394): the reference's observer gets
  // a host MRTree the device run cannot provide -> ConfigError, loudly; the
  // device observer gets the same leaf sets at the same points.
  for (int lt = 0; lt <= 1; ++lt) {
    const CaseSpec& s = find_case("lax_liu_6");
    const SchemeConfig sc = SchemeConfig::mr_preset();
    const int L = 6;
    const long n = s.steps_for_level(L);
    std::vector<std::pair<long, std::vector<NodeKey>>> ref_samples, dev_samples;
    std::vector<std::string> ref_mesh, dev_mesh;
    MROptions o;
    o.epsilon = s.mr_epsilon;
    o.local_time = lt == 1;
    o.on_sample = [&](long steps, const MRTree& tree) {
      ref_samples.emplace_back(steps, tree.leaves());
      std::ostringstream os;
      os.precision(12);
      for (NodeKey k : tree.leaves()) {  // driver.cpp:47-60 dump_tree_mesh text
        const NodeId id = unpack_key(k);
        const double h = tree.dx(id.level);
        os << id.level;
        for (int a = 0; a < tree.dim(); ++a) os << ' ' << tree.origin() + id.idx[a] * h;
        for (int a = 0; a < tree.dim(); ++a) os << ' ' << tree.origin() + (id.idx[a] + 1) * h;
        os << '\n';
      }
      ref_mesh.push_back(os.str());
    };
    MRRunResult r = run_mr(s, L, n, sc, o);
    bool threw = false;
    try {
      gpu::run_mr(s, L, n, sc, o);
    } catch (const ConfigError&) {
      threw = true;
    }
    const std::string tag = lt ? "run_mr (MRLT) sampled" : "run_mr sampled";
    report(tag + ": MROptions::on_sample raises ConfigError", threw);
    MROptions od = o;
    od.on_sample = nullptr;
    gpu::MRDeviceResult g = gpu::run_mr(s, L, n, sc, od, nullptr,
                                        [&](long steps, gpu::MRDevice& tree) {
                                          dev_samples.emplace_back(steps, tree.leaves());
                                          dev_mesh.push_back(gpu::tree_mesh_text(tree));
                                        });
    report(tag + ": sample points and leaf sets", ref_samples == dev_samples);
    report(tag + ": mesh dump text", ref_mesh == dev_mesh);
    report(tag + ": final state", same_grid(r.tree.to_uniform(L), g.grid));
    report(tag + ": leaves_per_step", r.report.leaves_per_step == g.report.leaves_per_step);
    report(tag + ": cells_per_step", r.report.cells_per_step == g.report.cells_per_step);
    report(tag + ": max_cfl", r.report.max_cfl == g.report.max_cfl);
    report(tag + ": fallbacks", r.report.fallbacks == g.report.fallbacks);
  }
  // MRTree::refine(eps, buffer_radius_per_level) (mr_tree.hpp:141)
  for (int variant = 0; variant < 3; ++variant) {
    const CaseSpec& s = find_case("lax_liu_6");
    const SchemeConfig sc = SchemeConfig::mr_preset();
    const int L = 7;
    UniformGrid init(2, L, s.origin, s.extent);
    init_case(s, init);
    const double eps = s.mr_epsilon * (variant == 2 ? 0.5 : 1.0);
    const std::vector<int> buffer =
        variant == 0 ? std::vector<int>(L + 1, 1)
                     : (variant == 1 ? std::vector<int>{0, 0, 1, 1, 2, 2, 3} : std::vector<int>{});
    MRTree tree = MRTree::from_uniform(init, 0.0, s.bc);
    tree.coarsen(s.mr_epsilon);
    tree.refine(eps, buffer);
    af_mr_options o{};
    o.eps = s.mr_epsilon;
    o.lt_gap = 3;
    gpu::MRDevice dev(2, L, s.origin, s.extent, s.gas, s.bc, sc, o);
    dev.build(init);
    dev.refine(eps, buffer);
    const std::string tag = "MRTree::refine(eps, buffer) variant " + std::to_string(variant);
    report(tag + " leaves", tree.leaves() == dev.leaves());
    report(tag + " to_uniform", same_grid(tree.to_uniform(L), dev.to_uniform(L)));
  }
  // reference_solution (cases.hpp:58-59): computed on the device on a miss,
  // the cache interchangeable with the reference's, CacheCorrupt on a mismatch
  {
    const CaseSpec& s = find_case("lax_liu_6");
    const SchemeConfig sc = SchemeConfig::mr_preset();
    const int L = 7;
    const std::string dref = "/tmp/af_shim_cache_ref", ddev = "/tmp/af_shim_cache_dev";
    std::filesystem::remove_all(dref);
    std::filesystem::remove_all(ddev);
    const UniformGrid a = reference_solution(s, L, sc, dref);
    const UniformGrid b = gpu::reference_solution(s, L, sc, ddev);
    report("reference_solution lax_liu_6 L=7 (device miss path)", same_grid(a, b));
    const std::string pa = reference_cache_path(s, L, sc, dref), pb = reference_cache_path(s, L, sc, ddev);
    report("reference_solution: meta key text identical",
           read_text_file(pa + ".meta") == read_text_file(pb + ".meta"));
    // each side reads the other's cache
    report("reference_solution: the reference accepts the device cache",
           same_grid(reference_solution(s, L, sc, ddev), a));
    report("reference_solution: the device shim accepts the reference cache",
           same_grid(gpu::reference_solution(s, L, sc, dref), a));
    bool corrupt = false;
    try {
      gpu::reference_solution(s, L, SchemeConfig::amr_preset(), dref + "/../af_shim_cache_ref");
      // same directory, another scheme with another flux name: a fresh file, no throw
      write_text_file(pa + ".meta", "hash=0\nstale\n");
      gpu::reference_solution(s, L, sc, dref);
    } catch (const CacheCorrupt&) {
      corrupt = true;
    }
    report("reference_solution: CacheCorrupt on a stale key", corrupt);
    std::filesystem::remove_all(dref);
    std::filesystem::remove_all(ddev);
  }
  for (int variant = 0; variant < 4; ++variant)
    amr_case(variant == 3 ? "ellipsoid3d" : "lax_liu_6", variant == 3 ? 5 : 8, variant != 1,
             variant == 2);
  std::printf("%s (%d failures)\n", failures ? "SHIM PARITY FAILED" : "SHIM PARITY OK", failures);
  return failures ? 1 : 0;
}
