// af_amr.h — the AMR patch path of libafgpu (host side, not part of the ABI).
//
// PatchHierarchy (amr.hpp:123-242) on the device: a level is a dense field
// over its index space plus a patch-id map (af_amr_kernels.cuh). The box
// lists, level times and the Berger-Rigoutsos clustering live on the host;
// everything that touches a cell value runs in a kernel.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "af_internal.h"

namespace af {

struct ABox {  // Box (amr.hpp:19-66): half-open [lo, hi), z = [0,1) in 2D
  int lo[3] = {0, 0, 0};
  int hi[3] = {0, 0, 1};
  long volume() const {
    if (hi[0] <= lo[0] || hi[1] <= lo[1] || hi[2] <= lo[2]) return 0;
    return (long)(hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
  }
  int extent(int a) const { return hi[a] - lo[a]; }
};

// cluster (amr.hpp:110-111, amr_cluster.cpp:79-232): signature-based
// recursive bisection of the set cells of `flags` (n0 x n1 x n2, x fastest)
// into disjoint boxes of fill ratio >= efficiency that stay inside `allowed`
// (nullable), sorted by (z, y, x) corner. Integer work on a mask that is
// already on the host for the box lists; runs on the host.
std::vector<ABox> amr_cluster(const uint8_t* flags, const uint8_t* allowed, int dim, int n0, int n1,
                              int n2, double efficiency);

// The same clustering with the masks staying on the device (summed-area
// tables + breadth-first bisection, af_amr_kernels.cuh); only the box list
// comes back. d_flags/d_allowed: device masks of an n x n (x n) level.
class DeviceCluster {
 public:
  explicit DeviceCluster(cudaStream_t stream) : stream_(stream) {}
  ~DeviceCluster();
  DeviceCluster(const DeviceCluster&) = delete;
  DeviceCluster& operator=(const DeviceCluster&) = delete;
  std::vector<ABox> run(int dim, const uint8_t* d_flags, const uint8_t* d_allowed, int n,
                        double efficiency, long* launches);

 private:
  cudaStream_t stream_;
  long sat_cap_ = 0;
  int *Sf_ = nullptr, *Sa_ = nullptr;
  void *qa_ = nullptr, *qb_ = nullptr, *out_ = nullptr;
  void* h_pin_ = nullptr;  // pinned readback buffer
  int* hdr_ = nullptr;  // [0] accepted boxes, [1] overflow, [2 + level] frontier sizes
  int cap_ = 0;
};

typedef void (*amr_ic_fn)(double x, double y, double z, double* q5, void* user);

class Amr {
 public:
  Amr(const af_config& cfg, const af_amr_options& opt);
  ~Amr();
  Amr(const Amr&) = delete;
  Amr& operator=(const Amr&) = delete;

  int n_levels() const { return (int)lv_.size(); }
  int cells_per_axis(int l) const { return 1 << (base_exp_ + l); }
  double dx(int l) const { return cfg_.extent / cells_per_axis(l); }
  const std::vector<ABox>& boxes(int l) const { return lv_[l].boxes; }
  double time(int l) const { return lv_[l].t; }
  double time_old(int l) const { return lv_[l].t_old; }

  void initialize(amr_ic_fn ic, void* user);
  void sync_ghosts(int l, double tau);
  void remesh(int l);
  af_step_diag update_level(int l, double dt);  // synchronises
  void average_down(int l);
  void flux_correct(int l);
  void total_conserved(double out5[5]);
  // l1_error_amr (amr.hpp:244-245): reference = a uniform solution at ref_level (AoS)
  void l1_error(int ref_level, const double* ref_aos, double out5[5]);
  long total_cells() const;
  long composite_cells() const;
  bool properly_nested();
  std::string dump_boxes() const;
  void assemble_level(int l, double* aos);
  // every patch of level l, box after box, AoS; ghost = 0 interiors, 2 the
  // blocks with their ghost layers as the patch sees them; old: data_old
  void patch_data(int l, int ghost, int old, double* aos);
  long patch_data_cells(int l, int ghost) const;

  // run_amr's cycle loop (amr_solver.cpp:24-133) for n_steps finest steps of
  // size dt_finest; cells/leaves_per_step (capacity n_steps) may be null
  void run(long n_steps, double dt_finest, long* cells_per_step, long* leaves_per_step,
           af_run_diag* diag);
  long kernel_launches() const { return launches_; }
  long cell_updates() const { return cell_updates_; }  // patch cells x stages, every update_level
  double remesh_seconds() const { return remesh_seconds_; }  // host time inside remesh()
  long remesh_calls() const { return remesh_calls_; }
  // CUDA events around the stepping kernels of every update_level (primitives,
  // predictor, faces, update; the RK2 midpoint sync included)
  void set_profile(bool on) { profile_ = on; }
  void stage_stats(double* ms, long* launches, long* updates) {
    check();
    if (ms) *ms = stage_ms_;
    if (launches) *launches = stage_launches_;
    if (updates) *updates = stage_updates_;
  }
  const af_error& last_error() const { return err_; }
  af_error& error_slot() { return err_; }

 private:
  struct Level {
    std::vector<ABox> boxes;
    double t = 0.0, t_old = 0.0;
    int n = 0;
    long cells = 0;
    int *pid = nullptr, *pid_new = nullptr;
    double *U = nullptr, *Uold = nullptr, *G = nullptr, *Gold = nullptr;
    int* d_boxes = nullptr;
    long* d_off = nullptr;  // four prefix arrays: interiors, shells, blocks, faces per (box, axis)
    int box_cap = 0;
    long total = 0;  // cells of the boxes
    long tot1 = 0, tot2 = 0, totF = 0;
    // flux registers of the pair (this level, next finer)
    int* regbase = nullptr;
    uint8_t* regmask = nullptr;
    int nslots = 0, slot_cap = 0;
    long* slot_cell = nullptr;
    uint8_t *slot_face = nullptr, *has = nullptr;
    double *Rc = nullptr, *Rf = nullptr;
  };
  struct Call {  // one asynchronous update_level
    int level;
    double dt;
  };

  template <int D> void sync_t(int l, double tau);
  template <int D> void remesh_t(int l);
  template <int D, int S> void update_t(int l, double dt);
  template <int D> void rebuild_domain_t(int l, bool into_new);
  template <int D>
  std::vector<ABox> cluster_device(const uint8_t* d_flags, const uint8_t* d_allowed, int n, double eff) {
    return clusterer_->run(D, d_flags, d_allowed, n, eff, &launches_);
  }
  void update_async(int l, double dt);
  void alloc_level(Level& L, int l);
  void free_level(Level& L);
  void upload_boxes(Level& L);
  void ensure_scratch(long cells, int n);
  void save_level(int l, bool restore);  // data_old = data (or the ghosts back from data_old)
  void rebuild_registers(int l);
  void clear_registers(int l);
  void check();            // synchronise, fold the records, throw a pending error
  void fold_records();
  void advance(int l, double dt, std::vector<long>* cps, std::vector<long>* lps);
  [[noreturn]] void raise_nonphysical(int tag);
  void launch_count(int k = 1) { launches_ += k; }

  af_config cfg_;
  af_amr_options opt_;
  int base_exp_;
  int dim_;
  std::vector<Level> lv_;
  std::vector<Level> spare_;  // allocations of popped levels, by index
  cudaStream_t stream_ = nullptr;
  int* d_err_ = nullptr;      // [0] code, [1] cell / tag
  int* d_flag_ = nullptr;     // any / bad / counters
  void* d_rec_ = nullptr;     // ARec[kRecCap]
  std::vector<Call> calls_;
  // folded diagnostics
  double wave_max_ = 0.0, cfl_max_ = 0.0;
  long fallbacks_ = 0;
  af_step_diag last_diag_{};
  // scratch sized for the largest level in use
  long scr_cells_ = 0;
  double *W_ = nullptr, *DU_ = nullptr, *F_ = nullptr;
  uint8_t *m_flags_ = nullptr, *m_tmp_ = nullptr, *m_nest_ = nullptr, *m_allowed_ = nullptr,
          *m_masked_ = nullptr;
  DeviceCluster* clusterer_ = nullptr;
  int* d_cb_ = nullptr;  // nest boxes of remesh
  long* d_cboff_ = nullptr;
  long cb_cap_ = 0;
  long launches_ = 0;
  long cell_updates_ = 0;
  double remesh_seconds_ = 0.0, cluster_seconds_ = 0.0;
  long remesh_calls_ = 0;
  bool profile_ = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events_;
  double stage_ms_ = 0.0;
  long stage_launches_ = 0, stage_updates_ = 0;
  af_error err_{};
  std::string prefix_;  // "cycle N: " while run() is stepping
};

}  // namespace af
