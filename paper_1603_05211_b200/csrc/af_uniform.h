// af_uniform.h — host class behind af_uniform_* (see af_uniform.cu).
#pragma once

#include <cuda.h>

#include "af_comm.h"
#include <vector>

#include "af_internal.h"

namespace af {

struct StageArgs;
struct UGrid;

// Tolerance-mode 3D stage kernels, compiled with FMA contraction in their own
// translation unit (af_fv3d_tol.cu).
void fv3d_tol_setup();
void fv3d_tol_launch(int scheme, dim3 grid, cudaStream_t stream, const StageArgs& a,
                     const UGrid& g, const CUtensorMap& tm, const CUtensorMap& tb);

// the slab [z0, z0+nz) of rank `rank` among n_ranks (af_uniform.cu); host arithmetic only
bool slab_extent(int dim, int level, int n_ranks, int rank, int* z0, int* nz);

class Uniform {
 public:
  Uniform(const af_config& cfg, Comm* comm);
  ~Uniform();
  Uniform(const Uniform&) = delete;
  Uniform& operator=(const Uniform&) = delete;

  void set_stream(cudaStream_t s);
  void set_numerics(int numerics);
  void upload(const double* aos);
  void download(double* aos);
  void step(double dt, af_step_diag* diag);
  // rk2_stage (step.hpp:62-64) on AoS states (host or device); optional
  // FluxField capture (step.hpp:16-50). Overwrites the solver's buffers.
  void rk2_stage(const double* base, const double* eval, double* out, double stage_dt,
                 double* capture, af_step_diag* diag);
  void run(long n_steps, double cfl, double fixed_dt, double* dt_hist, af_run_diag* diag);
  double speed_sum();
  void sync();
  // Lockstep run of a locally emulated slab decomposition (all ranks on one
  // GPU and one stream; halos move by device-to-device copies, the CFL
  // reduction by a max over the ranks' records). Exercises exactly the
  // per-rank code of the NCCL path except the transport itself.
  static void run_group(const std::vector<Uniform*>& ranks, long n_steps, double cfl,
                        double fixed_dt, double* dt_hist, af_run_diag* diag);

  const UGrid& grid() const { return g_; }
  long launches() const { return launches_; }
  const af_error& last_error() const { return last_; }
  af_error& last_error() { return last_; }

 private:
  void reset_error_();
  void free_records_();
  void ensure_records_(long n);
  void ensure_staging_();
  void exchange_halos_(double* q, cudaStream_t st = nullptr);
  void allreduce_max_(unsigned long long* bits);
  void launch_stage_(const StageArgs& a, int zbeg = -1, int zend = -1);
  bool launch_tile3d_(const StageArgs& a, int zbeg, int zend);
  void stage3d_overlapped_(const StageArgs& a, double* eval);
  const CUtensorMap* tensor_map_(const double* buf, bool own = false);
  void launch_hancock_(const StageArgs& a);
  void launch_speed_sum_(const double* q, unsigned long long* target);
  void launch_flux_capture_(const double* q, double* dst);
  void enqueue_steps_(long n_steps, double cfl, double fixed_dt);
  void check_error_();
  void upload_to_(const double* aos, double* dst);
  void download_from_(const double* src, double* aos);
  void collect_(long n_steps, double* dt_hist, af_run_diag* rd, af_step_diag* sd);

  af_config cfg_;
  Comm* comm_;
  UGrid g_{};
  double dx_ = 0.0, inv_dx_ = 0.0;
  double* d_u_ = nullptr;
  double* d_mid_ = nullptr;
  const double* hk_u0_ = nullptr;  // MUSCL-Hancock: the input buffer of even steps
  const double* hk_m0_ = nullptr;  // ... and of odd steps
  double* d_stage_ = nullptr;
  double* d_cap_ = nullptr;        // FluxField capture staging (rk2_stage)
  long cap_cap_ = 0;
  const double* err_eval_ = nullptr;  // rk2_stage: the stage's eval buffer for the error scan
  bool seam_msg_ = false;             // rk2_stage: the reference's message has no step prefix
  size_t stage_bytes_ = 0;
  int* d_err_ = nullptr;
  RunRecords rec_{};
  long rec_cap_ = 0;
  cudaStream_t stream_ = nullptr;
  cudaStream_t own_stream_ = nullptr;
  long launches_ = 0;
  af_error last_{};
  int numerics_ = AF_NUMERICS_EXACT;
  int tile_slots_ = 296;      // resident fv3d_tile CTAs on the device
  bool tile_exact_ = true;   // AF_FV3D_TILE=0: exact mode on the legacy fv3d_stage
  CUtensorMap tm_[2];      // TMA descriptors of d_u_ / d_mid_ (4D: x, y, component, plane)
  CUtensorMap tmo_[2];     // the same buffers with the owned-tile box (base values)
  const double* tm_base_[2] = {nullptr, nullptr};
  // halo exchange overlapped with the interior planes (3D, NCCL ranks)
  cudaStream_t comm_stream_ = nullptr;
  cudaEvent_t ev_ready_ = nullptr, ev_halo_ = nullptr;
  bool overlap_ = false;
};

}  // namespace af
