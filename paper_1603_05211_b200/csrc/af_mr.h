// af_mr.h — host class behind af_mr_* (see af_mr.cu).
#pragma once

#include <string>
#include <vector>

#include "af_comm.h"
#include "af_internal.h"
#include "af_mr_types.h"

namespace af {

struct MRStageArgs;

// Tolerance-mode full-tile stage kernels (af_mr_full_tol.cu, FMA contraction).
void mr_full_tol_setup();
void mr_full_tol_launch(int scheme, dim3 grid, cudaStream_t stream, bool pdl,
                        const MRStageArgs& a, const MRLevels& g, int lcode);

// One contiguous run of whole rows in a halo exchange (af_mr_dist.cu).
struct MR_XSeg {
  long cell;   // first cell (concatenated level index)
  long cells;  // contiguous cells
  long pos;    // offset in the peer's packed section
};

class MR {
 public:
  // AF_NUMERICS_EXACT (bit-identical) / AF_NUMERICS_TOLERANCE (the full-tile
  // 2D stage kernel with the tolerance physics; 1e-10 relative L1)
  void set_numerics(int numerics);
  // comm: null or one rank for a single GPU; otherwise this rank's slab of
  // the spatial decomposition.
  MR(const af_config& cfg, const af_mr_options& opt, Comm* comm = nullptr);
  void local_rows(int level, int* lo, int* hi) const;  // slab rows this rank owns
  std::string dump();  // MRTree::dump text (af_io.cu)
  ~MR();
  MR(const MR&) = delete;
  MR& operator=(const MR&) = delete;

  void set_stream(cudaStream_t s);
  // MRTree::from_uniform + set_min_leaf_level + coarsen(eps) (mr_solver.cpp:406-410)
  void build(const double* aos);
  void refine(int top);              // MRTree::refine (+ LT buffer when top >= 0)
  void refine(double eps, const int* buffer, int n);  // MRTree::refine(eps, buffer)
  void add_virtual_leaves();         // marks the virtual set (and counts it)
  void evolve_global(double dt, af_step_diag* d);
  void advance_local(int top, double t, double dt, af_step_diag* d);
  void coarsen();                    // MRTree::coarsen
  void remove_virtual_leaves();
  void run(long n_steps, double cfl, double fixed_dt, af_mr_cycle* cycles, long max_cycles,
           af_run_diag* rd);
  void counts(long* leaves, long* nodes, long* internals);
  int coarsest_leaf_level();
  long leaf_keys(uint64_t* keys, long cap);
  void to_uniform(int level, double* aos);
  void details(int level, double* out);
  double leaf_speed_sum();
  double max_cfl() const { return max_cfl_; }  // MRSolver::max_cfl (mr_solver.hpp)
  long fallbacks() const { return fallbacks_; }

  long launches() const { return launches_; }
  // device bytes of the per-cell arrays: now, peak, and as dense level grids
  void memory(unsigned long long* now, unsigned long long* peak, unsigned long long* dense) const;
  void profile(bool on);
  void stage_stats(double* ms, long* launches, long* updates);
  af_error& last_error() { return last_; }

 private:
  void refine_(const std::vector<int>& radius, const double* eps);
  void predict_fill_(int lo, int hi, int from = 1);
  void project_range_(int lo, int top);
  void build_lists_();
  bool ml_grid_(int lo, int hi, bool leaf, dim3* grid, int mult = 1, int cap = 148 * 8) const;
  int level_tiles_(int l) const { return g_.ntx[l] * g_.nty[l] * g_.ntz[l]; }
  void cycle_stats_(long* leaves, long* nodes, double* smax);
  int pre_() const;
  int coarsen_pre_(int l) const;  // kPreV for a sweep's levels below the finest       // prefetch permissions of the next launch (kPreList | kPreSt)
  long v_only_at_ = -1;   // launches_ right after a launch that writes only values
  int small_hi_ = 0;
  bool pdl_ = true;             // programmatic dependent launches (AF_MR_NO_PDL turns off)
  bool full_sweeps_ = false;    // AF_MR_FULL_SWEEPS: never skip a coarsen sweep; check the skip test
  void stage_(int lo, int hi, double tau, double sdt, int stage, long step);
  void step_levels_(int lo, int hi, double t, double dt, int sub);
  void build_registers_(int top);
  void check_error_(long step);
  void collect_stage_records_(af_step_diag* d);
  void apply_registers_(int coarse_level);
  struct StageRec {
    int slot;
    double step_dt;
    int lo, hi;
  };
  std::vector<StageRec> stage_records_;
  // CUDA graph of the global-time-step evolve (parameters are cycle-invariant:
  // counts, dt and the step index live in device memory)
  bool fixed_grids_ = false;
  double* d_dt_ = nullptr;
  int* d_step3_ = nullptr;
  double* h_dt_step_ = nullptr;
  cudaGraphExec_t graph_exec_ = nullptr;
  size_t graph_records_ = 0;
  long graph_launches_ = 0, graph_stage_launches_ = 0, graph_stage_updates_ = 0;
  std::vector<StageRec> graph_recs_;
  size_t graph_events_ = 0;
  void evolve_global_graph_(double dt);
  struct GraphCache {
    cudaGraphExec_t exec = nullptr;
    std::vector<StageRec> recs;
    long launches = 0;
    size_t events = 0;
  };
  GraphCache graphs_[2];
  // Whole-cycle graph of a global-time-step run (run_batch_graph_): refine
  // with the gradedness fixpoint and coarsen with its sweep loop as WHILE
  // conditional nodes, CFL dt and cycle records on the device. One launch per
  // cycle, one host synchronisation per batch of cycles.
  struct CycleGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    double cfl = -1.0, fixed_dt = -1.0;
    std::vector<cudaGraphNode_t> ev_nodes;  // event-record nodes, in capture order
    long launches_fixed = 0;                // kernels outside the WHILE bodies
    long grade_body = 0, sweep_body = 0;    // kernels per WHILE iteration
  };
  CycleGraph cyc_[2];
  cudaStream_t side_stream_ = nullptr;
  cudaStream_t fork_stream_ = nullptr;
  bool swap_ = false;
  // AF_MR_PHASES: event marks between the phases of the captured cycle graph
  // (one cycle per batch), averaged and printed at destruction
  void phase_(const char* name);
  bool phases_ = false;
  std::vector<std::pair<const char*, cudaEvent_t>> phase_ev_;
  std::vector<double> phase_ms_;
  long phase_n_ = 0;
  bool cycle_capture_ = false;              // capturing the whole-cycle graph (swap allowed)                       // stage_: output buffer becomes the state (no commit copy)      // cycle graph: work beside the prediction refresh
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  cudaEvent_t ev_aux_[4] = {nullptr, nullptr, nullptr, nullptr};  // cycle_end / re-sweep decision forks
  bool in_body_ = false;                    // capturing a WHILE body
  double* d_ckV_ = nullptr;                 // batch checkpoint (replay on failure)
  uint8_t* d_ckSt_ = nullptr;
  af_mr_cycle* d_cycrec_ = nullptr;
  af_mr_cycle* h_cycrec_ = nullptr;
  long long* d_cycctl_ = nullptr;           // [0] step index, [1] record slot
  unsigned long long* d_acc_ = nullptr;     // max_cfl, max wave, fallbacks, grade/sweep iterations
  unsigned long long* h_small_ = nullptr;   // pinned staging
  template <class F>
  void capture_while_(F&& body, cudaGraphConditionalHandle h = 0, bool have_h = false);
  cudaGraphConditionalHandle make_cond_(unsigned def);
  void build_lists_enqueue_();
  void note_event_node_();
  std::vector<cudaGraphNode_t> ev_nodes_;  // event-record nodes of the capture in progress
  void enqueue_cycle_(double cfl, double fixed_dt, long* grade_body, long* sweep_body);
  CycleGraph& cycle_graph_(double cfl, double fixed_dt);
  void invalidate_graphs_();
  bool run_batch_graph_(long B, double cfl, double fixed_dt, long& done, long& cycle, double& t,
                        af_mr_cycle* cycles, long max_cycles);
  void cycle_sync_(long n_steps, double cfl, double fixed_dt, long& done, long& cycle, double& t,
                   af_mr_cycle* cycles, long max_cycles);
  // ---- spatial decomposition (af_mr_dist.cu) ----
  Comm* comm_ = nullptr;
  int nranks_ = 1, rank_ = 0;
  bool dist_ = false;
  int lp_ = 0;  // partition level: levels >= lp_ are split in slabs of rows
  int halo_ = 2;  // halo rows kept per level
  using XSeg = MR_XSeg;
  struct Peer {
    int rank = 0;
    std::vector<XSeg> send, recv;
    long send_cells = 0, recv_cells = 0;
    XSeg* d_send = nullptr;
    XSeg* d_recv = nullptr;
    uint8_t* sbuf = nullptr;
    uint8_t* rbuf = nullptr;
  };
  std::vector<Peer> peers_;
  unsigned long long* d_xred_ = nullptr;
  enum { XV = 1, XST = 2, XMARK = 4 };
  enum { RED_MAX = 0, RED_SUM = 1, RED_MIN = 2 };
  void part_rows_(int r, int l, int* lo, int* hi) const;
  // Windowed arrays (ranks): each per-cell array reserves its full virtual
  // size but maps physical memory only for every level's window rows (the
  // region plus the tile and stencil overhang); global indexing is unchanged.
  bool windows_ = false;
  std::vector<std::vector<std::pair<long, long>>> win_;  // per level: cell ranges [c0, c1)
  struct WinMap {
    unsigned long long base = 0;
    size_t reserved = 0;
    std::vector<std::pair<unsigned long long, size_t>> maps;  // address, bytes
    std::vector<unsigned long long> handles;
  };
  std::vector<WinMap> wmaps_;
  void win_setup_();
  void* walloc_(size_t elem, int ncomp);
  void wfree_all_();
  void wset_(void* p, size_t elem, int ncomp, int value, int lev_lo, int lev_hi);
  void wtohost_(void* dst, const void* src, size_t elem, int ncomp);
  void dist_setup_();
  void dist_free_();
  void exchange_(int mask);
  void allreduce_(unsigned long long* v, int k, int op);
  // ---- storage of the per-cell arrays (af_mr_storage.cu) ----
  static constexpr int kBrickShift3 = 6;  // 64^3-cell bricks: 2 MiB per value component
  int storage_ = 0;                       // AF_MR_STORAGE_*
  struct SpArr {                          // one sparse value array (VMM)
    unsigned long long base = 0;
    size_t reserved = 0, coarse_bytes = 0;
    int ncomp = 0;
    long mapped = 0;
    std::vector<unsigned long long> coarse;  // per component: the always-mapped coarse block
    std::vector<unsigned long long> bricks;  // [brick * ncomp + c]: its page (0 = unmapped)
  };
  std::vector<SpArr> sp_;
  long sp_nbricks_ = 0;
  size_t sp_brick_bytes_ = 0, sp_now_ = 0, sp_peak_ = 0;
  size_t cell_bytes_ = 0;       // dense per-cell allocations
  size_t cell_elem_bytes_ = 0;  // bytes per cell over all per-cell arrays
  uint8_t* d_need_ = nullptr;
  std::vector<uint8_t> h_need_;
  void storage_setup_(const af_mr_options& o);
  int sp_level_(long gb, long* b) const;
  void* sp_alloc_(int ncomp);
  SpArr* sp_find_(const void* p);
  void sp_map_(SpArr& a, long gb);
  void sp_unmap_(SpArr& a, long gb);
  void sp_map_all_(const void* p);
  void sparse_sync_();
  void sp_free_all_();
  bool sp_set_(void* p, int value, int lev_lo, int lev_hi);
  bool sp_tohost_(void* dst, const void* src);
  void* calloc_(size_t elem, int ncomp, bool sparse);
  double norms_host_[5] = {1, 1, 1, 1, 1};
  double eps_at_(int child_level) const;

  af_config cfg_;
  af_mr_options opt_;
  std::vector<double> eps_level_;
  int D_, L_, NC_;
  MRLevels g_{};
  uint8_t* d_st_ = nullptr;
  uint8_t* d_mark_ = nullptr;    // virtual parents
  uint8_t* d_flag_ = nullptr;
  uint8_t* d_flag2_ = nullptr;
  double* d_V_ = nullptr;        // value_at field
  double* d_Vs_ = nullptr;       // stage output
  double* d_Qold_ = nullptr;     // step-start leaf values
  double* d_VQold_ = nullptr;    // virtual q_old snapshots (LT)
  double* d_det_ = nullptr;
  double* d_norms_ = nullptr;
  int* d_tiles_ = nullptr;       // per-level leaf-tile lists (tile_off_ regions)
  int* d_band_ = nullptr;        // per-level band-tile lists
  int* d_pband_ = nullptr;       // band tiles holding an absent cell (prediction work)
  int* d_lpart_ = nullptr;       // leaf tiles that are not full (mr_stage_kernel)
  int* d_lfull_ = nullptr;       // full leaf tiles (mr_stage_full2d)
  uint8_t* d_tflag_ = nullptr;
  int* d_tleaf_ = nullptr;  // leaves per tile (mr_tile_flags_all -> mr_tile_lists_all)
  int* d_tile_count_ = nullptr;  // [0..16] band counts, [17..33] leaf-tile counts
  unsigned long long* d_lpl_ = nullptr;  // leaves per level
  int* d_err_ = nullptr;
  int* d_flagi_ = nullptr;
  // flux registers (local time stepping)
  int* d_regbase_ = nullptr;
  uint8_t* d_regmask_ = nullptr;
  double* d_regc_ = nullptr;
  double* d_regf_ = nullptr;
  uint8_t* d_regfc_ = nullptr;
  uint8_t* d_regff_ = nullptr;
  int* d_regcount_ = nullptr;
  int* d_regerr_ = nullptr;
  unsigned long long* d_badkey_ = nullptr;
  long reg_cap_ = 0;
  int reg_fine_ = 0;  // fine slots per register: 2 substeps x 2^(d-1) sub-faces
  bool registers_built_ = false;
  unsigned long long* d_red_ = nullptr;  // scratch reductions
  std::vector<long> tile_off_;           // per-level offset into d_tiles_
  std::vector<int> tile_count_;  // leaf tiles per level
  std::vector<int> band_count_;  // band tiles per level
  std::vector<int> pband_count_; // band tiles with an absent cell per level
  std::vector<int> full_count_;  // full leaf tiles per level
  bool pband_ok_ = false;        // statuses unchanged since the lists were built
  int numerics_ = 0;             // AF_NUMERICS_EXACT / AF_NUMERICS_TOLERANCE
  bool fresh_ = false;
  bool coarse_stale_ = false;  // internal values below min_leaf-1 not projected (refresh_coarse_)
  void refresh_coarse_();
  bool lists_valid_ = false;
  double phase_s_[4] = {0, 0, 0, 0};
  double phase_t0_ = 0.0;
  double evolve_gpu_ms_ = 0.0;           // every absent band cell holds its current prediction
  std::vector<long> leaves_per_level_;
  std::vector<double> t_old_, t_new_;
  int min_leaf_ = 0;
  cudaStream_t stream_ = nullptr, own_stream_ = nullptr;
  long launches_ = 0;
  bool virtuals_ = false;
  // per-run accumulators (MRSolver::max_cfl_, fallbacks_)
  double max_cfl_ = 0.0;
  long fallbacks_ = 0;
  double max_wave_ = 0.0;
  long cur_step_ = 0;
  // stage-kernel timing
  bool profile_ = false;
  std::vector<cudaEvent_t> ev_pool_;
  size_t ev_used_ = 0;
  double stage_ms_ = 0.0;
  long stage_launches_ = 0, stage_updates_ = 0;
  void harvest_events_();
  double step_dt_ = 0.0;
  int sub_ = 0;
  af_error last_{};
};

}  // namespace af
