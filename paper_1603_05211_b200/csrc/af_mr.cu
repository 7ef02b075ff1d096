// af_mr.cu — host side of the adaptive MR solver (af_mr_* of af_gpu.h).
//
// Mirrors MRTree (mr_tree.cpp), MRSolver::step_levels (mr_solver.cpp:232-316)
// and the run_mr cycle (mr_solver.cpp:318-400) on per-level dense grids:
//   refine  = details -> split flags [-> LT buffer dilation] -> apply ->
//             gradedness fixpoint (decide-all / apply passes)
//   evolve  = per stage: stage kernels for every stepping level (all reads
//             before any write, as the reference's two-pass stage), commit,
//             project_range (finest first), prediction refresh (top-down)
//   coarsen = finest-first level sweeps repeated until nothing merges
// Host synchronisation happens only where the reference makes a decision
// that depends on data (fixpoint loops, per-cycle counts and errors).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <chrono>
#include <cstdlib>

#include "af_mr.h"
#include "af_mr_full.cuh"
#include "af_mr_stage.cuh"

namespace af {

namespace {

constexpr int kGrid = 148 * 8;
constexpr int kStageGrid = 148 * 2;  // stage kernel: 2 resident blocks per SM
constexpr long kFullMin = 148 * 2 * 4;  // full tiles that justify mr_stage_full2d

inline unsigned grid_for(long n, int block = 256) {
  long b = (n + block - 1) / block;
  return (unsigned)std::max<long>(1, std::min<long>(b, kGrid));
}

// Level-L cells of rows [r0, r1) from a compact AoS holding those rows.
template <int D>
__global__ void mr_upload_finest(const double* __restrict__ aos, double* V, MRLevels g, int r0,
                                 int r1) {
  AF_PDL_ENTRY();
  const long rowlen = D == 3 ? 1L << (2 * g.L) : 1L << g.L;
  const long cells = (long)(r1 - r0) * rowlen, comp = g.total_cells;
  const int n = 1 << g.L;
  for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < cells;
       u += (long)gridDim.x * blockDim.x) {
    const double* q = aos + 5 * u;
    // the uniform array is row-major; the level may be bricked (MRLevels::bsh)
    const long x = u + (long)r0 * rowlen;
    const long off = g.cell_off[g.L],
               c = mr_idx(g, D, n, (int)(x & (n - 1)), (int)((x >> g.L) & (n - 1)),
                          D == 3 ? (int)(x >> (2 * g.L)) : 0);
    V[off + c] = q[0];
    V[comp + off + c] = q[1];
    V[2 * comp + off + c] = q[2];
    if (D == 3) V[3 * comp + off + c] = q[3];
    V[(D + 1) * comp + off + c] = q[4];
  }
}

// Level-l cells of rows [r0, r1) into a compact AoS.
template <int D>
__global__ void mr_download_level(const double* V, double* __restrict__ aos, MRLevels g, int l,
                                  int r0, int r1) {
  AF_PDL_ENTRY();
  const long rowlen = D == 3 ? 1L << (2 * l) : 1L << l;
  const long cells = (long)(r1 - r0) * rowlen, comp = g.total_cells;
  const int n = 1 << l;
  for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < cells;
       u += (long)gridDim.x * blockDim.x) {
    double* q = aos + 5 * u;
    const long x = u + (long)r0 * rowlen;  // row-major output, possibly bricked level
    const long off = g.cell_off[l],
               c = mr_idx(g, D, n, (int)(x & (n - 1)), (int)((x >> l) & (n - 1)),
                          D == 3 ? (int)(x >> (2 * l)) : 0);
    q[0] = V[off + c];
    q[1] = V[comp + off + c];
    q[2] = V[2 * comp + off + c];
    q[3] = D == 3 ? V[3 * comp + off + c] : 0.0;
    q[4] = V[(D + 1) * comp + off + c];
  }
}

// One component of level l in row-major order (details of a bricked level).
template <int D>
__global__ void mr_level_rowmajor(const double* src, double* __restrict__ dst, MRLevels g, int l) {
  AF_PDL_ENTRY();
  const int n = 1 << l;
  const long cells = mr_cells(D, l);
  for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < cells;
       u += (long)gridDim.x * blockDim.x)
    dst[u] = src[g.cell_off[l] + mr_idx(g, D, n, (int)(u & (n - 1)), (int)((u >> l) & (n - 1)),
                                        D == 3 ? (int)(u >> (2 * l)) : 0)];
}

// Virtual q_old snapshot (mr_solver.cpp:251-266): VQold = V at the virtual
// children of the stepping leaves of level l-1.
template <int D>
__global__ void mr_virtual_snapshot(const double* V, double* VQ, const uint8_t* st,
                                    const uint8_t* mark, MRLevels g, int l) {
  AF_PDL_ENTRY();
  const int n = 1 << l, pn = n >> 1;
  const long cells = mr_cells(D, l), off = g.cell_off[l], poff = g.cell_off[l - 1];
  const long comp = g.total_cells;
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < cells;
       c += (long)gridDim.x * blockDim.x) {
    if (g.dist && !row_in_region(g, l, mr_row(g, D, l, c))) continue;  // this rank's rows
    if (st[off + c] != ST_ABSENT) continue;
    int i, j, k;
  mr_ijk(g, D, l, c, i, j, k);
    if (!mark[poff + mr_idx(g, D, pn, i >> 1, j >> 1, k >> 1)]) continue;
    for (int m = 0; m < D + 2; ++m) VQ[m * comp + off + c] = V[m * comp + off + c];
  }
}

// ---- whole-cycle graph helpers (MR::run_batch_graph_) ---------------------
// Re-arms a WHILE conditional node: continue while flags[0] (both == 0) or
// flags[0] && flags[1] (both == 1); clears the flags for the next iteration
// and counts the iteration in iters[0].
__global__ void mr_while_cond(cudaGraphConditionalHandle h, int* flags, int both,
                              unsigned long long* iters) {
  AF_PDL_ENTRY();
  const bool go = both ? (flags[0] != 0 && flags[1] != 0) : flags[0] != 0;
  flags[0] = 0;
  flags[1] = 0;
  ++iters[0];
  cudaGraphSetConditional(h, go ? 1u : 0u);
}

// Device part of the run_mr cycle head (mr_solver.cpp:339-374) for a global
// step: dt from the CFL rule (cfl * dx_L / smax, the host's operation order)
// or the fixed dt; the step index for error records; the cycle record.
// ctl[0] = global step index, ctl[1] = record slot in the batch.
__global__ void mr_cycle_begin(const unsigned long long* red, const unsigned long long* lpl,
                               int L, int D, double cfl, double fixed_dt, double dx_L,
                               double* dt_out, int* step3, long long* ctl, af_mr_cycle* rec,
                               unsigned long long* srec, int nsrec) {
  AF_PDL_ENTRY();
  for (int i = 0; i < nsrec; ++i) srec[i] = 0;  // this cycle's stage records (stage_)
  const double smax = __longlong_as_double((long long)red[3]);
  double dt = fixed_dt;
  if (cfl > 0.0) dt = cfl * dx_L / smax;
  *dt_out = dt;
  *step3 = (int)(3 * ctl[0]);
  af_mr_cycle r;
  r.leaves = (long)red[0];
  r.nodes = (long)(red[0] + red[1] + (red[2] << D));
  r.sub = 1;
  r.top = L;
  r.dt = dt;
  long upd = 0;
  for (int l = 0; l <= L; ++l) upd += 2 * (long)lpl[l];
  r.updates = upd;
  rec[ctl[1]] = r;
}

// collect_stage_records_ for the two stages of a global step, accumulated on
// the device: acc[0] = max_cfl bits, acc[1] = max wave speed bits,
// acc[2] = fallbacks (std::max order and expressions as on the host).
__global__ void mr_cycle_end(const unsigned long long* srec, const unsigned long long* lpl, int L,
                             double extent, const double* dt_p, unsigned long long* acc,
                             long long* ctl) {
  AF_PDL_ENTRY();
  const double dt = *dt_p;
  double mc = __longlong_as_double((long long)acc[0]);
  double mw = __longlong_as_double((long long)acc[1]);
  double ws = 0.0;
  unsigned long long fbs = 0;
  for (int r = 0; r < 2; ++r) {
    for (int l = 0; l <= L; ++l) {
      if (!lpl[l]) continue;
      const double w = __longlong_as_double((long long)srec[r * 17 + l]);
      const double dx = extent / static_cast<double>(1 << l);
      const double c = w * dt / dx;
      mc = mc < c ? c : mc;
      ws = ws < w ? w : ws;
    }
    fbs += srec[r * 17 + 16];
  }
  mw = mw < ws ? ws : mw;
  acc[0] = (unsigned long long)__double_as_longlong(mc);
  acc[1] = (unsigned long long)__double_as_longlong(mw);
  acc[2] += fbs;
  ++ctl[0];
  ++ctl[1];
}

// Kernel launch with the programmatic-dependent-launch attribute when `pdl`
// (see AF_PDL_ENTRY): the launch overlaps the predecessor's tail.
template <class... P, class... A>
void launch_k(bool pdl, cudaStream_t s, void (*kern)(P...), dim3 grid, unsigned block,
              size_t smem, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  AF_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...));
}

std::string fmt_f(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%f", v);
  return b;
}

double as_d(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}

constexpr int kTX2 = 32, kTY2 = 8;
constexpr int kMaxStageRecords = 2048;
constexpr long kCycBatch = 64;  // cycles per graph batch (one host synchronisation)
constexpr int kTX3 = 8, kTY3 = 8, kTZ3 = 4;

}  // namespace

MR::MR(const af_config& c, const af_mr_options& o, Comm* comm) : cfg_(c), opt_(o) {
  if (c.dim != 2 && c.dim != 3) throw Error(AF_E_CONFIG, "dim must be 2 or 3");
  if (c.level < 2 || c.level > 15) throw Error(AF_E_CONFIG, "level must be in [2, 15]");
  if (c.flux != AF_FLUX_AUSM_PLUS && c.flux != AF_FLUX_AUSMDV)
    throw Error(AF_E_CONFIG, "unknown flux");
  if (c.integrator != AF_INTEGRATOR_RK2)  // MRSolver::stage is RK2 (mr_solver.cpp:284-316)
    throw Error(AF_E_UNSUPPORTED, "the MR path steps with RK2");
  if (c.limiter != AF_LIMITER_MINMOD && c.limiter != AF_LIMITER_VAN_ALBADA)
    throw Error(AF_E_CONFIG, "unknown limiter");
  for (int f = 0; f < 6; ++f)
    if (c.bc[f] < 0 || c.bc[f] > 2) throw Error(AF_E_CONFIG, "unknown boundary condition");
  D_ = c.dim;
  L_ = c.level;
  NC_ = D_ + 2;
  reg_fine_ = 2 * (1 << (D_ - 1));
  if (o.eps_level) eps_level_.assign(o.eps_level, o.eps_level + L_ + 1);
  opt_.eps_level = nullptr;
  AF_CUDA(cudaSetDevice(c.device));
  g_.dim = D_;
  g_.L = L_;
  g_.nc = NC_;
  for (int f = 0; f < 6; ++f) g_.bc[f] = c.bc[f];
  long tot = 0;
  for (int l = 0; l <= L_; ++l) {
    g_.cell_off[l] = tot;
    tot += mr_cells(D_, l);
    const double dx = c.extent / static_cast<double>(1 << l);  // mr_tree.hpp:73
    g_.inv_dx[l] = 1.0 / dx;
  }
  g_.cell_off[L_ + 1] = tot;
  g_.total_cells = tot;
  for (int l = 0; l <= L_; ++l) g_.eps_l[l] = eps_at_(l);
  if (o.local_time) {
    AF_CUDA(cudaMalloc(&d_regcount_, sizeof(int)));
    AF_CUDA(cudaMalloc(&d_regerr_, sizeof(int)));
    AF_CUDA(cudaMalloc(&d_badkey_, sizeof(unsigned long long)));
  }
  AF_CUDA(cudaMalloc(&d_norms_, sizeof(double) * 5));
  AF_CUDA(cudaMalloc(&d_err_, 4 * sizeof(int)));
  AF_CUDA(cudaMalloc(&d_flagi_, 2 * sizeof(int)));
  AF_CUDA(cudaMalloc(&d_red_, sizeof(unsigned long long) * (64 + 17 * kMaxStageRecords)));
  tile_off_.assign(L_ + 2, 0);
  tile_count_.assign(L_ + 1, 0);
  band_count_.assign(L_ + 1, 0);
  pband_count_.assign(L_ + 1, 0);
  full_count_.assign(L_ + 1, 0);
  long toff = 0;
  for (int l = 0; l <= L_; ++l) {
    tile_off_[l] = toff;
    g_.tile_off[l] = toff;
    const int n = 1 << l;
    const int tx = D_ == 2 ? kTX2 : kTX3, ty = D_ == 2 ? kTY2 : kTY3, tz = D_ == 2 ? 1 : kTZ3;
    g_.ntx[l] = (n + tx - 1) / tx;
    g_.nty[l] = (n + ty - 1) / ty;
    g_.ntz[l] = D_ == 3 ? (n + tz - 1) / tz : 1;
    toff += (long)g_.ntx[l] * g_.nty[l] * g_.ntz[l];
  }
  tile_off_[L_ + 1] = toff;
  g_.tile_off[L_ + 1] = toff;
  // the coarsest levels (at most kTinyCells cells) run as one single-CTA
  // launch (mr_*_tiny); with ranks every level is a launch of its own
  small_hi_ = -1;
  if (!std::getenv("AF_MR_NO_TINY"))
    for (int l = 0; l <= L_; ++l)
      if (mr_cells(D_, l) <= kTinyCells) small_hi_ = l;
  full_sweeps_ = std::getenv("AF_MR_FULL_SWEEPS") != nullptr;
  pdl_ = std::getenv("AF_MR_NO_PDL") == nullptr;
  phases_ = std::getenv("AF_MR_PHASES") != nullptr;
  // spatial decomposition: one slab of rows per rank from the partition level
  // lp_ up (levels below are replicated); one rank owns everything
  if (comm && comm->n > 1) {
    if (comm->local && !comm->group)
      throw Error(AF_E_ARGUMENT, "MR ranks of a local group need af_comm_create_local");
    comm_ = comm;
    nranks_ = comm->n;
    rank_ = comm->rank;
    dist_ = true;
    int ml = o.min_leaf_level;
    if (o.local_time) ml = std::max(ml, std::max(0, L_ - o.lt_gap));
    lp_ = 0;
    while ((1 << lp_) < 4 * nranks_ && lp_ < ml) ++lp_;
    if ((1 << lp_) < nranks_)
      throw Error(AF_E_CONFIG, "more ranks than slab rows at the minimum leaf level");
    // halo depth: the stencil reach (2), or the LT refine buffer radius
    // 2^(l-top-1) at l = L-1 with top >= min leaf level (mr_solver.cpp:358-362)
    halo_ = 2;
    if (o.local_time) halo_ = std::max(2, 1 << std::max(0, L_ - ml - 2));
  }
  g_.lp = lp_;
  g_.count_rep = rank_ == 0 ? 1 : 0;
  g_.dist = dist_ ? 1 : 0;
  for (int l = 0; l <= L_; ++l) {
    part_rows_(rank_, l, &g_.own_lo[l], &g_.own_hi[l]);
    const int n = 1 << l;
    int ml = o.min_leaf_level;
    if (o.local_time) ml = std::max(ml, std::max(0, L_ - o.lt_gap));
    if (!dist_ || l < lp_ || (l == lp_ && lp_ == ml)) {
      // replicated levels, and the partition level when leaves can sit there
      // (their parents' details read the whole level): every row
      g_.reg_lo[l] = 0;
      g_.reg_hi[l] = n;
    } else {
      int lo = g_.own_lo[l] - halo_, hi = g_.own_hi[l] + halo_;
      if (c.bc[2 * (D_ - 1)] != AF_BC_PERIODIC) {
        lo = std::max(lo, 0);
        hi = std::min(hi, n);
      } else if (hi - lo >= n) {
        lo = 0;
        hi = n;
      }
      g_.reg_lo[l] = lo;
      g_.reg_hi[l] = hi;
    }
  }
  // cell order and padding of the level arrays (dense / bricks / sparse bricks)
  storage_setup_(o);
  // per-cell arrays: windowed with ranks (AF_MR_NO_WINDOWS maps everything);
  // the value arrays as sparse bricks with AF_MR_STORAGE_SPARSE
  windows_ = dist_ && std::getenv("AF_MR_NO_WINDOWS") == nullptr;
  win_setup_();
  const bool sp = storage_ == AF_MR_STORAGE_SPARSE;
  d_st_ = static_cast<uint8_t*>(calloc_(1, 1, false));
  d_mark_ = static_cast<uint8_t*>(calloc_(1, 1, false));
  d_flag_ = static_cast<uint8_t*>(calloc_(1, 1, false));
  d_flag2_ = static_cast<uint8_t*>(calloc_(1, 1, false));
  d_V_ = static_cast<double*>(calloc_(8, NC_, sp));
  d_Vs_ = static_cast<double*>(calloc_(8, NC_, sp));
  d_Qold_ = static_cast<double*>(calloc_(8, NC_, sp));
  d_det_ = static_cast<double*>(calloc_(8, 1, sp));
  if (o.local_time) {
    d_VQold_ = static_cast<double*>(calloc_(8, NC_, sp));
    d_regbase_ = static_cast<int*>(calloc_(4, 1, false));
    d_regmask_ = static_cast<uint8_t*>(calloc_(1, 1, false));
  }
  {  // stream-ordered scratch allocations keep their memory
    cudaMemPool_t pool;
    AF_CUDA(cudaDeviceGetDefaultMemPool(&pool, c.device));
    unsigned long long keep = ~0ull;
    AF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  AF_CUDA(cudaMalloc(&d_tiles_, sizeof(int) * toff));
  AF_CUDA(cudaMalloc(&d_band_, sizeof(int) * toff));
  AF_CUDA(cudaMalloc(&d_pband_, sizeof(int) * toff));
  AF_CUDA(cudaMalloc(&d_lpart_, sizeof(int) * toff));
  AF_CUDA(cudaMalloc(&d_lfull_, sizeof(int) * toff));
  AF_CUDA(cudaMalloc(&d_tflag_, toff));
  AF_CUDA(cudaMalloc(&d_tleaf_, sizeof(int) * toff));
  AF_CUDA(cudaMalloc(&d_tile_count_, sizeof(int) * 85));
  AF_CUDA(cudaMemset(d_tile_count_, 0, sizeof(int) * 85));
  g_.dcnt = d_tile_count_;
  AF_CUDA(cudaMalloc(&d_dt_, sizeof(double)));
  AF_CUDA(cudaMalloc(&d_step3_, sizeof(int)));
  AF_CUDA(cudaMallocHost(&h_dt_step_, 64));
  AF_CUDA(cudaMalloc(&d_lpl_, sizeof(unsigned long long) * 17));
  AF_CUDA(cudaStreamCreateWithFlags(&own_stream_, cudaStreamNonBlocking));
  stream_ = own_stream_;
  wset_(d_st_, 1, 1, ST_ABSENT, 0, L_);
  wset_(d_mark_, 1, 1, 0, 0, L_);
  wset_(d_V_, 8, NC_, 0, 0, L_);
  wset_(d_Vs_, 8, NC_, 0, 0, L_);
  wset_(d_Qold_, 8, NC_, 0, 0, L_);
  AF_CUDA(cudaMemsetAsync(d_err_, 0, 4 * sizeof(int), stream_));
  AF_CUDA(cudaMemsetAsync(d_err_ + 1, 0x7f, sizeof(int), stream_));
  t_old_.assign(L_ + 1, 0.0);
  t_new_.assign(L_ + 1, 0.0);
  leaves_per_level_.assign(L_ + 1, 0);
  std::memset(&last_, 0, sizeof(last_));
  last_.step = -1;
  if (D_ == 3) {
    for (auto fn : {(const void*)mr_stage_kernel<3, 0, kTX3, kTY3, kTZ3>,
                    (const void*)mr_stage_kernel<3, 1, kTX3, kTY3, kTZ3>,
                    (const void*)mr_stage_kernel<3, 2, kTX3, kTY3, kTZ3>,
                    (const void*)mr_stage_kernel<3, 3, kTX3, kTY3, kTZ3>})
      AF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)MRTile<3, kTX3, kTY3, kTZ3>::smem_bytes));
  } else {
    for (auto fn : {(const void*)mr_stage_full2d<0>, (const void*)mr_stage_full2d<1>,
                    (const void*)mr_stage_full2d<2>, (const void*)mr_stage_full2d<3>})
      AF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)MRFull2::smem_bytes));
    mr_full_tol_setup();
  }
  if (dist_) dist_setup_();
}

MR::~MR() {
  if (std::getenv("AF_MR_TIMING"))
    std::fprintf(stderr, "AF_MR_TIMING refine %.3f ms, virtual+counts+dt %.3f ms, evolve %.3f ms, "
                 "coarsen+lists %.3f ms (totals); evolve GPU span %.3f ms\n", 1e3 * phase_s_[0],
                 1e3 * phase_s_[1], 1e3 * phase_s_[2], 1e3 * phase_s_[3], evolve_gpu_ms_);
  cudaSetDevice(cfg_.device);
  if (own_stream_) cudaStreamSynchronize(own_stream_);
  if (phase_n_ > 0) {
    double tot = 0.0;
    for (size_t i = 1; i < phase_ms_.size(); ++i) tot += phase_ms_[i];
    std::fprintf(stderr, "AF_MR_PHASES: %ld cycles, %.1f us/cycle between the first and last mark\n",
                 phase_n_, 1e3 * tot / phase_n_);
    for (size_t i = 1; i < phase_ms_.size(); ++i)
      std::fprintf(stderr, "  %-30s %8.1f us\n", phase_ev_[i].first, 1e3 * phase_ms_[i] / phase_n_);
  }
  for (auto& pe : phase_ev_) cudaEventDestroy(pe.second);
  for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
  dist_free_();
  for (GraphCache& gc : graphs_)
    if (gc.exec) cudaGraphExecDestroy(gc.exec);
  for (CycleGraph& cg : cyc_) {
    if (cg.exec) cudaGraphExecDestroy(cg.exec);
    if (cg.graph) cudaGraphDestroy(cg.graph);
  }
  if (side_stream_) cudaStreamDestroy(side_stream_);
  if (fork_stream_) cudaStreamDestroy(fork_stream_);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  for (cudaEvent_t e : ev_aux_)
    if (e) cudaEventDestroy(e);
  if (h_cycrec_) cudaFreeHost(h_cycrec_);
  if (h_small_) cudaFreeHost(h_small_);
  for (void* p : {(void*)d_ckV_, (void*)d_ckSt_, (void*)d_cycrec_, (void*)d_cycctl_, (void*)d_acc_})
    cudaFree(p);
  if (h_dt_step_) cudaFreeHost(h_dt_step_);
  if (!sp_.empty()) {  // sparse value arrays: VMM reservations, not cudaMalloc
    sp_free_all_();
    d_V_ = d_Vs_ = d_Qold_ = d_VQold_ = d_det_ = nullptr;
  }
  if (windows_) {
    wfree_all_();
  } else {
    for (void* p : {(void*)d_st_, (void*)d_mark_, (void*)d_flag_, (void*)d_flag2_, (void*)d_V_,
                    (void*)d_Vs_, (void*)d_Qold_, (void*)d_VQold_, (void*)d_det_,
                    (void*)d_regbase_, (void*)d_regmask_})
      cudaFree(p);
  }
  for (void* p : {(void*)d_norms_, (void*)d_tiles_, (void*)d_tile_count_, (void*)d_err_,
                  (void*)d_band_, (void*)d_pband_, (void*)d_lpart_, (void*)d_lfull_, (void*)d_tflag_, (void*)d_tleaf_, (void*)d_lpl_, (void*)d_dt_, (void*)d_step3_,
                  (void*)d_flagi_, (void*)d_red_, (void*)d_regc_, (void*)d_regf_, (void*)d_regfc_,
                  (void*)d_regff_, (void*)d_regcount_, (void*)d_regerr_, (void*)d_badkey_})
    cudaFree(p);
  if (own_stream_) cudaStreamDestroy(own_stream_);
}

void MR::set_stream(cudaStream_t s) { stream_ = s ? s : own_stream_; }

void MR::invalidate_graphs_() {
  AF_CUDA(cudaStreamSynchronize(stream_));
  for (GraphCache& gc : graphs_) {
    if (gc.exec) cudaGraphExecDestroy(gc.exec);
    gc = GraphCache{};
  }
  for (CycleGraph& cg : cyc_) {
    if (cg.exec) cudaGraphExecDestroy(cg.exec);
    if (cg.graph) cudaGraphDestroy(cg.graph);
    cg = CycleGraph{};
  }
}

void MR::set_numerics(int numerics) {
  if (numerics != AF_NUMERICS_EXACT && numerics != AF_NUMERICS_TOLERANCE)
    throw Error(AF_E_ARGUMENT, "unknown numerics mode");
  if (numerics != numerics_) {  // captured cycle graphs hold the other kernels
    numerics_ = numerics;
    invalidate_graphs_();
  }
}

double MR::eps_at_(int child_level) const {
  return eps_level_.empty() ? opt_.eps : eps_level_[child_level];
}

#define AF_MR_LAUNCH(kern, grid, ...)                                   \
  do {                                                                  \
    if (D_ == 3)                                                        \
      launch_k(pdl_, stream_, kern<3>, dim3(grid), 256, 0, __VA_ARGS__); \
    else                                                                \
      launch_k(pdl_, stream_, kern<2>, dim3(grid), 256, 0, __VA_ARGS__); \
    ++launches_;                                                        \
    AF_CUDA(cudaGetLastError());                                        \
  } while (0)

// multi-level launch of a per-level kernel over levels [lo, hi] (band or leaf lists)
#define AF_ML_LAUNCH_M(kern, lo, hi, leaf, mult, ...)                                    \
  do {                                                                             \
    dim3 grid_;                                                                    \
    if (ml_grid_((lo), (hi), (leaf), &grid_, (mult))) {                           \
      const int AF_L = -(std::max((lo), 0) + 1);                                   \
      const int* AF_T = (leaf) ? d_tiles_ : d_band_;                               \
      const int AF_S = (std::min((hi), L_) << 3) | ((leaf) ? 1 : 0);              \
      if (D_ == 3)                                                                 \
        launch_k(pdl_, stream_, kern<3>, grid_, 256, 0, __VA_ARGS__, AF_T, AF_S);   \
      else                                                                         \
        launch_k(pdl_, stream_, kern<2>, grid_, 256, 0, __VA_ARGS__, AF_T, AF_S);   \
      ++launches_;                                                                 \
      AF_CUDA(cudaGetLastError());                                                 \
    }                                                                              \
  } while (0)

#define AF_ML_LAUNCH(kern, lo, hi, leaf, ...) AF_ML_LAUNCH_M(kern, lo, hi, leaf, 1, __VA_ARGS__)

// band / leaf tile list of level l and a grid for it
#define AF_BAND(l) d_band_ + tile_off_[l], (fixed_grids_ ? -1 : band_count_[l])
#define AF_PBAND(l) d_pband_ + tile_off_[l], (fixed_grids_ ? -3 : pband_count_[l])
#define AF_LEAFT(l) d_tiles_ + tile_off_[l], (fixed_grids_ ? -2 : tile_count_[l])
// per-level tile-list grid: the live count, or in graph capture (device-side
// counts) the level's tile total as the cycle-invariant bound
#define AF_TGRIDL(l, cnt, mult)                                                        \
  ((unsigned)std::max(1, std::min((fixed_grids_ ? level_tiles_(l) : (cnt)) * (mult), kGrid)))
#define AF_TGRID(l, cnt) AF_TGRIDL(l, cnt, 1)
#define AF_HAS(cnt) (fixed_grids_ || (cnt) > 0)

// Prefetch permissions of the next launch (kPreList | kPreSt, af_mr_types.h):
// granted when the launch just before it in stream order writes neither
// (v_only_at_ marks a value-only launch; any later launch revokes it).
// A coarsen sweep's level below the finest: the previous launch is the next
// finer level of the same sweep, which writes only statuses of levels l+1 and
// l+2 (and the merge flags), so values, lists and level-l statuses may be read
// before the PDL wait (mr_coarsen_level). Not with ranks (halo exchanges sit
// between the levels) or a launch that is not the sweep's continuation.
int MR::coarsen_pre_(int l) const {
  static const bool off = std::getenv("AF_MR_NO_PRE") != nullptr;
  return (!off && !g_.dist && l < L_ - 1) ? kPreV : 0;
}

int MR::pre_() const {
  static const bool off = std::getenv("AF_MR_NO_PRE") != nullptr;
  return !off && launches_ == v_only_at_ ? (kPreList | kPreSt) : 0;
}

// Prediction refresh over the band tiles, coarsest level first: the tiny
// levels in one single-CTA launch, then one launch per level. (Cooperative
// launches with grid-wide barriers between levels were slower on B200 inside
// the cycle graph than per-level launches with programmatic dependent launch.)
// Only levels above `from` can hold stale predictions: a prediction at level
// l reads level l-1 only, so after values of levels [lo, hi] change (stage
// commit + projection) the refresh starts at lo+1.
void MR::predict_fill_(int lo, int hi, int from) {
  // levels <= min_leaf are complete (build coarsens above it, refine only
  // adds): no absent cells there
  const int f = std::max({1, from, min_leaf_ + 1});
  const uint8_t* vm = virtuals_ ? d_mark_ : nullptr;
  // dist_: the small levels of a rank are windowed, so every level is its own launch
  const int small = dist_ ? -1 : small_hi_;
  if (f <= small) {
    const int to = std::min(small_hi_, L_);
    if (D_ == 3)
      launch_k(pdl_, stream_, mr_predict_tiny<3>, dim3(1), kTinyThreads, 0, d_V_,
               (const uint8_t*)d_st_, vm, g_, f, to, lo, hi);
    else
      launch_k(pdl_, stream_, mr_predict_tiny<2>, dim3(1), kTinyThreads, 0, d_V_,
               (const uint8_t*)d_st_, vm, g_, f, to, lo, hi);
    AF_CUDA(cudaGetLastError());
    v_only_at_ = ++launches_;
  }
  // While the statuses are those the lists were built from, only the band
  // tiles holding an absent cell have anything to predict (a dense level has
  // none); after merges every band tile is visited.
  for (int l = std::max(f, small + 1); l <= L_; ++l)
    if (pband_ok_) {
      if (AF_HAS(pband_count_[l])) {
        const int pre = pre_();
        AF_MR_LAUNCH(mr_predict_level, AF_TGRID(l, pband_count_[l]), d_V_, d_st_, vm, g_, l, lo,
                     hi, AF_PBAND(l), pre);
        v_only_at_ = launches_;
      }
    } else if (AF_HAS(band_count_[l])) {
      const int pre = pre_();
      AF_MR_LAUNCH(mr_predict_level, AF_TGRID(l, band_count_[l]), d_V_, d_st_, vm, g_, l, lo, hi,
                   AF_BAND(l), pre);
      v_only_at_ = launches_;
    }
  fresh_ = (!virtuals_ || (lo == 0 && hi >= L_)) && from <= 1;
}

// project_range (mr_solver.cpp:268-282): internals of levels [lo, top-1], finest first.
void MR::project_range_(int lo, int top) {
  // Internal values below min_leaf-1 are read by nothing on the cycle path
  // (details from min_leaf-1 up feed refine; merges start at min_leaf);
  // to_uniform and dump bring them up to date on demand (refresh_coarse_).
  if (lo < min_leaf_ - 1) {
    lo = min_leaf_ - 1;
    coarse_stale_ = true;
  }
  const int hi = std::min(top - 1, L_ - 1);
  if (g_.dist) {
    // owned rows of the split levels, then the halo rows (leaf values the
    // stage just committed and these projections) from their owners, then
    // the replicated levels below the partition level on every rank
    for (int l = hi; l >= std::max(lo, lp_); --l)
      if (AF_HAS(band_count_[l]))
        AF_MR_LAUNCH(mr_project_level, AF_TGRID(l, band_count_[l]), d_V_, d_st_, g_, l,
                     AF_BAND(l), 0);
    exchange_(XV);
    for (int l = std::min(hi, lp_ - 1); l >= lo; --l)
      if (AF_HAS(band_count_[l]))
        AF_MR_LAUNCH(mr_project_level, AF_TGRID(l, band_count_[l]), d_V_, d_st_, g_, l,
                     AF_BAND(l), 0);
    fresh_ = false;
    return;
  }
  for (int l = hi; l >= std::max(lo, small_hi_ + 1); --l)
    if (AF_HAS(band_count_[l])) {
      const int pre = pre_();
      AF_MR_LAUNCH(mr_project_level, AF_TGRID(l, band_count_[l]), d_V_, d_st_, g_, l, AF_BAND(l),
                   pre);
      v_only_at_ = launches_;
    }
  const int shi = std::min(hi, small_hi_);
  if (shi >= lo) {
    if (D_ == 3)
      launch_k(pdl_, stream_, mr_project_tiny<3>, dim3(1), kTinyThreads, 0, d_V_,
               (const uint8_t*)d_st_, g_, shi, lo);
    else
      launch_k(pdl_, stream_, mr_project_tiny<2>, dim3(1), kTinyThreads, 0, d_V_,
               (const uint8_t*)d_st_, g_, shi, lo);
    AF_CUDA(cudaGetLastError());
    v_only_at_ = ++launches_;
  }
  fresh_ = false;
}

void MR::build_lists_() {
  build_lists_enqueue_();
  int h[85];
  unsigned long long lp[17];
  AF_CUDA(cudaMemcpyAsync(h, d_tile_count_, sizeof h, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaMemcpyAsync(lp, d_lpl_, sizeof lp, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  if (g_.dist) allreduce_(lp, L_ + 1, RED_SUM);  // leaves per level over all ranks
  for (int l = 0; l <= L_; ++l) {
    band_count_[l] = h[l];
    tile_count_[l] = h[17 + l];
    pband_count_[l] = h[34 + l];
    full_count_[l] = h[68 + l];
    leaves_per_level_[l] = (long)lp[l];
    g_.band_cnt[l] = h[l];
    g_.leaf_cnt[l] = h[17 + l];
  }
  lists_valid_ = true;
}

// Band / leaf tile lists and leaves per level, device side only (counts in
// d_tile_count_ == g_.dcnt and d_lpl_).
void MR::build_lists_enqueue_() {
  // (the counts and leaves per level are cleared by mr_tile_flags_all)
  const long nt = tile_off_[L_ + 1];
  const unsigned gw = (unsigned)std::max<long>(1, std::min<long>((nt + 7) / 8, kGrid));
  const unsigned gt = grid_for(nt);
  if (D_ == 3) {
    launch_k(pdl_, stream_, mr_tile_flags_all<3>, dim3(gw), 256, 0, d_st_, g_, d_tflag_, d_tleaf_,
             d_tile_count_, d_lpl_);
    launch_k(pdl_, stream_, mr_tile_lists_all<3>, dim3(gt), 256, 0, (const uint8_t*)d_tflag_,
             (const int*)d_tleaf_, g_, d_band_, d_tiles_, d_pband_, d_lpart_, d_lfull_,
             d_tile_count_, d_lpl_);
  } else {
    launch_k(pdl_, stream_, mr_tile_flags_all<2>, dim3(gw), 256, 0, d_st_, g_, d_tflag_, d_tleaf_,
             d_tile_count_, d_lpl_);
    launch_k(pdl_, stream_, mr_tile_lists_all<2>, dim3(gt), 256, 0, (const uint8_t*)d_tflag_,
             (const int*)d_tleaf_, g_, d_band_, d_tiles_, d_pband_, d_lpart_, d_lfull_,
             d_tile_count_, d_lpl_);
  }
  launches_ += 2;
  AF_CUDA(cudaGetLastError());
  pband_ok_ = true;
}

// Grid of a multi-level launch over levels [lo, hi]: the total tile count of
// the lists (or its bound during capture), capped. False when all are empty.
bool MR::ml_grid_(int lo, int hi, bool leaf, dim3* grid, int mult, int cap) const {
  // one flat range over the tiles of levels [lo, hi] (for_each_tile)
  if (hi < lo) return false;
  long sum = 0;
  for (int l = std::max(lo, 0); l <= std::min(hi, L_); ++l)
    sum += fixed_grids_ ? level_tiles_(l)  // graph capture: a cycle-invariant bound
                        : (leaf ? tile_count_[l] : band_count_[l]);
  if (!sum) return false;
  *grid = dim3((unsigned)std::min<long>(sum * mult, cap));
  return true;
}

void MR::build(const double* aos) {
  if (!aos) throw Error(AF_E_ARGUMENT, "null state pointer");
  const long cells = mr_cells(D_, L_);
  const long rowlen = D_ == 3 ? 1L << (2 * L_) : 1L << L_;
  // this rank's rows of level L (every row on one rank), staged through a
  // scratch buffer: the caller's array may be host or device memory
  int r0 = 0, r1 = 1 << L_;
  if (dist_) part_rows_(rank_, L_, &r0, &r1);
  const long ucells = (long)(r1 - r0) * rowlen;
  sp_map_all_(d_V_);  // from_uniform fills and projects every level (sparse: all bricks)
  double* stage = nullptr;
  AF_CUDA(cudaMallocAsync((void**)&stage, sizeof(double) * 5 * ucells, stream_));
  AF_CUDA(cudaMemcpyAsync(stage, aos + 5 * (long)r0 * rowlen, sizeof(double) * 5 * ucells,
                          cudaMemcpyDefault, stream_));
  AF_MR_LAUNCH(mr_upload_finest, grid_for(ucells), (const double*)stage, d_V_, g_, r0, r1);
  AF_CUDA(cudaFreeAsync(stage, stream_));
  // from_uniform (mr_tree.cpp:29-71): leaves at L, internals above.
  wset_(d_st_, 1, 1, ST_INTERNAL, 0, L_ - 1);
  wset_(d_st_, 1, 1, ST_LEAF, L_, L_);
  wset_(d_mark_, 1, 1, 0, 0, L_);
  AF_CUDA(cudaMemsetAsync(d_err_, 0, 4 * sizeof(int), stream_));
  AF_CUDA(cudaMemsetAsync(d_err_ + 1, 0x7f, sizeof(int), stream_));
  virtuals_ = false;
  // with ranks: owned projections, the halo rows from their owners, the
  // replicated levels on every rank (project_range_)
  build_lists_();
  project_range_(0, L_);
  // set_norms_from (mr_tree.cpp:73-87)
  AF_CUDA(cudaMemsetAsync(d_red_, 0, sizeof(unsigned long long) * 8, stream_));
  AF_MR_LAUNCH(mr_norm_kernel, grid_for(cells), d_V_, g_, d_red_);
  unsigned long long nb[5] = {0, 0, 0, 0, 0};
  AF_CUDA(cudaMemcpyAsync(nb, d_red_, 8 * NC_, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  if (g_.dist) allreduce_(nb, NC_, RED_MAX);  // per-component max over all ranks' rows
  double n[5] = {0, 0, 0, 0, 0};
  n[0] = as_d(nb[0]);
  for (int a = 0; a < D_; ++a) n[1 + a] = as_d(nb[1 + a]);
  n[4] = as_d(nb[D_ + 1]);
  const double global = std::max({n[0], n[1], n[2], n[3], n[4], 1e-300});
  for (double& v : n)
    if (v < 1e-12 * global) v = global;
  std::memcpy(norms_host_, n, sizeof n);
  AF_CUDA(cudaMemcpyAsync(d_norms_, norms_host_, sizeof n, cudaMemcpyHostToDevice, stream_));
  min_leaf_ = opt_.min_leaf_level;
  if (opt_.local_time) min_leaf_ = std::max(min_leaf_, std::max(0, L_ - opt_.lt_gap));
  max_cfl_ = 0.0;
  fallbacks_ = 0;
  max_wave_ = 0.0;
  const bool timing = std::getenv("AF_MR_TIMING") && std::getenv("AF_MR_TIMING")[0] == '2';
  auto now_ms = [&] {
    AF_CUDA(cudaStreamSynchronize(stream_));
    return 1e3 * std::chrono::duration<double>(
                     std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t0 = timing ? now_ms() : 0.0;
  coarsen();
  build_lists_();
  sparse_sync_();  // sparse bricks: release what the coarsened tree does not reach
  if (timing) std::fprintf(stderr, "build: initial coarsen + lists %.3f ms\n", now_ms() - t0);
}

void MR::refine(int top) {
  std::vector<int> radius;
  if (top >= 0) {  // LT buffer radii (mr_solver.cpp:358-362)
    radius.assign(L_ + 1, 1);
    for (int l = 0; l <= L_; ++l)
      if (l > top + 1) radius[l] = 1 << (l - top - 1);
  }
  refine_(radius, nullptr);
}

// MRTree::refine(eps, buffer_radius_per_level) (mr_tree.hpp:141,
// mr_tree.cpp:361-402): one threshold for every level, and a Chebyshev
// dilation of the split set by buffer[l] leaves at level l (none when the
// buffer is empty; levels past its end or with a radius <= 0 do not dilate).
void MR::refine(double eps, const int* buffer, int n) {
  if (n < 0 || (n > 0 && !buffer)) throw Error(AF_E_ARGUMENT, "bad buffer radius array");
  std::vector<int> radius(buffer, buffer + n);
  for (int r : radius)
    if (dist_ && r > halo_)
      throw Error(AF_E_CONFIG, "refine buffer radius exceeds the decomposition's halo rows");
  refine_(radius, &eps);
}

void MR::refine_(const std::vector<int>& radius, const double* eps) {
  registers_built_ = false;
  if (!lists_valid_) build_lists_();
  sparse_sync_();  // sparse bricks: map what this cycle can reach (af_mr_storage.cu)
  wset_(d_flag_, 1, 1, 0, 0, L_);
  wset_(d_flag2_, 1, 1, 0, 0, L_);
  // details with the refine flags of their leaf children (one launch)
  for (int l = 1; l <= L_ - 1; ++l) g_.eps_l[l] = eps ? *eps : eps_at_(l);
  AF_ML_LAUNCH_M(mr_detail_level, std::max(0, min_leaf_ - 1), L_ - 2, false, 1 << D_, d_V_,
                 d_st_, d_det_, g_, AF_L, d_norms_, d_flag_);
  uint8_t* split = d_flag_;
  if (!radius.empty()) {
    for (int l = 1; l <= L_ - 1; ++l) {
      const int r = l < (int)radius.size() ? std::max(0, radius[l]) : 0;
      if (band_count_[l])
        AF_MR_LAUNCH(mr_dilate_level, AF_TGRID(l, band_count_[l]), d_st_, d_flag_, d_flag2_, g_, l,
                     r, AF_BAND(l));
    }
    split = d_flag2_;
  }
  AF_CUDA(cudaMemsetAsync(d_flagi_, 0, sizeof(int), stream_));
  AF_ML_LAUNCH(mr_apply_split_level, 1, L_ - 1, false, d_st_, split, g_, AF_L, d_flagi_);
  // enforce_gradedness (mr_tree.cpp:404-444)
  if (g_.dist) {
    // one decide/apply pass per round: the neighbours' splits arrive through
    // the status halo, and the fixpoint test is over all ranks
    exchange_(XST);
    for (;;) {
      AF_ML_LAUNCH(mr_grade_flag_level, 0, L_ - 1, false, d_st_, d_flag_, g_, AF_L);
      AF_CUDA(cudaMemsetAsync(d_flagi_, 0, sizeof(int), stream_));
      AF_ML_LAUNCH(mr_apply_split_level, 0, L_ - 1, false, d_st_, d_flag_, g_, AF_L, d_flagi_);
      exchange_(XST);
      int changed = 0;
      AF_CUDA(cudaMemcpyAsync(&changed, d_flagi_, sizeof(int), cudaMemcpyDeviceToHost, stream_));
      AF_CUDA(cudaStreamSynchronize(stream_));
      unsigned long long ch = changed ? 1 : 0;
      allreduce_(&ch, 1, RED_MAX);
      if (!ch) break;
    }
    build_lists_();
    lists_valid_ = true;
    predict_fill_(1, 0);
    return;
  }
  for (;;) {
    // two decide/apply passes per host check: the fixpoint usually needs one
    // pass plus the verifying one, so this saves a synchronisation
    AF_ML_LAUNCH(mr_grade_flag_level, 0, L_ - 1, false, d_st_, d_flag_, g_, AF_L);
    AF_ML_LAUNCH(mr_apply_split_level, 0, L_ - 1, false, d_st_, d_flag_, g_, AF_L, d_flagi_);
    AF_ML_LAUNCH(mr_grade_flag_level, 0, L_ - 1, false, d_st_, d_flag_, g_, AF_L);
    AF_CUDA(cudaMemsetAsync(d_flagi_, 0, sizeof(int), stream_));
    AF_ML_LAUNCH(mr_apply_split_level, 0, L_ - 1, false, d_st_, d_flag_, g_, AF_L, d_flagi_);
    int changed = 0;
    AF_CUDA(cudaMemcpyAsync(&changed, d_flagi_, sizeof(int), cudaMemcpyDeviceToHost, stream_));
    AF_CUDA(cudaStreamSynchronize(stream_));
    if (!changed) break;
  }
  build_lists_();
  lists_valid_ = true;
  predict_fill_(1, 0);  // predictions for band cells the splits brought in
}

void MR::add_virtual_leaves() {
  wset_(d_mark_, 1, 1, 0, 0, L_);
  if (!lists_valid_) build_lists_();
  // with ranks, leaves in halo rows mark owned parents too: scan the band;
  // the stage reads the marks of halo parents (MRLT interpolation, registers)
  AF_ML_LAUNCH(mr_virtual_mark_level, 1, L_, !g_.dist, d_st_, d_mark_, g_, AF_L);
  if (g_.dist) exchange_(XMARK);
  virtuals_ = true;
}

void MR::remove_virtual_leaves() {
  const bool was_fresh = fresh_;
  virtuals_ = false;
  // former virtual positions read as fresh predictions again (a no-op when
  // every virtual was just refreshed, as after a global step)
  if (!was_fresh) predict_fill_(1, 0);
  fresh_ = true;
}

void MR::counts(long* leaves, long* nodes, long* internals) {
  AF_CUDA(cudaMemsetAsync(d_red_, 0, sizeof(unsigned long long) * 3, stream_));
  launch_k(pdl_, stream_, mr_count_kernel, dim3(grid_for(g_.total_cells)), 256, 0,
      d_st_, virtuals_ ? d_mark_ : nullptr, g_.total_cells, d_red_, g_);
  ++launches_;
  unsigned long long h[3];
  AF_CUDA(cudaMemcpyAsync(h, d_red_, sizeof h, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  if (g_.dist) allreduce_(h, 3, RED_SUM);
  if (leaves) *leaves = (long)h[0];
  if (internals) *internals = (long)h[1];
  if (nodes) *nodes = (long)(h[0] + h[1] + (h[2] << D_));
}

// counts (leaves, nodes incl. virtual) and the CFL speed in one synchronisation
void MR::cycle_stats_(long* leaves, long* nodes, double* smax) {
  AF_CUDA(cudaMemsetAsync(d_red_, 0, sizeof(unsigned long long) * 4, stream_));
  const uint8_t* vm = virtuals_ ? d_mark_ : nullptr;
  if (!g_.dist) {  // one pass over the cells
    if (D_ == 3)
      launch_k(pdl_, stream_, mr_count_speed_kernel<3>, dim3(grid_for(g_.total_cells)), 256, 0,
               (const uint8_t*)d_st_, vm, g_.total_cells, d_red_, g_, (const double*)d_V_,
               cfg_.gamma, smax ? 1 : 0);
    else
      launch_k(pdl_, stream_, mr_count_speed_kernel<2>, dim3(grid_for(g_.total_cells)), 256, 0,
               (const uint8_t*)d_st_, vm, g_.total_cells, d_red_, g_, (const double*)d_V_,
               cfg_.gamma, smax ? 1 : 0);
    ++launches_;
  } else {
    launch_k(pdl_, stream_, mr_count_kernel, dim3(grid_for(g_.total_cells)), 256, 0, d_st_, vm,
             g_.total_cells, d_red_, g_);
    ++launches_;
    if (smax)
      AF_ML_LAUNCH(mr_leaf_speed_kernel, 0, L_, true, d_V_, d_st_, g_, AF_L, cfg_.gamma, d_red_ + 3);
  }
  unsigned long long h[4];
  AF_CUDA(cudaMemcpyAsync(h, d_red_, sizeof h, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  if (g_.dist) {
    allreduce_(h, 3, RED_SUM);
    allreduce_(h + 3, 1, RED_MAX);  // non-negative double: max of the bit patterns
  }
  *leaves = (long)h[0];
  *nodes = (long)(h[0] + h[1] + (h[2] << D_));
  if (smax) *smax = as_d(h[3]);
}

int MR::coarsest_leaf_level() {
  if (!lists_valid_) {  // a coarsen since the last list build changed the counts
    build_lists_();
    lists_valid_ = true;
  }
  for (int l = 0; l <= L_; ++l)
    if (leaves_per_level_[l]) return l;
  return L_;
}

double MR::leaf_speed_sum() {
  AF_CUDA(cudaMemsetAsync(d_red_, 0, sizeof(unsigned long long), stream_));
  AF_ML_LAUNCH(mr_leaf_speed_kernel, 0, L_, true, d_V_, d_st_, g_, AF_L, cfg_.gamma, d_red_);
  unsigned long long b = 0;
  AF_CUDA(cudaMemcpyAsync(&b, d_red_, 8, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  if (g_.dist) allreduce_(&b, 1, RED_MAX);
  return as_d(b);
}

// One RK stage for the leaves of levels [lo, hi] (MRSolver::stage,
// mr_solver.cpp:163-193): all levels read the same state, then commit.
void MR::stage_(int lo, int hi, double tau, double sdt, int stage, long step) {
  MRStageArgs a{};
  a.eval = d_V_;
  a.base = d_Qold_;
  a.snap = stage == 1 ? d_Qold_ : nullptr;  // stage 1 writes the q_old snapshot
  a.out = d_Vs_;
  a.st = d_st_;
  a.gamma = cfg_.gamma;
  a.gm1 = cfg_.gamma - 1.0;
  a.sdt = sdt;
  a.step3 = (int)(3 * std::max(step, 0L));
  if (fixed_grids_) {
    a.dt_dev = d_dt_;
    a.dt_scale = stage == 1 ? 0.5 : 1.0;  // step_levels: stage(dt/2), stage(dt)
    a.step3_dev = d_step3_;
  }
  a.stage = stage;
  a.post_check = stage == 2;
  // graph capture of a global step (a failing batch is replayed on the
  // synchronous path, which commits through the guarded copy)
  // MRLT substeps of the finest level alone (lo = hi = L) swap as well: the
  // stage writes every leaf of L, the level has no internal cells, and its
  // absent cells (virtual leaves, predictions) are copied over after the
  // swap (mr_copy_absent_tiles over the band tiles holding one)
  const bool swap_fine = !g_.dist && lo == L_ && hi >= L_ && pband_ok_ && !cycle_capture_ &&
                         std::getenv("AF_MR_NO_SWAP") == nullptr;
  swap_ = (!g_.dist && lo == 0 && hi >= L_ && std::getenv("AF_MR_NO_SWAP") == nullptr) ||
          swap_fine;
  a.post_stops = swap_ ? 1 : 0;
  a.err = d_err_;
  a.lo = lo;
  a.hi = hi;
  a.vmark = d_mark_;
  a.vq_old = d_VQold_;
  a.reg_stage = stage == 2 && registers_built_;
  a.step_dt = step_dt_;
  a.share = D_ == 3 ? 0.25 : 0.5;  // mr_solver.cpp:239
  a.sub = sub_;
  a.regbase = d_regbase_;
  a.regmask = d_regmask_;
  a.regc = d_regc_;
  a.regf = d_regf_;
  a.regfc = d_regfc_;
  a.regff = d_regff_;
  a.regerr = d_regerr_;
  a.tflag = std::getenv("AF_MR_NO_FULL") ? nullptr : d_tflag_;  // full-tile fast path
  for (int lv = 0; lv <= L_ && lv < 17; ++lv) {
    const double denom = t_new_[lv] - t_old_[lv];
    a.theta[lv] = denom > 0.0 ? std::clamp((tau - t_old_[lv]) / denom, 0.0, 1.0) : 1.0;
  }
  const int slot = (int)(stage_records_.size());
  if (slot >= kMaxStageRecords) throw Error(AF_E_CONFIG, "too many stages per cycle");
  stage_records_.push_back({slot, 0.0, lo, hi});
  unsigned long long* wave = d_red_ + 64 + slot * 17;
  unsigned long long* fb = d_red_ + 64 + slot * 17 + 16;
  // (in the cycle graph mr_cycle_begin clears both stages' records)
  if (!cycle_capture_) AF_CUDA(cudaMemsetAsync(wave, 0, sizeof(unsigned long long) * 17, stream_));
  a.wave = wave;
  a.fb = fb;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (profile_) {
    while (ev_pool_.size() < ev_used_ + 2) {
      cudaEvent_t e;
      AF_CUDA(cudaEventCreate(&e));
      ev_pool_.push_back(e);
    }
    e0 = ev_pool_[ev_used_++];
    e1 = ev_pool_[ev_used_++];
    AF_CUDA(cudaEventRecordWithFlags(e0, stream_, fixed_grids_ ? cudaEventRecordExternal : 0));
    note_event_node_();
  }
  // one launch for every stepping level (one flat range of leaf tiles);
  // all levels read the same state and write only their own leaves
  for (int l = std::max(lo, 0); l <= std::min(hi, L_); ++l)
    if (tile_count_[l] && profile_) {
      ++stage_launches_;
      stage_updates_ += leaves_per_level_[l];
    }
  // Full 2D tiles (every cell and face neighbour a leaf of the level) run on
  // mr_stage_full2d, the other leaf tiles on mr_stage_kernel (AF_MR_NO_FULLK:
  // every leaf tile on mr_stage_kernel, with its own full-tile fast path).
  // A few full tiles are not worth a second launch (cfg2's sparse levels):
  // the split is used when the last list build found at least kFullMin of
  // them among the stepping levels (host counts; also at graph capture).
  long nfull_host = 0;
  for (int l = std::max(lo, 0); l <= std::min(hi, L_); ++l) nfull_host += full_count_[l];
  const bool fullk = D_ == 2 && !g_.dist && a.tflag && !std::getenv("AF_MR_NO_FULLK") &&
                     (nfull_host >= kFullMin || std::getenv("AF_MR_FULLK"));
  long nfull = 0, npart = 0;
  for (int l = std::max(lo, 0); l <= std::min(hi, L_); ++l) {
    const long tot = fixed_grids_ ? level_tiles_(l) : tile_count_[l];
    const long fu = fixed_grids_ ? level_tiles_(l) : full_count_[l];
    nfull += fu;
    npart += fixed_grids_ ? tot : tot - fu;
  }
  if (fullk && nfull > 0) {
    MRStageArgs f = a;
    f.tiles = d_lfull_;
    f.ntiles = (std::min(hi, L_) << 3) | 4;
    const dim3 gf((unsigned)std::min<long>(nfull, kStageGrid));
    const int lcode = -(std::max(lo, 0) + 1);
    const int sch = cfg_.limiter | (cfg_.flux << 1);
    const size_t smf = MRFull2::smem_bytes;
    if (numerics_ == AF_NUMERICS_TOLERANCE) {
      mr_full_tol_launch(sch, gf, stream_, pdl_, f, g_, lcode);
    } else switch (sch) {
      case 0: launch_k(pdl_, stream_, mr_stage_full2d<0>, gf, MRFull2::NT, smf, f, g_, lcode); break;
      case 1: launch_k(pdl_, stream_, mr_stage_full2d<1>, gf, MRFull2::NT, smf, f, g_, lcode); break;
      case 2: launch_k(pdl_, stream_, mr_stage_full2d<2>, gf, MRFull2::NT, smf, f, g_, lcode); break;
      default: launch_k(pdl_, stream_, mr_stage_full2d<3>, gf, MRFull2::NT, smf, f, g_, lcode); break;
    }
    ++launches_;
    AF_CUDA(cudaGetLastError());
  }
  dim3 grid;
  const bool part_only = fullk;
  if (part_only ? npart > 0 && (grid = dim3((unsigned)std::min<long>(npart, kStageGrid)), true)
                : ml_grid_(lo, hi, true, &grid, 1, kStageGrid)) {
    a.tiles = part_only ? d_lpart_ : d_tiles_;
    a.ntiles = (std::min(hi, L_) << 3) | (part_only ? 3 : 1);
    const int lcode = -(std::max(lo, 0) + 1);
    const int sch = cfg_.limiter | (cfg_.flux << 1);  // scheme code (af_physics.cuh)
    const unsigned b2 = kTX2 * kTY2, b3 = kTX3 * kTY3 * kTZ3;
    const size_t sm2 = MRTile<2, kTX2, kTY2, 1>::smem_bytes;
    const size_t sm3 = MRTile<3, kTX3, kTY3, kTZ3>::smem_bytes;
#define AF_ST(S)                                                                           \
  do {                                                                                     \
    if (D_ == 2)                                                                           \
      launch_k(pdl_, stream_, mr_stage_kernel<2, S, kTX2, kTY2, 1>, grid, b2, sm2, a, g_,   \
               lcode);                                                                     \
    else                                                                                   \
      launch_k(pdl_, stream_, mr_stage_kernel<3, S, kTX3, kTY3, kTZ3>, grid, b3, sm3, a, g_, \
               lcode);                                                                     \
  } while (0)
    switch (sch) {
      case 0: AF_ST(0); break;
      case 1: AF_ST(1); break;
      case 2: AF_ST(2); break;
      default: AF_ST(3); break;
    }
#undef AF_ST
    ++launches_;
    AF_CUDA(cudaGetLastError());
  }
  if (profile_) {
    AF_CUDA(cudaEventRecordWithFlags(e1, stream_, fixed_grids_ ? cudaEventRecordExternal : 0));
    note_event_node_();
  }
  if (swap_) {
    // Every leaf steps (levels 0..L): the output buffer becomes the state.
    // The projection and prediction that follow write every other cell a
    // later stage reads (internal nodes, and the absent band cells), so no
    // commit copy is needed; two stages per step swap back. Off the cycle
    // graph (whose failing batches are replayed from a checkpoint) a guarded
    // kernel puts the committed leaf values back when the stage failed, as
    // the skipped commit copy leaves them.
    std::swap(d_V_, d_Vs_);
    if (!cycle_capture_) {
      AF_ML_LAUNCH(mr_copy_leaves_tiles, lo, hi, true, d_Vs_, d_V_, d_st_, g_, AF_L, d_err_,
                   (stage == 2 ? 1 : 0) | 2);
      v_only_at_ = launches_;
    }
    if (swap_fine && AF_HAS(pband_count_[L_])) {
      AF_MR_LAUNCH(mr_copy_absent_tiles, AF_TGRID(L_, pband_count_[L_]), d_Vs_, d_V_, d_st_, g_,
                   L_, AF_PBAND(L_));
      v_only_at_ = launches_;
    }
    return;
  }
  AF_ML_LAUNCH(mr_copy_leaves_tiles, lo, hi, true, d_Vs_, d_V_, d_st_, g_, AF_L, d_err_,
               stage == 2);
  v_only_at_ = launches_;
}

// MRSolver::step_levels (mr_solver.cpp:232-316). `sub` is which of the
// parent's two substeps this call is (the fine register slot).
void MR::step_levels_(int lo, int hi, double t, double dt, int sub) {
  const int top = std::min(hi, L_);
  // (the q_old snapshot of the stepping leaves is written by stage 1)
  for (int l = lo; l <= top; ++l) {
    t_old_[l] = t;
    t_new_[l] = t + dt;
  }
  // refresh_virtuals + the virtual q_old snapshot (mr_solver.cpp:251-266);
  // nothing to refresh when every prediction is current and all levels step
  if (!(fresh_ && lo == 0 && top >= L_)) predict_fill_(lo, top, lo + 1);
  if (d_VQold_)
    for (int l = lo + 1; l <= std::min(top + 1, L_); ++l)
      AF_MR_LAUNCH(mr_virtual_snapshot, grid_for(mr_cells(D_, l)), d_V_, d_VQold_, d_st_,
                   d_mark_, g_, l);
  const size_t r0 = stage_records_.size();
  step_dt_ = dt;
  sub_ = sub;
  stage_(lo, top, t, 0.5 * dt, 1, cur_step_);
  phase_("stage 1");
  project_range_(lo, top);
  phase_("project 1");
  predict_fill_(lo, top, lo + 1);
  phase_("predict 1");
  step_dt_ = dt;
  sub_ = sub;
  stage_(lo, top, t + 0.5 * dt, dt, 2, cur_step_);
  phase_("stage 2");
  project_range_(lo, top);
  phase_("project 2");
  predict_fill_(lo, top, lo + 1);
  phase_("predict 2");
  for (size_t r = r0; r < stage_records_.size(); ++r) stage_records_[r].step_dt = dt;
  bool deeper = false;
  for (int l = top + 1; l <= L_; ++l) deeper = deeper || leaves_per_level_[l] > 0;
  if (deeper) {
    if (!opt_.local_time) throw Error(AF_E_CONFIG, "finer leaves outside the stepping set");
    step_levels_(top + 1, top + 1, t, 0.5 * dt, 0);
    step_levels_(top + 1, top + 1, t + 0.5 * dt, 0.5 * dt, 1);
    apply_registers_(top);
    project_range_(lo, top + 1);
    predict_fill_(1, 0, lo + 1);
  }
}

void MR::evolve_global(double dt, af_step_diag* d) {
  stage_records_.clear();
  if (!lists_valid_) build_lists_();
  lists_valid_ = true;
  if (fresh_ && !g_.dist && !std::getenv("AF_MR_NO_GRAPH"))
    evolve_global_graph_(dt);
  else
    step_levels_(0, L_, 0.0, dt, 0);
  collect_stage_records_(d);
}

// The global step's launch sequence is identical every cycle once the counts,
// dt and the step index are read from device memory, so it is captured once
// into a CUDA graph and replayed (one launch instead of ~45 per cycle).
void MR::evolve_global_graph_(double dt) {
  h_dt_step_[0] = dt;
  reinterpret_cast<int*>(h_dt_step_ + 1)[0] = (int)(3 * std::max(cur_step_, 0L));
  AF_CUDA(cudaMemcpyAsync(d_dt_, h_dt_step_, sizeof(double), cudaMemcpyHostToDevice, stream_));
  AF_CUDA(cudaMemcpyAsync(d_step3_, h_dt_step_ + 1, sizeof(int), cudaMemcpyHostToDevice, stream_));
  // one cached graph per profiling mode (events are part of the graph)
  GraphCache& gc = graphs_[profile_ ? 1 : 0];
  graph_exec_ = gc.exec;
  graph_recs_ = gc.recs;
  graph_launches_ = gc.launches;
  graph_events_ = gc.events;
  if (!graph_exec_) {
    harvest_events_();
    const long l0 = launches_, s0 = stage_launches_, u0 = stage_updates_;
    fixed_grids_ = true;
    cudaGraph_t graph = nullptr;
    AF_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    try {
      step_levels_(0, L_, 0.0, dt, 0);
    } catch (...) {
      fixed_grids_ = false;
      cudaStreamEndCapture(stream_, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    AF_CUDA(cudaStreamEndCapture(stream_, &graph));
    fixed_grids_ = false;
    AF_CUDA(cudaGraphInstantiate(&graph_exec_, graph, 0));
    AF_CUDA(cudaGraphDestroy(graph));
    graph_recs_ = stage_records_;
    graph_launches_ = launches_ - l0;
    graph_stage_launches_ = stage_launches_ - s0;
    graph_stage_updates_ = stage_updates_ - u0;
    graph_events_ = ev_used_;
    gc = GraphCache{graph_exec_, graph_recs_, graph_launches_, graph_events_};
    launches_ = l0;
    stage_launches_ = s0;
    stage_updates_ = u0;
  }
  AF_CUDA(cudaGraphLaunch(graph_exec_, stream_));
  launches_ += graph_launches_;
  if (profile_) {
    // the stage updates of this cycle (leaf counts differ from the capture's)
    for (int l = 0; l <= L_; ++l)
      if (tile_count_[l]) {
        stage_launches_ += 2;
        stage_updates_ += 2 * leaves_per_level_[l];
      }
    ev_used_ = graph_events_;
  }
  stage_records_ = graph_recs_;
  for (StageRec& r : stage_records_) r.step_dt = dt;
  fresh_ = true;
}

void MR::advance_local(int top, double t, double dt, af_step_diag* d) {
  stage_records_.clear();
  if (!lists_valid_) build_lists_();
  lists_valid_ = true;
  if (opt_.local_time && !registers_built_) build_registers_(top);
  step_levels_(0, top, t, dt, 0);
  collect_stage_records_(d);
}

// Reads the per-stage wave/fallback records of the last evolve and folds
// them into the MRSolver accumulators (mr_solver.cpp:176-178); checks errors.
void MR::profile(bool on) {
  profile_ = on;
  stage_ms_ = 0.0;
  stage_launches_ = 0;
  stage_updates_ = 0;
}

void MR::harvest_events_() {
  if (!ev_used_) return;
  AF_CUDA(cudaStreamSynchronize(stream_));
  for (size_t e = 0; e + 1 < ev_used_; e += 2) {
    float ms = 0.f;
    AF_CUDA(cudaEventElapsedTime(&ms, ev_pool_[e], ev_pool_[e + 1]));
    stage_ms_ += ms;
  }
  ev_used_ = 0;
}

void MR::stage_stats(double* ms, long* launches, long* updates) {
  harvest_events_();
  if (ms) *ms = stage_ms_;
  if (launches) *launches = stage_launches_;
  if (updates) *updates = stage_updates_;
}

void MR::collect_stage_records_(af_step_diag* d) {
  check_error_(cur_step_);
  harvest_events_();
  const size_t ns = stage_records_.size();
  if (!ns) return;
  std::vector<unsigned long long> h(ns * 17);
  AF_CUDA(cudaMemcpyAsync(h.data(), d_red_ + 64, 8 * ns * 17, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  if (g_.dist)  // per record: 16 level maxima (wave-speed bits), then the fallback sum
    for (size_t r = 0; r < ns; ++r) {
      allreduce_(&h[r * 17], 16, RED_MAX);
      allreduce_(&h[r * 17 + 16], 1, RED_SUM);
    }
  double ws = 0.0;
  long fbs = 0;
  for (size_t r = 0; r < ns; ++r) {
    const StageRec& sr = stage_records_[r];
    for (int l = sr.lo; l <= std::min(sr.hi, L_); ++l) {
      if (!leaves_per_level_[l]) continue;
      const double w = as_d(h[r * 17 + l]);
      const double dx = cfg_.extent / static_cast<double>(1 << l);
      max_cfl_ = std::max(max_cfl_, w * sr.step_dt / dx);
      ws = std::max(ws, w);
    }
    fbs += (long)h[r * 17 + 16];
  }
  fallbacks_ += fbs;
  max_wave_ = std::max(max_wave_, ws);
  if (d) {
    d->max_wave_speed = ws;
    d->fallbacks = fbs;
  }
}

// Register slots for the leaves of levels [top, L-1] with an INTERNAL
// neighbour (valid until the tree changes at the end of the cycle).
void MR::build_registers_(int top) {
  if (!d_regbase_) throw Error(AF_E_CONFIG, "registers need local_time");
  wset_(d_regmask_, 1, 1, 0, 0, L_);
  AF_CUDA(cudaMemsetAsync(d_regcount_, 0, sizeof(int), stream_));
  for (int l = std::max(top, 0); l <= L_ - 1; ++l)
    AF_MR_LAUNCH(mr_reg_build_level, grid_for(mr_cells(D_, l)), d_st_, g_, l, d_regbase_,
                 d_regmask_, d_regcount_);
  int count = 0;
  AF_CUDA(cudaMemcpyAsync(&count, d_regcount_, sizeof(int), cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  static const bool dbg = std::getenv("AF_MR_DEBUG_REGS") != nullptr;
  if (dbg) std::fprintf(stderr, "registers: %d (capacity %ld)\n", count, reg_cap_);
  if (count > reg_cap_) {
    // stream-ordered, geometric growth: no device-wide synchronisation and
    // few reallocations while the interface grows over the first cycles
    for (void* p : {(void*)d_regc_, (void*)d_regf_, (void*)d_regfc_, (void*)d_regff_})
      if (p) AF_CUDA(cudaFreeAsync(p, stream_));
    // physical memory stays with the pool between reallocations (mapping
    // fresh memory is what makes a reallocation slow), and the capacity
    // grows 4x so that happens a few times per run at most
    cudaMemPool_t pool;
    AF_CUDA(cudaDeviceGetDefaultMemPool(&pool, cfg_.device));
    unsigned long long keep = ~0ull;
    AF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    // first allocation: room for an interface a quarter (2D) / sixteenth (3D)
    // of the level below the finest
    const long guess = reg_cap_ ? 0 : mr_cells(D_, L_ - 1) / (D_ == 3 ? 16 : 4);
    reg_cap_ = std::max<long>({2L * count, 4 * reg_cap_, guess, 1L << 16});
    AF_CUDA(cudaMallocAsync((void**)&d_regc_, sizeof(double) * NC_ * reg_cap_, stream_));
    AF_CUDA(cudaMallocAsync((void**)&d_regf_, sizeof(double) * NC_ * reg_fine_ * reg_cap_,
                            stream_));
    AF_CUDA(cudaMallocAsync((void**)&d_regfc_, reg_cap_, stream_));
    AF_CUDA(cudaMallocAsync((void**)&d_regff_, reg_cap_, stream_));
  }
  if (count) {  // only the slots this cycle uses
    AF_CUDA(cudaMemsetAsync(d_regfc_, 0, count, stream_));
    AF_CUDA(cudaMemsetAsync(d_regff_, 0, count, stream_));
    AF_CUDA(cudaMemsetAsync(d_regf_, 0, sizeof(double) * NC_ * reg_fine_ * count, stream_));
  }
  AF_CUDA(cudaMemsetAsync(d_regerr_, 0, sizeof(int), stream_));
  AF_CUDA(cudaMemsetAsync(d_badkey_, 0xff, sizeof(unsigned long long), stream_));
  registers_built_ = true;
}

// apply_registers (mr_solver.cpp:210-230) for the cells of `coarse_level`.
void MR::apply_registers_(int coarse_level) {
  if (!registers_built_) return;
  const double dx = cfg_.extent / static_cast<double>(1 << coarse_level);
  AF_MR_LAUNCH(mr_reg_apply_level, grid_for(mr_cells(D_, coarse_level)), d_V_, d_st_, g_,
               coarse_level, d_regbase_, d_regmask_, d_regc_, d_regf_, d_regfc_, d_regff_,
               1.0 / dx, d_badkey_, d_err_);
}

void MR::coarsen() {
  registers_built_ = false;
  if (!lists_valid_) {
    build_lists_();
    lists_valid_ = true;
  }
  bool clean = false;  // the previous sweep raised no re-sweep flag
  pband_ok_ = false;   // merges turn leaves into absent cells
  for (;;) {
    AF_CUDA(cudaMemsetAsync(d_flagi_, 0, 2 * sizeof(int), stream_));
    for (int l = L_ - 1; l >= min_leaf_; --l) {
      if (band_count_[l])
        AF_MR_LAUNCH(mr_coarsen_level, AF_TGRIDL(l, band_count_[l], 1 << D_), d_V_, d_st_, g_, l,
                     eps_at_(l + 1), d_norms_, d_flagi_, AF_BAND(l), coarsen_pre_(l));
      // the next level's merge_allowed reads this level's status in halo rows
      if (g_.dist) exchange_(XST);
    }
    int merged[2] = {0, 0};
    AF_CUDA(cudaMemcpyAsync(merged, d_flagi_, sizeof merged, cudaMemcpyDeviceToHost, stream_));
    AF_CUDA(cudaStreamSynchronize(stream_));
    if (g_.dist) {
      unsigned long long m2[2] = {(unsigned long long)merged[0], (unsigned long long)merged[1]};
      allreduce_(m2, 2, RED_MAX);
      merged[0] = (int)m2[0];
      merged[1] = (int)m2[1];
    }
    if (full_sweeps_ && clean && merged[0])
      throw Error(AF_E_INTERNAL, "coarsen: a sweep after a clean sweep merged (skip test unsound)");
    if (!merged[0]) break;
    clean = !merged[1];
    lists_valid_ = false;
    predict_fill_(1, 0, min_leaf_ + 1);  // merges only create absent cells above min_leaf
    // coarsen's while(merged) loop (mr_tree.cpp:474-510): the next sweep is
    // skipped when no merge can have changed a candidate's detail (merged[1],
    // see coarsen_level_dev); it would find nothing to merge.
    if (!merged[1] && !full_sweeps_) break;
  }
}

void MR::check_error_(long step) {
  int h[4];
  AF_CUDA(cudaMemcpyAsync(h, d_err_, sizeof h, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  if (g_.dist) {  // a failure on any rank stops every rank with the same report
    unsigned long long f[3] = {h[0] ? 1ull : 0ull, h[2] ? 1ull : 0ull, (unsigned)h[3]};
    allreduce_(f, 3, RED_MAX);
    unsigned long long code = (unsigned)h[1];
    allreduce_(&code, 1, RED_MIN);
    h[0] = (int)f[0];
    h[2] = (int)f[1];
    h[3] = (int)f[2];
    h[1] = (int)code;
  }
  if (!h[0] && !h[2]) return;
  if (d_badkey_) {
    unsigned long long bk = ~0ull;
    int regerr = 0;
    AF_CUDA(cudaMemcpy(&bk, d_badkey_, sizeof bk, cudaMemcpyDeviceToHost));
    AF_CUDA(cudaMemcpy(&regerr, d_regerr_, sizeof regerr, cudaMemcpyDeviceToHost));
    if (g_.dist) {
      allreduce_(&bk, 1, RED_MIN);
      unsigned long long re = regerr ? 1 : 0;
      allreduce_(&re, 1, RED_MAX);
      regerr = (int)re;
    }
    if (bk != ~0ull) {
      const unsigned long long ck = bk >> 3;
      const unsigned long long mask = (1ull << 15) - 1;
      const std::string node = "level " + std::to_string(ck >> 45) + " (" +
                               std::to_string((ck >> 30) & mask) + "," +
                               std::to_string((ck >> 15) & mask) + "," +
                               std::to_string(ck & mask) + ")";
      std::memset(&last_, 0, sizeof(last_));
      last_.status = AF_E_REGISTER_MISMATCH;
      last_.step = step;
      last_.level = (int)(ck >> 45);
      std::snprintf(last_.message, sizeof last_.message,
                    "interface flux register at %s is missing a side", node.c_str());
      throw Error(AF_E_REGISTER_MISMATCH, last_.message);
    }
    if (regerr) throw Error(AF_E_REGISTER_MISMATCH, "flux register slot missing");
  }
  const int lvl_lo = h[3] ? ((h[3] - 1) >> 8) : 0;
  const int lvl_hi = h[3] ? ((h[3] - 1) & 255) : L_;
  const int kind = h[1] % 3;  // 0/1 pass-1 of stage 1/2, 2 post-step
  const double* src = d_V_;
  std::vector<double> hv((size_t)NC_ * g_.total_cells);
  std::vector<uint8_t> hs(g_.total_cells);
  wtohost_(hv.data(), kind == 2 ? d_Vs_ : src, 8, NC_);
  wtohost_(hs.data(), d_st_, 1, 1);
  const double gm1 = cfg_.gamma - 1.0;
  const long comp = g_.total_cells;
  std::memset(&last_, 0, sizeof(last_));
  last_.status = AF_E_NONPHYSICAL;
  last_.step = step;
  last_.stage = kind == 2 ? 2 : kind + 1;
  const std::string pre = step >= 0 ? "step " + std::to_string(step) + ": " : "";
  std::string msg = pre + "non-physical state";
  // leaves in ascending pack_key order: level, then i, then j, then k
  // (with ranks: this rank's rows; the global first is the minimum key)
  bool found = false;
  for (int l = lvl_lo; l <= std::min(lvl_hi, L_) && !found; ++l) {
    const int n = 1 << l;
    const int nk = D_ == 3 ? n : 1;
    for (int i = 0; i < n && !found; ++i)
      for (int j = 0; j < n && !found; ++j)
        for (int k = 0; k < nk && !found; ++k) {
          const long c = g_.cell_off[l] + mr_idx(g_, D_, n, i, j, k);
          if (hs[c] != ST_LEAF || !row_owned(g_, l, D_ == 3 ? k : j)) continue;
          const double rho = hv[c];
          double msq = hv[comp + c] * hv[comp + c] + hv[2 * comp + c] * hv[2 * comp + c];
          if (D_ == 3) msq = msq + hv[3 * comp + c] * hv[3 * comp + c];
          const double inv = 1.0 / rho;
          const double p = gm1 * (hv[(NC_ - 1) * comp + c] - 0.5 * msq * inv);
          if (!(rho > 1e-12) || !(rho > 1e-12 && p > 1e-12)) {
            found = true;
            last_.level = l;
            last_.i = i;
            last_.j = j;
            last_.k = k;
            last_.rho = rho;
            last_.p = p;
          }
        }
  }
  if (g_.dist) {
    const auto key_of = [](const af_error& e) {
      return ((unsigned long long)e.level << 45) | ((unsigned long long)e.i << 30) |
             ((unsigned long long)e.j << 15) | (unsigned long long)e.k;
    };
    unsigned long long key = found ? key_of(last_) : ~0ull;
    allreduce_(&key, 1, RED_MIN);
    unsigned long long v[2] = {0, 0};
    if (found && key_of(last_) == key) {
      std::memcpy(&v[0], &last_.rho, 8);
      std::memcpy(&v[1], &last_.p, 8);
    }
    allreduce_(v, 2, RED_SUM);  // only the owner contributes
    found = key != ~0ull;
    if (found) {
      const unsigned long long m15 = (1ull << 15) - 1;
      last_.level = (int)(key >> 45);
      last_.i = (int)((key >> 30) & m15);
      last_.j = (int)((key >> 15) & m15);
      last_.k = (int)(key & m15);
      std::memcpy(&last_.rho, &v[0], 8);
      std::memcpy(&last_.p, &v[1], 8);
    }
  }
  if (found) {
    const std::string node = "level " + std::to_string(last_.level) + " (" +
                             std::to_string(last_.i) + "," + std::to_string(last_.j) + "," +
                             std::to_string(last_.k) + ")";
    msg = kind == 2 ? pre + "post-step " + node
                    : pre + node + ": rho=" + fmt_f(last_.rho) + " p=" + fmt_f(last_.p);
  }
  std::snprintf(last_.message, sizeof last_.message, "%s", msg.c_str());
  throw Error(AF_E_NONPHYSICAL, last_.message);
}

// ------------------------------------------------------- whole-cycle graph --
// Appends a WHILE conditional node to the graph being captured on stream_
// and captures body(handle) into it (on side_stream_). The handle is 1 at
// every graph launch; the body ends with mr_while_cond, which re-arms it.
// During a capture: remember the event-record node just added to stream_.
void MR::note_event_node_() {
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  AF_CUDA(cudaStreamGetCaptureInfo(stream_, &cs, nullptr, nullptr, &deps, &ndeps));
  if (cs != cudaStreamCaptureStatusActive) return;
  if (ndeps != 1) throw Error(AF_E_CUDA, "event record node: unexpected capture dependencies");
  ev_nodes_.push_back(deps[0]);
}

// The handle of a WHILE node: `def` on every graph launch (1: the body runs
// at least once), or with def = 0 set by a kernel ahead of the node.
cudaGraphConditionalHandle MR::make_cond_(unsigned def) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t graph = nullptr;
  AF_CUDA(cudaStreamGetCaptureInfo(stream_, &cs, nullptr, &graph, nullptr, nullptr));
  cudaGraphConditionalHandle h;
  AF_CUDA(cudaGraphConditionalHandleCreate(&h, graph, def, cudaGraphCondAssignDefault));
  return h;
}

template <class F>
void MR::capture_while_(F&& body, cudaGraphConditionalHandle h, bool have_h) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t graph = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  if (!have_h) h = make_cond_(1);
  AF_CUDA(cudaStreamGetCaptureInfo(stream_, &cs, nullptr, &graph, &deps, &ndeps));
  cudaGraphNodeParams p{};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  AF_CUDA(cudaGraphAddNode(&node, graph, deps, ndeps, &p));
  AF_CUDA(cudaStreamUpdateCaptureDependencies(stream_, &node, 1,
                                              cudaStreamSetCaptureDependencies));
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  cudaStream_t outer = stream_;
  stream_ = side_stream_;
  in_body_ = true;
  try {
    AF_CUDA(cudaStreamBeginCaptureToGraph(side_stream_, bodyg, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
    body(h);
    AF_CUDA(cudaStreamEndCapture(side_stream_, &bodyg));
  } catch (...) {
    cudaGraph_t g2 = nullptr;
    cudaStreamEndCapture(side_stream_, &g2);
    stream_ = outer;
    in_body_ = false;
    throw;
  }
  stream_ = outer;
  in_body_ = false;
}

// One run_mr cycle with a global step (mr_solver.cpp:339-395), enqueued with
// device-side counts only (fixed grids): refine + enforce_gradedness (WHILE),
// lists, predictions, virtual leaves, counts/CFL dt (mr_cycle_begin), the two
// RK stages, stage records (mr_cycle_end), coarsen sweeps (WHILE), lists.
void MR::phase_(const char* name) {
  if (!phases_ || !cycle_capture_) return;
  cudaEvent_t e;
  AF_CUDA(cudaEventCreate(&e));
  AF_CUDA(cudaEventRecordWithFlags(e, stream_, cudaEventRecordExternal));
  phase_ev_.push_back({name, e});
}

void MR::enqueue_cycle_(double cfl, double fixed_dt, long* grade_body, long* sweep_body) {
  const double dx_L = cfg_.extent / static_cast<double>(1 << L_);
  phase_("start");
  wset_(d_flag_, 1, 1, 0, 0, L_);
  for (int l = 1; l <= L_ - 1; ++l) g_.eps_l[l] = eps_at_(l);
  AF_ML_LAUNCH_M(mr_detail_level, std::max(0, min_leaf_ - 1), L_ - 2, false, 1 << D_, d_V_,
                 d_st_, d_det_, g_, AF_L, d_norms_, d_flag_);
  AF_ML_LAUNCH(mr_apply_split_level, 1, L_ - 1, false, d_st_, d_flag_, g_, AF_L, d_flagi_);
  AF_CUDA(cudaMemsetAsync(d_flagi_, 0, 2 * sizeof(int), stream_));
  long b0 = launches_;
  capture_while_([&](cudaGraphConditionalHandle h) {  // enforce_gradedness (mr_tree.cpp:404-444)
    AF_ML_LAUNCH(mr_grade_flag_level, 0, L_ - 1, false, d_st_, d_flag_, g_, AF_L);
    AF_ML_LAUNCH(mr_apply_split_level, 0, L_ - 1, false, d_st_, d_flag_, g_, AF_L, d_flagi_);
    launch_k(pdl_, stream_, mr_while_cond, dim3(1), 1, 0, h, d_flagi_, 0, d_acc_ + 3);
    ++launches_;
    AF_CUDA(cudaGetLastError());
  });
  *grade_body = launches_ - b0;
  phase_("refine+grade");
  build_lists_enqueue_();
  phase_("lists");
  // Fork: the prediction refresh (writes values of absent cells) runs beside
  // add_virtual_leaves / counts / CFL speed / cycle record (statuses, marks,
  // leaf values); both finish before the first stage.
  AF_CUDA(cudaEventRecord(ev_fork_, stream_));
  predict_fill_(1, 0);
  cudaStream_t main = stream_;
  stream_ = fork_stream_;
  AF_CUDA(cudaStreamWaitEvent(stream_, ev_fork_, 0));
  wset_(d_mark_, 1, 1, 0, 0, L_);
  AF_ML_LAUNCH(mr_virtual_mark_level, 1, L_, true, d_st_, d_mark_, g_, AF_L);
  AF_CUDA(cudaMemsetAsync(d_red_, 0, sizeof(unsigned long long) * 4, stream_));
  // counts and the CFL speed in one pass (mr_cycle_begin ignores the speed
  // under a fixed dt)
  if (D_ == 3)
    launch_k(pdl_, stream_, mr_count_speed_kernel<3>, dim3(grid_for(g_.total_cells)), 256, 0,
             (const uint8_t*)d_st_, (const uint8_t*)d_mark_, g_.total_cells, d_red_, g_,
             (const double*)d_V_, cfg_.gamma, 1);
  else
    launch_k(pdl_, stream_, mr_count_speed_kernel<2>, dim3(grid_for(g_.total_cells)), 256, 0,
             (const uint8_t*)d_st_, (const uint8_t*)d_mark_, g_.total_cells, d_red_, g_,
             (const double*)d_V_, cfg_.gamma, 1);
  ++launches_;
  launch_k(pdl_, stream_, mr_cycle_begin, dim3(1), 1, 0, d_red_, d_lpl_, L_, D_, cfl, fixed_dt,
           dx_L, d_dt_, d_step3_, d_cycctl_, d_cycrec_, d_red_ + 64, 2 * 17);
  ++launches_;
  AF_CUDA(cudaGetLastError());
  AF_CUDA(cudaEventRecord(ev_join_, stream_));
  stream_ = main;
  AF_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
  virtuals_ = true;
  phase_("predict || virtual+counts+dt");
  // the global step: dt and the step index come from mr_cycle_begin
  stage_records_.clear();
  cur_step_ = 0;
  step_levels_(0, L_, 0.0, 0.0, 0);
  cur_step_ = -1;
  // the stage records (mr_cycle_end) beside the coarsen sweep; joined at the
  // end of the cycle
  AF_CUDA(cudaEventRecord(ev_aux_[0], stream_));
  AF_CUDA(cudaStreamWaitEvent(fork_stream_, ev_aux_[0], 0));
  launch_k(pdl_, fork_stream_, mr_cycle_end, dim3(1), 1, 0, d_red_ + 64, d_lpl_, L_, cfg_.extent,
           d_dt_, d_acc_, d_cycctl_);
  ++launches_;
  AF_CUDA(cudaGetLastError());
  AF_CUDA(cudaEventRecord(ev_aux_[1], fork_stream_));
  virtuals_ = false;
  // coarsen (mr_tree.cpp:473-510): the first sweep and its prediction
  // refresh unconditionally, further sweeps (a WHILE node) only while one
  // merged and another can (the re-sweep test of coarsen_level_dev)
  AF_CUDA(cudaMemsetAsync(d_flagi_, 0, 2 * sizeof(int), stream_));
  pband_ok_ = false;  // merges turn leaves into absent cells
  phase_("cycle end");
  for (int l = L_ - 1; l >= min_leaf_; --l)
    AF_MR_LAUNCH(mr_coarsen_level, AF_TGRIDL(l, 0, 1 << D_), d_V_, d_st_, g_, l, eps_at_(l + 1),
                 d_norms_, d_flagi_, AF_BAND(l), coarsen_pre_(l));
  phase_("coarsen sweep");
  // the re-sweep decision (mr_while_cond reads the sweep's flags) beside the
  // prediction refresh
  const cudaGraphConditionalHandle hc = make_cond_(0);
  AF_CUDA(cudaEventRecord(ev_aux_[2], stream_));
  AF_CUDA(cudaStreamWaitEvent(fork_stream_, ev_aux_[2], 0));
  launch_k(pdl_, fork_stream_, mr_while_cond, dim3(1), 1, 0, hc, d_flagi_, full_sweeps_ ? 0 : 1,
           d_acc_ + 5);
  ++launches_;
  AF_CUDA(cudaGetLastError());
  AF_CUDA(cudaEventRecord(ev_aux_[3], fork_stream_));
  predict_fill_(1, 0, min_leaf_ + 1);
  AF_CUDA(cudaStreamWaitEvent(stream_, ev_aux_[3], 0));
  phase_("predict after coarsen");
  b0 = launches_;
  capture_while_(
      [&](cudaGraphConditionalHandle h) {
        for (int l = L_ - 1; l >= min_leaf_; --l)
          AF_MR_LAUNCH(mr_coarsen_level, AF_TGRIDL(l, 0, 1 << D_), d_V_, d_st_, g_, l,
                       eps_at_(l + 1), d_norms_, d_flagi_, AF_BAND(l), coarsen_pre_(l));
        predict_fill_(1, 0, min_leaf_ + 1);  // a no-op recompute when nothing merged
        launch_k(pdl_, stream_, mr_while_cond, dim3(1), 1, 0, h, d_flagi_, full_sweeps_ ? 0 : 1,
                 d_acc_ + 4);
        ++launches_;
        AF_CUDA(cudaGetLastError());
      },
      hc, true);
  *sweep_body = launches_ - b0;
  AF_CUDA(cudaStreamWaitEvent(stream_, ev_aux_[1], 0));  // mr_cycle_end
  phase_("re-sweeps");
  // no list rebuild here: the next refine works on this cycle's post-refine
  // lists, a superset of the coarsened tree's band (every node it holds
  // existed then), and rebuilds them after its splits
}

MR::CycleGraph& MR::cycle_graph_(double cfl, double fixed_dt) {
  CycleGraph& cg = cyc_[profile_ ? 1 : 0];
  if (cg.exec && cg.cfl == cfl && cg.fixed_dt == fixed_dt) return cg;
  if (cg.exec) {
    AF_CUDA(cudaStreamSynchronize(stream_));
    cudaGraphExecDestroy(cg.exec);
    cudaGraphDestroy(cg.graph);
    cg = CycleGraph{};
  }
  if (!side_stream_) {
    AF_CUDA(cudaStreamCreateWithFlags(&side_stream_, cudaStreamNonBlocking));
    AF_CUDA(cudaStreamCreateWithFlags(&fork_stream_, cudaStreamNonBlocking));
    AF_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    AF_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    for (cudaEvent_t& e : ev_aux_) AF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    AF_CUDA(cudaMalloc(&d_ckV_, sizeof(double) * NC_ * g_.total_cells));
    AF_CUDA(cudaMalloc(&d_ckSt_, g_.total_cells));
    AF_CUDA(cudaMalloc(&d_cycrec_, sizeof(af_mr_cycle) * kCycBatch));
    AF_CUDA(cudaMallocHost(&h_cycrec_, sizeof(af_mr_cycle) * kCycBatch));
    AF_CUDA(cudaMalloc(&d_cycctl_, 2 * sizeof(long long)));
    AF_CUDA(cudaMalloc(&d_acc_, 8 * sizeof(unsigned long long)));
    AF_CUDA(cudaMallocHost(&h_small_, 32 * sizeof(unsigned long long)));
  }
  harvest_events_();
  const size_t ev0 = ev_used_;
  const long l0 = launches_, s0 = stage_launches_, u0 = stage_updates_;
  long gb = 0, sb = 0;
  ev_nodes_.clear();
  fixed_grids_ = true;
  AF_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
  cycle_capture_ = true;
  try {
    enqueue_cycle_(cfl, fixed_dt, &gb, &sb);
    cycle_capture_ = false;
  } catch (...) {
    cycle_capture_ = false;
    fixed_grids_ = false;
    in_body_ = false;
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(stream_, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    throw;
  }
  AF_CUDA(cudaStreamEndCapture(stream_, &cg.graph));
  fixed_grids_ = false;
  AF_CUDA(cudaGraphInstantiate(&cg.exec, cg.graph, 0));
  cg.launches_fixed = launches_ - l0 - gb - sb;
  cg.grade_body = gb;
  cg.sweep_body = sb;
  launches_ = l0;
  stage_launches_ = s0;
  stage_updates_ = u0;
  cg.ev_nodes = ev_nodes_;  // the stage-timing event nodes, rebound to fresh events per launch
  if (cg.ev_nodes.size() != ev_used_ - ev0)
    throw Error(AF_E_CUDA, "cycle graph: stage event nodes not captured");
  ev_used_ = ev0;  // the captured records never ran
  cg.cfl = cfl;
  cg.fixed_dt = fixed_dt;
  lists_valid_ = true;
  fresh_ = true;
  virtuals_ = false;
  registers_built_ = false;
  return cg;
}

// B global-step cycles as B launches of the cycle graph and one host
// synchronisation. Returns false (state restored to the batch start) when a
// stage failed inside the batch; the caller replays it synchronously.
bool MR::run_batch_graph_(long B, double cfl, double fixed_dt, long& done, long& cycle, double& t,
                          af_mr_cycle* cycles, long max_cycles) {
  if (!lists_valid_) build_lists_();
  CycleGraph& cg = cycle_graph_(cfl, fixed_dt);
  const size_t vbytes = sizeof(double) * NC_ * g_.total_cells;
  AF_CUDA(cudaMemcpyAsync(d_ckV_, d_V_, vbytes, cudaMemcpyDeviceToDevice, stream_));
  AF_CUDA(cudaMemcpyAsync(d_ckSt_, d_st_, g_.total_cells, cudaMemcpyDeviceToDevice, stream_));
  long long* hc = reinterpret_cast<long long*>(h_small_);
  unsigned long long* ha = h_small_ + 2;
  int* he = reinterpret_cast<int*>(h_small_ + 16);
  hc[0] = done;
  hc[1] = 0;
  std::memcpy(&ha[0], &max_cfl_, 8);
  std::memcpy(&ha[1], &max_wave_, 8);
  ha[2] = ha[3] = ha[4] = 0;
  AF_CUDA(cudaMemcpyAsync(d_cycctl_, hc, 2 * sizeof(long long), cudaMemcpyHostToDevice, stream_));
  AF_CUDA(cudaMemcpyAsync(d_acc_, ha, 5 * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                          stream_));
  const size_t ev_start = ev_used_;
  for (long b = 0; b < B; ++b) {
    if (profile_ && !cg.ev_nodes.empty()) {
      while (ev_pool_.size() < ev_used_ + cg.ev_nodes.size()) {
        cudaEvent_t e;
        AF_CUDA(cudaEventCreate(&e));
        ev_pool_.push_back(e);
      }
      for (size_t i = 0; i < cg.ev_nodes.size(); ++i)
        AF_CUDA(cudaGraphExecEventRecordNodeSetEvent(cg.exec, cg.ev_nodes[i], ev_pool_[ev_used_ + i]));
      ev_used_ += cg.ev_nodes.size();
    }
    AF_CUDA(cudaGraphLaunch(cg.exec, stream_));
  }
  AF_CUDA(cudaMemcpyAsync(h_cycrec_, d_cycrec_, sizeof(af_mr_cycle) * B, cudaMemcpyDeviceToHost,
                          stream_));
  AF_CUDA(cudaMemcpyAsync(ha, d_acc_, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          stream_));
  AF_CUDA(cudaMemcpyAsync(he, d_err_, 4 * sizeof(int), cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  if (he[0] || he[2]) {
    ev_used_ = ev_start;
    AF_CUDA(cudaMemcpyAsync(d_V_, d_ckV_, vbytes, cudaMemcpyDeviceToDevice, stream_));
    AF_CUDA(cudaMemcpyAsync(d_st_, d_ckSt_, g_.total_cells, cudaMemcpyDeviceToDevice, stream_));
    AF_CUDA(cudaMemsetAsync(d_err_, 0, 4 * sizeof(int), stream_));
    AF_CUDA(cudaMemsetAsync(d_err_ + 1, 0x7f, sizeof(int), stream_));
    lists_valid_ = false;
    fresh_ = true;
    virtuals_ = false;
    return false;
  }
  launches_ += B * cg.launches_fixed + (long)ha[3] * cg.grade_body + (long)ha[4] * cg.sweep_body;
  if (phases_ && phase_ev_.size() > 1) {
    phase_ms_.resize(phase_ev_.size(), 0.0);
    for (size_t i = 1; i < phase_ev_.size(); ++i) {
      float ms = 0.f;
      AF_CUDA(cudaEventElapsedTime(&ms, phase_ev_[i - 1].second, phase_ev_[i].second));
      phase_ms_[i] += ms;
    }
    ++phase_n_;
  }
  static const bool dbg = std::getenv("AF_MR_DEBUG_LOOPS") != nullptr;
  if (dbg)
    std::fprintf(stderr, "batch of %ld cycles: %llu gradedness passes, %llu coarsen sweeps\n", B,
                 ha[3], ha[4]);
  std::memcpy(&max_cfl_, &ha[0], 8);
  std::memcpy(&max_wave_, &ha[1], 8);
  fallbacks_ += (long)ha[2];
  for (long b = 0; b < B; ++b) {
    const af_mr_cycle& r = h_cycrec_[b];
    if (cycles && cycle < max_cycles) cycles[cycle] = r;
    const double t_cycle = cfl > 0.0 ? t : static_cast<double>(done) * fixed_dt;
    t = t_cycle + static_cast<double>(r.sub) * r.dt;
    if (profile_) {
      stage_launches_ += 2;
      stage_updates_ += r.updates;
    }
    ++done;
    ++cycle;
  }
  build_lists_();  // host-side counts for the caller
  fresh_ = true;
  virtuals_ = false;
  return true;
}

void MR::run(long n_steps, double cfl, double fixed_dt, af_mr_cycle* cycles, long max_cycles,
             af_run_diag* rd) {
  if (n_steps < 0) throw Error(AF_E_ARGUMENT, "n_steps must be >= 0");
  if (!(cfl > 0.0) && !(fixed_dt > 0.0))
    throw Error(AF_E_ARGUMENT, "either cfl or fixed_dt must be positive");
  long done = 0, cycle = 0;
  double t = 0.0;
  // global time step: whole cycles replay as one graph each (run_batch_graph_)
  // (sparse bricks re-map between cycles: host-driven cycles)
  const bool graph = !opt_.local_time && !dist_ && storage_ != AF_MR_STORAGE_SPARSE &&
                     !std::getenv("AF_MR_NO_GRAPH") &&
                     !std::getenv("AF_MR_NO_CYCLE_GRAPH") && !std::getenv("AF_MR_TIMING");
  while (done < n_steps) {
    if (graph) {
      const long B = phases_ ? 1 : std::min<long>(n_steps - done, kCycBatch);
      if (run_batch_graph_(B, cfl, fixed_dt, done, cycle, t, cycles, max_cycles)) continue;
      // a stage failed inside the batch: replay it cycle by cycle from the
      // checkpoint; the synchronous path throws the reference's error there
      for (long b = 0; b < B; ++b)
        cycle_sync_(n_steps, cfl, fixed_dt, done, cycle, t, cycles, max_cycles);
      throw Error(AF_E_INTERNAL, "a failure inside a graph batch did not recur on replay");
    }
    cycle_sync_(n_steps, cfl, fixed_dt, done, cycle, t, cycles, max_cycles);
  }
  if (rd) {
    rd->max_wave_speed = max_wave_;
    rd->max_cfl = max_cfl_;
    rd->fallbacks = fallbacks_;
    rd->steps_done = done;
    rd->t = t;
  }
}

// One run_mr cycle (mr_solver.cpp:339-395) driven from the host.
void MR::cycle_sync_(long n_steps, double cfl, double fixed_dt, long& done, long& cycle,
                     double& t, af_mr_cycle* cycles, long max_cycles) {
  const double dx_L = cfg_.extent / static_cast<double>(1 << L_);
  long sub = 1;
  int top = L_;
  if (opt_.local_time) {  // mr_solver.cpp:345-354
    top = std::max(coarsest_leaf_level(), min_leaf_);
    long span = 1L << (L_ - top);
    while (span > n_steps - done) {
      span >>= 1;
      ++top;
    }
    sub = span;
  }
  const bool timing = std::getenv("AF_MR_TIMING") != nullptr;
  auto tick = [&](int slot) {
    if (!timing) return;
    AF_CUDA(cudaStreamSynchronize(stream_));
    const double now = std::chrono::duration<double>(
        std::chrono::steady_clock::now().time_since_epoch()).count();
    if (slot > 0) phase_s_[slot - 1] += now - phase_t0_;
    static const bool per_cycle = std::getenv("AF_MR_TIMING")[0] == '2';
    if (per_cycle && slot > 0)
      std::fprintf(stderr, "cycle %ld phase %d: %.3f ms\n", cycle, slot, 1e3 * (now - phase_t0_));
    phase_t0_ = now;
  };
  tick(0);
  refine(opt_.local_time ? top : -1);
  tick(1);
  add_virtual_leaves();
  long leaves = 0, nodes = 0;
  double smax = 0.0;
  cycle_stats_(&leaves, &nodes, cfl > 0.0 ? &smax : nullptr);
  double dt = fixed_dt;
  if (cfl > 0.0) dt = cfl * dx_L / smax;
  tick(2);
  cudaEvent_t te0 = nullptr, te1 = nullptr;
  if (timing) {
    cudaEventCreate(&te0);
    cudaEventCreate(&te1);
    cudaEventRecord(te0, stream_);
  }
  if (cycles && cycle < max_cycles) {
    cycles[cycle].leaves = leaves;
    cycles[cycle].nodes = nodes;
    cycles[cycle].sub = sub;
    cycles[cycle].top = top;
    cycles[cycle].dt = dt;
    long upd = 0;
    for (int l = 0; l <= L_; ++l)
      upd += 2 * leaves_per_level_[l] * (l > top ? (1L << (l - top)) : 1L);
    cycles[cycle].updates = upd;
  }
  const double t_cycle = cfl > 0.0 ? t : static_cast<double>(done) * fixed_dt;
  cur_step_ = done;
  if (opt_.local_time) build_registers_(top);
  if (timing && std::getenv("AF_MR_TIMING")[0] == '2') {
    AF_CUDA(cudaStreamSynchronize(stream_));
    std::fprintf(stderr, "cycle %ld registers built: %.3f ms since phase 2\n", cycle,
                 1e3 * (std::chrono::duration<double>(
                            std::chrono::steady_clock::now().time_since_epoch()).count() -
                        phase_t0_));
  }
  if (opt_.local_time)
    advance_local(top, t_cycle, static_cast<double>(sub) * dt, nullptr);
  else
    evolve_global(dt, nullptr);
  if (timing) {
    cudaEventRecord(te1, stream_);
    cudaEventSynchronize(te1);
    float ems = 0.f;
    cudaEventElapsedTime(&ems, te0, te1);
    evolve_gpu_ms_ += ems;
    cudaEventDestroy(te0);
    cudaEventDestroy(te1);
  }
  tick(3);
  cur_step_ = -1;
  registers_built_ = false;
  remove_virtual_leaves();
  coarsen();
  build_lists_();
  tick(4);
  lists_valid_ = true;
  done += sub;
  t = t_cycle + static_cast<double>(sub) * dt;
  ++cycle;
}

long MR::leaf_keys(uint64_t* keys, long cap) {
  std::vector<uint8_t> hs(g_.total_cells);
  wtohost_(hs.data(), d_st_, 1, 1);
  AF_CUDA(cudaStreamSynchronize(stream_));
  std::vector<uint64_t> out;
  for (int l = 0; l <= L_; ++l) {
    const int n = 1 << l;
    const long cells = mr_cells(D_, l);
    for (long c = 0; c < cells; ++c) {
      if (hs[g_.cell_off[l] + c] != ST_LEAF) continue;
      int ii, jj, kk;
      mr_ijk(g_, D_, l, c, ii, jj, kk);
      const uint64_t i = (uint64_t)ii, j = (uint64_t)jj, k = (uint64_t)kk;
      if (!row_counted(g_, l, (int)(D_ == 3 ? k : j))) continue;  // this rank's leaves
      out.push_back(((uint64_t)l << 45) | (i << 30) | (j << 15) | k);  // pack_key
    }
  }
  std::sort(out.begin(), out.end());
  if (keys)
    for (long q = 0; q < (long)out.size() && q < cap; ++q) keys[q] = out[q];
  return (long)out.size();
}

// The projections project_range_ skipped (levels below min_leaf-1), finest first.
void MR::refresh_coarse_() {
  if (!coarse_stale_) return;
  if (!lists_valid_) build_lists_();
  for (int l = std::min(min_leaf_ - 2, L_ - 1); l >= 0; --l)
    if (AF_HAS(band_count_[l]))
      AF_MR_LAUNCH(mr_project_level, AF_TGRID(l, band_count_[l]), d_V_, d_st_, g_, l, AF_BAND(l), 0);
  coarse_stale_ = false;
}

// With ranks, only this rank's rows (af_mr_local_rows) are written.
void MR::to_uniform(int level, double* aos) {
  if (level < 0 || level > L_) throw Error(AF_E_LEVEL_MISMATCH, "to_uniform: bad level");
  if (level < min_leaf_ - 1) refresh_coarse_();
  const long rowlen = D_ == 3 ? 1L << (2 * level) : 1L << level;
  int r0 = 0, r1 = 1 << level;
  if (dist_) local_rows(level, &r0, &r1);
  const long cells = (long)(r1 - r0) * rowlen;
  if (cells <= 0) return;
  sp_map_all_(d_V_);  // dense predictions below (sparse: every brick, trimmed at the next refine)
  // value_at for every cell: the band keeps predictions current only near the
  // tree; absent cells farther away get theirs here, coarsest first
  // (MRTree::to_uniform / value_at, mr_tree.cpp:171-180,608-621)
  for (int l = std::max(1, min_leaf_ + 1); l <= level; ++l)
    AF_MR_LAUNCH(mr_predict_level, grid_for(mr_cells(D_, l)), d_V_, (const uint8_t*)d_st_,
                 (const uint8_t*)(virtuals_ ? d_mark_ : nullptr), g_, l, 0, L_, (const int*)nullptr,
                 0, 0);
  fresh_ = false;
  double* tmp = nullptr;
  AF_CUDA(cudaMallocAsync((void**)&tmp, sizeof(double) * 5 * cells, stream_));
  AF_MR_LAUNCH(mr_download_level, grid_for(cells), (const double*)d_V_, tmp, g_, level, r0, r1);
  AF_CUDA(cudaMemcpyAsync(aos + 5 * (long)r0 * rowlen, tmp, sizeof(double) * 5 * cells,
                          cudaMemcpyDefault, stream_));
  AF_CUDA(cudaFreeAsync(tmp, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
}

void MR::details(int level, double* out) {
  if (level < 0 || level >= L_) throw Error(AF_E_LEVEL_MISMATCH, "details: bad level");
  const long cells = mr_cells(D_, level);
  sp_map_all_(d_V_);
  sp_map_all_(d_det_);
  AF_CUDA(cudaMemsetAsync(d_det_ + g_.cell_off[level], 0xff, sizeof(double) * cells, stream_));
  AF_MR_LAUNCH(mr_detail_level, grid_for(cells), d_V_, d_st_, d_det_, g_, level, d_norms_,
               (uint8_t*)nullptr, (const int*)nullptr, 0);
  if (g_.bsh && level > g_.bsh) {  // bricked level: back to row-major order
    double* tmp = nullptr;
    AF_CUDA(cudaMallocAsync((void**)&tmp, sizeof(double) * cells, stream_));
    AF_MR_LAUNCH(mr_level_rowmajor, grid_for(cells), (const double*)d_det_, tmp, g_, level);
    AF_CUDA(cudaMemcpyAsync(out, tmp, sizeof(double) * cells, cudaMemcpyDefault, stream_));
    AF_CUDA(cudaFreeAsync(tmp, stream_));
  } else {
    AF_CUDA(cudaMemcpyAsync(out, d_det_ + g_.cell_off[level], sizeof(double) * cells,
                            cudaMemcpyDefault, stream_));
  }
  AF_CUDA(cudaStreamSynchronize(stream_));
}

}  // namespace af
