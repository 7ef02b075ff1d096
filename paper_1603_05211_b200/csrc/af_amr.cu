// af_amr.cu — the AMR patch path: PatchHierarchy
// (amr_hierarchy.cpp), flag_cells + cluster (amr_cluster.cpp) and the run_amr
// cycle (amr_solver.cpp) on the device. Layout and kernels: af_amr_kernels.cuh.
#include "af_amr.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <tuple>

#include "af_amr_kernels.cuh"
#include "af_cases.h"

namespace af {

namespace {

constexpr int kRecCap = 1 << 16;

inline unsigned blocks_for(long n) { return (unsigned)((n + 255) / 256); }

std::string f6(double v) {  // std::to_string(double)
  char b[64];
  std::snprintf(b, sizeof b, "%f", v);
  return b;
}

// ---------------------------------------------------------------- cluster --
struct ClusterJob {
  const uint8_t* flags;
  const uint8_t* allowed;
  int dim;
  int n[3];
  double efficiency;
  std::vector<ABox>* out;
  bool flag(int i, int j, int k) const { return flags[((size_t)k * n[1] + j) * n[0] + i] != 0; }
  bool ok(int i, int j, int k) const { return allowed[((size_t)k * n[1] + j) * n[0] + i] != 0; }
};

// tight bounding box of the flagged cells of `region` and their count
ABox shrink(const ClusterJob& J, const ABox& region, long& flagged) {
  ABox b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = INT32_MAX;
    b.hi[a] = INT32_MIN;
  }
  flagged = 0;
  for (int k = region.lo[2]; k < region.hi[2]; ++k)
    for (int j = region.lo[1]; j < region.hi[1]; ++j)
      for (int i = region.lo[0]; i < region.hi[0]; ++i) {
        if (!J.flag(i, j, k)) continue;
        ++flagged;
        const int c[3] = {i, j, k};
        for (int a = 0; a < 3; ++a) {
          b.lo[a] = std::min(b.lo[a], c[a]);
          b.hi[a] = std::max(b.hi[a], c[a] + 1);
        }
      }
  return b;
}

bool inside_allowed(const ClusterJob& J, const ABox& b) {
  if (!J.allowed) return true;
  for (int k = b.lo[2]; k < b.hi[2]; ++k)
    for (int j = b.lo[1]; j < b.hi[1]; ++j)
      for (int i = b.lo[0]; i < b.hi[0]; ++i)
        if (!J.ok(i, j, k)) return false;
  return true;
}

void bisect(const ClusterJob& J, const ABox& region) {
  long flagged = 0;
  const ABox b = shrink(J, region, flagged);
  if (flagged == 0) return;
  const long vol = b.volume();
  const double fill = (double)flagged / (double)vol;
  if ((fill >= J.efficiency && inside_allowed(J, b)) || vol == 1) {
    J.out->push_back(b);
    return;
  }
  int axis = -1, cut = -1, best = -1;
  for (int a = 0; a < J.dim; ++a) {
    if (b.extent(a) < 2) continue;
    std::vector<long> sig((size_t)b.extent(a), 0);
    for (int k = b.lo[2]; k < b.hi[2]; ++k)
      for (int j = b.lo[1]; j < b.hi[1]; ++j)
        for (int i = b.lo[0]; i < b.hi[0]; ++i)
          if (J.flag(i, j, k)) ++sig[(size_t)((a == 0 ? i : a == 1 ? j : k) - b.lo[a])];
    int score = 0;
    const int off = propose_cut_t(sig.data(), (int)sig.size(), &score);
    const int pos = off < 0 ? -1 : b.lo[a] + off;
    if (pos > b.lo[a] && pos < b.hi[a] && score > best) {
      best = score;
      axis = a;
      cut = pos;
    }
  }
  if (axis < 0) {  // halve the longest axis (the first among equals)
    for (int a = 0; a < J.dim; ++a)
      if (axis < 0 || b.extent(a) > b.extent(axis)) axis = a;
    if (b.extent(axis) < 2) {
      J.out->push_back(b);
      return;
    }
    cut = b.lo[axis] + b.extent(axis) / 2;
  }
  ABox lo = b, hi = b;
  lo.hi[axis] = cut;
  hi.lo[axis] = cut;
  bisect(J, lo);
  bisect(J, hi);
}

}  // namespace

std::vector<ABox> amr_cluster(const uint8_t* flags, const uint8_t* allowed, int dim, int n0, int n1,
                              int n2, double efficiency) {
  std::vector<ABox> out;
  ClusterJob J{flags, allowed, dim, {n0, n1, n2}, efficiency, &out};
  ABox all;
  all.hi[0] = n0;
  all.hi[1] = n1;
  all.hi[2] = n2;
  bisect(J, all);
  std::sort(out.begin(), out.end(), [](const ABox& a, const ABox& b) {
    return std::tie(a.lo[2], a.lo[1], a.lo[0]) < std::tie(b.lo[2], b.lo[1], b.lo[0]);
  });
  return out;
}

// ------------------------------------------------------- device clustering --
namespace {
constexpr int kClusterLevels = 4000;  // frontier counters (the bisection depth bound)
constexpr int kClusterChunk = 12;     // levels launched between two looks at the frontier
}  // namespace

DeviceCluster::~DeviceCluster() {
  cudaFree(Sf_);
  cudaFree(Sa_);
  cudaFree(qa_);
  cudaFree(qb_);
  cudaFree(out_);
  cudaFree(hdr_);
  cudaFreeHost(h_pin_);
}

std::vector<ABox> DeviceCluster::run(int dim, const uint8_t* d_flags, const uint8_t* d_allowed, int n,
                                     double efficiency, long* launches) {
  const long np = n + 1;
  const long sat = dim == 3 ? np * np * np : np * np;
  const long cells = dim == 3 ? (long)n * n * n : (long)n * n;
  if (sat > sat_cap_) {
    AF_CUDA(cudaStreamSynchronize(stream_));
    cudaFree(Sf_);
    cudaFree(Sa_);
    AF_CUDA(cudaMalloc(&Sf_, sizeof(int) * sat));
    AF_CUDA(cudaMalloc(&Sa_, sizeof(int) * sat));
    sat_cap_ = sat;
  }
  const int want = (int)std::min<long>(cells + 2, 1 << 20);
  if (want > cap_) {
    AF_CUDA(cudaStreamSynchronize(stream_));
    cudaFree(qa_);
    cudaFree(qb_);
    cudaFree(out_);
    AF_CUDA(cudaMalloc(&qa_, sizeof(CBox) * want));
    AF_CUDA(cudaMalloc(&qb_, sizeof(CBox) * want));
    AF_CUDA(cudaMalloc(&out_, sizeof(CBox) * want));
    cap_ = want;
  }
  if (!hdr_) AF_CUDA(cudaMalloc(&hdr_, sizeof(int) * (kClusterLevels + 2)));
  auto sat_build = [&](const uint8_t* mask, int* S) {
    const long rows = dim == 3 ? (long)n * n : n;
    if (dim == 3) {
      amr_sat_x_kernel<3><<<(unsigned)((rows + 127) / 128), 128, 0, stream_>>>(mask, n, S);
      amr_sat_y_kernel<3><<<(unsigned)((np * n + 127) / 128), 128, 0, stream_>>>(n, S);
      amr_sat_z_kernel<<<(unsigned)((np * np + 127) / 128), 128, 0, stream_>>>(n, S);
      *launches += 3;
    } else {
      amr_sat_x_kernel<2><<<(unsigned)((rows + 127) / 128), 128, 0, stream_>>>(mask, n, S);
      amr_sat_y_kernel<2><<<(unsigned)((np + 127) / 128), 128, 0, stream_>>>(n, S);
      *launches += 2;
    }
  };
  sat_build(d_flags, Sf_);
  if (d_allowed) sat_build(d_allowed, Sa_);
  CBox root;
  for (int a = 0; a < 3; ++a) {
    root.lo[a] = 0;
    root.hi[a] = a < dim ? n : 1;
  }
  AF_CUDA(cudaMemsetAsync(hdr_, 0, sizeof(int) * (kClusterLevels + 2), stream_));
  const int one = 1;
  AF_CUDA(cudaMemcpyAsync(hdr_ + 2, &one, sizeof(int), cudaMemcpyHostToDevice, stream_));
  AF_CUDA(cudaMemcpyAsync(qa_, &root, sizeof(CBox), cudaMemcpyHostToDevice, stream_));
  const size_t smem = sizeof(int) * (size_t)n;
  if (smem > 48 * 1024) {
    AF_CUDA(cudaFuncSetAttribute(amr_cluster_level_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    AF_CUDA(cudaFuncSetAttribute(amr_cluster_level_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  // pinned landing zone: the counters and the first boxes in one round trip
  constexpr int kBoxPrefix = 2048;
  if (!h_pin_)
    AF_CUDA(cudaMallocHost(&h_pin_, sizeof(int) * (kClusterLevels + 2) + sizeof(CBox) * kBoxPrefix));
  int* hdr = static_cast<int*>(h_pin_);
  CBox* hbox = reinterpret_cast<CBox*>(hdr + kClusterLevels + 2);
  int level = 0;
  for (;;) {
    for (int k = 0; k < kClusterChunk && level < kClusterLevels - 1; ++k, ++level) {
      const CBox* in = static_cast<const CBox*>((level & 1) ? qb_ : qa_);
      CBox* next = static_cast<CBox*>((level & 1) ? qa_ : qb_);
      if (dim == 3)
        amr_cluster_level_kernel<3><<<592, 128, smem, stream_>>>(in, hdr_ + 2 + level, next, hdr_ + 3 + level,
                                                                 static_cast<CBox*>(out_), hdr_, cap_, Sf_,
                                                                 d_allowed ? Sa_ : nullptr, n, efficiency, hdr_ + 1);
      else
        amr_cluster_level_kernel<2><<<592, 128, smem, stream_>>>(in, hdr_ + 2 + level, next, hdr_ + 3 + level,
                                                                 static_cast<CBox*>(out_), hdr_, cap_, Sf_,
                                                                 d_allowed ? Sa_ : nullptr, n, efficiency, hdr_ + 1);
      ++*launches;
    }
    AF_CUDA(cudaGetLastError());
    AF_CUDA(cudaMemcpyAsync(hdr, hdr_, sizeof(int) * (size_t)(3 + level), cudaMemcpyDeviceToHost, stream_));
    AF_CUDA(cudaMemcpyAsync(hbox, out_, sizeof(CBox) * (size_t)std::min(cap_, kBoxPrefix), cudaMemcpyDeviceToHost,
                            stream_));
    AF_CUDA(cudaStreamSynchronize(stream_));
    if (hdr[1]) throw Error(AF_E_INTERNAL, "cluster: box queue overflow");
    if (hdr[(size_t)2 + level] == 0) break;
    if (level >= kClusterLevels - 1) throw Error(AF_E_INTERNAL, "cluster: bisection deeper than its bound");
  }
  std::vector<CBox> got((size_t)hdr[0]);
  if ((int)got.size() <= kBoxPrefix) {
    std::copy(hbox, hbox + got.size(), got.begin());
  } else {
    AF_CUDA(cudaMemcpyAsync(got.data(), out_, sizeof(CBox) * got.size(), cudaMemcpyDeviceToHost, stream_));
    AF_CUDA(cudaStreamSynchronize(stream_));
  }
  std::vector<ABox> out(got.size());
  for (size_t i = 0; i < got.size(); ++i)
    for (int a = 0; a < 3; ++a) {
      out[i].lo[a] = got[i].lo[a];
      out[i].hi[a] = got[i].hi[a];
    }
  std::sort(out.begin(), out.end(), [](const ABox& a, const ABox& b) {
    return std::tie(a.lo[2], a.lo[1], a.lo[0]) < std::tie(b.lo[2], b.lo[1], b.lo[0]);
  });
  return out;
}

// -------------------------------------------------------------- hierarchy --
namespace {
template <int D, class LevelT>
ALv<D> view(const LevelT& L) {
  ALv<D> v;
  v.n = L.n;
  v.cells = L.cells;
  v.pid = L.pid;
  v.ring = nullptr;
  v.U = L.U;
  v.Uold = L.Uold;
  v.G = L.G;
  v.Gold = L.Gold;
  v.boxes = L.d_boxes;
  v.nb = (int)L.boxes.size();
  v.off0 = L.d_off;
  v.off1 = L.d_off + (v.nb + 1);
  v.off2 = L.d_off + 2 * (v.nb + 1);
  v.offF = L.d_off + 3 * (v.nb + 1);
  v.tot0 = L.total;
  v.tot1 = L.tot1;
  v.tot2 = L.tot2;
  v.totF = L.totF;
  return v;
}
__global__ void amr_clear_regs_kernel(double* Rc, double* Rf, uint8_t* has, long nvals, int nslots) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nvals;
       i += (long)gridDim.x * blockDim.x) {
    Rc[i] = 0.0;
    Rf[i] = 0.0;
    if (i < nslots) has[i] = 0;
  }
}
}  // namespace

#define AMR_VIEW(D, L) view<D>(L)

Amr::Amr(const af_config& cfg, const af_amr_options& opt) : cfg_(cfg), opt_(opt) {
  dim_ = cfg.dim;
  base_exp_ = cfg.level;
  if (dim_ != 2 && dim_ != 3) throw Error(AF_E_CONFIG, "amr: dim must be 2 or 3");
  if (base_exp_ < 0 || opt.max_levels < 0 || base_exp_ + opt.max_levels > (dim_ == 3 ? 9 : 14))
    throw Error(AF_E_CONFIG, "amr: base level / max_levels out of range");
  AF_CUDA(cudaSetDevice(cfg.device));
  AF_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  AF_CUDA(cudaMalloc(&d_err_, 4 * sizeof(int)));
  AF_CUDA(cudaMemset(d_err_, 0, 4 * sizeof(int)));
  AF_CUDA(cudaMalloc(&d_flag_, 4 * sizeof(int)));
  AF_CUDA(cudaMalloc(&d_rec_, sizeof(ARec) * kRecCap));
  AF_CUDA(cudaMemset(d_rec_, 0, sizeof(ARec) * kRecCap));
  spare_.resize((size_t)opt.max_levels + 1);
  clusterer_ = new DeviceCluster(stream_);
  // level 0: one patch over the whole domain (amr_hierarchy.cpp:41-56)
  Level L;
  alloc_level(L, 0);
  ABox all;
  const int n = cells_per_axis(0);
  all.hi[0] = n;
  all.hi[1] = n;
  all.hi[2] = dim_ == 3 ? n : 1;
  L.boxes.push_back(all);
  lv_.push_back(L);
  if (dim_ == 3) rebuild_domain_t<3>(0, false); else rebuild_domain_t<2>(0, false);
}

Amr::~Amr() {
  cudaStreamSynchronize(stream_);
  if (std::getenv("AF_AMR_TRACE"))
    std::fprintf(stderr, "AF_AMR_TRACE: remesh %.4f s in %ld calls, of which clustering (tables, bisection, "
                 "box list round trip) %.4f s; %ld launches\n", remesh_seconds_, remesh_calls_, cluster_seconds_,
                 launches_);
  for (Level& L : lv_) free_level(L);
  for (Level& L : spare_) free_level(L);
  delete clusterer_;
  cudaFree(d_cb_);
  cudaFree(d_cboff_);
  cudaFree(d_err_);
  cudaFree(d_flag_);
  cudaFree(d_rec_);
  cudaFree(W_);
  cudaFree(DU_);
  cudaFree(F_);
  cudaFree(m_flags_);
  cudaFree(m_tmp_);
  cudaFree(m_nest_);
  cudaFree(m_allowed_);
  cudaFree(m_masked_);
  cudaStreamDestroy(stream_);
}

void Amr::alloc_level(Level& L, int l) {
  if (spare_[l].U) {  // reuse the arrays of a level popped earlier
    L = spare_[l];
    spare_[l] = Level();
    L.boxes.clear();
    return;
  }
  L.n = cells_per_axis(l);
  L.cells = dim_ == 3 ? (long)L.n * L.n * L.n : (long)L.n * L.n;
  const size_t fb = sizeof(double) * (size_t)(dim_ + 2) * (size_t)L.cells;
  AF_CUDA(cudaMalloc(&L.pid, sizeof(int) * L.cells));
  AF_CUDA(cudaMalloc(&L.pid_new, sizeof(int) * L.cells));
  AF_CUDA(cudaMalloc(&L.U, fb));
  AF_CUDA(cudaMalloc(&L.Uold, fb));
  AF_CUDA(cudaMalloc(&L.G, fb));
  AF_CUDA(cudaMalloc(&L.Gold, fb));
  AF_CUDA(cudaMalloc(&L.regbase, sizeof(int) * L.cells));
  AF_CUDA(cudaMalloc(&L.regmask, L.cells));
  AF_CUDA(cudaMemsetAsync(L.pid, 0xff, sizeof(int) * L.cells, stream_));
  AF_CUDA(cudaMemsetAsync(L.regmask, 0, L.cells, stream_));
  AF_CUDA(cudaMemsetAsync(L.U, 0, fb, stream_));
  AF_CUDA(cudaMemsetAsync(L.Uold, 0, fb, stream_));
  AF_CUDA(cudaMemsetAsync(L.G, 0, fb, stream_));
  AF_CUDA(cudaMemsetAsync(L.Gold, 0, fb, stream_));
  ensure_scratch(L.cells, L.n);
}

void Amr::free_level(Level& L) {
  cudaFree(L.pid);
  cudaFree(L.pid_new);
  cudaFree(L.U);
  cudaFree(L.Uold);
  cudaFree(L.G);
  cudaFree(L.Gold);
  cudaFree(L.d_boxes);
  cudaFree(L.d_off);
  cudaFree(L.regbase);
  cudaFree(L.regmask);
  cudaFree(L.slot_cell);
  cudaFree(L.slot_face);
  cudaFree(L.has);
  cudaFree(L.Rc);
  cudaFree(L.Rf);
  L = Level();
}

void Amr::ensure_scratch(long cells, int n) {
  if (cells <= scr_cells_) return;
  AF_CUDA(cudaStreamSynchronize(stream_));
  cudaFree(W_);
  cudaFree(DU_);
  cudaFree(F_);
  cudaFree(m_flags_);
  cudaFree(m_tmp_);
  cudaFree(m_nest_);
  cudaFree(m_allowed_);
  cudaFree(m_masked_);
  const int nc = dim_ + 2;
  const long np = n + 2;
  const long padded = dim_ == 3 ? np * np * np : np * np;
  const long per = dim_ == 3 ? (long)(n + 1) * n * n : (long)(n + 1) * n;
  AF_CUDA(cudaMalloc(&W_, sizeof(double) * nc * cells));
  AF_CUDA(cudaMalloc(&DU_, sizeof(double) * nc * padded));
  AF_CUDA(cudaMalloc(&F_, sizeof(double) * nc * dim_ * per));
  AF_CUDA(cudaMalloc(&m_flags_, cells));
  AF_CUDA(cudaMalloc(&m_tmp_, cells));
  AF_CUDA(cudaMalloc(&m_nest_, cells));
  AF_CUDA(cudaMalloc(&m_allowed_, cells));
  AF_CUDA(cudaMalloc(&m_masked_, cells));
  scr_cells_ = cells;
}

static ABc bc_of(const af_config& c) {
  ABc b;
  for (int i = 0; i < 6; ++i) b.bc[i] = c.bc[i];
  return b;
}

void Amr::upload_boxes(Level& L) {
  const int nb = (int)L.boxes.size();
  std::vector<int> bx((size_t)6 * nb);
  const size_t stride = (size_t)nb + 1;
  std::vector<long> off(3 * stride + (size_t)nb * dim_ + 1, 0);
  long* o0 = off.data();
  long* o1 = o0 + stride;
  long* o2 = o1 + stride;
  long* oF = o2 + stride;
  for (int i = 0; i < nb; ++i) {
    const ABox& b = L.boxes[i];
    long v1 = 1, v2 = 1;
    for (int a = 0; a < 3; ++a) {
      bx[6 * i + a] = b.lo[a];
      bx[6 * i + 3 + a] = b.hi[a];
      v1 *= b.extent(a) + (a < dim_ ? 2 : 0);
      v2 *= b.extent(a) + (a < dim_ ? 4 : 0);
    }
    o0[i + 1] = o0[i] + b.volume();
    o1[i + 1] = o1[i] + v1;
    o2[i + 1] = o2[i] + v2;
    for (int a = 0; a < dim_; ++a)
      oF[i * dim_ + a + 1] = oF[i * dim_ + a] + b.volume() / b.extent(a) * (b.extent(a) + 1);
  }
  L.total = o0[nb];
  L.tot1 = o1[nb];
  L.tot2 = o2[nb];
  L.totF = oF[(size_t)nb * dim_];
  if (nb + 1 > L.box_cap) {
    AF_CUDA(cudaStreamSynchronize(stream_));
    cudaFree(L.d_boxes);
    cudaFree(L.d_off);
    L.box_cap = 2 * (nb + 1) + 64;
    AF_CUDA(cudaMalloc(&L.d_boxes, sizeof(int) * 6 * L.box_cap));
    AF_CUDA(cudaMalloc(&L.d_off, sizeof(long) * 7 * L.box_cap));
  }
  // pageable sources: the copies are staged before the calls return
  AF_CUDA(cudaMemcpyAsync(L.d_boxes, bx.data(), sizeof(int) * 6 * nb, cudaMemcpyHostToDevice, stream_));
  AF_CUDA(cudaMemcpyAsync(L.d_off, off.data(), sizeof(long) * off.size(), cudaMemcpyHostToDevice, stream_));
}

void Amr::save_level(int l, bool restore) {
  Level& L = lv_[l];
  if (dim_ == 3)
    amr_save_kernel<3><<<blocks_for(L.tot2), 256, 0, stream_>>>(AMR_VIEW(3, L), bc_of(cfg_), restore ? 1 : 0, d_err_);
  else
    amr_save_kernel<2><<<blocks_for(L.tot2), 256, 0, stream_>>>(AMR_VIEW(2, L), bc_of(cfg_), restore ? 1 : 0, d_err_);
  launch_count();
}

// rebuild_domain (amr_hierarchy.cpp:58-62): the patch-id map of the level's
// boxes (into pid_new while the old map is still needed) and the position lists
template <int D>
void Amr::rebuild_domain_t(int l, bool into_new) {
  Level& L = lv_[l];
  upload_boxes(L);
  int* pid = into_new ? L.pid_new : L.pid;
  AF_CUDA(cudaMemsetAsync(pid, 0xff, sizeof(int) * L.cells, stream_));
  if (L.total)
    amr_setpid_kernel<D><<<blocks_for(L.total), 256, 0, stream_>>>(L.d_boxes, L.d_off,
                                                                   (int)L.boxes.size(), L.total, L.n, pid);
  launch_count();
  AF_CUDA(cudaGetLastError());
}

template <int D>
void Amr::sync_t(int l, double tau) {
  Level& L = lv_[l];
  double theta = 1.0;
  if (l > 0) {  // amr_hierarchy.cpp:184-188
    const Level& C = lv_[l - 1];
    const double denom = C.t - C.t_old;
    theta = denom > 0.0 ? std::min(std::max((tau - C.t_old) / denom, 0.0), 1.0) : 1.0;
  }
  const ALv<D> fine = AMR_VIEW(D, L);
  const ALv<D> coarse = l > 0 ? AMR_VIEW(D, lv_[l - 1]) : fine;
  amr_sync_kernel<D><<<blocks_for(L.tot2), 256, 0, stream_>>>(fine, coarse, l > 0, bc_of(cfg_), theta,
                                                               cfg_.gamma - 1.0, d_err_);
  launch_count();
  AF_CUDA(cudaGetLastError());
}

void Amr::sync_ghosts(int l, double tau) {
  if (l < 0 || l >= n_levels()) throw Error(AF_E_ARGUMENT, "sync_ghosts: no such level");
  if (dim_ == 3) sync_t<3>(l, tau); else sync_t<2>(l, tau);
}

void Amr::initialize(amr_ic_fn ic, void* user) {
  if (!ic) throw Error(AF_E_ARGUMENT, "initialize: null initial condition");
  // fill_from_ic (amr_hierarchy.cpp:109-122): the patch interiors from the
  // initial condition at the cell centres, data_old = data
  auto fill = [&](int l) {
    Level& L = lv_[l];
    const double h = dx(l);
    std::vector<double> aos((size_t)5 * L.total);
    size_t t = 0;
    for (const ABox& b : L.boxes)
      for (int k = b.lo[2]; k < b.hi[2]; ++k)
        for (int j = b.lo[1]; j < b.hi[1]; ++j)
          for (int i = b.lo[0]; i < b.hi[0]; ++i, ++t)
            ic(cfg_.origin + (i + 0.5) * h, cfg_.origin + (j + 0.5) * h,
               dim_ == 3 ? cfg_.origin + (k + 0.5) * h : 0.0, &aos[5 * t], user);
    double* d = nullptr;
    AF_CUDA(cudaMalloc(&d, sizeof(double) * aos.size()));
    AF_CUDA(cudaMemcpyAsync(d, aos.data(), sizeof(double) * aos.size(), cudaMemcpyHostToDevice, stream_));
    if (dim_ == 3)
      amr_put_kernel<3><<<blocks_for(L.total), 256, 0, stream_>>>(L.d_boxes, L.d_off, (int)L.boxes.size(),
                                                                  L.total, L.n, L.cells, d, L.U);
    else
      amr_put_kernel<2><<<blocks_for(L.total), 256, 0, stream_>>>(L.d_boxes, L.d_off, (int)L.boxes.size(),
                                                                  L.total, L.n, L.cells, d, L.U);
    launch_count();
    save_level(l, false);
    AF_CUDA(cudaStreamSynchronize(stream_));
    cudaFree(d);
  };
  fill(0);
  for (int pass = 0; pass < opt_.max_levels + 2; ++pass) {
    remesh(0);
    for (int l = 1; l < n_levels(); ++l) fill(l);
    if (n_levels() == opt_.max_levels + 1 && pass > 0) break;
  }
  for (int l = 0; l < n_levels(); ++l) {
    sync_ghosts(l, 0.0);
    save_level(l, false);
  }
  check();
}

// remesh (amr_hierarchy.cpp:216-342)
template <int D>
void Amr::remesh_t(int l) {
  const int deepest = n_levels() - 1;
  const int top = std::min(deepest + 1, opt_.max_levels);
  const ABc b = bc_of(cfg_);
  const double gm1 = cfg_.gamma - 1.0;
  std::vector<std::vector<ABox>> fresh((size_t)top + 2);
  for (int m = top; m >= l + 1; --m) {
    const int src = m - 1;
    if (src > deepest) continue;
    Level& S = lv_[src];
    sync_ghosts(src, S.t);
    const unsigned g = blocks_for(S.cells);
    AF_CUDA(cudaMemsetAsync(m_tmp_, 0, S.cells, stream_));
    amr_flag_kernel<D><<<blocks_for(S.total), 256, 0, stream_>>>(AMR_VIEW(D, S), b, gm1, opt_.eps_rho, opt_.eps_p,
                                                                m_tmp_);
    const uint8_t* nest = nullptr;
    if (m + 1 <= top && !fresh[m + 1].empty()) {
      // the next finer level's new boxes, coarsened twice and dilated, stay covered
      std::vector<int> cb;
      std::vector<long> cboff(1, 0);
      for (const ABox& fb : fresh[m + 1]) {
        int lo[3], hi[3];
        long vol = 1;
        for (int a = 0; a < 3; ++a) {
          lo[a] = std::max(fb.lo[a] >> 2, 0);
          hi[a] = std::min((fb.hi[a] + 3) >> 2, a < D ? S.n : 1);
          if (a >= D) {
            lo[a] = 0;
            hi[a] = 1;
          }
          vol *= std::max(hi[a] - lo[a], 0);
        }
        if (vol == 0) continue;
        cb.insert(cb.end(), {lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]});
        cboff.push_back(cboff.back() + vol);
      }
      if ((long)cb.size() > cb_cap_) {
        AF_CUDA(cudaStreamSynchronize(stream_));
        cudaFree(d_cb_);
        cudaFree(d_cboff_);
        cb_cap_ = 2 * (long)cb.size() + 384;
        AF_CUDA(cudaMalloc(&d_cb_, sizeof(int) * cb_cap_));
        AF_CUDA(cudaMalloc(&d_cboff_, sizeof(long) * (cb_cap_ / 6 + 2)));
      }
      AF_CUDA(cudaMemcpyAsync(d_cb_, cb.data(), sizeof(int) * cb.size(), cudaMemcpyHostToDevice, stream_));
      AF_CUDA(cudaMemcpyAsync(d_cboff_, cboff.data(), sizeof(long) * cboff.size(), cudaMemcpyHostToDevice, stream_));
      AF_CUDA(cudaMemsetAsync(m_masked_, 0, S.cells, stream_));
      if (cboff.back())
        amr_setbox_kernel<D><<<blocks_for(cboff.back()), 256, 0, stream_>>>(d_cb_, d_cboff_, (int)(cb.size() / 6),
                                                                            cboff.back(), S.n, m_masked_);
      amr_dilate_kernel<D><<<g, 256, 0, stream_>>>(m_masked_, S.n, b, 1, nullptr, m_nest_);
      launch_count(2);
      nest = m_nest_;
    }
    amr_dilate_kernel<D><<<g, 256, 0, stream_>>>(m_tmp_, S.n, b, 1, nest, m_flags_);
    amr_allowed_kernel<D><<<g, 256, 0, stream_>>>(S.pid, S.n, b, m_flags_, m_allowed_, m_masked_, d_flag_);
    launch_count(3);
    const auto tc0 = std::chrono::steady_clock::now();
    const std::vector<ABox> clustered = cluster_device<D>(m_masked_, m_allowed_, S.n, opt_.cluster_efficiency);
    cluster_seconds_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - tc0).count();
    for (const ABox& cbx : clustered) {
      ABox r;  // Box::refined (amr.hpp:49-64)
      for (int a = 0; a < D; ++a) {
        r.lo[a] = 2 * cbx.lo[a];
        r.hi[a] = 2 * cbx.hi[a];
      }
      fresh[m].push_back(r);
    }
  }

  // the new levels bottom-up: previous values where refined before, the
  // coarse interpolation elsewhere
  int new_top = l;
  for (int m = l + 1; m <= top && !fresh[m].empty(); ++m) {
    const bool had = m <= deepest;
    if (!had) {
      Level L;
      alloc_level(L, m);
      lv_.push_back(L);
    }
    Level& L = lv_[m];
    L.boxes = fresh[m];
    L.t = lv_[l].t;
    L.t_old = lv_[l].t;
    rebuild_domain_t<D>(m, /*into_new=*/true);
    ALv<D> nv = AMR_VIEW(D, L);
    nv.pid = L.pid_new;
    amr_build_kernel<D><<<blocks_for(L.total), 256, 0, stream_>>>(nv, L.pid, had ? 1 : 0,
                                                                 AMR_VIEW(D, lv_[m - 1]), b, gm1, d_err_);
    launch_count();
    std::swap(L.pid, L.pid_new);
    sync_ghosts(m, L.t);
    save_level(m, false);  // data_old = data, interiors and the fresh ghosts
    new_top = m;
  }
  while (n_levels() - 1 > new_top) {
    const int idx = n_levels() - 1;
    AF_CUDA(cudaStreamSynchronize(stream_));
    spare_[idx] = lv_.back();
    spare_[idx].boxes.clear();
    lv_.pop_back();
  }
  // registers of the rebuilt pairs restart; pairs below l keep accumulating
  for (int m = l; m < n_levels(); ++m) rebuild_registers(m);
  // NestingViolation (amr_hierarchy.cpp:340-341), reported by the next check()
  for (int m = std::max(l, 1); m < n_levels(); ++m) {
    amr_nested_kernel<D><<<blocks_for(lv_[m].total), 256, 0, stream_>>>(AMR_VIEW(D, lv_[m]), lv_[m - 1].pid,
                                                                        d_err_ + 2);
    launch_count();
  }
  AF_CUDA(cudaGetLastError());
}

void Amr::remesh(int l) {
  if (l < 0 || l >= n_levels()) throw Error(AF_E_ARGUMENT, "remesh: no such level");
  // a stage that failed earlier in the cycle is reported against the boxes it
  // ran on, so before they change (remesh synchronises for the flag masks anyway)
  check();
  const auto t0 = std::chrono::steady_clock::now();
  if (dim_ == 3) remesh_t<3>(l); else remesh_t<2>(l);
  remesh_seconds_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  ++remesh_calls_;
}

void Amr::rebuild_registers(int l) {
  Level& L = lv_[l];
  L.nslots = 0;
  if (l + 1 >= n_levels()) return;
  const Level& Fn = lv_[l + 1];
  // every register face is a coarse face of a fine box's surface: an upper
  // bound the host knows without asking the device
  long bound = 0;
  for (const ABox& fb : Fn.boxes)
    for (int a = 0; a < dim_; ++a) {
      long area = 1;
      for (int t = 0; t < dim_; ++t)
        if (t != a) area *= fb.extent(t) / 2;
      bound += 2 * area;
    }
  if (bound > L.slot_cap) {
    AF_CUDA(cudaStreamSynchronize(stream_));
    cudaFree(L.slot_cell);
    cudaFree(L.slot_face);
    cudaFree(L.has);
    cudaFree(L.Rc);
    cudaFree(L.Rf);
    L.slot_cap = (int)(bound + bound / 2 + 64);
    AF_CUDA(cudaMalloc(&L.slot_cell, sizeof(long) * L.slot_cap));
    AF_CUDA(cudaMalloc(&L.slot_face, L.slot_cap));
    AF_CUDA(cudaMalloc(&L.has, L.slot_cap));
    AF_CUDA(cudaMalloc(&L.Rc, sizeof(double) * (dim_ + 2) * L.slot_cap));
    AF_CUDA(cudaMalloc(&L.Rf, sizeof(double) * (dim_ + 2) * L.slot_cap));
  }
  L.nslots = (int)bound;  // slots past the device's count stay unused (face 0xff)
  const ABc b = bc_of(cfg_);
  AF_CUDA(cudaMemsetAsync(d_flag_, 0, 2 * sizeof(int), stream_));
  AF_CUDA(cudaMemsetAsync(L.slot_face, 0xff, L.nslots, stream_));
  if (dim_ == 3)
    amr_reg_alloc_kernel<3><<<blocks_for(L.total), 256, 0, stream_>>>(AMR_VIEW(3, L), Fn.pid, b, L.regbase, L.regmask,
                                                                      d_flag_, L.slot_cell, L.slot_face, L.nslots,
                                                                      d_err_);
  else
    amr_reg_alloc_kernel<2><<<blocks_for(L.total), 256, 0, stream_>>>(AMR_VIEW(2, L), Fn.pid, b, L.regbase, L.regmask,
                                                                      d_flag_, L.slot_cell, L.slot_face, L.nslots,
                                                                      d_err_);
  launch_count();
  clear_registers(l);
  AF_CUDA(cudaGetLastError());
}

void Amr::clear_registers(int l) {
  Level& L = lv_[l];
  if (!L.nslots) return;
  const long nvals = (long)(dim_ + 2) * L.nslots;
  amr_clear_regs_kernel<<<std::min<unsigned>(blocks_for(nvals), 1184), 256, 0, stream_>>>(L.Rc, L.Rf, L.has,
                                                                                         nvals, L.nslots);
  launch_count();
}

// update_level (amr_hierarchy.cpp:464-528)
template <int D, int S>
void Amr::update_t(int l, double dt) {
  Level& L = lv_[l];
  if ((int)calls_.size() >= kRecCap) check();
  const int call = (int)calls_.size();
  calls_.push_back({l, dt});
  ARec* rec = static_cast<ARec*>(d_rec_) + call;
  const ABc b = bc_of(cfg_);
  const ALv<D> v = AMR_VIEW(D, L);
  const int n = L.n;
  const double h = dx(l), inv_dx = 1.0 / h, gamma = cfg_.gamma;
  const unsigned gc = blocks_for(L.total), gb = blocks_for(L.tot2), gf = blocks_for(L.totF);

  cell_updates_ += L.total * (cfg_.integrator == AF_INTEGRATOR_MUSCL_HANCOCK ? 1 : 2);
  L.t_old = L.t;
  save_level(l, false);  // p.data_old = p.data
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (profile_) {
    AF_CUDA(cudaEventCreate(&e0));
    AF_CUDA(cudaEventCreate(&e1));
    AF_CUDA(cudaEventRecord(e0, stream_));
  }
  auto stepped = [&](int kernels) {
    if (!profile_) return;
    AF_CUDA(cudaEventRecord(e1, stream_));
    events_.emplace_back(e0, e1);
    stage_launches_ += kernels;
    stage_updates_ += L.total * (cfg_.integrator == AF_INTEGRATOR_MUSCL_HANCOCK ? 1 : 2);
  };

  auto registers = [&] {  // accumulate_registers, fine side then coarse side
    if (l > 0 && lv_[l - 1].nslots) {
      Level& C = lv_[l - 1];
      amr_reg_fine_kernel<D><<<blocks_for(C.nslots), 256, 0, stream_>>>(
          C.slot_cell, C.slot_face, C.nslots, C.n, n, F_, dt * (D == 3 ? 0.25 : 0.5), C.Rf, C.has, d_err_);
      launch_count();
    }
    if (l + 1 < n_levels() && L.nslots) {
      amr_reg_coarse_kernel<D><<<blocks_for(L.nslots), 256, 0, stream_>>>(
          L.slot_cell, L.slot_face, L.nslots, n, F_, dt, L.Rc, L.has, d_err_);
      launch_count();
    }
  };

  if (cfg_.integrator == AF_INTEGRATOR_MUSCL_HANCOCK) {
    amr_prims_kernel<D><<<gb, 256, 0, stream_>>>(v, b, W_, gamma, rec, d_err_, 2 * call + 1);
    amr_predict_kernel<D, S><<<blocks_for(L.tot1), 256, 0, stream_>>>(v, b, W_, DU_, 0.5 * dt / h,
                                                                     gamma - 1.0, rec, d_err_);
    amr_faces_hancock<D, S><<<gf, 256, 0, stream_>>>(v, b, W_, DU_, F_, gamma, rec, d_err_);
    amr_update_kernel<D><<<gc, 256, 0, stream_>>>(v, L.U, F_, inv_dx, dt, d_err_);
    launch_count(4);
    stepped(4);
    registers();
  } else {
    // stage 1 of every patch, the midpoint ghosts, stage 2 (the patch blocks
    // keep the ghosts of time t afterwards: out = saved)
    amr_prims_kernel<D><<<gb, 256, 0, stream_>>>(v, b, W_, gamma, rec, d_err_, 2 * call);
    amr_faces_rk2<D, S><<<gf, 256, 0, stream_>>>(v, b, W_, F_, gamma, rec, d_err_);
    amr_update_kernel<D><<<gc, 256, 0, stream_>>>(v, L.Uold, F_, inv_dx, 0.5 * dt, d_err_);
    launch_count(3);
    sync_ghosts(l, L.t + 0.5 * dt);
    amr_prims_kernel<D><<<gb, 256, 0, stream_>>>(v, b, W_, gamma, rec, d_err_, 2 * call + 1);
    amr_faces_rk2<D, S><<<gf, 256, 0, stream_>>>(v, b, W_, F_, gamma, rec, d_err_);
    amr_update_kernel<D><<<gc, 256, 0, stream_>>>(v, L.Uold, F_, inv_dx, dt, d_err_);
    launch_count(3);
    stepped(7);
    save_level(l, true);
    registers();
  }
  L.t += dt;
  AF_CUDA(cudaGetLastError());
}

void Amr::update_async(int l, double dt) {
  if (l < 0 || l >= n_levels()) throw Error(AF_E_ARGUMENT, "update_level: no such level");
  const int sch = cfg_.limiter | (cfg_.flux << 1);
#define AMR_UPD(D)                                  \
  switch (sch) {                                    \
    case 0: update_t<D, 0>(l, dt); break;           \
    case 1: update_t<D, 1>(l, dt); break;           \
    case 2: update_t<D, 2>(l, dt); break;           \
    default: update_t<D, 3>(l, dt); break;          \
  }
  if (dim_ == 3) {
    AMR_UPD(3)
  } else {
    AMR_UPD(2)
  }
#undef AMR_UPD
}

af_step_diag Amr::update_level(int l, double dt) {
  check();
  update_async(l, dt);
  check();
  return last_diag_;
}

void Amr::fold_records() {
  if (calls_.empty()) return;
  std::vector<ARec> rec(calls_.size());
  AF_CUDA(cudaMemcpyAsync(rec.data(), d_rec_, sizeof(ARec) * rec.size(), cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  for (size_t i = 0; i < calls_.size(); ++i) {
    double wave;
    std::memcpy(&wave, &rec[i].wave, sizeof wave);
    last_diag_.max_wave_speed = wave;
    last_diag_.fallbacks = (long)rec[i].fallbacks;
    wave_max_ = std::max(wave_max_, wave);
    cfl_max_ = std::max(cfl_max_, wave * calls_[i].dt / dx(calls_[i].level));
    fallbacks_ += (long)rec[i].fallbacks;
  }
  AF_CUDA(cudaMemsetAsync(d_rec_, 0, sizeof(ARec) * calls_.size(), stream_));
}

void Amr::check() {
  int err[4] = {0, 0, 0, 0};
  AF_CUDA(cudaMemcpyAsync(err, d_err_, sizeof err, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  for (auto& e : events_) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, e.first, e.second) == cudaSuccess) stage_ms_ += ms;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  events_.clear();
  if (err[0] == 1) raise_nonphysical(err[1]);
  fold_records();
  calls_.clear();
  if (err[0] == 2)
    throw Error(AF_E_INTERNAL, prefix_ + "no coarse donor under a fine ghost or new cell (MissingBracketingStates)");
  if (err[0] == 3)
    throw Error(AF_E_REGISTER_MISMATCH, prefix_ + "flux register is missing a side");
  if (err[2])
    throw Error(AF_E_INTERNAL, "remesh produced an improperly nested hierarchy");
}

// The reference's NonPhysicalState text: the first offending cell in the
// order build_primitives walks the first offending patch's block
// (step.cpp:26-38), with update_level's "level L patch P: " prefix where it
// adds one (amr_hierarchy.cpp:480-483, 514-517). The kernels stopped at the
// failure, so G still holds the field the failing stage read.
void Amr::raise_nonphysical(int tag) {
  const int call = tag >> 1, stage2 = tag & 1;
  const int l = calls_.at((size_t)call).level;
  calls_.clear();
  Level& L = lv_[l];
  std::string msg = "non-physical state";
  for (size_t pi = 0; pi < L.boxes.size(); ++pi) {
    const ABox one = L.boxes[pi];
    // the block of this patch with its ghosts; the failing stage read the
    // synced field, so every position is a G read
    const int g = 2;
    long cells = 1;
    int ext[3];
    for (int a = 0; a < 3; ++a) {
      ext[a] = one.extent(a) + (a < dim_ ? 2 * g : 0);
      cells *= ext[a];
    }
    std::vector<double> aos((size_t)5 * cells);
    {
      int bx[6] = {one.lo[0], one.lo[1], one.lo[2], one.hi[0], one.hi[1], one.hi[2]};
      long off[2] = {0, cells};
      int* d_b = nullptr;
      long* d_o = nullptr;
      double* d_a = nullptr;
      AF_CUDA(cudaMalloc(&d_b, sizeof bx));
      AF_CUDA(cudaMalloc(&d_o, sizeof off));
      AF_CUDA(cudaMalloc(&d_a, sizeof(double) * aos.size()));
      AF_CUDA(cudaMemcpy(d_b, bx, sizeof bx, cudaMemcpyHostToDevice));
      AF_CUDA(cudaMemcpy(d_o, off, sizeof off, cudaMemcpyHostToDevice));
      if (dim_ == 3)
        amr_get_kernel<3><<<blocks_for(cells), 256, 0, stream_>>>(d_b, d_o, 1, cells, AMR_VIEW(3, L), bc_of(cfg_), g,
                                                                  0, 1, d_a);
      else
        amr_get_kernel<2><<<blocks_for(cells), 256, 0, stream_>>>(d_b, d_o, 1, cells, AMR_VIEW(2, L), bc_of(cfg_), g,
                                                                  0, 1, d_a);
      AF_CUDA(cudaMemcpyAsync(aos.data(), d_a, sizeof(double) * aos.size(), cudaMemcpyDeviceToHost, stream_));
      AF_CUDA(cudaStreamSynchronize(stream_));
      cudaFree(d_b);
      cudaFree(d_o);
      cudaFree(d_a);
    }
    const double gm1 = cfg_.gamma - 1.0;
    long t = 0;
    bool found = false;
    for (int k = 0; k < ext[2] && !found; ++k)
      for (int j = 0; j < ext[1] && !found; ++j)
        for (int i = 0; i < ext[0]; ++i, ++t) {
          const double* q = &aos[5 * t];
          const double inv_rho = 1.0 / q[0];
          const double kin = 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) * inv_rho;
          const double p = gm1 * (q[4] - kin);
          if ((q[0] > 1e-12) && (p > 1e-12)) continue;
          const int li = i - g, lj = j - g, lk = dim_ == 3 ? k - g : 0;
          const bool ghost = li < 0 || li >= one.extent(0) || lj < 0 || lj >= one.extent(1) ||
                             lk < 0 || lk >= one.extent(2);
          std::string cs = "(" + std::to_string(li) + "," + std::to_string(lj);
          if (dim_ == 3) cs += "," + std::to_string(lk);
          cs += ")";
          msg = "cell " + cs + (ghost ? " (ghost)" : "") + ": rho=" + f6(q[0]) + " p=" + f6(p);
          const bool wrapped = cfg_.integrator == AF_INTEGRATOR_MUSCL_HANCOCK || stage2;
          if (wrapped) msg = "level " + std::to_string(l) + " patch " + std::to_string(pi) + ": " + msg;
          err_.i = li;
          err_.j = lj;
          err_.k = lk;
          err_.level = l;
          err_.is_ghost = ghost;
          err_.rho = q[0];
          err_.p = p;
          found = true;
          break;
        }
    if (found) break;
  }
  throw Error(AF_E_NONPHYSICAL, prefix_ + msg);
}

void Amr::average_down(int l) {
  if (l + 1 >= n_levels()) return;
  const Level& Fn = lv_[l + 1];
  Level& C = lv_[l];
  if (std::fabs(Fn.t - C.t) > 1e-12 * std::max(1.0, std::fabs(C.t)))
    throw Error(AF_E_LEVEL_MISMATCH, "average_down: levels at t=" + f6(C.t) + " and t=" + f6(Fn.t));
  if (dim_ == 3)
    amr_average_down_kernel<3><<<blocks_for(C.total), 256, 0, stream_>>>(AMR_VIEW(3, C), AMR_VIEW(3, lv_[l + 1]), d_err_);
  else
    amr_average_down_kernel<2><<<blocks_for(C.total), 256, 0, stream_>>>(AMR_VIEW(2, C), AMR_VIEW(2, lv_[l + 1]), d_err_);
  launch_count();
  AF_CUDA(cudaGetLastError());
}

void Amr::flux_correct(int l) {
  if (l >= n_levels()) return;
  Level& L = lv_[l];
  if (!L.nslots) return;
  if (opt_.flux_correction) {
    const double inv_h = 1.0 / dx(l);
    if (dim_ == 3)
      amr_flux_correct_kernel<3><<<blocks_for(L.nslots), 256, 0, stream_>>>(AMR_VIEW(3, L), L.regbase, L.regmask,
                                                                           L.slot_cell, L.slot_face, L.Rc, L.Rf, L.has,
                                                                           L.nslots, inv_h, d_err_);
    else
      amr_flux_correct_kernel<2><<<blocks_for(L.nslots), 256, 0, stream_>>>(AMR_VIEW(2, L), L.regbase, L.regmask,
                                                                           L.slot_cell, L.slot_face, L.Rc, L.Rf, L.has,
                                                                           L.nslots, inv_h, d_err_);
    launch_count();
  }
  clear_registers(l);
  AF_CUDA(cudaGetLastError());
}

void Amr::total_conserved(double out5[5]) {
  check();
  double* d = nullptr;
  AF_CUDA(cudaMalloc(&d, sizeof(double) * 5));
  for (int m = 0; m < 5; ++m) out5[m] = 0.0;
  for (int l = 0; l < n_levels(); ++l) {
    Level& L = lv_[l];
    AF_CUDA(cudaMemsetAsync(d, 0, sizeof(double) * 5, stream_));
    const int* fp = l + 1 < n_levels() ? lv_[l + 1].pid : nullptr;
    const unsigned g = std::min<unsigned>(blocks_for(L.total), 1184);
    if (dim_ == 3)
      amr_sum_kernel<3><<<g, 256, 0, stream_>>>(AMR_VIEW(3, L), fp, d);
    else
      amr_sum_kernel<2><<<g, 256, 0, stream_>>>(AMR_VIEW(2, L), fp, d);
    launch_count();
    double s[5] = {0, 0, 0, 0, 0};
    AF_CUDA(cudaMemcpyAsync(s, d, sizeof(double) * (dim_ + 2), cudaMemcpyDeviceToHost, stream_));
    AF_CUDA(cudaStreamSynchronize(stream_));
    const double h = dx(l), vol = dim_ == 3 ? h * h * h : h * h;
    out5[0] += s[0] * vol;
    out5[1] += s[1] * vol;
    out5[2] += s[2] * vol;
    if (dim_ == 3) out5[3] += s[3] * vol;
    out5[4] += s[dim_ + 1] * vol;
  }
  cudaFree(d);
}

void Amr::l1_error(int ref_level, const double* ref_aos, double out5[5]) {
  if (!ref_aos || !out5) throw Error(AF_E_ARGUMENT, "l1_error_amr: null pointer");
  check();
  for (int m = 0; m < 5; ++m) out5[m] = 0.0;
  double* d = nullptr;
  AF_CUDA(cudaMalloc(&d, sizeof(double) * 5));
  for (int l = 0; l < n_levels(); ++l) {
    const int res = base_exp_ + l;
    if (ref_level < res) {
      cudaFree(d);
      throw Error(AF_E_LEVEL_MISMATCH, "reference too coarse for hierarchy level " + std::to_string(l));
    }
    Level& L = lv_[l];
    double* r = nullptr;
    AF_CUDA(cudaMalloc(&r, sizeof(double) * 5 * L.cells));
    restrict_to_level(dim_, ref_level, res, ref_aos, r);  // device, bit-exact (af_io.cu)
    AF_CUDA(cudaMemsetAsync(d, 0, sizeof(double) * 5, stream_));
    const int* fp = l + 1 < n_levels() ? lv_[l + 1].pid : nullptr;
    const unsigned g = std::min<unsigned>(blocks_for(L.total), 1184);
    if (dim_ == 3)
      amr_l1_kernel<3><<<g, 256, 0, stream_>>>(AMR_VIEW(3, L), fp, r, d);
    else
      amr_l1_kernel<2><<<g, 256, 0, stream_>>>(AMR_VIEW(2, L), fp, r, d);
    launch_count();
    double s[5];
    AF_CUDA(cudaMemcpyAsync(s, d, sizeof s, cudaMemcpyDeviceToHost, stream_));
    AF_CUDA(cudaStreamSynchronize(stream_));
    cudaFree(r);
    const double h = dx(l), vol = dim_ == 3 ? h * h * h : h * h;
    for (int m = 0; m < 5; ++m) out5[m] += s[m] * vol;
  }
  cudaFree(d);
}

long Amr::total_cells() const {
  long c = 0;
  for (const Level& L : lv_)
    for (const ABox& b : L.boxes) c += b.volume();
  return c;
}

long Amr::composite_cells() const {  // amr_hierarchy.cpp:590-598
  long c = 0;
  for (int l = 0; l < n_levels(); ++l) {
    long dom = 0, fine = 0;
    for (const ABox& b : lv_[l].boxes) dom += b.volume();
    if (l + 1 < n_levels())
      for (const ABox& b : lv_[l + 1].boxes) fine += b.volume();
    c += dom - fine / (1 << dim_);
  }
  return c;
}

bool Amr::properly_nested() {
  if (n_levels() < 2) return true;
  AF_CUDA(cudaMemsetAsync(d_flag_, 0, sizeof(int), stream_));
  for (int l = 1; l < n_levels(); ++l) {
    const Level& Fn = lv_[l];
    if (dim_ == 3)
      amr_nested_kernel<3><<<blocks_for(Fn.total), 256, 0, stream_>>>(AMR_VIEW(3, Fn), lv_[l - 1].pid, d_flag_);
    else
      amr_nested_kernel<2><<<blocks_for(Fn.total), 256, 0, stream_>>>(AMR_VIEW(2, Fn), lv_[l - 1].pid, d_flag_);
    launch_count();
  }
  int bad = 0;
  AF_CUDA(cudaMemcpyAsync(&bad, d_flag_, sizeof(int), cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  return !bad;
}

std::string Amr::dump_boxes() const {  // amr_hierarchy.cpp:618-629
  std::string s;
  for (int l = 0; l < n_levels(); ++l)
    for (const ABox& b : lv_[l].boxes) {
      s += std::to_string(l);
      for (int a = 0; a < dim_; ++a) s += " " + std::to_string(b.lo[a]);
      for (int a = 0; a < dim_; ++a) s += " " + std::to_string(b.hi[a]);
      s += "\n";
    }
  return s;
}

long Amr::patch_data_cells(int l, int ghost) const {
  long c = 0;
  for (const ABox& b : lv_[l].boxes) {
    long v = 1;
    for (int a = 0; a < 3; ++a) v *= b.extent(a) + (a < dim_ ? 2 * ghost : 0);
    c += v;
  }
  return c;
}

void Amr::patch_data(int l, int ghost, int old, double* aos) {
  if (l < 0 || l >= n_levels() || !aos) throw Error(AF_E_ARGUMENT, "patch_data: bad argument");
  check();
  Level& L = lv_[l];
  const int nb = (int)L.boxes.size();
  std::vector<long> off((size_t)nb + 1, 0);
  for (int i = 0; i < nb; ++i) {
    long v = 1;
    for (int a = 0; a < 3; ++a) v *= L.boxes[i].extent(a) + (a < dim_ ? 2 * ghost : 0);
    off[i + 1] = off[i] + v;
  }
  const long total = off[nb];
  long* d_o = nullptr;
  double* d_a = nullptr;
  AF_CUDA(cudaMalloc(&d_o, sizeof(long) * (nb + 1)));
  AF_CUDA(cudaMalloc(&d_a, sizeof(double) * 5 * total));
  AF_CUDA(cudaMemcpyAsync(d_o, off.data(), sizeof(long) * (nb + 1), cudaMemcpyHostToDevice, stream_));
  if (dim_ == 3)
    amr_get_kernel<3><<<blocks_for(total), 256, 0, stream_>>>(L.d_boxes, d_o, nb, total, AMR_VIEW(3, L), bc_of(cfg_),
                                                              ghost, old, 0, d_a);
  else
    amr_get_kernel<2><<<blocks_for(total), 256, 0, stream_>>>(L.d_boxes, d_o, nb, total, AMR_VIEW(2, L), bc_of(cfg_),
                                                              ghost, old, 0, d_a);
  launch_count();
  AF_CUDA(cudaMemcpyAsync(aos, d_a, sizeof(double) * 5 * total, cudaMemcpyDefault, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  cudaFree(d_o);
  cudaFree(d_a);
}

void Amr::assemble_level(int l, double* aos) {  // amr_hierarchy.cpp:600-616
  if (l < 0 || l >= n_levels() || !aos) throw Error(AF_E_ARGUMENT, "assemble_level: bad argument");
  long dom = 0;
  for (const ABox& b : lv_[l].boxes) dom += b.volume();
  if (dom != lv_[l].cells)
    throw Error(AF_E_LEVEL_MISMATCH,
                "assemble_level: level " + std::to_string(l) + " does not cover the domain");
  check();
  Level& L = lv_[l];
  const int n = L.n;
  const int bx[6] = {0, 0, 0, n, n, dim_ == 3 ? n : 1};
  const long off[2] = {0, L.cells};
  int* d_b = nullptr;
  long* d_o = nullptr;
  double* d_a = nullptr;
  AF_CUDA(cudaMalloc(&d_b, sizeof bx));
  AF_CUDA(cudaMalloc(&d_o, sizeof off));
  AF_CUDA(cudaMalloc(&d_a, sizeof(double) * 5 * L.cells));
  AF_CUDA(cudaMemcpyAsync(d_b, bx, sizeof bx, cudaMemcpyHostToDevice, stream_));
  AF_CUDA(cudaMemcpyAsync(d_o, off, sizeof off, cudaMemcpyHostToDevice, stream_));
  if (dim_ == 3)
    amr_get_kernel<3><<<blocks_for(L.cells), 256, 0, stream_>>>(d_b, d_o, 1, L.cells, AMR_VIEW(3, L), bc_of(cfg_), 0, 0,
                                                                2, d_a);
  else
    amr_get_kernel<2><<<blocks_for(L.cells), 256, 0, stream_>>>(d_b, d_o, 1, L.cells, AMR_VIEW(2, L), bc_of(cfg_), 0, 0,
                                                                2, d_a);
  launch_count();
  AF_CUDA(cudaMemcpyAsync(aos, d_a, sizeof(double) * 5 * L.cells, cudaMemcpyDefault, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  cudaFree(d_b);
  cudaFree(d_o);
  cudaFree(d_a);
}

// AmrDriver::advance (amr_solver.cpp:24-60)
void Amr::advance(int l, double dt, std::vector<long>* cps, std::vector<long>* lps) {
  const bool lt = opt_.time_refine != 0;
  const int r = (lt && l > 0) ? 2 : 1;
  for (int sub = 0; sub < r; ++sub) {
    sync_ghosts(l, lv_[l].t);
    if ((sub > 0 || l == 0) && l < opt_.max_levels) remesh(l);
    update_async(l, dt);
    if (l == n_levels() - 1) {
      cps->push_back(total_cells());
      lps->push_back(composite_cells());
    }
    if (l + 1 < n_levels()) {
      sync_ghosts(l, lv_[l].t);
      advance(l + 1, lt ? 0.5 * dt : dt, cps, lps);
      average_down(l);
      flux_correct(l);
    }
  }
}

void Amr::run(long n_steps, double dt_finest, long* cells_per_step, long* leaves_per_step,
              af_run_diag* diag) {
  const bool lt = opt_.time_refine != 0;
  const long per_cycle = lt ? (1l << opt_.max_levels) : 1;
  if (n_steps % per_cycle != 0)
    throw Error(AF_E_CONFIG, "n_steps=" + std::to_string(n_steps) + " is not a multiple of the " +
                                 std::to_string(per_cycle) + " substeps of one time-refined cycle");
  const long cycles = n_steps / per_cycle;
  const double dt0 = lt ? dt_finest * (double)per_cycle : dt_finest;
  std::vector<long> cps, lps;
  wave_max_ = 0.0;
  cfl_max_ = 0.0;
  fallbacks_ = 0;
  long done = 0;
  try {
    for (long cycle = 0; cycle < cycles; ++cycle) {
      prefix_ = "cycle " + std::to_string(cycle) + ": ";
      advance(0, dt0, &cps, &lps);
      check();
      while ((long)cps.size() < (cycle + 1) * per_cycle) {  // pad_samples
        cps.push_back(total_cells());
        lps.push_back(composite_cells());
      }
      done = (cycle + 1) * per_cycle;
    }
  } catch (...) {
    prefix_.clear();
    throw;
  }
  prefix_.clear();
  for (long i = 0; i < n_steps && i < (long)cps.size(); ++i) {
    if (cells_per_step) cells_per_step[i] = cps[(size_t)i];
    if (leaves_per_step) leaves_per_step[i] = lps[(size_t)i];
  }
  if (diag) {
    diag->max_wave_speed = wave_max_;
    diag->max_cfl = cfl_max_;
    diag->fallbacks = fallbacks_;
    diag->steps_done = done;
    diag->t = lv_[0].t;
  }
}

}  // namespace af

// ------------------------------------------------------------------ C ABI --
struct af_amr {
  af::Amr* impl;
  std::string text;
};

namespace {
template <class F>
af_status amr_guard(af_amr* h, F&& f) {
  af_error* e = h ? &h->impl->error_slot() : nullptr;
  auto rec = [&](af_status st, const char* msg) {
    if (e) {
      if (st != AF_E_NONPHYSICAL) {
        std::memset(e, 0, sizeof *e);
        e->step = -1;
        e->level = -1;
      }
      e->status = st;
      std::snprintf(e->message, sizeof e->message, "%s", msg);
    }
    return st;
  };
  try {
    f();
    return AF_OK;
  } catch (const af::Error& x) {
    return rec(x.status, x.what());
  } catch (const std::exception& x) {
    return rec(AF_E_ARGUMENT, x.what());
  }
}
}  // namespace

extern "C" {

af_status af_amr_create(const af_config* cfg, const af_amr_options* opt, af_amr** out) {
  if (!cfg || !opt || !out) return AF_E_ARGUMENT;
  *out = nullptr;
  try {
    af_amr* h = new af_amr{new af::Amr(*cfg, *opt), {}};
    *out = h;
    return AF_OK;
  } catch (const af::Error& x) {
    return x.status;
  } catch (const std::exception&) {
    return AF_E_ARGUMENT;
  }
}
af_status af_amr_destroy(af_amr* h) {
  if (!h) return AF_OK;
  delete h->impl;
  delete h;
  return AF_OK;
}
af_status af_amr_initialize(af_amr* h, af_amr_ic ic, void* user) {
  if (!h) return AF_E_ARGUMENT;
  return amr_guard(h, [&] { h->impl->initialize(ic, user); });
}
af_status af_amr_initialize_case(af_amr* h, int kind, uint64_t seed, double gamma) {
  if (!h) return AF_E_ARGUMENT;
  return amr_guard(h, [&] {
    struct Ctx {
      int kind;
      double gamma;
      af_case_params cp;
    } ctx;
    ctx.kind = kind;
    ctx.gamma = gamma;
    af_rng rng;
    af_case_draw(kind, seed, &ctx.cp, &rng);
    double probe[5];
    if (af_case_point(kind, &ctx.cp, gamma, 0.25, 0.25, 0.25, probe) != 0)
      throw af::Error(AF_E_CONFIG, "af_amr_initialize_case: this case has no position form");
    h->impl->initialize(
        [](double x, double y, double z, double* q, void* u) {
          const Ctx* c = static_cast<const Ctx*>(u);
          af_case_point(c->kind, &c->cp, c->gamma, x, y, z, q);
        },
        &ctx);
  });
}
af_status af_amr_sync_ghosts(af_amr* h, int level, double tau) {
  if (!h) return AF_E_ARGUMENT;
  return amr_guard(h, [&] { h->impl->sync_ghosts(level, tau); });
}
af_status af_amr_remesh(af_amr* h, int level) {
  if (!h) return AF_E_ARGUMENT;
  return amr_guard(h, [&] { h->impl->remesh(level); });
}
af_status af_amr_update_level(af_amr* h, int level, double dt, af_step_diag* diag) {
  if (!h) return AF_E_ARGUMENT;
  return amr_guard(h, [&] {
    const af_step_diag d = h->impl->update_level(level, dt);
    if (diag) *diag = d;
  });
}
af_status af_amr_average_down(af_amr* h, int level) {
  if (!h) return AF_E_ARGUMENT;
  return amr_guard(h, [&] { h->impl->average_down(level); });
}
af_status af_amr_flux_correct(af_amr* h, int level) {
  if (!h) return AF_E_ARGUMENT;
  return amr_guard(h, [&] { h->impl->flux_correct(level); });
}
af_status af_amr_run(af_amr* h, long n_steps, double dt_finest, long* cells_per_step,
                     long* leaves_per_step, af_run_diag* diag) {
  if (!h) return AF_E_ARGUMENT;
  return amr_guard(h, [&] { h->impl->run(n_steps, dt_finest, cells_per_step, leaves_per_step, diag); });
}
af_status af_amr_n_levels(const af_amr* h, int* n) {
  if (!h || !n) return AF_E_ARGUMENT;
  *n = h->impl->n_levels();
  return AF_OK;
}
af_status af_amr_level_info(const af_amr* h, int level, int* n_patches, long* cells, double* t,
                            double* t_old) {
  if (!h || level < 0 || level >= h->impl->n_levels()) return AF_E_ARGUMENT;
  const auto& bx = h->impl->boxes(level);
  if (n_patches) *n_patches = (int)bx.size();
  if (cells) {
    long c = 0;
    for (const auto& b : bx) c += b.volume();
    *cells = c;
  }
  if (t) *t = h->impl->time(level);
  if (t_old) *t_old = h->impl->time_old(level);
  return AF_OK;
}
af_status af_amr_boxes(const af_amr* h, int level, int* boxes6, int capacity) {
  if (!h || !boxes6 || level < 0 || level >= h->impl->n_levels()) return AF_E_ARGUMENT;
  const auto& bx = h->impl->boxes(level);
  if ((int)bx.size() > capacity) return AF_E_ARGUMENT;
  for (size_t i = 0; i < bx.size(); ++i)
    for (int a = 0; a < 3; ++a) {
      boxes6[6 * i + a] = bx[i].lo[a];
      boxes6[6 * i + 3 + a] = bx[i].hi[a];
    }
  return AF_OK;
}
af_status af_amr_patch_data_cells(const af_amr* h, int level, int ghost, long* cells) {
  if (!h || !cells || level < 0 || level >= h->impl->n_levels()) return AF_E_ARGUMENT;
  *cells = h->impl->patch_data_cells(level, ghost);
  return AF_OK;
}
af_status af_amr_patch_data(af_amr* h, int level, int ghost, int old, double* aos) {
  if (!h) return AF_E_ARGUMENT;
  return amr_guard(h, [&] { h->impl->patch_data(level, ghost, old, aos); });
}
af_status af_amr_assemble_level(af_amr* h, int level, double* aos) {
  if (!h) return AF_E_ARGUMENT;
  return amr_guard(h, [&] { h->impl->assemble_level(level, aos); });
}
af_status af_amr_total_conserved(af_amr* h, double out5[5]) {
  if (!h || !out5) return AF_E_ARGUMENT;
  return amr_guard(h, [&] { h->impl->total_conserved(out5); });
}
af_status af_amr_l1_error(af_amr* h, int ref_level, const double* ref_aos, double out5[5]) {
  if (!h) return AF_E_ARGUMENT;
  return amr_guard(h, [&] { h->impl->l1_error(ref_level, ref_aos, out5); });
}
af_status af_amr_counts(const af_amr* h, long* total_cells, long* composite_cells) {
  if (!h) return AF_E_ARGUMENT;
  if (total_cells) *total_cells = h->impl->total_cells();
  if (composite_cells) *composite_cells = h->impl->composite_cells();
  return AF_OK;
}
af_status af_amr_properly_nested(af_amr* h, int* nested) {
  if (!h || !nested) return AF_E_ARGUMENT;
  return amr_guard(h, [&] { *nested = h->impl->properly_nested() ? 1 : 0; });
}
af_status af_amr_dump_boxes(af_amr* h, const char** text) {
  if (!h || !text) return AF_E_ARGUMENT;
  return amr_guard(h, [&] {
    h->text = h->impl->dump_boxes();
    *text = h->text.c_str();
  });
}
af_status af_amr_last_error(const af_amr* h, af_error* err) {
  if (!h || !err) return AF_E_ARGUMENT;
  *err = h->impl->last_error();
  return AF_OK;
}
af_status af_amr_kernel_launches(const af_amr* h, long* count) {
  if (!h || !count) return AF_E_ARGUMENT;
  *count = h->impl->kernel_launches();
  return AF_OK;
}
af_status af_amr_remesh_stats(const af_amr* h, double* seconds, long* calls) {
  if (!h) return AF_E_ARGUMENT;
  if (seconds) *seconds = h->impl->remesh_seconds();
  if (calls) *calls = h->impl->remesh_calls();
  return AF_OK;
}
af_status af_amr_profile(af_amr* h, int enable) {
  if (!h) return AF_E_ARGUMENT;
  h->impl->set_profile(enable != 0);
  return AF_OK;
}
af_status af_amr_stage_stats(af_amr* h, double* ms, long* launches, long* updates) {
  if (!h) return AF_E_ARGUMENT;
  return amr_guard(h, [&] { h->impl->stage_stats(ms, launches, updates); });
}
af_status af_amr_cell_updates(const af_amr* h, long* updates) {
  if (!h || !updates) return AF_E_ARGUMENT;
  *updates = h->impl->cell_updates();
  return AF_OK;
}
af_status af_amr_cluster_device(const unsigned char* flags, const unsigned char* allowed, int dim,
                                int n, double efficiency, int* boxes6, int capacity, int* n_boxes) {
  if (!flags || !n_boxes || (dim != 2 && dim != 3) || n < 1) return AF_E_ARGUMENT;
  try {
    const size_t cells = dim == 3 ? (size_t)n * n * n : (size_t)n * n;
    unsigned char *d_f = nullptr, *d_a = nullptr;
    AF_CUDA(cudaMalloc(&d_f, cells));
    AF_CUDA(cudaMemcpy(d_f, flags, cells, cudaMemcpyHostToDevice));
    if (allowed) {
      AF_CUDA(cudaMalloc(&d_a, cells));
      AF_CUDA(cudaMemcpy(d_a, allowed, cells, cudaMemcpyHostToDevice));
    }
    std::vector<af::ABox> out;
    long launches = 0;
    {
      af::DeviceCluster dc(nullptr);
      out = dc.run(dim, d_f, d_a, n, efficiency, &launches);
    }
    cudaFree(d_f);
    cudaFree(d_a);
    *n_boxes = (int)out.size();
    if (boxes6) {
      if ((int)out.size() > capacity) return AF_E_ARGUMENT;
      for (size_t i = 0; i < out.size(); ++i)
        for (int a = 0; a < 3; ++a) {
          boxes6[6 * i + a] = out[i].lo[a];
          boxes6[6 * i + 3 + a] = out[i].hi[a];
        }
    }
    return AF_OK;
  } catch (const af::Error& x) {
    return x.status;
  } catch (const std::exception&) {
    return AF_E_ARGUMENT;
  }
}
af_status af_amr_cluster(const unsigned char* flags, const unsigned char* allowed, int dim, int n0,
                         int n1, int n2, double efficiency, int* boxes6, int capacity, int* n_boxes) {
  if (!flags || !n_boxes || (dim != 2 && dim != 3) || n0 < 1 || n1 < 1 || n2 < 1) return AF_E_ARGUMENT;
  try {
    const std::vector<af::ABox> out = af::amr_cluster(flags, allowed, dim, n0, n1, n2, efficiency);
    *n_boxes = (int)out.size();
    if (boxes6) {
      if ((int)out.size() > capacity) return AF_E_ARGUMENT;
      for (size_t i = 0; i < out.size(); ++i)
        for (int a = 0; a < 3; ++a) {
          boxes6[6 * i + a] = out[i].lo[a];
          boxes6[6 * i + 3 + a] = out[i].hi[a];
        }
    }
    return AF_OK;
  } catch (const std::exception&) {
    return AF_E_ARGUMENT;
  }
}

}  // extern "C"
