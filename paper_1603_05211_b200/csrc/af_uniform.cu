// af_uniform.cu — host side of the uniform FV solver (af_uniform_* of af_gpu.h).
//
// Mirrors run_uniform's step loop (unigrid.cpp:33-47) and step_block's RK2
// (step.cpp:237-251): per step, stage(u,u,mid,dt/2) then stage(u,mid,u,dt).
// The ghost fill (grid.cpp:9-62) is folded into the kernels' index mapping;
// only inter-rank halo planes are exchanged (NCCL send/recv over NVLink).
// Δt (CFL rule) is reduced on the device by the previous step's stage-2
// epilogue, so a multi-step run issues no host synchronisation and can be
// captured in a CUDA graph.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "af_comm.h"
#include "af_uniform.h"
#include "af_fv3d.cuh"
#include "af_hancock.cuh"
#include "af_uniform_kernels.cuh"

namespace af {

namespace {

constexpr int kTY = 8;

// 3D stage tile (af_fv3d.cuh): 16x15 columns, 8 warps (751 faces per plane =
// 24 warp units, 3 per warp), two CTAs per SM (128 registers).
constexpr int kT3 = 16, kT3Y = 15, kW3 = 8;
using Geo3 = Fv3dGeom<kT3, kT3Y, kW3>;

// cuTensorMapEncodeTiled through the runtime's driver entry point (the
// library does not link libcuda, so it still loads without a driver).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    AF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p)
      throw Error(AF_E_CUDA, "driver entry point missing: cuTensorMapEncodeTiled");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

__global__ void aos_to_soa(const double* __restrict__ aos, double* __restrict__ soa, UGrid g) {
  const long cells = g.plane * g.nzl;
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < cells;
       c += (long)gridDim.x * blockDim.x) {
    const long off = (c / g.plane + 2) * g.zs + c % g.plane;
    const double* q = aos + 5 * c;
    if (g.ncomp == 5) {
#pragma unroll
      for (int m = 0; m < 5; ++m) soa[m * g.cs + off] = q[m];
    } else {  // 2D: drop mom2 (identically zero in the reference)
      soa[off] = q[0];
      soa[g.cs + off] = q[1];
      soa[2 * g.cs + off] = q[2];
      soa[3 * g.cs + off] = q[4];
    }
  }
}

__global__ void soa_to_aos(const double* __restrict__ soa, double* __restrict__ aos, UGrid g) {
  const long cells = g.plane * g.nzl;
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < cells;
       c += (long)gridDim.x * blockDim.x) {
    const long off = (c / g.plane + 2) * g.zs + c % g.plane;
    double* q = aos + 5 * c;
    if (g.ncomp == 5) {
#pragma unroll
      for (int m = 0; m < 5; ++m) q[m] = soa[m * g.cs + off];
    } else {
      q[0] = soa[off];
      q[1] = soa[g.cs + off];
      q[2] = soa[2 * g.cs + off];
      q[3] = 0.0;
      q[4] = soa[3 * g.cs + off];
    }
  }
}

std::string fmt_f(double v) {  // std::to_string(double) == "%f"
  char b[64];
  std::snprintf(b, sizeof b, "%f", v);
  return b;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace

// Contiguous slabs of the slab axis (z in 3D, y in 2D); 2D slabs stay multiples
// of the tile height. Pure host arithmetic: false when a rank would be empty.
bool slab_extent(int dim, int level, int n_ranks, int rank, int* z0, int* nz) {
  if (dim < 2 || dim > 3 || level < 0 || level > 30 || n_ranks < 1 || rank < 0 ||
      rank >= n_ranks)
    return false;
  const int n = 1 << level;
  const int quantum = dim == 2 ? kTY : 2;
  const int units = n / quantum;
  if (units < n_ranks) return false;
  const int lo_u = (int)((long)units * rank / n_ranks);
  const int hi_u = (int)((long)units * (rank + 1) / n_ranks);
  *z0 = lo_u * quantum;
  *nz = (hi_u - lo_u) * quantum;
  return true;
}

Uniform::Uniform(const af_config& c, Comm* comm) : cfg_(c), comm_(comm) {
  if (c.dim != 2 && c.dim != 3) throw Error(AF_E_CONFIG, "dim must be 2 or 3");
  if (c.level < 3 || c.level > 15)
    throw Error(AF_E_CONFIG, "level must be in [3, 15] (>= 8 cells per axis)");
  if (c.flux != AF_FLUX_AUSM_PLUS && c.flux != AF_FLUX_AUSMDV)
    throw Error(AF_E_CONFIG, "unknown flux");
  if (c.integrator != AF_INTEGRATOR_RK2 && c.integrator != AF_INTEGRATOR_MUSCL_HANCOCK)
    throw Error(AF_E_CONFIG, "unknown integrator");
  if (c.limiter != AF_LIMITER_MINMOD && c.limiter != AF_LIMITER_VAN_ALBADA)
    throw Error(AF_E_CONFIG, "unknown limiter");
  for (int f = 0; f < 6; ++f)
    if (c.bc[f] < 0 || c.bc[f] > 2) throw Error(AF_E_CONFIG, "unknown boundary condition");
  if (!(c.gamma > 1.0)) throw Error(AF_E_CONFIG, "gamma must exceed 1");
  AF_CUDA(cudaSetDevice(c.device));
  const int n = 1 << c.level;
  g_.dim = c.dim;
  g_.n = n;
  g_.nranks = comm ? comm->n : 1;
  const int rank = comm ? comm->rank : 0;
  if (!slab_extent(c.dim, c.level, g_.nranks, rank, &g_.zlo, &g_.nzl))
    throw Error(AF_E_CONFIG, "too many ranks for this mesh");
  for (int f = 0; f < 6; ++f) g_.bc[f] = c.bc[f];
  g_.ncomp = c.dim == 3 ? 5 : 4;
  g_.plane = c.dim == 3 ? (long)n * n : (long)n;
  g_.cs = g_.plane;
  g_.zs = g_.ncomp * g_.plane;
  g_.total = g_.zs * (g_.nzl + 4);
  dx_ = c.extent / static_cast<double>(n);  // grid.hpp:98
  inv_dx_ = 1.0 / dx_;                      // step.cpp:62
  AF_CUDA(cudaMalloc(&d_u_, sizeof(double) * g_.total));
  AF_CUDA(cudaMalloc(&d_mid_, sizeof(double) * g_.total));
  AF_CUDA(cudaMemset(d_u_, 0, sizeof(double) * g_.total));
  AF_CUDA(cudaMemset(d_mid_, 0, sizeof(double) * g_.total));
  AF_CUDA(cudaMalloc(&d_err_, 2 * sizeof(int)));
  AF_CUDA(cudaStreamCreateWithFlags(&own_stream_, cudaStreamNonBlocking));
  stream_ = own_stream_;
  reset_error_();
  std::memset(&last_, 0, sizeof(last_));
  last_.step = -1;
  // NCCL ranks in 3D: the halo exchange runs on its own stream, overlapped
  // with the interior planes of each stage (stage3d_overlapped_)
  overlap_ = comm && comm->n > 1 && !comm->local && c.dim == 3 && g_.nzl >= 6 &&
             !std::getenv("AF_UNIFORM_NO_OVERLAP");
  if (overlap_) {
    AF_CUDA(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking));
    AF_CUDA(cudaEventCreateWithFlags(&ev_ready_, cudaEventDisableTiming));
    AF_CUDA(cudaEventCreateWithFlags(&ev_halo_, cudaEventDisableTiming));
  }
  const size_t sm3 = Fv3d<1, 32, kTY>::smem_bytes;
  for (auto fn : {(const void*)fv3d_stage<0, 32, kTY>, (const void*)fv3d_stage<1, 32, kTY>,
                  (const void*)fv3d_stage<2, 32, kTY>, (const void*)fv3d_stage<3, 32, kTY>,
                  (const void*)fv3d_stage<0, 16, kTY>, (const void*)fv3d_stage<1, 16, kTY>,
                  (const void*)fv3d_stage<2, 16, kTY>, (const void*)fv3d_stage<3, 16, kTY>,
                  (const void*)fv3d_stage<0, 8, kTY>, (const void*)fv3d_stage<1, 8, kTY>,
                  (const void*)fv3d_stage<2, 8, kTY>, (const void*)fv3d_stage<3, 8, kTY>})
    AF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3));
  const size_t smh = Hk<3, 8, 8, 4>::smem_bytes;
  for (auto fn : {(const void*)hancock_step<3, 0, 8, 8, 4>, (const void*)hancock_step<3, 1, 8, 8, 4>,
                  (const void*)hancock_step<3, 2, 8, 8, 4>, (const void*)hancock_step<3, 3, 8, 8, 4>})
    AF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smh));
  const char* te = std::getenv("AF_FV3D_TILE");
  tile_exact_ = !(te && te[0] == '0');
  if (c.dim == 3 && n >= kT3) {
    for (auto fn : {(const void*)fv3d_tile<0, kT3, kT3Y, kW3, 0>, (const void*)fv3d_tile<1, kT3, kT3Y, kW3, 0>,
                    (const void*)fv3d_tile<2, kT3, kT3Y, kW3, 0>, (const void*)fv3d_tile<3, kT3, kT3Y, kW3, 0>})
      AF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)Geo3::smem_bytes));
    fv3d_tol_setup();
    int per_sm = 0, sms = 0;
    AF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, fv3d_tile<1, kT3, kT3Y, kW3, 0>, Geo3::NT, Geo3::smem_bytes));
    AF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    tile_slots_ = std::max(1, per_sm * sms);
    // TMA descriptors: the slab allocation as a 4D tensor (x, y, component,
    // local plane); one (TX+4) x (TY+4) x 5 x 1 box per halo plane
    for (int b = 0; b < 2; ++b) {
      double* base = b == 0 ? d_u_ : d_mid_;
      const cuuint64_t dims[4] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)g_.ncomp,
                                  (cuuint64_t)(g_.nzl + 4)};
      const cuuint64_t strides[3] = {(cuuint64_t)n * 8, (cuuint64_t)g_.cs * 8,
                                     (cuuint64_t)g_.zs * 8};
      const cuuint32_t box[4] = {(cuuint32_t)Geo3::HX, (cuuint32_t)Geo3::HY, 5, 1};
      const cuuint32_t es[4] = {1, 1, 1, 1};
      const cuuint32_t obox[4] = {(cuuint32_t)kT3, (cuuint32_t)kT3Y, 5, 1};
      for (int own = 0; own < 2; ++own) {
        const CUresult r = encode_tiled()(own ? &tmo_[b] : &tm_[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                                          4, base, dims, strides, own ? obox : box, es,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw Error(AF_E_CUDA, "cuTensorMapEncodeTiled failed");
      }
      tm_base_[b] = base;
    }
  }
}

void Uniform::set_numerics(int numerics) {
  if (numerics != AF_NUMERICS_EXACT && numerics != AF_NUMERICS_TOLERANCE)
    throw Error(AF_E_ARGUMENT, "unknown numerics mode");
  numerics_ = numerics;
}

const CUtensorMap* Uniform::tensor_map_(const double* buf, bool own) {
  for (int b = 0; b < 2; ++b)
    if (tm_base_[b] == buf) return own ? &tmo_[b] : &tm_[b];
  return nullptr;
}

// The 3D RK2 stage on the TMA-fed 16x16 tile kernel (af_fv3d.cuh); false when
// the mesh is too small for it or the legacy kernel is selected.
bool Uniform::launch_tile3d_(const StageArgs& a, int zbeg, int zend) {
  const int n = g_.n;
  if (g_.dim != 3 || n < kT3) return false;
  // AF_FV3D_TILE=0 runs exact mode on the legacy 32x8 fv3d_stage instead
  // (bit-identical; tools/gpu/fv3d_check.py compares the two).
  if (numerics_ == AF_NUMERICS_EXACT && !tile_exact_) return false;
  const CUtensorMap* tm = tensor_map_(a.eval);
  const CUtensorMap* tb = tensor_map_(a.base, true);
  if (!tm || !tb) return false;
  const long tiles = (long)(n / kT3) * ((n + kT3Y - 1) / kT3Y);
  const int nz = zend - zbeg;
  // z chunks per tile column: all CTAs take about the same time, so pick the
  // count that minimises waves x (chunk planes + the 3-plane prologue) over
  // the resident CTA slots (wave quantisation against prologue overhead)
  int chunks = 1;
  if (const char* e = std::getenv("AF_FV3D_CHUNKS")) chunks = std::max(1, std::atoi(e));
  else {
    const long slots = (long)tile_slots_;
    double best = 1e300;
    for (int c = 1; c <= 16 && c <= std::max(1, nz / 8); ++c) {
      const long zc = (nz + c - 1) / c;
      const long cc = (nz + zc - 1) / zc;
      const double cost = (double)((tiles * cc + slots - 1) / slots) * (double)(zc + 3);
      if (cost < best * 0.999) {
        best = cost;
        chunks = (int)cc;
      }
    }
  }
  StageArgs b = a;
  b.zbeg = zbeg;
  b.zend = zend;
  b.zchunk = (nz + chunks - 1) / chunks;
  chunks = (nz + b.zchunk - 1) / b.zchunk;
  dim3 grid((unsigned)tiles, (unsigned)chunks);
  const int sch = cfg_.limiter | (cfg_.flux << 1);
  if (numerics_ == AF_NUMERICS_TOLERANCE) {
    fv3d_tol_launch(sch, grid, stream_, b, g_, *tm, *tb);
  } else {
#define AF_T3(S) \
  fv3d_tile<S, kT3, kT3Y, kW3, 0><<<grid, Geo3::NT, Geo3::smem_bytes, stream_>>>(b, g_, *tm, *tb)
    switch (sch) {
      case 0: AF_T3(0); break;
      case 1: AF_T3(1); break;
      case 2: AF_T3(2); break;
      default: AF_T3(3); break;
    }
#undef AF_T3
  }
  ++launches_;
  AF_CUDA(cudaGetLastError());
  return true;
}

Uniform::~Uniform() {
  cudaSetDevice(cfg_.device);
  if (own_stream_) cudaStreamSynchronize(own_stream_);
  cudaFree(d_u_);
  cudaFree(d_mid_);
  cudaFree(d_err_);
  cudaFree(d_stage_);
  cudaFree(d_cap_);
  free_records_();
  if (comm_stream_) {
    cudaStreamSynchronize(comm_stream_);
    cudaStreamDestroy(comm_stream_);
  }
  if (ev_ready_) cudaEventDestroy(ev_ready_);
  if (ev_halo_) cudaEventDestroy(ev_halo_);
  if (own_stream_) cudaStreamDestroy(own_stream_);
}

void Uniform::set_stream(cudaStream_t s) { stream_ = s ? s : own_stream_; }

void Uniform::reset_error_() {
  // flag = 0, first failing stage = 0x7f7f7f7f (larger than any step*2+1)
  AF_CUDA(cudaMemsetAsync(d_err_, 0, sizeof(int), stream_));
  AF_CUDA(cudaMemsetAsync(d_err_ + 1, 0x7f, sizeof(int), stream_));
}

void Uniform::free_records_() {
  cudaFree(rec_.smax);
  cudaFree(rec_.wave_u);
  cudaFree(rec_.wave_mid);
  cudaFree(rec_.fb);
  cudaFree(rec_.dt);
  rec_ = RunRecords{};
  rec_cap_ = 0;
}

void Uniform::ensure_records_(long n) {
  if (n <= rec_cap_) return;
  AF_CUDA(cudaStreamSynchronize(stream_));
  free_records_();
  const long cap = std::max<long>(n, 64);
  AF_CUDA(cudaMalloc(&rec_.smax, sizeof(unsigned long long) * (cap + 1)));
  AF_CUDA(cudaMalloc(&rec_.wave_u, sizeof(unsigned long long) * cap));
  AF_CUDA(cudaMalloc(&rec_.wave_mid, sizeof(unsigned long long) * cap));
  AF_CUDA(cudaMalloc(&rec_.fb, sizeof(unsigned long long) * cap));
  AF_CUDA(cudaMalloc(&rec_.dt, sizeof(double) * cap));
  rec_cap_ = cap;
}

void Uniform::ensure_staging_() {
  const size_t need = sizeof(double) * 5 * g_.plane * g_.nzl;
  if (stage_bytes_ >= need) return;
  AF_CUDA(cudaStreamSynchronize(stream_));
  cudaFree(d_stage_);
  d_stage_ = nullptr;
  AF_CUDA(cudaMalloc(&d_stage_, need));
  stage_bytes_ = need;
}

void Uniform::upload(const double* aos) {
  upload_to_(aos, d_u_);
  reset_error_();
}

void Uniform::upload_to_(const double* aos, double* dst) {
  if (!aos) throw Error(AF_E_ARGUMENT, "null state pointer");
  const size_t bytes = sizeof(double) * 5 * g_.plane * g_.nzl;
  const double* src = aos;
  if (!is_device_ptr(aos)) {
    ensure_staging_();
    AF_CUDA(cudaMemcpyAsync(d_stage_, aos, bytes, cudaMemcpyHostToDevice, stream_));
    src = d_stage_;
  }
  aos_to_soa<<<4 * 148, 256, 0, stream_>>>(src, dst, g_);
  ++launches_;
  AF_CUDA(cudaGetLastError());
}

void Uniform::download(double* aos) { download_from_(d_u_, aos); }

void Uniform::download_from_(const double* q, double* aos) {
  if (!aos) throw Error(AF_E_ARGUMENT, "null state pointer");
  const size_t bytes = sizeof(double) * 5 * g_.plane * g_.nzl;
  if (is_device_ptr(aos)) {
    soa_to_aos<<<4 * 148, 256, 0, stream_>>>(q, aos, g_);
    ++launches_;
    AF_CUDA(cudaGetLastError());
    AF_CUDA(cudaStreamSynchronize(stream_));
    return;
  }
  ensure_staging_();
  soa_to_aos<<<4 * 148, 256, 0, stream_>>>(q, d_stage_, g_);
  ++launches_;
  AF_CUDA(cudaGetLastError());
  AF_CUDA(cudaMemcpyAsync(aos, d_stage_, bytes, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
}

// Halo planes of `q` along the slab axis: 2 planes to each neighbour, one
// NCCL message per direction (per-plane SoA keeps them contiguous).
void Uniform::exchange_halos_(double* q, cudaStream_t st) {
  if (!comm_ || comm_->n == 1) return;
  if (!st) st = stream_;
  if (comm_->local) throw Error(AF_E_ARGUMENT, "ranks of a local group run via af_uniform_run_group");
  const int r = comm_->rank, P = comm_->n;
  const bool periodic = g_.bc[2 * (g_.dim - 1)] == AF_BC_PERIODIC &&
                        g_.bc[2 * (g_.dim - 1) + 1] == AF_BC_PERIODIC;
  const int lo = r > 0 ? r - 1 : (periodic ? P - 1 : -1);
  const int hi = r < P - 1 ? r + 1 : (periodic ? 0 : -1);
  const size_t cnt = (size_t)2 * g_.zs;
  ncclComm_t nc = comm_->nccl;
  auto ck = [](ncclResult_t e) {
    if (e != ncclSuccess) throw Error(AF_E_NCCL, ncclGetErrorString(e));
  };
  // Posting order (top->hi, low halo<-lo, bottom->lo, high halo<-hi) keeps the
  // pairwise send/recv matching right when lo == hi (two periodic ranks).
  ck(ncclGroupStart());
  if (hi >= 0) ck(ncclSend(q + (long)g_.nzl * g_.zs, cnt, ncclDouble, hi, nc, st));
  if (lo >= 0) ck(ncclRecv(q, cnt, ncclDouble, lo, nc, st));
  if (lo >= 0) ck(ncclSend(q + 2 * g_.zs, cnt, ncclDouble, lo, nc, st));
  if (hi >= 0) ck(ncclRecv(q + (long)(g_.nzl + 2) * g_.zs, cnt, ncclDouble, hi, nc, st));
  ck(ncclGroupEnd());
}

// dispatch on the scheme code sch = limiter | flux << 1
#define AF_SCHEME(M, TX) \
  switch (sch) {         \
    case 0: M(0, TX); break; \
    case 1: M(1, TX); break; \
    case 2: M(2, TX); break; \
    default: M(3, TX); break; \
  }

// One MUSCL-Hancock step (af_hancock.cuh): eval -> out.
void Uniform::launch_hancock_(const StageArgs& a) {
  const int n = g_.n;
  const int sch = cfg_.limiter | (cfg_.flux << 1);
  if (g_.dim == 3) {
    const unsigned tiles = (unsigned)((long)(n / 8) * (n / 8) * ((g_.nzl + 3) / 4));
    const size_t sm = Hk<3, 8, 8, 4>::smem_bytes;
#define AF_H3(S, TX) hancock_step<3, S, 8, 8, 4><<<tiles, 256, sm, stream_>>>(a, g_)
    AF_SCHEME(AF_H3, 8);
#undef AF_H3
  } else {
    const int tx = n >= 32 ? 32 : (n >= 16 ? 16 : 8);
    const unsigned tiles = (unsigned)((n / tx) * (g_.nzl / kTY));
#define AF_H2(S, TX) \
  hancock_step<2, S, TX, kTY, 1><<<tiles, TX * kTY, Hk<2, TX, kTY, 1>::smem_bytes, stream_>>>(a, g_)
    if (tx == 32) {
      AF_SCHEME(AF_H2, 32);
    } else if (tx == 16) {
      AF_SCHEME(AF_H2, 16);
    } else {
      AF_SCHEME(AF_H2, 8);
    }
#undef AF_H2
  }
  ++launches_;
  AF_CUDA(cudaGetLastError());
}

// Launch with the programmatic-stream-serialization attribute (PDL): the
// kernel's launch overlaps its predecessor's tail; the kernel waits
// (griddepcontrol.wait) before it reads anything. Used for the small 2D
// launches, where launch latency is the step's cost (cfg1).
template <class... P, class... A>
void launch_pdl(cudaStream_t s, void (*kern)(P...), dim3 grid, unsigned block, size_t smem,
                A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  AF_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...));
}

void Uniform::launch_stage_(const StageArgs& a0, int zbeg, int zend) {
  StageArgs a = a0;
  a.zbeg = zbeg < 0 ? g_.zlo : zbeg;
  a.zend = zend < 0 ? g_.zlo + g_.nzl : zend;
  if (a.zend <= a.zbeg) return;
  if (launch_tile3d_(a, a.zbeg, a.zend)) return;
  const int n = g_.n;
  const int tx = n >= 32 ? 32 : (n >= 16 ? 16 : 8);
  const int sch = cfg_.limiter | (cfg_.flux << 1);  // scheme code (af_physics.cuh)
  if (g_.dim == 3) {
    const long tiles = (long)(n / tx) * (n / kTY);
    const long target = 148L * 2 * 8;
    const int nz = a.zend - a.zbeg;
    int chunks = (int)std::max<long>(1, std::min<long>(target / tiles, nz / 8));
    StageArgs b = a;
    b.zchunk = (nz + chunks - 1) / chunks;
    chunks = (nz + b.zchunk - 1) / b.zchunk;
    dim3 grid((unsigned)tiles, (unsigned)chunks);
#define AF_L3(L, TX)                                                                     \
  fv3d_stage<L, TX, kTY><<<grid, TX * kTY, Fv3d<L, TX, kTY>::smem_bytes, stream_>>>(b, g_)
    if (tx == 32) {
      AF_SCHEME(AF_L3, 32);
    } else if (tx == 16) {
      AF_SCHEME(AF_L3, 16);
    } else {
      AF_SCHEME(AF_L3, 8);
    }
#undef AF_L3
  } else {
    const unsigned tiles = (unsigned)((n / tx) * (g_.nzl / kTY));
#define AF_L2(L, TX) \
  launch_pdl(stream_, fv2d_stage<L, TX, kTY>, dim3(tiles), TX * kTY, Fv2d<L, TX, kTY>::smem_bytes, a, g_)
    if (tx == 32) {
      AF_SCHEME(AF_L2, 32);
    } else if (tx == 16) {
      AF_SCHEME(AF_L2, 16);
    } else {
      AF_SCHEME(AF_L2, 8);
    }
#undef AF_L2
  }
  ++launches_;
  AF_CUDA(cudaGetLastError());
}

void Uniform::launch_speed_sum_(const double* q, unsigned long long* target) {
  if (g_.dim == 3)
    speed_sum_kernel<3><<<2 * 148, 256, 0, stream_>>>(q, g_, cfg_.gamma, target, d_err_);
  else
    launch_pdl(stream_, speed_sum_kernel<2>, dim3(2 * 148), 256, 0, q, g_, cfg_.gamma, target,
               (const int*)d_err_);
  ++launches_;
  AF_CUDA(cudaGetLastError());
}

// Enqueues n_steps RK2 steps (no host synchronisation).
void Uniform::enqueue_steps_(long n_steps, double cfl, double fixed_dt) {
  ensure_records_(n_steps);
  AF_CUDA(cudaMemsetAsync(rec_.smax, 0, sizeof(unsigned long long) * (n_steps + 1), stream_));
  AF_CUDA(cudaMemsetAsync(rec_.wave_u, 0, sizeof(unsigned long long) * n_steps, stream_));
  AF_CUDA(cudaMemsetAsync(rec_.wave_mid, 0, sizeof(unsigned long long) * n_steps, stream_));
  AF_CUDA(cudaMemsetAsync(rec_.fb, 0, sizeof(unsigned long long) * n_steps, stream_));
  RunRecords r = rec_;
  r.err = d_err_;
  StageArgs a{};
  a.dx = dx_;
  a.inv_dx = inv_dx_;
  a.gamma = cfg_.gamma;
  a.gm1 = cfg_.gamma - 1.0;
  a.cfl = cfl;
  a.fixed_dt = fixed_dt;
  a.use_cfl = cfl > 0.0 ? 1 : 0;
  a.r = r;
  if (a.use_cfl) {
    launch_speed_sum_(d_u_, rec_.smax);
    if (comm_ && comm_->n > 1) allreduce_max_(rec_.smax);
  }
  hk_u0_ = d_u_;
  hk_m0_ = d_mid_;
  if (cfg_.integrator == AF_INTEGRATOR_MUSCL_HANCOCK) {
    // muscl_hancock_step (step.cpp:148-235): one launch per step, u -> mid,
    // then the buffers swap roles (the step-s input is hk_u0_ for even s)
    for (long s = 0; s < n_steps; ++s) {
      a.step = (int)s;
      exchange_halos_(d_u_);
      a.stage = 1;
      a.dt_scale = 1.0;
      a.eval = d_u_;
      a.base = d_u_;
      a.out = d_mid_;
      launch_hancock_(a);
      std::swap(d_u_, d_mid_);
      if (a.use_cfl && comm_ && comm_->n > 1) allreduce_max_(rec_.smax + s + 1);
    }
    return;
  }
  for (long s = 0; s < n_steps; ++s) {
    a.step = (int)s;
    a.stage = 1;
    a.dt_scale = 0.5;
    a.eval = d_u_;
    a.base = d_u_;
    a.out = d_mid_;
    if (overlap_) {
      stage3d_overlapped_(a, d_u_);
    } else {
      exchange_halos_(d_u_);
      launch_stage_(a);
    }
    a.stage = 2;
    a.dt_scale = 1.0;
    a.eval = d_mid_;
    a.base = d_u_;
    a.out = d_u_;
    if (overlap_) {
      stage3d_overlapped_(a, d_mid_);
    } else {
      exchange_halos_(d_mid_);
      launch_stage_(a);
    }
    if (a.use_cfl && comm_ && comm_->n > 1) allreduce_max_(rec_.smax + s + 1);
  }
}

// One 3D RK stage with the halo exchange of `eval` overlapped: the interior
// planes [zlo+2, zlo+nzl-2) read no halo plane, so they run while NCCL moves
// the halo planes on comm_stream_; the two planes at each slab end follow
// once the halos have arrived. Per stage and neighbour the
// exchange carries 2 planes x 5 components x n^2 doubles (21 MB at 512^2).
void Uniform::stage3d_overlapped_(const StageArgs& a, double* eval) {
  AF_CUDA(cudaEventRecord(ev_ready_, stream_));
  AF_CUDA(cudaStreamWaitEvent(comm_stream_, ev_ready_, 0));
  exchange_halos_(eval, comm_stream_);
  AF_CUDA(cudaEventRecord(ev_halo_, comm_stream_));
  const int z0 = g_.zlo, z1 = g_.zlo + g_.nzl;
  launch_stage_(a, z0 + 2, z1 - 2);
  AF_CUDA(cudaStreamWaitEvent(stream_, ev_halo_, 0));
  launch_stage_(a, z0, z0 + 2);
  launch_stage_(a, z1 - 2, z1);
}

namespace {
struct GroupPtrs {
  unsigned long long* p[16];
};
__global__ void group_max_kernel(GroupPtrs g, int n) {
  unsigned long long m = 0;
  for (int r = 0; r < n; ++r) m = m > *g.p[r] ? m : *g.p[r];
  for (int r = 0; r < n; ++r) *g.p[r] = m;
}
}  // namespace

void Uniform::run_group(const std::vector<Uniform*>& R, long n_steps, double cfl,
                        double fixed_dt, double* dt_hist, af_run_diag* rd) {
  const int P = (int)R.size();
  if (P < 1 || P > 16) throw Error(AF_E_ARGUMENT, "group size must be in [1, 16]");
  if (!(cfl > 0.0) && !(fixed_dt > 0.0))
    throw Error(AF_E_ARGUMENT, "either cfl or fixed_dt must be positive");
  cudaStream_t st = R[0]->stream_;
  std::vector<StageArgs> A(P);
  for (int r = 0; r < P; ++r) {
    Uniform& u = *R[r];
    u.stream_ = st;
    u.ensure_records_(n_steps);
    AF_CUDA(cudaMemsetAsync(u.rec_.smax, 0, 8 * (n_steps + 1), st));
    AF_CUDA(cudaMemsetAsync(u.rec_.wave_u, 0, 8 * n_steps, st));
    AF_CUDA(cudaMemsetAsync(u.rec_.wave_mid, 0, 8 * n_steps, st));
    AF_CUDA(cudaMemsetAsync(u.rec_.fb, 0, 8 * n_steps, st));
    StageArgs& a = A[r];
    a = StageArgs{};
    a.dx = u.dx_;
    a.inv_dx = u.inv_dx_;
    a.gamma = u.cfg_.gamma;
    a.gm1 = u.cfg_.gamma - 1.0;
    a.cfl = cfl;
    a.fixed_dt = fixed_dt;
    a.use_cfl = cfl > 0.0 ? 1 : 0;
    a.r = u.rec_;
    a.r.err = u.d_err_;
  }
  const UGrid& g0 = R[0]->g_;
  const int axis = g0.dim - 1;
  const bool periodic = g0.bc[2 * axis] == AF_BC_PERIODIC && g0.bc[2 * axis + 1] == AF_BC_PERIODIC;
  // halo planes of buffer `which` (0 = u, 1 = mid) between neighbouring slabs
  auto exchange = [&](int which) {
    for (int r = 0; r < P; ++r) {
      const int hi = r < P - 1 ? r + 1 : (periodic ? 0 : -1);
      if (hi < 0 || P == 1) continue;
      Uniform& a = *R[r];
      Uniform& b = *R[hi];
      double* qa = which ? a.d_mid_ : a.d_u_;
      double* qb = which ? b.d_mid_ : b.d_u_;
      const size_t bytes = sizeof(double) * 2 * a.g_.zs;
      // a's top two planes -> b's low halo; b's bottom two planes -> a's high halo
      AF_CUDA(cudaMemcpyAsync(qb, qa + (long)a.g_.nzl * a.g_.zs, bytes, cudaMemcpyDeviceToDevice, st));
      AF_CUDA(cudaMemcpyAsync(qa + (long)(a.g_.nzl + 2) * a.g_.zs, qb + 2 * b.g_.zs, bytes,
                              cudaMemcpyDeviceToDevice, st));
    }
  };
  auto group_max = [&](long slot) {
    GroupPtrs gp{};
    for (int r = 0; r < P; ++r) gp.p[r] = R[r]->rec_.smax + slot;
    group_max_kernel<<<1, 1, 0, st>>>(gp, P);
    AF_CUDA(cudaGetLastError());
  };
  if (cfl > 0.0) {
    for (int r = 0; r < P; ++r) R[r]->launch_speed_sum_(R[r]->d_u_, R[r]->rec_.smax);
    group_max(0);
  }
  for (int r = 0; r < P; ++r) {
    R[r]->hk_u0_ = R[r]->d_u_;
    R[r]->hk_m0_ = R[r]->d_mid_;
  }
  const bool hancock = R[0]->cfg_.integrator == AF_INTEGRATOR_MUSCL_HANCOCK;
  for (long s = 0; s < n_steps && hancock; ++s) {
    exchange(0);
    for (int r = 0; r < P; ++r) {
      StageArgs& a = A[r];
      a.step = (int)s;
      a.stage = 1;
      a.dt_scale = 1.0;
      a.eval = R[r]->d_u_;
      a.base = R[r]->d_u_;
      a.out = R[r]->d_mid_;
      R[r]->launch_hancock_(a);
      std::swap(R[r]->d_u_, R[r]->d_mid_);
    }
    if (cfl > 0.0) group_max(s + 1);
  }
  // 3D: the interior planes of every rank first, then the exchange, then the
  // slab-end planes (the launch split of stage3d_overlapped_; on one stream
  // here, so it checks the split, not the overlap)
  const bool split = g0.dim == 3 && P > 1;
  auto stage_all = [&](int which) {
    for (int r = 0; r < P; ++r) {
      StageArgs& a = A[r];
      a.stage = which + 1;
      a.dt_scale = which ? 1.0 : 0.5;
      a.eval = which ? R[r]->d_mid_ : R[r]->d_u_;
      a.base = R[r]->d_u_;
      a.out = which ? R[r]->d_u_ : R[r]->d_mid_;
      const int z0 = R[r]->g_.zlo, z1 = z0 + R[r]->g_.nzl;
      if (split && z1 - z0 >= 6) R[r]->launch_stage_(a, z0 + 2, z1 - 2);
    }
    exchange(which);
    for (int r = 0; r < P; ++r) {
      StageArgs& a = A[r];
      const int z0 = R[r]->g_.zlo, z1 = z0 + R[r]->g_.nzl;
      if (split && z1 - z0 >= 6) {
        R[r]->launch_stage_(a, z0, z0 + 2);
        R[r]->launch_stage_(a, z1 - 2, z1);
      } else {
        R[r]->launch_stage_(a);
      }
    }
  };
  for (long s = 0; s < n_steps && !hancock; ++s) {
    for (int r = 0; r < P; ++r) A[r].step = (int)s;
    stage_all(0);
    stage_all(1);
    if (cfl > 0.0) group_max(s + 1);
  }
  // per-rank records -> the run's diagnostics (max/sum over ranks)
  af_run_diag total{};
  for (int r = 0; r < P; ++r) {
    af_run_diag d{};
    std::vector<double> dts(n_steps);
    R[r]->collect_(n_steps, dts.data(), &d, nullptr);
    if (r == 0 && dt_hist) std::memcpy(dt_hist, dts.data(), sizeof(double) * n_steps);
    total.max_wave_speed = std::max(total.max_wave_speed, d.max_wave_speed);
    total.fallbacks += d.fallbacks;
    total.steps_done = d.steps_done;
    total.t = d.t;
  }
  // max_cfl from the combined per-step wave maxima (unigrid.cpp:43)
  if (rd) {
    std::vector<double> ms(n_steps, 0.0), dts(n_steps);
    for (int r = 0; r < P; ++r) {
      std::vector<unsigned long long> wu(n_steps), wm(n_steps);
      AF_CUDA(cudaMemcpy(wu.data(), R[r]->rec_.wave_u, 8 * n_steps, cudaMemcpyDeviceToHost));
      AF_CUDA(cudaMemcpy(wm.data(), R[r]->rec_.wave_mid, 8 * n_steps, cudaMemcpyDeviceToHost));
      if (r == 0) AF_CUDA(cudaMemcpy(dts.data(), R[0]->rec_.dt, 8 * n_steps, cudaMemcpyDeviceToHost));
      for (long s = 0; s < n_steps; ++s) {
        double a, b;
        std::memcpy(&a, &wu[s], 8);
        std::memcpy(&b, &wm[s], 8);
        ms[s] = std::max(ms[s], std::max(a, b));
      }
    }
    double mc = 0.0;
    for (long s = 0; s < n_steps; ++s) mc = std::max(mc, ms[s] * dts[s] / R[0]->dx_);
    total.max_cfl = mc;
    *rd = total;
  }
}

void Uniform::allreduce_max_(unsigned long long* bits) {
  if (comm_->local) throw Error(AF_E_ARGUMENT, "ranks of a local group run via af_uniform_run_group");
  // max of non-negative doubles == max of their bit patterns
  const ncclResult_t e = ncclAllReduce(bits, bits, 1, ncclUint64, ncclMax, comm_->nccl, stream_);
  if (e != ncclSuccess) throw Error(AF_E_NCCL, ncclGetErrorString(e));
}

// Reads the device error record; on failure rebuilds the reference's
// message (first offender in build_primitives' scan order, step.cpp:22-38).
void Uniform::check_error_() {
  int h[2];
  AF_CUDA(cudaMemcpyAsync(h, d_err_, sizeof h, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  if (!h[0]) return;
  const long step = h[1] / 2;
  const int stage = h[1] % 2 + 1;
  const double* eval = stage == 1 ? d_u_ : d_mid_;
  if (cfg_.integrator == AF_INTEGRATOR_MUSCL_HANCOCK) eval = step % 2 ? hk_m0_ : hk_u0_;
  if (err_eval_) eval = err_eval_;
  std::vector<double> hs(g_.total);
  AF_CUDA(cudaMemcpy(hs.data(), eval, sizeof(double) * g_.total, cudaMemcpyDeviceToHost));
  std::memset(&last_, 0, sizeof(last_));
  last_.status = AF_E_NONPHYSICAL;
  last_.step = step;
  last_.stage = stage;
  last_.level = -1;
  const int n = g_.n, dim = g_.dim;
  const double gm1 = cfg_.gamma - 1.0;
  auto map = [&](int c, int axis, bool& flip) {
    flip = false;
    if (c >= 0 && c < n) return c;
    const int kind = c < 0 ? g_.bc[2 * axis] : g_.bc[2 * axis + 1];
    if (kind == AF_BC_OUTFLOW) return c < 0 ? 0 : n - 1;
    if (kind == AF_BC_PERIODIC) return ((c % n) + n) % n;
    while (c < 0 || c >= n) {
      if (c < 0) c = -1 - c;
      if (c >= n) c = 2 * n - 1 - c;
      flip = !flip;
    }
    return c;
  };
  const int gz = dim == 3 ? 2 : 0;
  const int nk = dim == 3 ? n : 1;
  bool found = false;
  // The slab owns global slab-axis range [zlo, zlo+nzl); ghosts beyond the
  // global domain are scanned by the owning edge rank.
  for (int k = -gz; k < nk + gz && !found; ++k)
    for (int j = -2; j < n + 2 && !found; ++j)
      for (int i = -2; i < n + 2 && !found; ++i) {
        const int sl = dim == 3 ? k : j;  // slab-axis coordinate
        bool f;
        const int msl = map(sl, dim - 1, f);
        if (msl < g_.zlo || msl >= g_.zlo + g_.nzl) continue;
        const int mi = map(i, 0, f);
        const int mj = dim == 3 ? map(j, 1, f) : msl;
        const long off = (long)(msl - g_.zlo + 2) * g_.zs + (dim == 3 ? (long)mj * n : 0) + mi;
        const double rho = hs[off];
        double msq = hs[g_.cs + off] * hs[g_.cs + off] + hs[2 * g_.cs + off] * hs[2 * g_.cs + off];
        if (dim == 3) msq = msq + hs[3 * g_.cs + off] * hs[3 * g_.cs + off];
        const double E = hs[(g_.ncomp - 1) * g_.cs + off];
        const double inv_rho = 1.0 / rho;
        const double kin = 0.5 * msq * inv_rho;
        const double p = gm1 * (E - kin);
        if (!(rho > 1e-12) || !(rho > 1e-12 && p > 1e-12)) {
          found = true;
          const bool ghost = i < 0 || i >= n || j < 0 || j >= n || (dim == 3 && (k < 0 || k >= n));
          last_.i = i;
          last_.j = j;
          last_.k = dim == 3 ? k : 0;
          last_.is_ghost = ghost;
          last_.rho = rho;
          last_.p = p;
          std::string cs = "(" + std::to_string(i) + "," + std::to_string(j);
          if (dim == 3) cs += "," + std::to_string(k);
          cs += ")";
          const std::string msg = (seam_msg_ ? std::string() : "step " + std::to_string(step) + ": ") + "cell " + cs +
                                  (ghost ? " (ghost)" : "") + ": rho=" + fmt_f(rho) +
                                  " p=" + fmt_f(p);
          std::snprintf(last_.message, sizeof last_.message, "%s", msg.c_str());
        }
      }
  if (!found)
    std::snprintf(last_.message, sizeof last_.message,
                  "step %ld: non-physical state on another rank", step);
  throw Error(AF_E_NONPHYSICAL, last_.message);
}

void Uniform::collect_(long n_steps, double* dt_hist, af_run_diag* rd, af_step_diag* sd) {
  check_error_();
  std::vector<unsigned long long> wu(n_steps), wm(n_steps), fb(n_steps);
  std::vector<double> dts(n_steps);
  AF_CUDA(cudaMemcpyAsync(wu.data(), rec_.wave_u, 8 * n_steps, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaMemcpyAsync(wm.data(), rec_.wave_mid, 8 * n_steps, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaMemcpyAsync(fb.data(), rec_.fb, 8 * n_steps, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaMemcpyAsync(dts.data(), rec_.dt, 8 * n_steps, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  auto asd = [](unsigned long long b) {
    double d;
    std::memcpy(&d, &b, 8);
    return d;
  };
  double max_ws = 0.0, max_cfl = 0.0, t = 0.0;
  long fbs = 0;
  for (long s = 0; s < n_steps; ++s) {
    const double ms = std::max(asd(wu[s]), asd(wm[s]));  // step.cpp:243
    max_ws = std::max(max_ws, ms);
    max_cfl = std::max(max_cfl, ms * dts[s] / dx_);  // unigrid.cpp:43
    fbs += (long)fb[s];
    t += dts[s];
  }
  if (dt_hist) std::memcpy(dt_hist, dts.data(), sizeof(double) * n_steps);
  if (rd) {
    rd->max_wave_speed = max_ws;
    rd->max_cfl = max_cfl;
    rd->fallbacks = fbs;
    rd->steps_done = n_steps;
    rd->t = t;
  }
  if (sd) {
    sd->max_wave_speed = max_ws;
    sd->fallbacks = fbs;
  }
}

void Uniform::launch_flux_capture_(const double* q, double* dst) {
  const int sch = cfg_.limiter | (cfg_.flux << 1);
  const unsigned grid = 148 * 8;
#define AF_CAP(D)                                                                         \
  switch (sch) {                                                                          \
    case 0: flux_capture_kernel<D, 0><<<grid, 256, 0, stream_>>>(q, g_, dst, cfg_.gamma); break; \
    case 1: flux_capture_kernel<D, 1><<<grid, 256, 0, stream_>>>(q, g_, dst, cfg_.gamma); break; \
    case 2: flux_capture_kernel<D, 2><<<grid, 256, 0, stream_>>>(q, g_, dst, cfg_.gamma); break; \
    default: flux_capture_kernel<D, 3><<<grid, 256, 0, stream_>>>(q, g_, dst, cfg_.gamma); break; \
  }
  if (g_.dim == 3) {
    AF_CAP(3)
  } else {
    AF_CAP(2)
  }
#undef AF_CAP
  ++launches_;
  AF_CUDA(cudaGetLastError());
}

// rk2_stage (step.hpp:62-64, step.cpp:93-109): out = base + stage_dt * rhs(eval)
// with eval's ghosts the configured boundary conditions (fill_ghosts,
// grid.cpp:9-62). base goes to d_u_, eval to d_mid_, the stage writes d_u_.
// capture: the stage's face fluxes in FluxField layout (step.hpp:16-50),
// recomputed by flux_capture (the same operations as the stage kernels, so the
// same bits). The reference's NonPhysicalState text has no step prefix here.
void Uniform::rk2_stage(const double* base, const double* eval, double* out, double stage_dt,
                        double* capture, af_step_diag* diag) {
  if (comm_ && comm_->n > 1)
    throw Error(AF_E_UNSUPPORTED, "rk2_stage: single-rank solvers only");
  if (!base || !eval || !out) throw Error(AF_E_ARGUMENT, "null state pointer");
  if (capture && numerics_ == AF_NUMERICS_TOLERANCE && g_.dim == 3)
    throw Error(AF_E_UNSUPPORTED, "rk2_stage: flux capture needs exact numerics");
  upload_to_(base, d_u_);
  upload_to_(eval, d_mid_);
  reset_error_();
  ensure_records_(1);
  AF_CUDA(cudaMemsetAsync(rec_.smax, 0, sizeof(unsigned long long) * 2, stream_));
  AF_CUDA(cudaMemsetAsync(rec_.wave_u, 0, sizeof(unsigned long long), stream_));
  AF_CUDA(cudaMemsetAsync(rec_.wave_mid, 0, sizeof(unsigned long long), stream_));
  AF_CUDA(cudaMemsetAsync(rec_.fb, 0, sizeof(unsigned long long), stream_));
  StageArgs a{};
  a.dx = dx_;
  a.inv_dx = inv_dx_;
  a.gamma = cfg_.gamma;
  a.gm1 = cfg_.gamma - 1.0;
  a.fixed_dt = stage_dt;
  a.use_cfl = 0;
  a.r = rec_;
  a.r.err = d_err_;
  a.step = 0;
  a.stage = 1;
  a.dt_scale = 1.0;
  a.eval = d_mid_;
  a.base = d_u_;
  a.out = d_u_;
  launch_stage_(a);
  if (capture) {
    const int n = g_.n, dim = g_.dim;
    const long per = dim == 3 ? (long)(n + 1) * n * n : (long)(n + 1) * n;
    const long faces = dim * per;
    double* dst = capture;
    if (!is_device_ptr(capture)) {
      if (cap_cap_ < faces) {
        cudaFree(d_cap_);
        AF_CUDA(cudaMalloc(&d_cap_, sizeof(double) * 5 * faces));
        cap_cap_ = faces;
      }
      dst = d_cap_;
    }
    launch_flux_capture_(d_mid_, dst);
    if (dst != capture)
      AF_CUDA(cudaMemcpyAsync(capture, dst, sizeof(double) * 5 * faces, cudaMemcpyDeviceToHost,
                              stream_));
  }
  err_eval_ = d_mid_;
  seam_msg_ = true;
  try {
    af_step_diag d{};
    collect_(1, nullptr, nullptr, &d);
    if (diag) *diag = d;
  } catch (...) {
    err_eval_ = nullptr;
    seam_msg_ = false;
    throw;
  }
  err_eval_ = nullptr;
  seam_msg_ = false;
  download_from_(d_u_, out);
}

void Uniform::step(double dt, af_step_diag* diag) {
  if (!(dt > 0.0)) throw Error(AF_E_ARGUMENT, "dt must be positive");
  enqueue_steps_(1, 0.0, dt);
  if (diag) collect_(1, nullptr, nullptr, diag);
}

void Uniform::run(long n_steps, double cfl, double fixed_dt, double* dt_hist, af_run_diag* rd) {
  if (n_steps < 0) throw Error(AF_E_ARGUMENT, "n_steps must be >= 0");
  if (n_steps == 0) {
    if (rd) *rd = af_run_diag{};
    return;
  }
  if (!(cfl > 0.0) && !(fixed_dt > 0.0))
    throw Error(AF_E_ARGUMENT, "either cfl or fixed_dt must be positive");
  enqueue_steps_(n_steps, cfl, fixed_dt);
  if (dt_hist || rd) collect_(n_steps, dt_hist, rd, nullptr);
}

double Uniform::speed_sum() {
  ensure_records_(1);
  AF_CUDA(cudaMemsetAsync(rec_.smax, 0, sizeof(unsigned long long), stream_));
  launch_speed_sum_(d_u_, rec_.smax);
  if (comm_ && comm_->n > 1) allreduce_max_(rec_.smax);
  unsigned long long b = 0;
  AF_CUDA(cudaMemcpyAsync(&b, rec_.smax, 8, cudaMemcpyDeviceToHost, stream_));
  AF_CUDA(cudaStreamSynchronize(stream_));
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}

void Uniform::sync() { check_error_(); }

}  // namespace af
