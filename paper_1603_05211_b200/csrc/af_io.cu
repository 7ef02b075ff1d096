// af_io.cu — the formats and compare path either side of the hot path
// (SURVEY.md §8(f) "next" #2-3):
//   * AFSN v1 snapshots (snapshot.hpp:10-22, snapshot.cpp:29-104), bit-exact
//     round trips, for checkpoint/resume of GPU runs and golden exchange;
//   * MRTree::dump (mr_tree.cpp:623-641) of the device tree;
//   * restrict_to_level (grid.cpp:64-93) and l1_error (metrics.cpp:134-148)
//     on the device.
// The ABI's cell layout is AoS, 5 doubles per cell (rho, mom0, mom1, mom2,
// rhoE; mom2 = 0 in 2D), x fastest.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "af_internal.h"
#include "af_mr.h"
#include "af_physics.cuh"

namespace af {

namespace {

constexpr char kMagic[4] = {'A', 'F', 'S', 'N'};
constexpr uint32_t kVersion = 1;

template <typename T>
void put(std::ostream& os, T v) {
  os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
T get(std::istream& is) {
  T v{};
  is.read(reinterpret_cast<char*>(&v), sizeof(T));
  return v;
}

// One coarsening step of restrict_to_level: s = 0; s += child (dk, dj, di
// order); coarse = s * w (grid.cpp:76-89).
__global__ void restrict_kernel(const double* fine, double* coarse, int dim, int nc) {
  const long cells = dim == 3 ? (long)nc * nc * nc : (long)nc * nc;
  const int nf = 2 * nc;
  const double w = dim == 3 ? 0.125 : 0.25;
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < cells;
       c += (long)gridDim.x * blockDim.x) {
    const int i = (int)(c % nc), j = (int)((c / nc) % nc), k = dim == 3 ? (int)(c / ((long)nc * nc)) : 0;
    double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    const int kcnt = dim == 3 ? 2 : 1;
    for (int dk = 0; dk < kcnt; ++dk)
      for (int dj = 0; dj < 2; ++dj)
        for (int di = 0; di < 2; ++di) {
          const long f = dim == 3 ? ((long)(2 * k + dk) * nf + 2 * j + dj) * nf + 2 * i + di
                                  : (long)(2 * j + dj) * nf + 2 * i + di;
#pragma unroll
          for (int m = 0; m < 5; ++m) s[m] = s[m] + fine[5 * f + m];
        }
#pragma unroll
    for (int m = 0; m < 5; ++m) coarse[5 * c + m] = s[m] * w;
  }
}

// sum over cells of |a - r| per component (fp64 atomics on a per-block sum;
// the association differs from the reference's sequential loop)
__global__ void l1_kernel(const double* a, const double* r, long cells, double* out) {
  __shared__ double red[5][8];
  double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < cells;
       c += (long)gridDim.x * blockDim.x)
#pragma unroll
    for (int m = 0; m < 5; ++m) s[m] += fabs(a[5 * c + m] - r[5 * c + m]);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < 5; ++m) {
    double v = s[m];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[m][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) v += red[threadIdx.x][w];
    atomicAdd(out + threadIdx.x, v);
  }
}

// device copy of an AoS array that may live on the host
struct DevArray {
  const double* p = nullptr;
  double* own = nullptr;
  DevArray(const double* src, size_t n) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeDevice) {
      p = src;
      return;
    }
    cudaGetLastError();
    AF_CUDA(cudaMalloc(&own, n * sizeof(double)));
    AF_CUDA(cudaMemcpy(own, src, n * sizeof(double), cudaMemcpyDefault));
    p = own;
  }
  ~DevArray() {
    if (own) cudaFree(own);
  }
};

long cells_of(int dim, int level) { return dim == 3 ? 1L << (3 * level) : 1L << (2 * level); }

}  // namespace

void snapshot_write(const char* path, const af_snapshot_header& h, const double* aos) {
  if (h.dim != 2 && h.dim != 3) throw Error(AF_E_ARGUMENT, "snapshot: dim must be 2 or 3");
  std::ofstream os(path, std::ios::binary | std::ios::trunc);
  if (!os) throw Error(AF_E_IO, std::string("cannot open snapshot for writing: ") + path);
  const uint64_t n = 1ull << h.level;
  os.write(kMagic, 4);
  put<uint32_t>(os, kVersion);
  put<uint32_t>(os, (uint32_t)h.dim);
  put<int32_t>(os, h.level);
  put<uint64_t>(os, n);
  put<double>(os, h.gamma);
  put<double>(os, h.time);
  put<double>(os, h.origin);
  put<double>(os, h.extent);
  const long nz = h.dim == 3 ? (long)n : 1;
  std::vector<double> row(n * (h.dim + 2));
  for (long k = 0; k < nz; ++k)
    for (long j = 0; j < (long)n; ++j) {
      size_t w = 0;
      for (long i = 0; i < (long)n; ++i) {
        const double* q = aos + 5 * ((k * (long)n + j) * (long)n + i);
        row[w++] = q[0];
        for (int c = 0; c < h.dim; ++c) row[w++] = q[1 + c];
        row[w++] = q[4];
      }
      os.write(reinterpret_cast<const char*>(row.data()), (std::streamsize)(w * sizeof(double)));
    }
  if (!os) throw Error(AF_E_IO, std::string("short write on snapshot: ") + path);
}

void snapshot_read(const char* path, af_snapshot_header* h, double* aos) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw Error(AF_E_IO, std::string("cannot open snapshot: ") + path);
  char magic[4];
  is.read(magic, 4);
  if (!is || std::memcmp(magic, kMagic, 4) != 0)
    throw Error(AF_E_IO, std::string("not a snapshot file: ") + path);
  const uint32_t version = get<uint32_t>(is);
  if (version != kVersion)
    throw Error(AF_E_IO, "unsupported snapshot version " + std::to_string(version));
  const uint32_t dim = get<uint32_t>(is);
  const int32_t level = get<int32_t>(is);
  const uint64_t n = get<uint64_t>(is);
  af_snapshot_header hh;
  hh.gamma = get<double>(is);
  hh.time = get<double>(is);
  hh.origin = get<double>(is);
  hh.extent = get<double>(is);
  if ((dim != 2 && dim != 3) || level < 0 || level > 30 || n != (uint64_t(1) << level))
    throw Error(AF_E_IO, std::string("inconsistent snapshot header: ") + path);
  hh.dim = (int)dim;
  hh.level = level;
  *h = hh;
  if (!aos) return;
  const long nz = dim == 3 ? (long)n : 1;
  std::vector<double> row(n * (dim + 2));
  for (long k = 0; k < nz; ++k)
    for (long j = 0; j < (long)n; ++j) {
      is.read(reinterpret_cast<char*>(row.data()), (std::streamsize)(row.size() * sizeof(double)));
      if (!is) throw Error(AF_E_IO, std::string("truncated snapshot payload: ") + path);
      size_t r = 0;
      for (long i = 0; i < (long)n; ++i) {
        double* q = aos + 5 * ((k * (long)n + j) * (long)n + i);
        q[0] = row[r++];
        q[1] = row[r++];
        q[2] = row[r++];
        q[3] = dim == 3 ? row[r++] : 0.0;
        q[4] = row[r++];
      }
    }
}

void restrict_to_level(int dim, int fine_level, int target, const double* fine, double* out) {
  if (dim != 2 && dim != 3) throw Error(AF_E_ARGUMENT, "restrict_to_level: dim must be 2 or 3");
  if (target > fine_level)
    throw Error(AF_E_LEVEL_MISMATCH, "restrict_to_level: target " + std::to_string(target) +
                                         " finer than input level " + std::to_string(fine_level));
  if (target < 0) throw Error(AF_E_ARGUMENT, "restrict_to_level: negative level");
  const long nf = cells_of(dim, fine_level);
  DevArray src(fine, 5 * (size_t)nf);
  double* a = nullptr;
  double* b = nullptr;
  AF_CUDA(cudaMalloc(&a, 5 * sizeof(double) * (size_t)nf));
  AF_CUDA(cudaMemcpy(a, src.p, 5 * sizeof(double) * (size_t)nf, cudaMemcpyDeviceToDevice));
  if (fine_level > target) AF_CUDA(cudaMalloc(&b, 5 * sizeof(double) * (size_t)cells_of(dim, fine_level - 1)));
  for (int l = fine_level; l > target; --l) {
    const long nc = cells_of(dim, l - 1);
    const unsigned grid = (unsigned)std::max<long>(1, std::min<long>((nc + 255) / 256, 148 * 8));
    restrict_kernel<<<grid, 256>>>(a, b, dim, 1 << (l - 1));
    AF_CUDA(cudaGetLastError());
    std::swap(a, b);
  }
  AF_CUDA(cudaMemcpy(out, a, 5 * sizeof(double) * (size_t)cells_of(dim, target), cudaMemcpyDefault));
  cudaFree(a);
  cudaFree(b);
}

void l1_error(int dim, int level, double extent, const double* sol, int ref_level,
              const double* ref, double* out5) {
  if (ref_level < level)
    throw Error(AF_E_LEVEL_MISMATCH, "l1_error: reference level " + std::to_string(ref_level) +
                                         " coarser than solution level " + std::to_string(level));
  const long cells = cells_of(dim, level);
  double* r = nullptr;
  AF_CUDA(cudaMalloc(&r, 5 * sizeof(double) * (size_t)cells));
  restrict_to_level(dim, ref_level, level, ref, r);
  DevArray a(sol, 5 * (size_t)cells);
  double* d = nullptr;
  AF_CUDA(cudaMalloc(&d, 5 * sizeof(double)));
  AF_CUDA(cudaMemset(d, 0, 5 * sizeof(double)));
  const unsigned grid = (unsigned)std::max<long>(1, std::min<long>((cells + 255) / 256, 148 * 4));
  l1_kernel<<<grid, 256>>>(a.p, r, cells, d);
  AF_CUDA(cudaGetLastError());
  double s[5];
  AF_CUDA(cudaMemcpy(s, d, sizeof s, cudaMemcpyDeviceToHost));
  cudaFree(d);
  cudaFree(r);
  const double dx = extent / static_cast<double>(1L << level);
  double v = dx * dx;
  if (dim == 3) v = v * dx;  // UniformGrid::cell_volume (grid.hpp:107-110)
  for (int m = 0; m < 5; ++m) out5[m] = s[m] * v;
}

// MRTree::dump (mr_tree.cpp:623-641): every node in ascending key order,
// "level i j k status rho mom0 mom1 mom2 rhoE" with 17 significant digits.
std::string MR::dump() {
  refresh_coarse_();
  std::vector<uint8_t> hs(g_.total_cells);
  std::vector<double> hv((size_t)NC_ * g_.total_cells);
  wtohost_(hs.data(), d_st_, 1, 1);
  wtohost_(hv.data(), d_V_, 8, NC_);
  std::vector<uint8_t> vm;
  if (virtuals_) {
    vm.resize(g_.total_cells);
    wtohost_(vm.data(), d_mark_, 1, 1);
  }
  const long comp = g_.total_cells;
  std::string out;
  char line[512];
  for (int l = 0; l <= L_; ++l) {
    const int n = 1 << l;
    const int nk = D_ == 3 ? n : 1;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < nk; ++k) {
          const long c = g_.cell_off[l] + mr_idx(g_, D_, n, i, j, k);
          const uint8_t st = hs[c];
          bool virt = false;
          if (st == ST_ABSENT) {  // virtual leaves: children of a marked leaf
            if (vm.empty() || l == 0) continue;
            const long pc = g_.cell_off[l - 1] + mr_idx(g_, D_, n >> 1, i >> 1, j >> 1, k >> 1);
            if (!vm[pc]) continue;
            virt = true;
          }
          if (!row_counted(g_, l, D_ == 3 ? k : j)) continue;  // this rank's nodes
          const double m2 = D_ == 3 ? hv[3 * comp + c] : 0.0;
          std::snprintf(line, sizeof line, "%d %d %d %d %s %.17g %.17g %.17g %.17g %.17g\n", l, i,
                        j, k, virt ? "virtual" : st == ST_LEAF ? "leaf" : "internal", hv[c],
                        hv[comp + c], hv[2 * comp + c], m2, hv[(NC_ - 1) * comp + c]);
          out += line;
        }
  }
  return out;
}

// Self-check of the fast-path division and square root (af_physics.cuh fdiv /
// fsqrt) against the IEEE operations on n random operand pairs whose binary
// exponents lie in [emin, emax]: out = {division mismatches, divisions left
// to the IEEE path, sqrt mismatches, sqrts left to the IEEE path}.
namespace {
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__device__ double rand_double(uint64_t& s, int emin, int emax) {
  s = mix64(s);
  const uint64_t m = s & ((1ull << 52) - 1);
  const int e = emin + (int)((s >> 52) % (uint64_t)(emax - emin + 1));
  uint64_t b = ((uint64_t)(e + 1023) << 52) | m;
  if (mix64(s) & 1) b |= 1ull << 63;
  return __longlong_as_double((long long)b);
}
__global__ void fastdiv_check_kernel(uint64_t seed, long n, int emin, int emax,
                                     unsigned long long* out) {
  unsigned long long c[4] = {0, 0, 0, 0};
  uint64_t s = mix64(seed ^ (blockIdx.x * 0x100000001ull + threadIdx.x));
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    const double a = rand_double(s, emin, emax), b = rand_double(s, emin, emax);
    bool ok = true;
    const double q = fdiv(a, b, ok);
    if (!ok) ++c[1];
    else if (__double_as_longlong(q) != __double_as_longlong(a / b)) ++c[0];
    const double x = fabs(rand_double(s, 2 * emin, 2 * emax));
    bool ok2 = true;
    const double r = fsqrt(x, ok2);
    if (!ok2) ++c[3];
    else if (__double_as_longlong(r) != __double_as_longlong(sqrt(x))) ++c[2];
  }
  for (int k = 0; k < 4; ++k)
    if (c[k]) atomicAdd(out + k, c[k]);
}
}  // namespace

}  // namespace af

extern "C" af_status af_check_division(long n, uint64_t seed, int emin, int emax,
                                       unsigned long long out[4]) {
  if (!out || n < 0 || emin > emax || emin < -1022 || emax > 1023 || 2 * emin < -1022 ||
      2 * emax > 1023)
    return AF_E_ARGUMENT;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 4 * sizeof(unsigned long long)) != cudaSuccess) return AF_E_CUDA;
  cudaMemset(d, 0, 4 * sizeof(unsigned long long));
  af::fastdiv_check_kernel<<<148 * 8, 256>>>(seed, n, emin, emax, d);
  const cudaError_t e = cudaMemcpy(out, d, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? AF_OK : AF_E_CUDA;
}
