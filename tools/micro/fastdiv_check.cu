// Checks the inline fast-path division / square root of af_physics.cuh
// (CUDA's own fast-path sequences with their validity tests, no slow-path
// branch) bit for bit against IEEE a/b and sqrt(x) on random operands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o fastdiv_check fastdiv_check.cu
#include <cstdio>
#include <cstdint>
#include "../../paper_1603_05211_b200/csrc/af_physics.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
// random double with exponent in [emin, emax], random sign and mantissa
__device__ double rnd(uint64_t& s, int emin, int emax) {
  s = mix(s);
  const uint64_t m = s & ((1ull << 52) - 1);
  const int e = emin + (int)((s >> 52) % (uint64_t)(emax - emin + 1));
  uint64_t b = ((uint64_t)(e + 1023) << 52) | m;
  if (mix(s) & 1) b |= 1ull << 63;
  return __longlong_as_double((long long)b);
}

__global__ void check(uint64_t seed, long n, int emin, int emax, unsigned long long* out) {
  unsigned long long bad_div = 0, bad_sqrt = 0, slow_div = 0, slow_sqrt = 0;
  uint64_t s = mix(seed ^ (blockIdx.x * 0x100000001ull + threadIdx.x));
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const double a = rnd(s, emin, emax), b = rnd(s, emin, emax);
    bool ok = true;
    const double q = af::fdiv(a, b, ok);
    if (!ok) ++slow_div;
    else if (__double_as_longlong(q) != __double_as_longlong(a / b)) ++bad_div;
    const double x = fabs(rnd(s, 2 * emin, 2 * emax));
    bool ok2 = true;
    const double r = af::fsqrt(x, ok2);
    if (!ok2) ++slow_sqrt;
    else if (__double_as_longlong(r) != __double_as_longlong(sqrt(x))) ++bad_sqrt;
  }
  atomicAdd(out + 0, bad_div);
  atomicAdd(out + 1, slow_div);
  atomicAdd(out + 2, bad_sqrt);
  atomicAdd(out + 3, slow_sqrt);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 4 * sizeof(unsigned long long));
  const int ranges[][2] = {{-4, 4}, {-40, 40}, {-300, 300}, {-1022, 1023}};
  for (auto& rg : ranges) {
    cudaMemset(d, 0, 4 * sizeof(unsigned long long));
    const long n = 4L << 30;
    check<<<148 * 16, 256>>>(12345 + rg[0], n, rg[0], rg[1], d);
    unsigned long long h[4];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    std::printf("exponents [%d,%d]: %ld divisions: %llu mismatches, %llu slow; %ld sqrts: %llu "
                "mismatches, %llu slow\n", rg[0], rg[1], n, h[0], h[1], n, h[2], h[3]);
  }
  return cudaGetLastError() != cudaSuccess;
}
