// Microbenchmark: fp64 pipe throughput on this GPU for the
// operations the FV stage is made of: DADD, DMUL, DFMA, IEEE division and
// sqrt (correctly rounded, as the parity build uses). 8 independent chains
// per thread, full occupancy; reports operations per second for the device.
#include <cstdio>

template <int OP>
__global__ void bench(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = 1.0 + 1e-3 * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = __dadd_rn(x[i], a);
      if (OP == 1) x[i] = __dmul_rn(x[i], b);
      if (OP == 2) x[i] = __fma_rn(x[i], b, a);
      if (OP == 3) x[i] = a / x[i] + 0.5;
      if (OP == 4) x[i] = sqrt(x[i]) + 0.25;
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"dadd", "dmul", "dfma", "ddiv (IEEE x/y)", "dsqrt (IEEE)"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int op = 0; op < 5; ++op) {
    const int iters = op >= 3 ? 2000 : 20000;
    const int blocks = sms * 8, threads = 256;
    auto run = [&]() {
      switch (op) {
        case 0: bench<0><<<blocks, threads>>>(out, iters, 1e-9, 0.9999999); break;
        case 1: bench<1><<<blocks, threads>>>(out, iters, 1e-9, 0.9999999); break;
        case 2: bench<2><<<blocks, threads>>>(out, iters, 1e-9, 0.9999999); break;
        case 3: bench<3><<<blocks, threads>>>(out, iters, 1.0, 0.0); break;
        default: bench<4><<<blocks, threads>>>(out, iters, 0.0, 0.0); break;
      }
    };
    run();
    cudaEventRecord(e0);
    run();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 8;
    printf("%-16s %.3e ops/s (%.2f per SM per clock at 1.965 GHz) %s\n", names[op], ops / (ms * 1e-3),
           ops / (ms * 1e-3) / sms / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
