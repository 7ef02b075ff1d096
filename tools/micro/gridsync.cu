// Microbenchmark: cost of cooperative grid.sync() on this GPU for a given
// grid (blocks x 256 threads), and of a launch-per-phase chain for comparison.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void syncs(int n, int* sink) {
  cg::grid_group grid = cg::this_grid();
  for (int i = 0; i < n; ++i) grid.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = n;
}
__global__ void empty(int* sink) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink += 1;
}

int main() {
  int* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int blocks : {64, 148, 296, 592}) {
    int n = 1000;
    void* args[] = {&n, &sink};
    cudaLaunchCooperativeKernel((void*)syncs, blocks, 256, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)syncs, blocks, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync blocks=%d: %.3f us/sync (%s)\n", blocks, ms * 1e3 / n,
           cudaGetErrorString(cudaGetLastError()));
  }
  // back-to-back empty launches (stream) and in a graph
  for (int blocks : {1, 296, 1184}) {
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 100; ++i) empty<<<blocks, 256, 0, s>>>(sink);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("graph of 100 empty kernels blocks=%d: %.3f us/kernel\n", blocks, ms * 1e3 / 100);
    cudaEventRecord(a, s);
    for (int i = 0; i < 100; ++i) empty<<<blocks, 256, 0, s>>>(sink);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("stream of 100 empty kernels blocks=%d: %.3f us/kernel\n", blocks, ms * 1e3 / 100);
  }
  return 0;
}
