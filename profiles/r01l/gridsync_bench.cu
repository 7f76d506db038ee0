// microbenchmark: cost of cooperative_groups grid.sync() with one 1024-thread CTA per SM (the
// k_tail launch shape), and of a plain kernel launch boundary, on B200
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_sync(int iters, int *x) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) atomicAdd(x + (blockIdx.x & 7), 1);
    g.sync();
  }
}
__global__ void k_empty(int *x) { if (threadIdx.x == 0 && blockIdx.x == 0) x[8] += 1; }
int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int *x;
  cudaMalloc(&x, 64 * sizeof(int));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int iters : {1, 1000, 10000}) {
    void *args[] = {&iters, &x};
    cudaLaunchCooperativeKernel((void *)k_sync, sms, 1024, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void *)k_sync, sms, 1024, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync x%d: %.2f us total, %.3f us per sync\n", iters, 1e3 * ms, 1e3 * ms / iters);
  }
  cudaStream_t s; cudaStreamCreate(&s);
  cudaGraph_t gr; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 1000; ++i) k_empty<<<sms, 1024, 0, s>>>(x);
  cudaStreamEndCapture(s, &gr);
  cudaGraphInstantiate(&ge, gr, 0);
  cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
  cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("graph of 1000 empty %dx1024 kernels: %.3f us per kernel\n", sms, ms);
  cudaEventRecord(a, s);
  for (int i = 0; i < 1000; ++i) k_empty<<<sms, 1024, 0, s>>>(x);
  cudaEventRecord(b, s); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("stream of 1000 empty %dx1024 kernels: %.3f us per kernel\n", sms, ms);
  return 0;
}
