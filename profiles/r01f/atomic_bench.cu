// microbenchmark: fp64 atomicAdd scatter throughput (L2-resident target), B200
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_scatter(int n, const int *__restrict__ idx, double *y, int reps) {
  for (int r = 0; r < reps; ++r)
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
      int j = idx[t];
      atomicAdd(y + 3 * j, 1.0); atomicAdd(y + 3 * j + 1, 1.0); atomicAdd(y + 3 * j + 2, 1.0);
    }
}
__global__ void k_scatter_red(int n, const int *__restrict__ idx, double *y, int reps) {
  for (int r = 0; r < reps; ++r)
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
      int j = idx[t];
      double *p = y + 3 * j;
      asm volatile("red.global.add.f64 [%0], %1;" :: "l"(p), "d"(1.0) : "memory");
      asm volatile("red.global.add.f64 [%0], %1;" :: "l"(p + 1), "d"(1.0) : "memory");
      asm volatile("red.global.add.f64 [%0], %1;" :: "l"(p + 2), "d"(1.0) : "memory");
    }
}
int main() {
  const int n = 2600000, m = 210000;
  int *hidx = new int[n];
  unsigned s = 1;
  for (int i = 0; i < n; ++i) { s = s * 1664525u + 1013904223u; int row = (int)((long long)i * m / n); int off = (int)(s >> 24) - 128; int j = row + off; hidx[i] = j < 0 ? 0 : (j >= m ? m - 1 : j); }
  int *idx; double *y;
  cudaMalloc(&idx, n * 4); cudaMalloc(&y, 3 * m * 8);
  cudaMemcpy(idx, hidx, n * 4, cudaMemcpyHostToDevice);
  cudaMemset(y, 0, 3 * m * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int v = 0; v < 2; ++v) {
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(a);
      if (v == 0) k_scatter<<<148 * 8, 256>>>(n, idx, y, 10); else k_scatter_red<<<148 * 8, 256>>>(n, idx, y, 10);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (w) printf("%s: %.1f us per pass of %d x 3 fp64 atomics (%.1f G atomics/s)\n", v ? "red" : "atom", 1000 * ms / 10, n, 3.0 * n * 10 / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
