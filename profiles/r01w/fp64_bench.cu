// fp64 throughput on B200: DFMA, DMUL and DADD issue rates with 8 independent chains per thread,
// 148 x 8 CTAs of 256 threads (the denominator of k_tag's ALU roofline)
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = __fma_rn(x[i], a, b);
      else if (OP == 1) x[i] = __dmul_rn(x[i], a);
      else x[i] = __dadd_rn(x[i], b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *o; cudaMalloc(&o, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096, grid = sms * 8, block = 256;
  const char *nm[3] = {"DFMA", "DMUL", "DADD"};
  for (int op = 0; op < 3; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (op == 0) k<0><<<grid, block>>>(o, iters, 0.999999, 1e-9);
      if (op == 1) k<1><<<grid, block>>>(o, iters, 0.999999, 1e-9);
      if (op == 2) k<2><<<grid, block>>>(o, iters, 0.999999, 1e-9);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = (double)grid * block * iters * 8;
      if (rep) printf("%s: %.2f Tinst/s (%.2f TFLOP/s counting FMA as 2)\n", nm[op], ops / (ms * 1e-3) / 1e12,
                      ops * (op == 0 ? 2 : 1) / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
