// FP64 issue-rate microbenchmark (DFMA/DMUL/DADD dependent chains, 8 ILP)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double *out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __fma_rn(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void dadd_kernel(double *out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __dadd_rn(x[i], a);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void latency_kernel(double *out, int iters, double a, double b, long long *cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x = __dadd_rn(x, a);
  long long t1 = clock64();
  double y = x;
  long long t2 = clock64();
  for (int it = 0; it < iters; ++it) y = __dmul_rn(y, b);
  long long t3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t3 - t2; }
  if (x + y == 12345.678) out[0] = x;
}
int main() {
  double *out; cudaMalloc(&out, 8); long long *cyc; cudaMallocManaged(&cyc, 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000, threads = 1024, blocks = sms * 2;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * 8;
    printf("DFMA: %.3f ms  %.2f TFLOP/s  %.1f DFMA/clk/SM (at %d MHz nominal)\n", ms, 2 * ops / ms / 1e9,
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    cudaEventRecord(e0); dadd_kernel<<<blocks, threads>>>(out, iters, 1e-7, 0); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("DADD: %.3f ms  %.1f DADD/clk/SM\n", ms, ops / (ms * 1e-3) / sms / (clk * 1e3));
  }
  latency_kernel<<<1, 32>>>(out, 1000, 1e-7, 0.9999, cyc); cudaDeviceSynchronize();
  printf("latency: DADD %.1f cycles, DMUL %.1f cycles\n", cyc[0] / 1000.0, cyc[1] / 1000.0);
  return 0;
}
