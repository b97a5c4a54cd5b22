// Dependent FP64 chain latencies on one warp: DADD->DADD, DMUL->DMUL, DMUL->DADD alternating,
// and the OU Euler step (mul, add, add, mul, add) (development aid).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chains(double *out, long long *cyc, int iters, double a, double b) {
  double x = threadIdx.x * 1e-9 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __dadd_rn(x, a);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x = __dmul_rn(x, b);
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) x = __dadd_rn(__dmul_rn(x, b), a);
  long long t3 = clock64();
  const double c0 = 0.0, h = 0.01, aE = 0.5;
  for (int i = 0; i < iters; ++i) {
    const double d = __dadd_rn(__dadd_rn(__dmul_rn(a, x), __dmul_rn(aE, x)), c0);
    x = __dadd_rn(x, __dmul_rn(h, d));
  }
  long long t4 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double *o; long long *c, h[4];
  cudaMalloc(&o, 256); cudaMalloc(&c, 32);
  const int iters = 100000;
  chains<<<1, 1>>>(o, c, iters, -1e-12, 1.0000000001);
  cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("DADD chain %.2f cyc/op, DMUL chain %.2f, DMUL->DADD pair %.2f cyc/pair, OU Euler step %.2f cyc/step\n",
         h[0] / (double)iters, h[1] / (double)iters, h[2] / (double)iters, h[3] / (double)iters);
  return 0;
}
