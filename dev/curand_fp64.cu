// Dynamic FP64 instruction count of curand_normal2_double per normal (the
// canonical-normal cost of SURVEY 8(d)); run under ncu with
// --metrics smsp__sass_thread_inst_executed_op_fp64_pred_on.sum (development aid).
#include <cstdio>
#include <curand_kernel.h>
__global__ void normals(double *out, int pairs) {
  curandStatePhilox4_32_10_t st;
  curand_init(1234, blockIdx.x * blockDim.x + threadIdx.x, 0, &st);
  double acc = 0.0;
  for (int i = 0; i < pairs; ++i) {
    double2 z = curand_normal2_double(&st);
    acc += z.x + z.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  const int threads = 128, blocks = 148, pairs = 1000;
  double *out;
  cudaMalloc(&out, threads * blocks * 8);
  normals<<<blocks, threads>>>(out, pairs);
  cudaDeviceSynchronize();
  printf("normals generated: %ld (+ %d accumulation DADD per pair)\n", (long)threads * blocks * pairs * 2, 2);
  return 0;
}
