// Read-bandwidth ceiling of the pipeline's access pattern: every CTA streams
// consecutive 51.2 KB rows (one 1-D bulk copy per step into a ring of
// shared-memory stages, mbarrier completion), no compute.  Reports GB/s for
// several CTA counts / stage depths (development aid).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512, 2) stream_kernel(const double *src, int64_t row_elems, int rows_per_cta,
                                                       int64_t cta_stride, int stages, uint32_t bytes, double *sink) {
  extern __shared__ __align__(128) double st[];
  __shared__ __align__(8) uint64_t bar[8];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int q = 0; q < stages; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[q])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const double *base = src + (int64_t)blockIdx.x * cta_stride;
  auto issue = [&](int j) {
    const int q = j % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[q])), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(st + (size_t)q * (bytes / 8))),
                 "l"(base + (int64_t)j * row_elems), "r"(bytes), "r"(smem_u32(&bar[q])));
  };
  if (tid == 0)
    for (int j = 0; j < stages && j < rows_per_cta; ++j) issue(j);
  double acc = 0.0;
  for (int j = 0; j < rows_per_cta; ++j) {
    const int q = j % stages;
    const uint32_t par = (j / stages) & 1;
    asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}" ::"r"(
                     smem_u32(&bar[q])),
                 "r"(par));
    acc += st[(size_t)q * (bytes / 8) + tid];
    __syncthreads();
    if (tid == 0 && j + stages < rows_per_cta) issue(j + stages);
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  const int64_t row_elems = 6400;  // 51.2 KB per CTA per step, as the pipeline's 16-CTA clusters
  const uint32_t bytes = row_elems * 8;
  const int rows = 500;
  const int max_ctas = 296;
  double *src, *sink;
  const size_t total = (size_t)max_ctas * rows * row_elems * 8;
  cudaMalloc(&src, total);
  cudaMemset(src, 0, total);
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int stages : {2, 3, 4}) {
    const size_t smem = (size_t)stages * bytes;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int ctas : {148, 224, 264, 296}) {
      if (stages > 2 && ctas > 148) continue;  // one CTA per SM above 2 stages
      for (int w = 0; w < 2; ++w)
        stream_kernel<<<ctas, 512, smem>>>(src, row_elems, rows, (int64_t)rows * row_elems, stages, bytes, sink);
      cudaEventRecord(e0);
      const int reps = 5;
      for (int r = 0; r < reps; ++r)
        stream_kernel<<<ctas, 512, smem>>>(src, row_elems, rows, (int64_t)rows * row_elems, stages, bytes, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gb = (double)ctas * rows * bytes * reps / 1e9;
      printf("stages %d ctas %3d: %.3f ms/launch, %.0f GB/s (%s)\n", stages, ctas, ms / reps, gb / (ms / 1e3),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
