// Max co-resident clusters for fine-sweep-like CTAs (512 threads, 2 per SM,
// ~100 KB shared each) at several cluster sizes, and where a full wave lands.
#include <cstdio>
#include <set>
#include <vector>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 2) probe(int *out, long long spin) {
  extern __shared__ double s[];
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) { s[0] = smid; out[blockIdx.x] = smid; }
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
}
__global__ void __launch_bounds__(1024, 1) probe1k(int *out, long long spin) {
  extern __shared__ double s[];
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) { s[0] = smid; out[blockIdx.x] = smid; }
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
}
template <typename K>
void run(K kern, int threads, int cl, size_t smem) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cfg.gridDim = dim3(cl);
  int n = 0;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
  // launch exactly n clusters, see how many distinct SMs they use
  cfg.gridDim = dim3(n * cl);
  int *d; cudaMalloc(&d, n * cl * sizeof(int));
  cudaLaunchKernelEx(&cfg, kern, d, 200000LL);
  cudaDeviceSynchronize();
  std::vector<int> h(n * cl);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  std::set<int> sms(h.begin(), h.end());
  printf("threads %4d cluster %2d smem %6zu: max active clusters %3d (%s) = %4d CTAs on %3zu SMs\n", threads, cl, smem, n,
         cudaGetErrorString(e), n * cl, sms.size());
  cudaFree(d);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  for (int cl : {1, 2, 4, 8, 16}) run(probe, 512, cl, 102400);
  for (int cl : {1, 2, 4, 8, 16}) run(probe1k, 1024, cl, 204800);
  return 0;
}
