// Which CTAs share an SM when 16-CTA clusters of 512 threads run two per SM?
#include <cstdio>
#include <vector>
#include <map>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 2) probe(int *out, long long spin) {
  extern __shared__ double s[];
  unsigned smid, rank;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    s[0] = smid;
    out[blockIdx.x * 2] = smid;
    out[blockIdx.x * 2 + 1] = blockIdx.x / 16;  // cluster index
  }
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
}
int main(int argc, char **argv) {
  const int clusters = 64, ctas = clusters * 16;
  int *d;
  cudaMalloc(&d, ctas * 2 * sizeof(int));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int pol = 0; pol < 3; ++pol) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = 100 * 1024;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr[1].val.clusterSchedulingPolicyPreference = (cudaClusterSchedulingPolicy)pol;
    cfg.attrs = attr; cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, probe, d, 2000000LL);
    cudaDeviceSynchronize();
    std::vector<int> h(ctas * 2);
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    // first wave: clusters 0..13; count SMs hosting 2 CTAs of the same cluster vs different
    std::map<int, std::vector<int>> bysm;
    for (int b = 0; b < 14 * 16; ++b) bysm[h[2 * b]].push_back(h[2 * b + 1]);
    int same = 0, diff = 0, single = 0;
    for (auto &kv : bysm) {
      if (kv.second.size() == 1) ++single;
      else if (kv.second[0] == kv.second[1]) ++same;
      else ++diff;
    }
    printf("policy %d (%s): first 14 clusters on %zu SMs: %d SMs with 2 CTAs of the same cluster, %d with two clusters, %d with one CTA\n",
           pol, cudaGetErrorString(e), bysm.size(), same, diff, single);
  }
  return 0;
}
