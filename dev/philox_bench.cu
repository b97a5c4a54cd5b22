// Philox-only throughput at the noise kernel's launch shape (development aid).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2310_11365_b200/csrc/npstream.cuh"
using namespace mmpr;

template <int BLOCKS>
__global__ void __launch_bounds__(32, 16) philox_only(const uint64_t *keys, int64_t words, unsigned long long *out) {
  const uint64_t k0 = keys[2 * blockIdx.x], k1 = keys[2 * blockIdx.x + 1];
  unsigned long long acc = 0;
  for (uint64_t sub = 0; sub * 32 * 4 * BLOCKS < (uint64_t)words; ++sub) {
    const uint64_t b0 = (sub * 32 + threadIdx.x) * BLOCKS;
#pragma unroll
    for (int b = 0; b < BLOCKS; ++b) {
      uint64_t w[4];
      np::philox_block(b0 + b, k0, k1, w);
      acc ^= w[0] ^ w[1] ^ w[2] ^ w[3];
    }
  }
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  const int streams = 6400;
  const int64_t words = 102400;  // ~1e5 normals per stream
  uint64_t *keys;
  unsigned long long *out;
  cudaMalloc(&keys, streams * 16);
  cudaMemset(keys, 7, streams * 16);
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    philox_only<2><<<streams, 32>>>(keys, words, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("philox-only (2 blocks/lane): %.3f ms  %.1f Gwords/s\n", ms, streams * (double)words / ms / 1e6);
    cudaEventRecord(e0);
    philox_only<4><<<streams, 32>>>(keys, words, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("philox-only (4 blocks/lane): %.3f ms  %.1f Gwords/s\n", ms, streams * (double)words / ms / 1e6);
  }
  return 0;
}
