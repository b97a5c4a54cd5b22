// Philox4x64 round multiply: __umul64hi + 64-bit multiply vs four
// mad.wide.u32 partial products (development aid).  Checks equality and
// times both at the noise kernel's launch shape.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2310_11365_b200/csrc/npstream.cuh"
using namespace mmpr;

// 64x64 -> 128 with one 32x32 product per partial
__device__ __forceinline__ void mul128(uint64_t a, uint64_t b, uint64_t &lo, uint64_t &hi) {
  asm("{\n\t"
      ".reg .u32 al, ah, bl, bh, p0l, p0h, tl, th, ul, uh;\n\t"
      ".reg .u64 p0, t, u, hh, x;\n\t"
      "mov.b64 {al, ah}, %2;\n\t"
      "mov.b64 {bl, bh}, %3;\n\t"
      "mul.wide.u32 p0, al, bl;\n\t"
      "mov.b64 {p0l, p0h}, p0;\n\t"
      "cvt.u64.u32 x, p0h;\n\t"
      "mad.wide.u32 t, ah, bl, x;\n\t"
      "mov.b64 {tl, th}, t;\n\t"
      "cvt.u64.u32 x, tl;\n\t"
      "mad.wide.u32 u, al, bh, x;\n\t"
      "mov.b64 {ul, uh}, u;\n\t"
      "mov.b64 %0, {p0l, ul};\n\t"
      "cvt.u64.u32 x, th;\n\t"
      "mad.wide.u32 hh, ah, bh, x;\n\t"
      "cvt.u64.u32 x, uh;\n\t"
      "add.u64 %1, hh, x;\n\t"
      "}"
      : "=l"(lo), "=l"(hi)
      : "l"(a), "l"(b));
}

__device__ __forceinline__ void philox_block_w(uint64_t b, uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t c0 = b + 1, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t lo0, hi0, lo1, hi1;
    mul128(c0, MMPR_PHILOX_M0, lo0, hi0);
    mul128(c2, MMPR_PHILOX_M1, lo1, hi1);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += MMPR_PHILOX_W0;
    k1 += MMPR_PHILOX_W1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

template <int V>
__global__ void __launch_bounds__(32, 16) philox_only(const uint64_t *keys, int64_t words, unsigned long long *out) {
  const uint64_t k0 = keys[2 * blockIdx.x], k1 = keys[2 * blockIdx.x + 1];
  unsigned long long acc = 0;
  for (uint64_t sub = 0; sub * 32 * 8 < (uint64_t)words; ++sub) {
    const uint64_t b0 = (sub * 32 + threadIdx.x) * 2;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      uint64_t w[4];
      if (V == 0) np::philox_block(b0 + b, k0, k1, w);
      else philox_block_w(b0 + b, k0, k1, w);
      acc ^= w[0] ^ w[1] ^ w[2] ^ w[3];
    }
  }
  out[blockIdx.x * 32 + threadIdx.x] = acc;
}

__global__ void check(const uint64_t *keys, int n, int *bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t a[4], b[4];
  const uint64_t k0 = keys[0] * (i + 1), k1 = keys[1] ^ (uint64_t)i * 0x9E3779B97F4A7C15ULL;
  np::philox_block((uint64_t)i * 7919u, k0, k1, a);
  philox_block_w((uint64_t)i * 7919u, k0, k1, b);
  for (int q = 0; q < 4; ++q)
    if (a[q] != b[q]) atomicAdd(bad, 1);
}

int main() {
  const int streams = 6400;
  const int64_t words = 102400;
  uint64_t *keys;
  unsigned long long *out;
  int *bad;
  cudaMalloc(&keys, streams * 16);
  cudaMemset(keys, 0x5b, streams * 16);
  cudaMalloc(&out, streams * 32 * 8);
  cudaMalloc(&bad, 4);
  cudaMemset(bad, 0, 4);
  check<<<4096, 256>>>(keys, 4096 * 256, bad);
  int hb = -1;
  cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  printf("mismatching words: %d of %d\n", hb, 4096 * 256 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(e0);
    philox_only<0><<<streams, 32>>>(keys, words, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("umul64hi: %.3f ms\n", ms);
    cudaEventRecord(e0);
    philox_only<1><<<streams, 32>>>(keys, words, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("mad.wide: %.3f ms\n", ms);
  }
  return 0;
}
