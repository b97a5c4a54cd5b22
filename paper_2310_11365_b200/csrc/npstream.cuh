// numpy-exact noise stream primitives on the device: SeedSequence key
// derivation, Philox4x64-10 and the ziggurat layer tables.
//
// Reference: NoisePlan._generator / normals / init_rng
// (/root/reference/pkg/src/mcparareal/particles.py:49-65), i.e.
// np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy))).
// The same algorithm is restated for the CPU in oracle/npstream.c (the
// checker); tests pin both against numpy 2.3.5.
#pragma once

#include <stdint.h>

#include "np_ziggurat_tables.h"

namespace mmpr {
namespace np {

// ---- SeedSequence (pool of four 32-bit words) -------------------------------
__host__ __device__ __forceinline__ uint32_t ss_hashmix(uint32_t v, uint32_t &h) {
  v ^= h;
  h *= 0x931e8875u;
  v *= h;
  return v ^ (v >> 16);
}

__host__ __device__ __forceinline__ uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  return r ^ (r >> 16);
}

// Key = SeedSequence(words).generate_state(2, uint64).
__host__ __device__ inline void seedseq_key(const uint32_t *w, int n, uint64_t &k0, uint64_t &k1) {
  uint32_t pool[4];
  uint32_t h = 0x43b0d7e5u;
#pragma unroll
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < n ? w[i] : 0u, h);
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], h));
  for (int s = 4; s < n; ++s)
#pragma unroll
    for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(w[s], h));
  uint32_t hb = 0x8b51f9ddu, o[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t v = pool[i] ^ hb;
    hb *= 0x58f38dedu;
    v *= hb;
    o[i] = v ^ (v >> 16);
  }
  k0 = (uint64_t)o[0] | ((uint64_t)o[1] << 32);
  k1 = (uint64_t)o[2] | ((uint64_t)o[3] << 32);
}

// numpy's coercion of one non-negative Python int to uint32 words
// (little-endian, 0 -> [0]); returns words appended.
__host__ __device__ __forceinline__ int push_int_words(uint32_t *w, int n, uint64_t v) {
  if (v == 0) {
    w[n++] = 0;
    return n;
  }
  while (v) {
    w[n++] = (uint32_t)(v & 0xffffffffu);
    v >>= 32;
  }
  return n;
}

// ---- Philox4x64-10 ---------------------------------------------------------
#define MMPR_PHILOX_M0 0xD2E7470EE14C6C93ULL
#define MMPR_PHILOX_M1 0xCA5A826395121157ULL
#define MMPR_PHILOX_W0 0x9E3779B97F4A7C15ULL
#define MMPR_PHILOX_W1 0xBB67AE8584CAA73BULL

// Block `b` of a fresh numpy Philox stream: counter (b + 1, 0, 0, 0).
__device__ __forceinline__ void philox_block(uint64_t b, uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t c0 = b + 1, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = MMPR_PHILOX_M0 * c0;
    const uint64_t hi0 = __umul64hi(MMPR_PHILOX_M0, c0);
    const uint64_t lo1 = MMPR_PHILOX_M1 * c2;
    const uint64_t hi1 = __umul64hi(MMPR_PHILOX_M1, c2);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += MMPR_PHILOX_W0;
    k1 += MMPR_PHILOX_W1;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

__device__ __forceinline__ uint64_t philox_word(uint64_t i, uint64_t k0, uint64_t k1) {
  uint64_t o[4];
  philox_block(i >> 2, k0, k1, o);
  const int q = (int)(i & 3);
  return q == 0 ? o[0] : q == 1 ? o[1] : q == 2 ? o[2] : o[3];
}

// next_double(): (w >> 11) * 2^-53
__device__ __forceinline__ double unit_double(uint64_t w) { return (double)(w >> 11) * 0x1.0p-53; }

}  // namespace np
}  // namespace mmpr
