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


// ---- libm log1p of the host numpy links against ----------------------------
// numpy's Marsaglia tail (random_standard_normal, the idx == 0 branch) calls
// npy_log1p = the C library's log1p.  On x86-64 glibc 2.39 resolves log1p
// through an ifunc to the FMA build of the fdlibm-derived s_log1p.c (parallel
// polynomial evaluation); this is that function with gcc's contraction
// pattern spelled out (__fma_rn where the FMA build fuses, _rn elsewhere).
// The same restatement in C (oracle/npstream.c log1p_restated) is pinned to
// the host libm in tests/test_oracle_npstream.py; this device function is
// pinned to the host libm in tests/test_gpu_noise.py.
__device__ __forceinline__ double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
               Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int32_t hx = __double2hiint(x);
  const int32_t ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -__longlong_as_double(0x7ff0000000000000LL) : __longlong_as_double(0x7ff8000000000000LL);
    if (ax < 0x3e200000) return ax < 0x3c900000 ? x : __fma_rn(-__dmul_rn(x, x), 0.5, x);
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return __dadd_rn(x, x);
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = __dadd_rn(1.0, x);
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
      c = __ddiv_rn(c, u);
    } else {
      u = x;
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
    } else {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double dk = (double)k;
  const double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = __fma_rn(dk, ln2_lo, c);
      return __fma_rn(dk, ln2_hi, c);
    }
    const double R = __dmul_rn(hfsq, __fma_rn(-0.66666666666666666, f, 1.0));
    if (k == 0) return __dsub_rn(f, R);
    return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(R, __fma_rn(dk, ln2_lo, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z4, z2);
  const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
  const double R = __fma_rn(z6, R4, __fma_rn(z4, R3, __fma_rn(z, Lp1, __dmul_rn(z2, R2))));
  const double sR = __dmul_rn(s, __dadd_rn(hfsq, R));
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, sR));
  return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(sR, __fma_rn(dk, ln2_lo, c))), f));
}

}  // namespace np
}  // namespace mmpr
