// Counter-based Philox noise generated in registers (NoiseMode.PHILOX /
// PHILOX_FRESH): the north-star noise supply of the fine propagator.
//
// The reference draws every (slice, step) row from its own numpy stream
// (NoisePlan.normals, /root/reference/pkg/src/mcparareal/particles.py:49-61),
// so element p depends on every earlier draw of the row and must be
// materialised in HBM (noise.cu).  This mode keeps the reference's normal
// transform -- numpy's 256-layer ziggurat over one 64-bit word per attempt
// (same layer tables, same wedge and Marsaglia-tail rules) -- but feeds it
// from Philox4x32-10 (Salmon et al., SC'11) addressed by the particle itself:
//
//   block(p, j, n, c3) = Philox4x32-10(counter = (p, j, n, c3), key = (k0, k1))
//   c3 = kfield + (draw << 24), kfield = 0 (PHILOX) or k + 1 (PHILOX_FRESH)
//
// Attempt a of particle p's step-j normal uses block draw = a: word
// lo|hi<<32 of outputs (0, 1) is the ziggurat word, outputs (2, 3) the wedge
// test's uniform.  Tail iteration t uses block draw = 128 + t (both words as
// the uniform pair).  Every increment is a pure function of (p, j, n, k), so
// any kernel geometry (cluster sweep, grid sweep, iteration pipeline)
// produces the same bits.  The key is SeedSequence((seed, 4)).generate_state
// (2, uint32) (noise.py).  Parity: oracle/npstream.c restates the generator
// (nps_counter_normals); tests pin the device bit for bit against it and the
// Philox4x32-10 core against curand's and the Random123 known answers.
#pragma once

#include <stdint.h>

#include "npstream.cuh"

namespace mmpr {
namespace cn {

#define MMPR_PHILOX32_M0 0xD2511F53u
#define MMPR_PHILOX32_M1 0xCD9E8D57u
#define MMPR_PHILOX32_W0 0x9E3779B9u
#define MMPR_PHILOX32_W1 0xBB67AE85u

struct CounterNoise {
  uint32_t k0, k1;  // Philox key
  uint32_t kfield;  // 0 (frozen) or iteration + 1 (fresh)
  int32_t n_base;   // global slice index of local slice 0
};

__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

// Philox4x32-10 in place: c <- Philox4x32-10(c, (k0, k1)).
__host__ __device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = mulhi32(MMPR_PHILOX32_M0, c[0]), lo0 = MMPR_PHILOX32_M0 * c[0];
    const uint32_t hi1 = mulhi32(MMPR_PHILOX32_M1, c[2]), lo1 = MMPR_PHILOX32_M1 * c[2];
    c[0] = hi1 ^ c[1] ^ k0;
    c[1] = lo1;
    c[2] = hi0 ^ c[3] ^ k1;
    c[3] = lo0;
    k0 += MMPR_PHILOX32_W0;
    k1 += MMPR_PHILOX32_W1;
  }
}

// Ziggurat layer tables in shared memory (lanes index them divergently).
struct ZigTables {
  uint64_t ki[256];
  double wi[256];
  double fi[256];
};
static_assert(sizeof(ZigTables) == 6144, "ZigTables layout");

static __constant__ uint64_t c_cn_ki[256] = {NPZ_KI_VALUES};
static __constant__ double c_cn_wi[256] = {NPZ_WI_VALUES};
static __constant__ double c_cn_fi[256] = {NPZ_FI_VALUES};

__device__ __forceinline__ void load_zig(ZigTables *z, int tid, int nthreads) {
  for (int i = tid; i < 256; i += nthreads) {
    z->ki[i] = c_cn_ki[i];
    z->wi[i] = c_cn_wi[i];
    z->fi[i] = c_cn_fi[i];
  }
}

__device__ __forceinline__ double unit53(uint64_t w) { return (double)(w >> 11) * 0x1.0p-53; }

// The rare paths (wedge test, Marsaglia tail, further attempts), kept out of
// line so the step loop's register budget only carries the fast path.
static __device__ __noinline__ double zig_slow(uint64_t w, uint64_t u, uint32_t p, uint32_t j, uint32_t n, uint32_t kf,
                                        uint32_t k0, uint32_t k1, const ZigTables *z) {
  for (uint32_t a = 0;;) {
    const int idx = (int)(w & 0xff);
    const uint64_t rabs = (w >> 9) & 0x000fffffffffffffULL;
    double x = __dmul_rn((double)rabs, z->wi[idx]);
    if ((w >> 8) & 1) x = -x;
    if (rabs < z->ki[idx]) return x;
    if (idx == 0) {
      for (uint32_t t = 0;; ++t) {
        uint32_t c[4] = {p, j, n, kf + ((128u + t) << 24)};
        philox4x32_10(c, k0, k1);
        const double xx = __dmul_rn(-NPZ_INV_R, np::glibc_log1p(-unit53((uint64_t)c[0] | ((uint64_t)c[1] << 32))));
        const double yy = -np::glibc_log1p(-unit53((uint64_t)c[2] | ((uint64_t)c[3] << 32)));
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx))
          return ((rabs >> 8) & 1) ? -__dadd_rn(NPZ_R, xx) : __dadd_rn(NPZ_R, xx);
      }
    }
    const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(z->fi[idx - 1], z->fi[idx]), unit53(u)), z->fi[idx]);
    if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) return x;
    ++a;
    uint32_t c[4] = {p, j, n, kf + (a << 24)};
    philox4x32_10(c, k0, k1);
    w = (uint64_t)c[0] | ((uint64_t)c[1] << 32);
    u = (uint64_t)c[2] | ((uint64_t)c[3] << 32);
  }
}

// Standard normal increment of particle p at step j of global slice n.
__device__ __forceinline__ double normal(const CounterNoise &cn, uint32_t p, uint32_t j, uint32_t n,
                                         const ZigTables *z) {
  uint32_t c[4] = {p, j, n, cn.kfield};
  philox4x32_10(c, cn.k0, cn.k1);
  const uint64_t w = (uint64_t)c[0] | ((uint64_t)c[1] << 32);
  const int idx = (int)(c[0] & 0xff);
  const uint64_t rabs = (w >> 9) & 0x000fffffffffffffULL;
  const double x = __dmul_rn((double)rabs, z->wi[idx]);
  if (rabs < z->ki[idx]) return ((c[0] >> 8) & 1) ? -x : x;
  return zig_slow(w, (uint64_t)c[2] | ((uint64_t)c[3] << 32), p, j, n, cn.kfield, cn.k0, cn.k1, z);
}

}  // namespace cn
}  // namespace mmpr
