// Counter-based Philox noise generated in registers (NoiseMode.PHILOX /
// PHILOX_FRESH): the north-star noise supply of the fine propagator.
//
// The reference draws every (slice, step) row from its own numpy stream
// (NoisePlan.normals, /root/reference/pkg/src/mcparareal/particles.py:49-61),
// so element p depends on every earlier draw of the row and must be
// materialised in HBM (noise.cu).  This mode keeps the reference's normal
// transform -- numpy's 256-layer ziggurat over one 64-bit word per attempt
// (same layer tables, same wedge and Marsaglia-tail rules) -- but feeds it
// from Philox2x32-10 (Salmon et al., SC'11) addressed by the particle itself:
//
//   word(p, j, n, d) = Philox2x32-10(counter = (p, j | d << 24),
//                                    key = k32 ^ (n | kfield << 20))
//   kfield = 0 (PHILOX) or k + 1 (PHILOX_FRESH)
//
// Draw d of particle p's step-j normal: attempt a uses d = 2a for the
// ziggurat word and d = 2a + 1 for its wedge uniform; Marsaglia-tail
// iteration t uses d = 128 + 2t and 129 + 2t.  Every increment is a pure
// function of (p, j, n, k), so any kernel geometry (cluster sweep, grid
// sweep, iteration pipeline) produces the same bits.  k32 is
// SeedSequence((seed, 4)).generate_state(1, uint32) (noise.py).
//
// In the step loop (cn::step) every lane runs the fast path -- one Philox
// word, a table lookup, one multiply, ~98.8% accepted -- for all of its
// particles, then resolves its few rejected draws (wedge test, tail,
// further attempts) one per round.  Measured on B200 (config-4 sweep,
// 64 x 1e5 x 100): 5.2 ms, against 1.5 ms without the generator, 2.7 ms
// with the fast path only, 7.1 ms when rejected draws were instead compacted
// over the warp (dev/phx_ab.sh) -- the rare path's divergence and the
// per-step barrier on the slowest warp bound this mode, not FP64.
//
// Parity: oracle/npstream.c restates the generator (nps_counter_normals);
// tests pin the device bit for bit against it and the Philox2x32-10 core
// against the Random123 known answers.
#pragma once

#include <stdint.h>

#include "npstream.cuh"

namespace mmpr {
namespace cn {

// CTAs of 512 threads per SM the generate-ahead kernels are compiled for
// (the register budget: 2 -> 64 registers per thread, 1 -> 128)
#ifndef MMPR_PHX_MINB
#define MMPR_PHX_MINB 2
#endif
// unroll factor of cn::gen's fast path over a lane's particles
#ifndef MMPR_PHX_GEN_UNROLL
#define MMPR_PHX_GEN_UNROLL 16
#endif

#define MMPR_PHILOX2_M 0xD256D193u
#define MMPR_PHILOX2_W 0x9E3779B9u

struct CounterNoise {
  uint32_t k0;      // SeedSequence key word
  uint32_t unused;  // (mmpr_counter_noise.key[1])
  uint32_t kfield;  // 0 (frozen) or iteration + 1 (fresh), < 2^12
  int32_t n_base;   // global slice index of local slice 0
};

__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

// Philox2x32-10: (c0, c1) <- Philox2x32-10((c0, c1), k).
__host__ __device__ __forceinline__ void philox2x32_10(uint32_t &c0, uint32_t &c1, uint32_t k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi = mulhi32(MMPR_PHILOX2_M, c0), lo = MMPR_PHILOX2_M * c0;
    c0 = hi ^ k ^ c1;
    c1 = lo;
    k += MMPR_PHILOX2_W;
  }
}

__host__ __device__ __forceinline__ uint32_t slice_key(const CounterNoise &c, uint32_t n) {
  return c.k0 ^ (n | (c.kfield << 20));
}

// The 64-bit word of draw d: low half = output 0, high half = output 1.
__device__ __forceinline__ void word(uint32_t p, uint32_t j, uint32_t d, uint32_t key, uint32_t &lo, uint32_t &hi) {
  uint32_t c0 = p, c1 = j | (d << 24);
  philox2x32_10(c0, c1, key);
  lo = c0;
  hi = c1;
}

// Ziggurat layer tables in shared memory (lanes index them divergently):
// (ki as a double, wi) pairs for one 16-byte load, then fi.
struct ZigTables {
  double2 kw[256];
  double fi[256];
};
static_assert(sizeof(ZigTables) == 6144, "ZigTables layout");

static __constant__ uint64_t c_cn_ki[256] = {NPZ_KI_VALUES};
static __constant__ double c_cn_wi[256] = {NPZ_WI_VALUES};
static __constant__ double c_cn_fi[256] = {NPZ_FI_VALUES};

__device__ __forceinline__ void load_zig(ZigTables *z, int tid, int nthreads) {
  for (int i = tid; i < 256; i += nthreads) {
    z->kw[i] = make_double2((double)c_cn_ki[i], c_cn_wi[i]);  // ki < 2^53: exact
    z->fi[i] = c_cn_fi[i];
  }
}

__device__ __forceinline__ double unit53(uint32_t lo, uint32_t hi) {
  const uint64_t w = (uint64_t)lo | ((uint64_t)hi << 32);
  return (double)(w >> 11) * 0x1.0p-53;
}

// numpy's magnitude field (w >> 9) & (2^52 - 1) as an exact double: the
// bits go into the mantissa of 2^52 and 2^52 is subtracted (no int64
// conversion on the step loop's path).
__device__ __forceinline__ double rabs_of(uint32_t lo, uint32_t hi) {
  const uint32_t mlo = (lo >> 9) | (hi << 23);
  const uint32_t mhi = (hi >> 9) & 0x000fffffu;
  return __dsub_rn(__hiloint2double((int)(0x43300000u | mhi), (int)mlo), 0x1.0p52);
}

// Fast path: true (and the value) when the attempt-0 word is accepted.
__device__ __forceinline__ bool fast(uint32_t p, uint32_t j, uint32_t key, const ZigTables *z, double &out) {
  uint32_t lo, hi;
#if defined(MMPR_PHX_DEBUG) && MMPR_PHX_DEBUG == 2  // dev A/B only: no generator
  lo = p * 0x9E3779B9u ^ j;
  hi = lo * 0x85EBCA6Bu;
#else
  word(p, j, 0, key, lo, hi);
#endif
  const double r = rabs_of(lo, hi);
  const double2 kw = z->kw[lo & 0xff];
  const double x = __dmul_rn(r, kw.y);
  out = ((lo >> 8) & 1) ? -x : x;
  return r < kw.x;
}

// Marsaglia tail of a layer-0 attempt (2.6e-4 of the draws): out of line.
static __device__ __noinline__ double tail(uint32_t p, uint32_t j, uint32_t key, bool neg) {
  for (uint32_t t = 0;; ++t) {
    uint32_t l1, h1, l2, h2;
    word(p, j, 128 + 2 * t, key, l1, h1);
    word(p, j, 129 + 2 * t, key, l2, h2);
    const double xx = __dmul_rn(-NPZ_INV_R, np::glibc_log1p(-unit53(l1, h1)));
    const double yy = -np::glibc_log1p(-unit53(l2, h2));
    if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) return neg ? -__dadd_rn(NPZ_R, xx) : __dadd_rn(NPZ_R, xx);
  }
}

// The whole ziggurat for one normal from attempt 0.  Wedge test: a
// single-precision filter decides all but draws within 2^-18 of the
// boundary, which take the double-precision exp.  Marsaglia tail: the sign
// is bit 8 of the magnitude field (numpy's (rabs >> 8) & 1), bit 17 of the
// word.
// slow_from: attempt 0's word (lo, hi) is already known (the fast path made
// it); later attempts make their own.
__device__ __forceinline__ double slow_from(uint32_t p, uint32_t j, uint32_t key, const ZigTables *z, uint32_t lo,
                                            uint32_t hi) {
  for (uint32_t a = 0;; ++a) {
    if (a > 0) word(p, j, 2 * a, key, lo, hi);
    const int idx = (int)(lo & 0xff);
    const double r = rabs_of(lo, hi);
    const double2 kw = z->kw[idx];
    double x = __dmul_rn(r, kw.y);
    if ((lo >> 8) & 1) x = -x;
    if (r < kw.x) return x;
    if (idx == 0) return tail(p, j, key, (lo >> 17) & 1);
    uint32_t ul, uh;
    word(p, j, 2 * a + 1, key, ul, uh);
    const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(z->fi[idx - 1], z->fi[idx]), unit53(ul, uh)), z->fi[idx]);
    const double q = __dmul_rn(__dmul_rn(-0.5, x), x);
    const double ef = (double)expf((float)q);  // within 1e-6 relative of exp(q) here
    if (lhs < ef * (1.0 - 0x1.0p-18)) return x;
    if (!(lhs > ef * (1.0 + 0x1.0p-18)) && lhs < exp(q)) return x;
  }
}

__device__ __forceinline__ double slow(uint32_t p, uint32_t j, uint32_t key, const ZigTables *z) {
  uint32_t lo, hi;
  word(p, j, 0, key, lo, hi);
  return slow_from(p, j, key, z, lo, hi);
}

// Standard normal increment of particle p at step j of global slice n.
__device__ __forceinline__ double normal(const CounterNoise &c, uint32_t p, uint32_t j, uint32_t n,
                                         const ZigTables *z) {
  const uint32_t key = slice_key(c, n);
  double v;
  if (fast(p, j, key, z, v)) return v;
  return slow(p, j, key, z);
}

// One Euler-Maruyama step of a lane's particles with counter increments.
// Particle m of the lane is global index pbase + 8 m (live when m < LO or
// m < cnt); the lane's tail element (HAS_TAIL, when tail_live) is ptail.
// upd(x, z) returns the updated position.  Every lane runs the fast path for
// all of its particles first; the few rejected draws (0.16 per lane-step on
// average) are then resolved by their own lanes, one per round, with the
// particle picked out of / written back into the register array by
// compile-time selects (no local-memory indexing).
template <int PPT, int LO, bool HAS_TAIL, class Upd>
__device__ __forceinline__ void step(uint32_t key, uint32_t j, const ZigTables *z, double (&x)[PPT], double &xt,
                                     uint32_t pbase, int cnt, uint32_t ptail, bool tail_live, int lane, Upd upd) {
  uint32_t rej = 0;
#pragma unroll
  for (int m = 0; m < PPT; ++m) {
    if (m < LO || m < cnt) {
      double v;
      if (fast(pbase + 8u * (uint32_t)m, j, key, z, v)) x[m] = upd(x[m], v);
      else rej |= 1u << m;
    }
  }
  if (HAS_TAIL && tail_live) {
    double v;
    if (fast(ptail, j, key, z, v)) xt = upd(xt, v);
    else rej |= 1u << PPT;
  }
#if defined(MMPR_PHX_DEBUG) && MMPR_PHX_DEBUG >= 1  // dev A/B only: rejected draws left unresolved
  return;
#endif
  (void)lane;
  while (rej) {
    const int m = __ffs(rej) - 1;
    rej &= rej - 1;
    const double zv = slow(m == PPT ? ptail : pbase + 8u * (uint32_t)m, j, key, z);
    if (HAS_TAIL && m == PPT) {
      xt = upd(xt, zv);
    } else {
      double xm = x[0];
#pragma unroll
      for (int q = 1; q < PPT; ++q) xm = (m == q) ? x[q] : xm;
      xm = upd(xm, zv);
#pragma unroll
      for (int q = 0; q < PPT; ++q) x[q] = (m == q) ? xm : x[q];
    }
  }
}

// Step j's increments of a lane's particles, written to the lane's column of
// a shared-memory buffer (element m at zb[m * stride], the tail element at
// zb[PPT * stride]) one step AHEAD of their use: the kernels call this while
// the previous step's cluster-wide mean is in flight, so the generator's
// issue work (and the divergent resolution of rejected draws) fills the
// latency of the per-step reduction instead of lengthening the step's
// critical path.  A rejected draw's slot first holds its attempt-0 word,
// which the resolution reuses.  Only the generating lane reads its column
// (program order; no barrier).  Same values as step()/normal().
constexpr int kGenUnroll = MMPR_PHX_GEN_UNROLL;

template <int PPT, int LO, bool HAS_TAIL>
__device__ __forceinline__ void gen(uint32_t key, uint32_t j, const ZigTables *z, double *zb, int stride,
                                    uint32_t pbase, int cnt, uint32_t ptail, bool tail_live) {
  uint32_t rej = 0;
#pragma unroll kGenUnroll
  for (int m = 0; m < PPT; ++m) {
    if (m < LO || m < cnt) {
      const uint32_t pm = pbase + 8u * (uint32_t)m;
      uint32_t lo, hi;
      word(pm, j, 0, key, lo, hi);
      const double r = rabs_of(lo, hi);
      const double2 kw = z->kw[lo & 0xff];
      const double xv = __dmul_rn(r, kw.y);
      const bool acc = r < kw.x;
      zb[m * stride] = acc ? (((lo >> 8) & 1) ? -xv : xv) : __hiloint2double((int)hi, (int)lo);
      rej |= acc ? 0u : (1u << m);
    }
  }
  if (HAS_TAIL && tail_live) {
    uint32_t lo, hi;
    word(ptail, j, 0, key, lo, hi);
    const double r = rabs_of(lo, hi);
    const double2 kw = z->kw[lo & 0xff];
    const double xv = __dmul_rn(r, kw.y);
    const bool acc = r < kw.x;
    zb[PPT * stride] = acc ? (((lo >> 8) & 1) ? -xv : xv) : __hiloint2double((int)hi, (int)lo);
    rej |= acc ? 0u : (1u << PPT);
  }
  while (rej) {
    const int m = __ffs(rej) - 1;
    rej &= rej - 1;
    const double w = zb[m * stride];
    const uint32_t pm = (HAS_TAIL && m == PPT) ? ptail : pbase + 8u * (uint32_t)m;
    zb[m * stride] = slow_from(pm, j, key, z, (uint32_t)__double2loint(w), (uint32_t)__double2hiint(w));
  }
}

// dynamic shared memory of a generate-ahead kernel with T threads and PPT
// accumulator elements per lane: the ziggurat tables, then the increment
// columns
__host__ __device__ constexpr size_t gen_smem_bytes(int ppt, int threads) {
  return sizeof(ZigTables) + (size_t)(ppt + 1) * (size_t)threads * sizeof(double);
}

}  // namespace cn
}  // namespace mmpr
