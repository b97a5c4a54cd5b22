// Shared device helpers for libmmpr (sm_100a).
//
//  * exact-arithmetic wrappers: every a*b+c that the reference evaluates with
//    numpy/Python as two roundings is written with __dmul_rn/__dadd_rn so
//    nvcc can never contract it into an FMA (bitwise parity with numpy);
//  * drift/diffusion of the supported model families, in the reference
//    factories' operation order (models.py:265-279, 339-372);
//  * numpy pairwise-summation tree geometry (numpy add.reduce on contiguous
//    float64: blocks of <= 128 with 8 interleaved accumulators, halves split
//    at a multiple of 8), which fixes the association order of every
//    np.mean / np.var the reference takes (models.py:65-67,
//    particles.py:201-202, coupling.py:68-69);
//  * PTX wrappers for clusters / DSMEM, mbarriers and bulk async copies.
#pragma once

#include <stdint.h>
#include <cuda_runtime.h>

#include "../../include/mmpr.h"

#define MMPR_FULL_MASK 0xffffffffu

namespace mmpr {

// ---------------------------------------------------------------------------
// exact IEEE helpers (no contraction)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }

// x**3 rounded once (numpy evaluates x**3 with its vectorised pow; both are
// within an ulp of the exact cube -- parity for cubic drifts is tolerance
// based).
__device__ __forceinline__ double cube(double x) {
  double p = __dmul_rn(x, x);
  double pe = __fma_rn(x, x, -p);
  double c = __dmul_rn(p, x);
  double ce = __fma_rn(p, x, -c);
  return __dadd_rn(c, __fma_rn(pe, x, ce));
}

// exponent field not all ones (integer pipe; keeps the FP64 pipe for the update)
__device__ __forceinline__ bool finite(double x) { return (__double2hiint(x) & 0x7ff00000) != 0x7ff00000; }

// ---------------------------------------------------------------------------
// model families (MEAN_OF_F, identity f)
// ---------------------------------------------------------------------------
struct ModelCoeffs {
  double drift, diff, drift_dx, diff_dx, diff_dxx;
};

// Drift a(x, s) exactly as the reference closures evaluate it.
__device__ __forceinline__ double drift(const mmpr_model &m, double x, double s) {
  const double *p = m.p;
  switch (m.kind) {
    case MMPR_MODEL_OU:  // a*x + a_E*s
      return add(mul(p[0], x), mul(p[1], s));
    case MMPR_MODEL_LINEAR:  // A*x + A_E*s + A_0
      return add(add(mul(p[0], x), mul(p[1], s)), p[2]);
    case MMPR_MODEL_DOUBLE_WELL:
    case MMPR_MODEL_DW_MULT: {  // -(4a x^3 - 2g x - beta s + tilt)
      double t = sub(sub(mul(p[0], cube(x)), mul(p[1], x)), mul(p[2], s));
      return -add(t, p[3]);
    }
    case MMPR_MODEL_CUBIC_MF:  // cE*s - c1*x - c3*(x*x*x)
      return sub(sub(mul(p[2], s), mul(p[0], x)), mul(p[1], mul(mul(x, x), x)));
    default:
      return __longlong_as_double(0x7ff8000000000000ULL);
  }
}

// Diffusion b(x, s).
__device__ __forceinline__ double diffusion(const mmpr_model &m, double x, double s) {
  const double *p = m.p;
  switch (m.kind) {
    case MMPR_MODEL_OU:
      return p[2];
    case MMPR_MODEL_LINEAR:
      return add(add(mul(p[3], x), mul(p[4], s)), p[5]);
    case MMPR_MODEL_DOUBLE_WELL:
      return p[4];
    case MMPR_MODEL_CUBIC_MF:
      return p[3];
    case MMPR_MODEL_DW_MULT:  // s0 * sqrt(1 + x*x)
      return mul(p[4], __dsqrt_rn(add(1.0, mul(x, x))));
    default:
      return __longlong_as_double(0x7ff8000000000000ULL);
  }
}

// True when b does not depend on x or s (b*sqrt(dt) can be hoisted: the
// reference multiplies the constant array np.full_like(x, B) by sqrt(dt),
// which is the same value for every particle).
__host__ __device__ __forceinline__ bool constant_diffusion(int kind) {
  return kind == MMPR_MODEL_OU || kind == MMPR_MODEL_DOUBLE_WELL || kind == MMPR_MODEL_CUBIC_MF;
}

// Scalar coefficients and x-derivatives at (x, s) for the moment closures
// (moments.py:52-68, 145-192).
__device__ inline ModelCoeffs coeffs(const mmpr_model &m, double x, double s) {
  const double *p = m.p;
  ModelCoeffs c;
  if (m.kind == MMPR_MODEL_ROTATOR) {
    // point statistic of a mass at x: (S, C) = (sin x, cos x) (models.py:86-96)
    // a = K (cos x S - sin x C) - sin x, a_x = K (-sin x S - cos x C) - cos x
    double sx, cx;
    sincos(x, &sx, &cx);
    c.drift = sub(mul(p[0], sub(mul(cx, sx), mul(sx, cx))), sx);
    c.drift_dx = sub(mul(p[0], sub(mul(-sx, sx), mul(cx, cx))), cx);
    c.diff = p[1];
    c.diff_dx = 0.0;
    c.diff_dxx = 0.0;
    return c;
  }
  c.drift = drift(m, x, s);
  c.diff = diffusion(m, x, s);
  switch (m.kind) {
    case MMPR_MODEL_OU:
      c.drift_dx = p[0]; c.diff_dx = 0.0; c.diff_dxx = 0.0;
      break;
    case MMPR_MODEL_LINEAR:
      c.drift_dx = p[0]; c.diff_dx = p[3]; c.diff_dxx = 0.0;
      break;
    case MMPR_MODEL_DOUBLE_WELL:  // -(12 a x^2 - 2 g)
      c.drift_dx = -sub(mul(p[5], mul(x, x)), p[1]); c.diff_dx = 0.0; c.diff_dxx = 0.0;
      break;
    case MMPR_MODEL_CUBIC_MF:  // -c1 - 3 c3 x^2
      c.drift_dx = sub(-p[0], mul(mul(3.0, p[1]), mul(x, x))); c.diff_dx = 0.0; c.diff_dxx = 0.0;
      break;
    case MMPR_MODEL_DW_MULT: {
      c.drift_dx = -sub(mul(p[5], mul(x, x)), p[1]);
      double q = add(1.0, mul(x, x));
      double r = __dsqrt_rn(q);
      c.diff_dx = div(mul(p[4], x), r);           // s0*x / sqrt(1+x^2)
      c.diff_dxx = div(p[4], mul(q, r));          // s0 / ((1+x^2) sqrt(1+x^2))
      break;
    }
    default:
      c.drift_dx = c.diff_dx = c.diff_dxx = __longlong_as_double(0x7ff8000000000000ULL);
  }
  return c;
}

// ---------------------------------------------------------------------------
// numpy pairwise-sum tree: padded perfect tree of 2^D leaf slots
// ---------------------------------------------------------------------------
#define MMPR_PW_BLOCK 128

__host__ __device__ __forceinline__ int64_t pw_split(int64_t n) {
  int64_t n2 = n / 2;
  return n2 - (n2 % 8);
}

// Depth of the deepest leaf (always on the right spine: right halves are
// never smaller than left halves).
__host__ __device__ inline int pw_depth(int64_t n) {
  int d = 0;
  while (n > MMPR_PW_BLOCK) {
    n -= pw_split(n);
    ++d;
  }
  return d;
}

// Leaf held by slot `s` of the padded depth-D tree over n elements: a leaf at
// depth d < D sits in the first slot of its 2^(D-d) sub-range, the other
// slots are empty (len 0).
__host__ __device__ inline void pw_leaf(int64_t n, int D, int64_t s, int64_t *off, int64_t *len) {
  int64_t o = 0, m = n;
  for (int level = 0; level < D; ++level) {
    if (m <= MMPR_PW_BLOCK) {
      int64_t below = s & ((int64_t(1) << (D - level)) - 1);
      if (below != 0) { *off = o; *len = 0; return; }
      break;
    }
    int64_t h = pw_split(m);
    if ((s >> (D - 1 - level)) & 1) { o += h; m -= h; } else { m = h; }
  }
  *off = o;
  *len = m;
}

// Pairwise combine with empty-slot semantics: an empty right child passes
// the left value through unchanged (a left child is never empty when its
// right sibling is populated).
struct PwVal {
  double v;
  int ok;
};

__device__ __forceinline__ PwVal pw_combine(PwVal l, PwVal r) {
  PwVal o;
  o.v = r.ok ? add(l.v, r.v) : l.v;
  o.ok = l.ok | r.ok;
  return o;
}

__device__ __forceinline__ PwVal shfl_xor(PwVal a, int lanemask) {
  PwVal b;
  b.v = __shfl_xor_sync(MMPR_FULL_MASK, a.v, lanemask);
  b.ok = __shfl_xor_sync(MMPR_FULL_MASK, a.ok, lanemask);
  return b;
}

// Combine (value from the lower lane block, value from the upper) in the
// fixed left/right order regardless of which lane evaluates it.
__device__ __forceinline__ PwVal pw_xor_level(PwVal mine, int lane, int lanemask) {
  PwVal other = shfl_xor(mine, lanemask);
  return (lane & lanemask) ? pw_combine(other, mine) : pw_combine(mine, other);
}

// ---------------------------------------------------------------------------
// PTX: cluster, DSMEM, mbarrier, bulk async copy
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ void st_cluster_v2(uint32_t addr, unsigned long long a, unsigned long long b) {
  asm volatile("st.shared::cluster.v2.u64 [%0], {%1, %2};" ::"r"(addr), "l"(a), "l"(b) : "memory");
}

// Bulk prefetch of global memory into L2 (no shared-memory destination).
// %globaltimer (ns): per-slice timestamps of the fine sweeps
__device__ __forceinline__ long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (long long)t;
}

__device__ __forceinline__ void prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Asynchronous 16-byte store into another CTA's shared memory that
// completes `bytes` transaction bytes on that CTA's mbarrier (no fence, no
// cluster barrier: the receiver waits on its own mbarrier).
__device__ __forceinline__ void st_async_v2(uint32_t remote_addr, unsigned long long a, unsigned long long b,
                                            uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.u64 [%0], {%1, %2}, [%3];" ::"r"(
                   remote_addr),
               "l"(a), "l"(b), "r"(remote_bar)
               : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t *bar, uint32_t parity) {
  uint32_t addr = smem_addr(bar);
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "MMPR_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra MMPR_WAIT_%=;\n}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> this CTA's shared memory, completion counted on
// `bar` (bytes and both addresses must be multiples of 16).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

}  // namespace mmpr
