/*
 * npstream.c -- CPU restatement of the noise stream behind the reference's
 * NoisePlan (TEST INFRASTRUCTURE: the checker for the GPU stream generator;
 * never linked into the product).
 *
 * Reference call site: mcparareal.particles.NoisePlan._generator/normals
 *   /root/reference/pkg/src/mcparareal/particles.py:49-61
 *     np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy)))
 *         .standard_normal(count)
 * That algorithm lives in the third-party dependency numpy (not vendored in
 * /root/reference; pinned here at numpy 2.3.5).  Its published pieces are
 * restated below:
 *   1. SeedSequence entropy pool (O'Neill's seed_seq hash mixing, pool of
 *      four 32-bit words) and generate_state(2, uint64) -> Philox key.
 *   2. Philox4x64-10 (Salmon et al., SC'11), counter pre-incremented before
 *      each 4-word block, words served in order from the block.
 *   3. numpy's 256-layer ziggurat standard normal over one 64-bit word per
 *      attempt (layer = low 8 bits, sign = bit 8, 52-bit mantissa above),
 *      wedge test with one extra uniform, Marsaglia tail from layer 0.
 *      Tables: np_ziggurat_tables.h (recovered by
 *      oracle/tools/extract_numpy_ziggurat.py).
 * Pinned against numpy itself in tests/test_oracle_npstream.py.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "np_ziggurat_tables.h"

static const uint64_t NPZ_KI[256] = {NPZ_KI_VALUES};
static const double NPZ_WI[256] = {NPZ_WI_VALUES};
static const double NPZ_FI[256] = {NPZ_FI_VALUES};

/* ---- 1. SeedSequence ---------------------------------------------------- */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

static uint32_t ss_hashmix(uint32_t v, uint32_t *h) {
  v ^= *h;
  *h *= SS_MULT_A;
  v *= *h;
  return v ^ (v >> 16);
}

static uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  return r ^ (r >> 16);
}

/* pool[4] from the assembled entropy words (no spawn key). */
void nps_seedseq_pool(const uint32_t *words, int n_words, uint32_t pool[4]) {
  uint32_t h = SS_INIT_A;
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < n_words ? words[i] : 0u, &h);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &h));
  for (int s = 4; s < n_words; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(words[s], &h));
}

/* generate_state(2, np.uint64): four 32-bit words, little-endian pairs. */
void nps_seedseq_key(const uint32_t *words, int n_words, uint64_t key[2]) {
  uint32_t pool[4], out[4], h = SS_INIT_B;
  nps_seedseq_pool(words, n_words, pool);
  for (int i = 0; i < 4; ++i) {
    uint32_t v = pool[i] ^ h;
    h *= SS_MULT_B;
    v *= h;
    out[i] = v ^ (v >> 16);
  }
  key[0] = (uint64_t)out[0] | ((uint64_t)out[1] << 32);
  key[1] = (uint64_t)out[2] | ((uint64_t)out[3] << 32);
}

/* ---- 2. Philox4x64-10 ---------------------------------------------------- */
static void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
  __uint128_t p = (__uint128_t)a * b;
  *hi = (uint64_t)(p >> 64);
  *lo = (uint64_t)p;
}

void nps_philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
  uint64_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL; }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, c[0], &hi0, &lo0);
    mulhilo64(0xCA5A826395121157ULL, c[2], &hi1, &lo1);
    uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
  }
  memcpy(out, c, sizeof c);
}

/* Word i of a fresh stream: block i/4 uses counter (i/4 + 1). */
uint64_t nps_word(const uint64_t key[2], uint64_t i) {
  uint64_t ctr[4] = {(i >> 2) + 1, 0, 0, 0}, out[4];
  if (ctr[0] == 0) ctr[1] = 1; /* carry (never reached in practice) */
  nps_philox4x64_10(ctr, key, out);
  return out[i & 3];
}

typedef struct { uint64_t key[2]; uint64_t pos; uint64_t buf[4]; } nps_stream;

static uint64_t next64(nps_stream *s) {
  if ((s->pos & 3) == 0) {
    uint64_t ctr[4] = {(s->pos >> 2) + 1, 0, 0, 0};
    nps_philox4x64_10(ctr, s->key, s->buf);
  }
  return s->buf[s->pos++ & 3];
}

static double next_unit(nps_stream *s) { return (double)(next64(s) >> 11) * (1.0 / 9007199254740992.0); }

/* ---- 3. ziggurat standard normal ---------------------------------------- */
static double standard_normal(nps_stream *s) {
  for (;;) {
    uint64_t r = next64(s);
    int layer = (int)(r & 0xff);
    r >>= 8;
    int negative = (int)(r & 1);
    uint64_t mant = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)mant * NPZ_WI[layer];
    if (negative) x = -x;
    if (mant < NPZ_KI[layer]) return x;
    if (layer == 0) {
      for (;;) {
        double xx = -NPZ_INV_R * log1p(-next_unit(s));
        double yy = -log1p(-next_unit(s));
        if (yy + yy > xx * xx) return ((mant >> 8) & 1) ? -(NPZ_R + xx) : NPZ_R + xx;
      }
    }
    if ((NPZ_FI[layer - 1] - NPZ_FI[layer]) * next_unit(s) + NPZ_FI[layer] < exp(-0.5 * x * x)) return x;
  }
}

/* Fill out[0..count) from the stream keyed by the SeedSequence entropy words;
 * returns the number of 64-bit words consumed. */
uint64_t nps_standard_normal_fill(const uint32_t *words, int n_words, int64_t count, double *out) {
  nps_stream s;
  memset(&s, 0, sizeof s);
  nps_seedseq_key(words, n_words, s.key);
  for (int64_t i = 0; i < count; ++i) out[i] = standard_normal(&s);
  return s.pos;
}

/* Same, from an explicit Philox key (used to cross-check key derivation). */
uint64_t nps_standard_normal_fill_key(const uint64_t key[2], int64_t count, double *out) {
  nps_stream s;
  memset(&s, 0, sizeof s);
  s.key[0] = key[0];
  s.key[1] = key[1];
  for (int64_t i = 0; i < count; ++i) out[i] = standard_normal(&s);
  return s.pos;
}

/* ---- 4. the host libm's log1p (numpy's tail draws call it) ---------------- */
/* nps_libm_log1p_fill: out[i] = log1p(x[i]) from the C library itself (what
 * numpy's npy_log1p resolves to).  nps_log1p_restated_fill: the restatement
 * of glibc 2.39's FMA build of s_log1p.c (fdlibm algorithm, parallel
 * polynomial) that the device uses (npstream.cuh np::glibc_log1p), compiled
 * with -ffp-contract=off and explicit fma() where the FMA build fuses.
 * tests/test_oracle_npstream.py pins the two against each other here and
 * tests/test_gpu_noise.py pins the device against nps_libm_log1p_fill. */
void nps_libm_log1p_fill(const double *x, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = log1p(x[i]);
}

static int32_t hiword(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return (int32_t)(u >> 32);
}

static double with_hiword(double x, int32_t h) {
  uint64_t u;
  memcpy(&u, &x, 8);
  u = (u & 0xffffffffULL) | ((uint64_t)(uint32_t)h << 32);
  memcpy(&x, &u, 8);
  return x;
}

static double log1p_restated(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
               Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int32_t hx = hiword(x), ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : NAN;
    if (ax < 0x3e200000) return ax < 0x3c900000 ? x : fma(-(x * x), 0.5, x);
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return x + x;
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = hiword(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
      c /= u;
    } else {
      u = x;
      hu = hiword(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hiword(u, hu | 0x3ff00000);
    } else {
      k += 1;
      u = with_hiword(u, hu | 0x3fe00000);
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double dk = (double)k, hfsq = (0.5 * f) * f;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = fma(dk, ln2_lo, c);
      return fma(dk, ln2_hi, c);
    }
    const double R = hfsq * fma(-0.66666666666666666, f, 1.0);
    if (k == 0) return f - R;
    return fma(dk, ln2_hi, -((R - fma(dk, ln2_lo, c)) - f));
  }
  const double s = f / (2.0 + f), z = s * s;
  const double z2 = z * z, z4 = z2 * z2, z6 = z4 * z2;
  const double R = fma(z6, fma(z, Lp7, Lp6), fma(z4, fma(z, Lp5, Lp4), fma(z, Lp1, z2 * fma(z, Lp3, Lp2))));
  const double sR = s * (hfsq + R);
  if (k == 0) return f - (hfsq - sR);
  return fma(dk, ln2_hi, -((hfsq - (sR + fma(dk, ln2_lo, c))) - f));
}

void nps_log1p_restated_fill(const double *x, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = log1p_restated(x[i]);
}

/* ---- 5. counter-based Philox mode (NoiseMode.PHILOX / PHILOX_FRESH) ------- */
/* The device generator of paper_2310_11365_b200/csrc/counter_noise.cuh,
 * restated: Philox2x32-10 (Salmon et al.) words addressed by
 * (p, j | draw << 24) under the slice key k32 ^ (n | kfield << 20), fed to
 * numpy's ziggurat transform (section 3's tables and rules; the tail's
 * log1p is the C library's, as on the device, which restates it).  Attempt
 * a: word = draw 2a, wedge uniform = draw 2a + 1; tail iteration t: draws
 * 128 + 2t and 129 + 2t.  This mode has no reference counterpart (the
 * reference's noise is numpy's stream); tests pin the device to this
 * restatement bit for bit and the engine's Philox-mode runs to the
 * reference's numpy-noise runs statistically. */
#define PH_M 0xD256D193u
#define PH_W 0x9E3779B9u

void nps_philox2x32_10(const uint32_t ctr[2], uint32_t key, uint32_t out[2]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], k = key;
  for (int r = 0; r < 10; ++r) {
    const uint64_t prod = (uint64_t)PH_M * c0;
    const uint32_t n0 = (uint32_t)(prod >> 32) ^ k ^ c1;
    c1 = (uint32_t)prod;
    c0 = n0;
    k += PH_W;
  }
  out[0] = c0;
  out[1] = c1;
}

static uint64_t ph_word(uint32_t p, uint32_t j, uint32_t d, uint32_t key) {
  const uint32_t ctr[2] = {p, j | (d << 24)};
  uint32_t o[2];
  nps_philox2x32_10(ctr, key, o);
  return (uint64_t)o[0] | ((uint64_t)o[1] << 32);
}

static double ph_unit(uint64_t w) { return (double)(w >> 11) * (1.0 / 9007199254740992.0); }

static double counter_normal(uint32_t p, uint32_t j, uint32_t key) {
  for (uint32_t a = 0;; ++a) {
    const uint64_t w = ph_word(p, j, 2 * a, key);
    const int idx = (int)(w & 0xff);
    const uint64_t rabs = (w >> 9) & 0x000fffffffffffffULL;
    double x = (double)rabs * NPZ_WI[idx];
    if ((w >> 8) & 1) x = -x;
    if (rabs < NPZ_KI[idx]) return x;
    if (idx == 0) {
      for (uint32_t t = 0;; ++t) {
        const double xx = -NPZ_INV_R * log1p(-ph_unit(ph_word(p, j, 128 + 2 * t, key)));
        const double yy = -log1p(-ph_unit(ph_word(p, j, 129 + 2 * t, key)));
        if (yy + yy > xx * xx) return ((rabs >> 8) & 1) ? -(NPZ_R + xx) : NPZ_R + xx;
      }
    }
    const double u = ph_unit(ph_word(p, j, 2 * a + 1, key));
    if ((NPZ_FI[idx - 1] - NPZ_FI[idx]) * u + NPZ_FI[idx] < exp(-0.5 * x * x)) return x;
  }
}

/* out[i] = increment of particle p0 + i at step j of global slice n */
void nps_counter_normals(const uint32_t key[2], uint32_t kfield, uint32_t n, uint32_t j, uint32_t p0, int64_t count,
                         double *out) {
  const uint32_t k = key[0] ^ (n | (kfield << 20));
  for (int64_t i = 0; i < count; ++i) out[i] = counter_normal(p0 + (uint32_t)i, j, k);
}
