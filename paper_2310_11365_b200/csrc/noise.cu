// numpy-exact standard-normal streams on sm_100a.
//
// Replaces NoisePlan.normals / init_rng
// (/root/reference/pkg/src/mcparareal/particles.py:49-65): every (slice,
// step[, iteration]) address is its own numpy stream
//   Generator(Philox(SeedSequence((seed, domain, n, j[, k])))).standard_normal(P)
// and this file reproduces those streams bit-for-bit: the Marsaglia tail
// uses the host libm's log1p restated (np::glibc_log1p), and a wedge test
// whose outcome CUDA's exp cannot decide the way glibc's would is counted
// (mmpr_noise_exp_ambiguous; tests assert the count stays 0).
//
// One CTA materialises one stream.  The stream is a variable-length parse of
// Philox words (a fast-accept word yields one normal; a wedge word consumes
// its successor as a uniform; a tail word consumes pairs of successors), so
// output i is not at word i.  Per chunk of 1024 words:
//   1. each thread generates one Philox4x64 block (4 consecutive words) and
//      classifies the words assuming each starts an attempt;
//   2. each warp parses its 128 words from entry offset 0 by walking only the
//      non-fast words (warp-uniform loop, ~3 iterations per chunk);
//   3. warp 0 stitches the 8 speculative parses with the chunk carry (falls
//      back to an exact sequential re-walk when a speculation is wrong);
//   4. every produced normal is written at its exact stream position.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "mmpr_device.cuh"
#include "npstream.cuh"
#include "counter_noise.cuh"
#include "capi_internal.h"

namespace mmpr {

__constant__ uint64_t c_zig_ki[256] = {NPZ_KI_VALUES};
__constant__ double c_zig_wi[256] = {NPZ_WI_VALUES};
__constant__ double c_zig_fi[256] = {NPZ_FI_VALUES};

// wedge tests decided inside the exp ambiguity band (see wedge_accepts)
__device__ unsigned long long g_exp_ambiguous = 0;

#define NF_THREADS 256
// streams at or above which one warp (not one CTA) materialises a stream
#define MMPR_WARP_STREAMS_MIN 256
#define NF_WARPS (NF_THREADS / 32)

// ---------------------------------------------------------------------------
// keys
// ---------------------------------------------------------------------------
__global__ void noise_keys_kernel(uint64_t seed, int fresh, int iteration, int n_offset, int n_slices,
                                  int steps, uint64_t *keys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n_slices * steps) return;
  const int n = n_offset + (int)(i / steps);
  const int j = (int)(i % steps);
  uint32_t w[8];
  int nw = np::push_int_words(w, 0, seed);
  nw = np::push_int_words(w, nw, fresh ? 2u : 1u);  // _DOMAIN_STEP_FRESH / _FROZEN
  nw = np::push_int_words(w, nw, (uint64_t)n);
  nw = np::push_int_words(w, nw, (uint64_t)j);
  if (fresh) nw = np::push_int_words(w, nw, (uint64_t)iteration);
  uint64_t k0, k1;
  np::seedseq_key(w, nw, k0, k1);
  keys[2 * i] = k0;
  keys[2 * i + 1] = k1;
}

struct EntropyWords {
  uint32_t w[16];
};

__global__ void entropy_key_kernel(EntropyWords e, int n, uint64_t *key) {
  uint64_t k0, k1;
  np::seedseq_key(e.w, n, k0, k1);
  key[0] = k0;
  key[1] = k1;
}

// ---------------------------------------------------------------------------
// stream parse helpers
// ---------------------------------------------------------------------------
// first set bit at position >= pos in a 128-bit mask, or -1
__device__ __forceinline__ int next_set128(const uint32_t m[4], int pos) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (pos < 32 * (k + 1)) {
      uint32_t v = m[k];
      if (pos > 32 * k) v &= ~((1u << (pos - 32 * k)) - 1u);
      if (v) return 32 * k + __ffs(v) - 1;
    }
  }
  return -1;
}

// clear bits [lo, hi) (hi <= 128)
__device__ __forceinline__ void clear_range128(uint32_t m[4], int lo, int hi) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int a = max(lo, 32 * k), b = min(hi, 32 * (k + 1));
    if (a < b) {
      const int n = b - a;
      const uint32_t bits = (n == 32) ? 0xffffffffu : (((1u << n) - 1u) << (a - 32 * k));
      m[k] &= ~bits;
    }
  }
}

// bits at positions >= e kept
__device__ __forceinline__ uint32_t mask_ge(int k, int e) {
  if (e <= 32 * k) return 0xffffffffu;
  if (e >= 32 * (k + 1)) return 0u;
  return ~((1u << (e - 32 * k)) - 1u);
}

// Exact sequential parse of one 128-word range from entry `e` (< 128) with
// token lengths `len`: start mask and exit (words consumed past the range).
__device__ int rewalk(const uint32_t na[4], const uint16_t *len, int e, uint32_t S[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) S[k] = mask_ge(k, e);
  int pos = e;
  for (;;) {
    const int b = next_set128(na, pos);
    if (b < 0) return 0;
    const int L = len[b];
    clear_range128(S, b + 1, min(b + L, 128));
    pos = b + L;
    if (pos >= 128) return pos - 128;
  }
}

// Parse from entry 0 when every non-fast word is a wedge (length 2): in a
// maximal run of wedge words starting at a, the words at odd offsets
// a+1, a+3, ... (up to one past the run) are consumed uniforms, the rest
// start attempts.  Runs are separated by parity of their start with one
// carry-propagating add (the simdjson odd-backslash trick).
__device__ __forceinline__ void wedge_parse(const uint32_t nf[4], uint32_t S[4], int &exit) {
  const uint64_t EVEN = 0x5555555555555555ULL, ODD = 0xAAAAAAAAAAAAAAAAULL;
  const uint64_t wl = (uint64_t)nf[0] | ((uint64_t)nf[1] << 32);
  const uint64_t wh = (uint64_t)nf[2] | ((uint64_t)nf[3] << 32);
  const uint64_t pl = wl << 1, ph = (wh << 1) | (wl >> 63);        // W << 1
  const uint64_t sl = wl & ~pl, sh = wh & ~ph;                      // run starts
  const uint64_t el = sl & EVEN, eh = sh & EVEN;                    // even-start runs
  const uint64_t al = wl + el;                                      // carry through runs
  const uint64_t ah = wh + eh + (al < wl ? 1ULL : 0ULL);
  const uint64_t rel = wl & ~al, reh = wh & ~ah;                    // even-start run bits
  const uint64_t rol = wl & ~rel, roh = wh & ~reh;                  // odd-start run bits
  const uint64_t cl = ((rel << 1) & ODD) | ((rol << 1) & EVEN);
  const uint64_t ch = ((((reh << 1) | (rel >> 63)) & ODD)) | ((((roh << 1) | (rol >> 63)) & EVEN));
  S[0] = ~(uint32_t)cl;
  S[1] = ~(uint32_t)(cl >> 32);
  S[2] = ~(uint32_t)ch;
  S[3] = ~(uint32_t)(ch >> 32);
  // a wedge starting at word 127 consumes word 0 of the next range
  exit = ((wh >> 63) & 1ULL) && ((S[3] >> 31) & 1u) ? 1 : 0;
}

// Tail attempt starting at stream word `wi` (layer 0, mantissa >= ki[0]):
// Marsaglia's tail over successive pairs of uniforms.  Rare (~2.6e-4 of the
// draws), so the successor words are recomputed from the counter.
__device__ __noinline__ double tail_token(uint64_t wi, uint64_t mant, uint64_t k0, uint64_t k1, int *len) {
  uint64_t i = wi + 1;
  for (;;) {
    const uint64_t a = np::philox_word(i++, k0, k1);
    const uint64_t b = np::philox_word(i++, k0, k1);
    const double xx = mul(-NPZ_INV_R, np::glibc_log1p(-np::unit_double(a)));
    const double yy = -np::glibc_log1p(-np::unit_double(b));
    if (add(yy, yy) > mul(xx, xx)) {
      const uint64_t L = i - wi;
      *len = (int)(L < 0xffffu ? L : 0xffffu);
      return ((mant >> 8) & 1) ? -add(NPZ_R, xx) : add(NPZ_R, xx);
    }
  }
}

// Wedge test of layer `layer` at x with the next word's uniform (fi: the
// fi table, constant or shared memory).
__device__ __forceinline__ bool wedge_accepts(int layer, double x, uint64_t next_word,
                                              const double *fi = c_zig_fi) {
  const double u = np::unit_double(next_word);
  const double lhs = add(mul(sub(fi[layer - 1], fi[layer]), u), fi[layer]);
  const double q = mul(mul(-0.5, x), x);  // in [-6.7, 0] for wedge draws
  // single-precision filter: expf((float)q) is within 1e-6 of exp(q)
  // relative here (rounding of q times |q|, plus expf's 2 ulp), so only
  // draws within 4e-6 of the boundary need the double-precision exp
  const double ef = (double)expf((float)q);
  if (lhs < ef * (1.0 - 0x1.0p-18)) return true;
  if (lhs > ef * (1.0 + 0x1.0p-18)) return false;
  // glibc's exp is within 0.52 ulp of exp(q) and CUDA's within 1 ulp, so
  // outside a 2^-50 relative band around CUDA's value both give the same
  // comparison; inside it (never observed) the draw is counted
  const double e = exp(q);
  if (fabs(sub(lhs, e)) <= mul(e, 0x1.0p-50)) atomicAdd(&g_exp_ambiguous, 1ULL);
  return lhs < e;
}

// ---------------------------------------------------------------------------
// stream fill kernel
// ---------------------------------------------------------------------------
#define NF_BPT 2                          // Philox blocks (rows) per thread per chunk
#define NF_RANGES (NF_WARPS * NF_BPT)     // 128-word ranges per chunk (<= 32)

__global__ void __launch_bounds__(NF_THREADS, 3)
normals_fill_kernel(const uint64_t *__restrict__ keys, int64_t count, double *__restrict__ out,
                    int64_t pitch, int affine, double loc, double scale) {
  __shared__ ulonglong2 zig[256];
  __shared__ __align__(16) uint32_t s_spec[NF_RANGES][4];  // speculative starts (entry 0)
  __shared__ __align__(16) uint32_t s_prod[NF_RANGES][4];  // words that yield a normal if they start
  __shared__ __align__(16) uint32_t s_nonfast[NF_RANGES][4];
  __shared__ __align__(16) uint32_t s_final[NF_RANGES][4];
  __shared__ __align__(16) uint16_t s_len[NF_RANGES * 128];
  __shared__ int s_exit[NF_RANGES];
  __shared__ int s_base[NF_RANGES];
  __shared__ int s_carry, s_total;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t k0 = keys[2 * blockIdx.x], k1 = keys[2 * blockIdx.x + 1];
  double *o = out + (int64_t)blockIdx.x * pitch;

  for (int i = tid; i < 256; i += NF_THREADS)
    zig[i] = make_ulonglong2(c_zig_ki[i], (unsigned long long)__double_as_longlong(c_zig_wi[i]));
  if (tid == 0) s_carry = 0;
  __syncthreads();

  const int sh = 4 * (lane & 7);
  int64_t produced = 0;
  for (uint64_t chunk = 0; produced < count; ++chunk) {
    double val[NF_BPT][4];
    uint32_t prod_nib[NF_BPT], tail_nib[NF_BPT];
#pragma unroll
    for (int r = 0; r < NF_BPT; ++r) {
      const uint64_t blk = (chunk * NF_BPT + r) * NF_THREADS + tid;
      const uint64_t word0 = blk * 4;
      uint64_t w[4];
      np::philox_block(blk, k0, k1, w);
      const uint64_t succ = __shfl_down_sync(MMPR_FULL_MASK, w[0], 1);
      uint32_t nonfast = 0, prod = 0, tails = 0;
      uint16_t lens[4] = {1, 1, 1, 1};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t rw = w[q];
        const int layer = (int)(rw & 0xff);
        const uint64_t mant = (rw >> 9) & 0x000fffffffffffffULL;
        const ulonglong2 z = zig[layer];
        const double wi = __longlong_as_double((long long)z.y);
        // (double)mant * wi rounded once: (2^52 + mant) * wi - 2^52 * wi
        double x = __fma_rn(__longlong_as_double((long long)(0x4330000000000000ULL | mant)), wi, -0x1.0p52 * wi);
        if ((rw >> 8) & 1) x = -x;
        val[r][q] = x;
        if (mant >= z.x) {
          nonfast |= 1u << q;
          if (layer != 0) {
            const uint64_t nx = (q < 3) ? w[q + 1] : (lane < 31 ? succ : np::philox_word(word0 + 4, k0, k1));
            if (wedge_accepts(layer, x, nx)) prod |= 1u << q;
            lens[q] = 2;
          } else {
            int L;
            tail_token(word0 + q, mant, k0, k1, &L);
            lens[q] = (uint16_t)L;
            tails |= 1u << q;
            prod |= 1u << q;
          }
        } else {
          prod |= 1u << q;
        }
      }
      prod_nib[r] = prod;
      tail_nib[r] = tails;
      const int range = r * NF_WARPS + warp;
      *reinterpret_cast<ushort4 *>(&s_len[range * 128 + 4 * lane]) = make_ushort4(lens[0], lens[1], lens[2], lens[3]);
      uint32_t NF[4], PR[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        NF[k] = __reduce_or_sync(MMPR_FULL_MASK, (lane >> 3) == k ? (nonfast << sh) : 0u);
        PR[k] = __reduce_or_sync(MMPR_FULL_MASK, (lane >> 3) == k ? (prod << sh) : 0u);
      }
      uint32_t S[4];
      int exit0 = 0;
      if (!__any_sync(MMPR_FULL_MASK, tails != 0)) {
        wedge_parse(NF, S, exit0);
      } else {  // a tail token in this range: general walk (warp-uniform)
        const uint64_t lp = (uint64_t)lens[0] | ((uint64_t)lens[1] << 16) | ((uint64_t)lens[2] << 32) |
                            ((uint64_t)lens[3] << 48);
#pragma unroll
        for (int k = 0; k < 4; ++k) S[k] = 0xffffffffu;
        int pos = 0;
        for (;;) {
          const int b = next_set128(NF, pos);
          if (b < 0) break;
          const uint64_t l = __shfl_sync(MMPR_FULL_MASK, lp, b >> 2);
          const int L = (int)((l >> (16 * (b & 3))) & 0xffff);
          clear_range128(S, b + 1, min(b + L, 128));
          pos = b + L;
          if (pos >= 128) {
            exit0 = pos - 128;
            break;
          }
        }
      }
      if (lane < 4) {
        s_spec[range][lane] = S[lane];
        s_prod[range][lane] = PR[lane];
        s_nonfast[range][lane] = NF[lane];
      }
      if (lane == 0) s_exit[range] = exit0;
    }
    __syncthreads();

    // stitch the NF_RANGES speculative parses in stream order (warp 0)
    if (warp == 0) {
      const int me = lane < NF_RANGES ? lane : 0;
      const int e = (me == 0) ? s_carry : s_exit[me - 1];
      bool ok = true;
      if (lane < NF_RANGES && e != 0) ok = e < 128 && ((s_spec[me][e >> 5] >> (e & 31)) & 1u);
      if (__all_sync(MMPR_FULL_MASK, ok)) {
        int cnt = 0;
        if (lane < NF_RANGES) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t F = s_spec[me][k] & mask_ge(k, e);
            s_final[me][k] = F;
            cnt += __popc(F & s_prod[me][k]);
          }
        }
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int v = __shfl_up_sync(MMPR_FULL_MASK, incl, d);
          if (lane >= d) incl += v;
        }
        if (lane < NF_RANGES) s_base[lane] = incl - cnt;
        const int tot = __shfl_sync(MMPR_FULL_MASK, incl, NF_RANGES - 1);
        __syncwarp();
        if (lane == 0) {
          s_total = tot;
          s_carry = s_exit[NF_RANGES - 1];
        }
      } else if (lane == 0) {
        int ent = s_carry, base = 0;
        for (int ri = 0; ri < NF_RANGES; ++ri) {
          uint32_t F[4];
          int ex;
          if (ent >= 128) {
            F[0] = F[1] = F[2] = F[3] = 0u;
            ex = ent - 128;
          } else if (ent == 0 || ((s_spec[ri][ent >> 5] >> (ent & 31)) & 1u)) {
#pragma unroll
            for (int k = 0; k < 4; ++k) F[k] = s_spec[ri][k] & mask_ge(k, ent);
            ex = s_exit[ri];
          } else {
            const uint32_t na[4] = {s_nonfast[ri][0], s_nonfast[ri][1], s_nonfast[ri][2], s_nonfast[ri][3]};
            ex = rewalk(na, &s_len[ri * 128], ent, F);
          }
          s_base[ri] = base;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            s_final[ri][k] = F[k];
            base += __popc(F[k] & s_prod[ri][k]);
          }
          ent = ex;
        }
        s_total = base;
        s_carry = ent;
      }
    }
    __syncthreads();

    // scatter this thread's normals to their stream positions
#pragma unroll
    for (int r = 0; r < NF_BPT; ++r) {
      const int range = r * NF_WARPS + warp;
      const uint4 F = *reinterpret_cast<const uint4 *>(s_final[range]);
      const uint32_t Fk[4] = {F.x, F.y, F.z, F.w};
      const int k = lane >> 3;
      int pre = 0;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        if (kk < k) pre += __popc(Fk[kk] & s_prod[range][kk]);
      const uint32_t Ok = Fk[k] & s_prod[range][k];
      pre += __popc(Ok & ((1u << sh) - 1u));
      const uint32_t nib = (Ok >> sh) & 0xfu;
      const int64_t base = produced + s_base[range] + pre;
      const uint64_t word0 = ((chunk * NF_BPT + r) * NF_THREADS + tid) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if ((nib >> q) & 1u) {
          const int64_t idx = base + __popc(nib & ((1u << q) - 1u));
          if (idx < count) {
            double v = val[r][q];
            if ((tail_nib[r] >> q) & 1u) {  // rare: recompute the tail value
              const uint64_t rw = np::philox_word(word0 + q, k0, k1);
              int L;
              v = tail_token(word0 + q, (rw >> 9) & 0x000fffffffffffffULL, k0, k1, &L);
            }
            o[idx] = affine ? add(loc, mul(scale, v)) : v;
          }
        }
      }
      (void)prod_nib;
    }
    produced += s_total;
    // s_final/s_base/s_total are rewritten only after the next chunk's first
    // barrier, which every thread reaches after finishing this scatter.
  }
}

// ---------------------------------------------------------------------------
// warp-per-stream fill (many streams): no block barriers at all
// ---------------------------------------------------------------------------
// Each warp owns one stream and walks it in sub-chunks of 32 lanes x 8
// consecutive words.  A lane parses its 8 words from an assumed entry with
// the wedge bit trick (or a short exact loop when a tail token is present);
// entries are then stitched lane to lane with shuffles until stable (an
// entry of 1 usually just truncates the speculative parse), the produced
// normals are counted with a warp scan and written at their exact positions.
#ifndef NW_WORDS
#define NW_WORDS 8  // words per lane and sub-chunk (8; 16 measured slower: 4.2 vs 3.3 ms)
#endif
#define NW_ALL ((1u << NW_WORDS) - 1u)

// Lane parse of 8 words from entry e (< 8) when all non-fast words are wedges.
__device__ __forceinline__ void wedge_parse8(uint32_t nf, int e, uint32_t &S, int &exit) {
  const uint32_t w = nf >> e;
  const int width = NW_WORDS - e;
  const uint32_t starts = w & ~(w << 1);
  const uint32_t re = w & ~(w + (starts & 0x55555555u));   // runs starting at even offsets
  const uint32_t ro = w & ~re;
  const uint32_t cov = ((re << 1) & 0xAAAAAAAAu) | ((ro << 1) & 0x55555555u);
  const uint32_t s_rel = ~cov & ((1u << width) - 1u);
  S = s_rel << e;
  exit = (((w & s_rel) >> (width - 1)) & 1u) ? 1 : 0;
}

// Exact lane parse from entry e with tail tokens present (rare path); the
// tail lengths were measured once by the work-list pass (tlen).
__device__ __noinline__ void general_parse8(uint32_t nf, uint32_t tt, int e, const uint16_t *tlen,
                                            uint32_t *S_out, int *exit_out) {
  uint32_t S = 0;
  int pos = e;
  while (pos < NW_WORDS) {
    S |= 1u << pos;
    int L = 1;
    if ((nf >> pos) & 1u) L = ((tt >> pos) & 1u) ? (int)tlen[pos] : 2;
    pos += L;
  }
  *S_out = S;
  *exit_out = pos - NW_WORDS;
}

__device__ __noinline__ uint64_t successor_word(uint64_t i, uint64_t k0, uint64_t k1) {
  return np::philox_word(i, k0, k1);
}

// One single-warp CTA per stream: the Philox key is CTA-uniform (uniform
// datapath for the key schedule), there is no block barrier in the loop,
// and up to 32 streams run per SM.
#ifndef NW_MINB
#define NW_MINB 16
#endif
// Segments (more streams than resident warps): a stream's sub-chunks are cut
// into `nseg` runs of `seg_subs`, one single-warp CTA per (stream, segment),
// CTAs laid out segment-major (grid y = segment).  A segment starts from the (produced, carry)
// state its predecessor leaves in the stream's LAST output slot -- a
// mailbox only the final segment writes a normal to: the host sizes the
// segments so that the earlier ones cannot produce `count` values (outputs
// <= words), and a clear kernel zeroes the mailboxes ahead of the launch.
// The CTAs of a 1-D grid are dispatched in index order (CUB's decoupled
// look-back relies on the same), so a predecessor is resident or finished
// before its successor starts; with more streams than resident warps it
// finished long before and the wait is one load.  The launch then ends in
// a full last wave instead of a ragged one (config 4: 2.7 waves of 2368
// warps; measured ~5%).  A bounded spin turns a broken assumption into a
// trap, not a hang.
#define NW_TAG_SHIFT 56
#define NW_CARRY_SHIFT 40

__device__ __noinline__ unsigned long long mailbox_wait(const double *mail, int seg) {
  const long long t0 = clock64();
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mail) : "memory");
    if ((int)(v >> NW_TAG_SHIFT) == seg) return v;
    __nanosleep(100);
    if (clock64() - t0 > (1LL << 33)) __trap();  // in-order dispatch assumption broken
  }
}

__global__ void noise_mailbox_clear_kernel(double *__restrict__ out, int64_t pitch, int64_t count, int n_streams) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_streams) reinterpret_cast<unsigned long long *>(out + (int64_t)i * pitch)[count - 1] = 0ULL;
}

template <bool AFFINE>
__global__ void __launch_bounds__(32, NW_MINB)
normals_fill_warp_kernel(const uint64_t *__restrict__ keys, int64_t count, double *__restrict__ out, int64_t pitch,
                         double loc, double scale, int nseg, int seg_subs) {
  __shared__ ulonglong2 zig[256];
  __shared__ double s_fi[256];
  __shared__ uint16_t s_tlen[32 * NW_WORDS];  // tail starts (lane-private slots): length in words
  __shared__ __align__(16) unsigned long long s_w[32 * NW_WORDS + 1];  // the sub-chunk's words + the next one's first
  const int lane = threadIdx.x;
#pragma unroll
  for (int i = lane; i < 256; i += 32) {
    // ki as the double 2^52 + ki (exact: ki < 2^52), so the fast-accept test
    // is one FP64 compare against the 2^52 + mant the transform builds anyway
    zig[i] = make_ulonglong2(0x4330000000000000ULL | c_zig_ki[i], (unsigned long long)__double_as_longlong(c_zig_wi[i]));
    s_fi[i] = c_zig_fi[i];
  }
  __syncwarp();
  // (stream, segment) = (blockIdx.x, blockIdx.y): both CTA-uniform special
  // registers, so the Philox key stays on the uniform datapath (an index
  // division would move the key schedule to the vector registers); CTAs are
  // dispatched x-fastest, i.e. segment-major
  const int seg = (int)blockIdx.y;
  double *o = out + (int64_t)blockIdx.x * pitch;
  int carry = 0;
  int64_t produced = 0;
  if (seg > 0) {  // the predecessor's state
    // (every lane polls: one lane polling and a shuffle made the compiler
    // precompute the ten round keys into 40 vector registers and spill them)
    const unsigned long long v = mailbox_wait(o + count - 1, seg);
    produced = (int64_t)(v & ((1ULL << NW_CARRY_SHIFT) - 1ULL));
    carry = (int)((v >> NW_CARRY_SHIFT) & 0xffffULL);
  }
  const uint64_t k0 = keys[2 * blockIdx.x], k1 = keys[2 * blockIdx.x + 1];
  // sub-chunks this segment may take (the last one runs to the end of the stream)
  int left = seg == nseg - 1 ? 0x7fffffff : seg_subs;
  const int next_tag = seg == nseg - 1 ? 0 : seg + 1;
  uint32_t m20, e52;  // opaque to the compiler, so they stay in registers (see the transform)
  asm volatile("mov.b32 %0, 0x000FFFFF;" : "=r"(m20));
  asm volatile("mov.b32 %0, 0x43300000;" : "=r"(e52));
  for (uint64_t sub = (uint64_t)seg * (uint64_t)seg_subs; left > 0 && produced < count; ++sub, --left) {
    const uint64_t word0 = (sub * 32 + lane) * NW_WORDS;
    // fast path for every word, branch-free, eight words (two Philox blocks)
    // at a time; the words go to shared memory for the rare-word loop below
    // (which indexes them instead of selecting among registers) and leave
    // the registers
    double x[NW_WORDS];
    uint32_t nf = 0;
#pragma unroll
    for (int g = 0; g < NW_WORDS; g += 8) {
      uint64_t w[8];
      np::philox_block(word0 / 4 + g / 4, k0, k1, w);
      np::philox_block(word0 / 4 + g / 4 + 1, k0, k1, w + 4);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint64_t rw = w[i];
        const ulonglong2 z = zig[rw & 0xff];
        const double wi = __longlong_as_double((long long)z.y);
        // 2^52 + mant, mant = (rw >> 9) & (2^52 - 1): the high half's mask and
        // exponent in one LOP3 (both constants in registers)
        uint32_t dhi;
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(dhi) : "r"((uint32_t)(rw >> 41)), "r"(m20), "r"(e52));
        const double d = __hiloint2double((int)dhi, (int)(uint32_t)(rw >> 9));
        const double v = __fma_rn(d, wi, -0x1.0p52 * wi);
        // sign bit 8 of the word -> sign of the double (one LOP3 on the high half)
        x[g + i] = __hiloint2double(__double2hiint(v) ^ (int)(((uint32_t)rw << 23) & 0x80000000u), __double2loint(v));
        nf |= (d >= __longlong_as_double((long long)z.x) ? 1u : 0u) << (g + i);
      }
      ulonglong2 *row = reinterpret_cast<ulonglong2 *>(&s_w[lane * NW_WORDS + g]);
      row[0] = make_ulonglong2(w[0], w[1]);
      row[1] = make_ulonglong2(w[2], w[3]);
      row[2] = make_ulonglong2(w[4], w[5]);
      row[3] = make_ulonglong2(w[6], w[7]);
    }
    // Rare words (~2.2%, ~0.2 per lane): each lane tests its own non-fast
    // words in order, all lanes together, so the wedge test's arithmetic runs
    // once per round for the warp; a tail token's value replaces the
    // fast-path value in the lane's registers, its length goes to a
    // lane-private slot.
    uint32_t pr = ~nf & NW_ALL, tt = 0;
    if (__any_sync(MMPR_FULL_MASK, nf != 0)) {
      // the last lane's last word: its successor opens the next sub-chunk
      if (lane == 31 && (nf >> (NW_WORDS - 1))) s_w[32 * NW_WORDS] = successor_word(word0 + NW_WORDS, k0, k1);
      __syncwarp();
      for (uint32_t rem = nf; __any_sync(MMPR_FULL_MASK, rem != 0);) {
        if (rem) {
          const int i = __ffs(rem) - 1;
          rem &= rem - 1;
          const uint64_t rw = s_w[lane * NW_WORDS + i];
          const int layer = (int)(rw & 0xff);
          const uint64_t mant = (rw >> 9) & 0x000fffffffffffffULL;
          if (layer != 0) {
            const uint64_t nx = s_w[lane * NW_WORDS + i + 1];
            const double wi = __longlong_as_double((long long)zig[layer].y);
            double v = __fma_rn(__longlong_as_double((long long)(0x4330000000000000ULL | mant)), wi, -0x1.0p52 * wi);
            if ((rw >> 8) & 1) v = -v;
            pr |= (wedge_accepts(layer, v, nx, s_fi) ? 1u : 0u) << i;
          } else {  // tail start: always produces
            int L;
            const double v = tail_token(word0 + i, mant, k0, k1, &L);
#pragma unroll
            for (int k = 0; k < NW_WORDS; ++k) x[k] = (i == k) ? v : x[k];
            s_tlen[lane * NW_WORDS + i] = (uint16_t)L;
            pr |= 1u << i;
            tt |= 1u << i;
          }
        }
      }
    }
    __syncwarp();  // the next sub-chunk overwrites the staged words
    // lane parse from entry 0, then the entries lane to lane.  Exits are 0 or
    // 1 unless a tail token is involved, and an entry of 1 onto a word that
    // starts an attempt in the entry-0 parse only drops word 0 (same
    // boundaries after it, same exit): then one ballot resolves every entry.
    // Anything else (entry onto a consumed word, tails, a long carry) takes
    // the exact stitch loop.
    uint32_t S;
    int ex;
    if (tt == 0) wedge_parse8(nf, 0, S, ex);
    else general_parse8(nf, tt, 0, &s_tlen[lane * NW_WORDS], &S, &ex);
    const uint32_t X = __ballot_sync(MMPR_FULL_MASK, ex != 0);
    const int e1 = lane == 0 ? carry : (int)((X >> ((lane + 31) & 31)) & 1u);
    const bool hard = ex > 1 || e1 > 1 || (e1 == 1 && !((S >> 1) & 1u));
    if (!__any_sync(MMPR_FULL_MASK, hard)) {
      S &= ~(uint32_t)e1;
      carry = (int)(X >> 31);
    } else {
      int ecur = 0;
      for (;;) {
        int e = __shfl_up_sync(MMPR_FULL_MASK, ex, 1);
        if (lane == 0) e = carry;
        bool changed = false;
        if (e != ecur) {
          changed = true;
          if (e >= NW_WORDS) {
            S = 0;
            ex = e - NW_WORDS;
          } else if (ecur == 0 && ((S >> e) & 1u)) {
            S &= ~((1u << e) - 1u);  // same attempt boundaries from e on: same exit
          } else if (tt == 0) {
            wedge_parse8(nf, e, S, ex);
          } else {
            general_parse8(nf, tt, e, &s_tlen[lane * NW_WORDS], &S, &ex);
          }
          ecur = e;
        }
        if (!__any_sync(MMPR_FULL_MASK, changed)) break;
      }
      carry = __shfl_sync(MMPR_FULL_MASK, ex, 31);
    }
    // output offsets: words dropped before this lane, from ballots of the bits of
    // the per-lane dropped count (0..NW_WORDS) instead of a five-step shuffle scan
    const uint32_t O = S & pr;
    const int cnt = __popc(O);
    const uint32_t dr = (uint32_t)(NW_WORDS - cnt);
    const uint32_t lt = (1u << lane) - 1u;
    int dropped_before = 0;
#pragma unroll
    for (int b = 0; (1 << b) <= NW_WORDS; ++b)
      dropped_before += __popc(__ballot_sync(MMPR_FULL_MASK, (dr >> b) & 1u) & lt) << b;
    const int incl = NW_WORDS * lane - dropped_before + cnt;
    const int total = __shfl_sync(MMPR_FULL_MASK, incl, 31);
    const int64_t base = produced + incl - cnt;
    if (produced + 32 * NW_WORDS <= count) {  // warp-uniform: no bound checks in this sub-chunk
      double *dst = o + base;  // produced values are consecutive from base
#pragma unroll
      for (int i = 0; i < NW_WORDS; ++i) {
        const uint32_t take = (O >> i) & 1u;
        if (take) *dst = AFFINE ? add(loc, mul(scale, x[i])) : x[i];
        dst += take;
      }
    } else {
#pragma unroll
      for (int i = 0; i < NW_WORDS; ++i) {
        const int64_t idx = base + __popc(O & ((1u << i) - 1u));
        if (((O >> i) & 1u) && idx < count) o[idx] = AFFINE ? add(loc, mul(scale, x[i])) : x[i];
      }
    }
    produced += total;
  }
  if (next_tag != 0 && lane == 0) {  // hand the stream's state to the next segment
    const unsigned long long v = ((unsigned long long)next_tag << NW_TAG_SHIFT) |
                                 ((unsigned long long)(carry < 0xffff ? carry : 0xffff) << NW_CARRY_SHIFT) |
                                 (unsigned long long)produced;
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(o + count - 1), "l"(v) : "memory");
  }
}

}  // namespace mmpr

using namespace mmpr;

extern "C" int mmpr_noise_keys(uint64_t master_seed, int32_t fresh, int32_t iteration, int32_t n_offset,
                               int32_t n_slices, int32_t steps, uint64_t *keys, void *stream) {
  if (n_slices < 0 || steps < 0 || n_offset < 0 || !keys) return MMPR_ERR_ARG;
  const int64_t total = (int64_t)n_slices * steps;
  if (total == 0) return MMPR_OK;
  const int threads = 128;
  const int64_t blocks = (total + threads - 1) / threads;
  noise_keys_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(master_seed, fresh, iteration,
                                                                           n_offset, n_slices, steps, keys); mmpr_launched();
  return mmpr_check_launch("noise_keys_kernel");
}

extern "C" int mmpr_entropy_key(const uint32_t *words, int32_t n_words, uint64_t *key_dev, void *stream) {
  if (!words || n_words < 1 || n_words > 16 || !key_dev) return MMPR_ERR_ARG;
  EntropyWords e;
  for (int i = 0; i < 16; ++i) e.w[i] = i < n_words ? words[i] : 0u;
  entropy_key_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(e, n_words, key_dev); mmpr_launched();
  return mmpr_check_launch("entropy_key_kernel");
}

extern "C" int mmpr_normals_fill(const uint64_t *keys, int32_t n_streams, int64_t count, double *out,
                                 int64_t pitch, int32_t affine, double loc, double scale, void *stream) {
  if (n_streams < 0 || count < 0 || !keys || !out || (n_streams > 1 && pitch < count)) return MMPR_ERR_ARG;
  if (n_streams == 0 || count == 0) return MMPR_OK;
  if (n_streams >= MMPR_WARP_STREAMS_MIN) {  // one single-warp CTA per (stream, segment)
    static int slots_dev[MMPR_MAX_DEVICES] = {};
    const int dev = mmpr_current_device();
    if (slots_dev[dev] == 0) {
      int sms = 0;
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) sms = 148;
      slots_dev[dev] = NW_MINB * sms;
    }
    // more streams than resident warps, and not so many that the waves are
    // nearly full anyway: eight segments per stream; the segments before the
    // last must not be able to reach the stream's last output slot
    const char *segs_env = getenv("MMPR_NOISE_SEGS");  // A/B and tests: 1 = unsegmented, N = force N segments
    int nseg = segs_env ? atoi(segs_env) : ((n_streams > slots_dev[dev] && n_streams < 8 * slots_dev[dev]) ? 8 : 1);
    if (nseg < 1 || nseg > 64) nseg = 1;
    int seg_subs = 0;
    for (; nseg > 1; --nseg) {
      seg_subs = (int)((count + count / 48) / ((int64_t)(32 * NW_WORDS) * nseg));
      if (seg_subs >= 4 && (int64_t)(nseg - 1) * seg_subs * (32 * NW_WORDS) < count - 1 &&
          (int64_t)nseg * n_streams < (int64_t)INT32_MAX && count < (1LL << NW_CARRY_SHIFT))
        break;
    }
    if (nseg > 1) {
      noise_mailbox_clear_kernel<<<(n_streams + 255) / 256, 256, 0, (cudaStream_t)stream>>>(out, pitch, count,
                                                                                             n_streams); mmpr_launched();
      const int st = mmpr_check_launch("noise_mailbox_clear_kernel");
      if (st != MMPR_OK) return st;
    }
    const dim3 grid((unsigned)n_streams, (unsigned)nseg, 1);
    if (affine) {
      normals_fill_warp_kernel<true><<<grid, 32, 0, (cudaStream_t)stream>>>(keys, count, out, pitch, loc, scale, nseg,
                                                                           seg_subs); mmpr_launched();
    } else {
      normals_fill_warp_kernel<false><<<grid, 32, 0, (cudaStream_t)stream>>>(keys, count, out, pitch, loc, scale, nseg,
                                                                            seg_subs); mmpr_launched();
    }
    return mmpr_check_launch("normals_fill_warp_kernel");
  }
  normals_fill_kernel<<<n_streams, NF_THREADS, 0, (cudaStream_t)stream>>>(keys, count, out, pitch, affine, loc,
                                                                          scale); mmpr_launched();
  return mmpr_check_launch("normals_fill_kernel");
}

namespace mmpr {
__global__ void log1p_kernel(const double *__restrict__ x, double *__restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = np::glibc_log1p(x[i]);
}
}  // namespace mmpr

extern "C" int mmpr_noise_exp_ambiguous(uint64_t *count, int32_t reset) {
  if (!count) return MMPR_ERR_ARG;
  unsigned long long v = 0;
  int st = mmpr_check(cudaMemcpyFromSymbol(&v, g_exp_ambiguous, sizeof v), "exp ambiguity counter");
  if (st != MMPR_OK) return st;
  *count = (uint64_t)v;
  if (reset) {
    v = 0;
    st = mmpr_check(cudaMemcpyToSymbol(g_exp_ambiguous, &v, sizeof v), "exp ambiguity counter");
  }
  return st;
}

extern "C" int mmpr_log1p_libm(const double *x, double *out, int64_t n, void *stream) {
  if (n < 0 || (n > 0 && (!x || !out))) return MMPR_ERR_ARG;
  if (n == 0) return MMPR_OK;
  const int64_t blocks = (n + 255) / 256;
  log1p_kernel<<<(unsigned)(blocks < 4736 ? blocks : 4736), 256, 0, (cudaStream_t)stream>>>(x, out, n); mmpr_launched();
  return mmpr_check_launch("log1p_kernel");
}

namespace mmpr {
__global__ void counter_normals_kernel(const cn::CounterNoise c, uint32_t n, uint32_t j0, int rows, int64_t p0,
                                       int64_t count, double *__restrict__ out, int64_t pitch) {
  __shared__ cn::ZigTables z;
  cn::load_zig(&z, threadIdx.x, blockDim.x);
  __syncthreads();
  const int64_t total = (int64_t)rows * count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / count);
    const int64_t q = i - (int64_t)r * count;
    out[r * pitch + q] = cn::normal(c, (uint32_t)(p0 + q), j0 + (uint32_t)r, n, &z);
  }
}
}  // namespace mmpr

extern "C" int mmpr_counter_normals_fill(const mmpr_counter_noise *noise, int32_t n, int32_t j0, int32_t rows,
                                         int64_t p0, int64_t count, double *out, int64_t pitch, void *stream) {
  if (!noise || n < 0 || n >= (1 << 20) || j0 < 0 || rows < 0 || j0 + rows > (1 << 24) || p0 < 0 || count < 0 ||
      p0 + count > (int64_t)UINT32_MAX || (rows > 1 && pitch < count) || noise->kfield >= (1u << 12))
    return MMPR_ERR_ARG;
  if (rows == 0 || count == 0) return MMPR_OK;
  if (!out) return MMPR_ERR_ARG;
  const cn::CounterNoise c{noise->key[0], 0u, noise->kfield, noise->slice_offset};
  const int64_t total = (int64_t)rows * count;
  const int64_t blocks = (total + 255) / 256;
  counter_normals_kernel<<<(unsigned)(blocks < 4736 ? blocks : 4736), 256, 0, (cudaStream_t)stream>>>(
      c, (uint32_t)n, (uint32_t)j0, rows, p0, count, out, pitch); mmpr_launched();
  return mmpr_check_launch("counter_normals_kernel");
}
