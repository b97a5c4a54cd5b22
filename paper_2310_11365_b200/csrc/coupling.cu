// Restriction and matching operators.
//
// restrict: particles.region_statistics / coupling.restrict
//   (/root/reference/pkg/src/mcparareal/particles.py:176-205,
//    /root/reference/pkg/src/mcparareal/coupling.py:26-29)
// match/lift: coupling.match / coupling.lift
//   (/root/reference/pkg/src/mcparareal/coupling.py:32-95)
//
// Region membership is searchsorted(seps, x, side="right") on the
// pre-transform positions (state.py:73-78).  Each region's members are
// compacted in index order (the array x[idx == i] numpy builds) and reduced
// with numpy's pairwise tree, so means and two-pass variances match
// np.mean/np.var bit for bit.  Matching consumes those same statistics, which
// makes match(restrict(u), u) the bitwise identity exactly as in the
// reference (coupling.py:82-83).
#include <cuda_runtime.h>
#include <stdlib.h>
#include <stdint.h>

#include "mmpr_device.cuh"
#include "capi_internal.h"
#include "fine_common.cuh"
#include "regions.cuh"

namespace mmpr {

#define RS_THREADS 1024
#define RS_MAX_CHUNKS 1024

__device__ __forceinline__ int region_of(const mmpr_partition &part, double v) {
  // number of separatrices <= v; NaN sorts last in numpy (last region)
  if (isnan(v)) return part.n_regions - 1;
  int r = 0;
#pragma unroll
  for (int i = 0; i < MMPR_MAX_REGIONS - 1; ++i)
    if (i < part.n_regions - 1 && part.seps[i] <= v) r = i + 1;
  return r;
}

// numpy pairwise sum of f(a[0..n)) by one 1024-thread CTA (all threads get
// the result).  mode 0: f = identity; mode 1: f(v) = (v - m)^2.
__device__ double cta_pairwise_sum(const double *__restrict__ a, int64_t n, int mode, double m, PwVal *s_wp,
                                   PwVal *s_chunk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int D = pw_depth(n);
  const int64_t nslots = int64_t(1) << D;
  const int64_t chunks = nslots > 128 ? nslots / 128 : 1;
  for (int64_t c = 0; c < chunks; ++c) {
    const int64_t s = c * 128 + (tid >> 3);
    const int j8 = tid & 7;
    int64_t off = 0, len = 0;
    if (s < nslots) pw_leaf(n, D, s, &off, &len);
    const int64_t cnt = len >> 3;
    double acc = 0.0;
    if (cnt > 0) {
      double v = a[off + j8];
      acc = mode ? mul(sub(v, m), sub(v, m)) : v;
      for (int64_t k = 1; k < cnt; ++k) {
        v = a[off + j8 + 8 * k];
        acc = add(acc, mode ? mul(sub(v, m), sub(v, m)) : v);
      }
    }
    // every lane of the group holds an equal cnt, so the shuffles are uniform
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 1));
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 2));
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 4));
    if (cnt == 0) acc = 0.0;
    for (int64_t i = cnt * 8; i < len; ++i) {
      const double v = a[off + i];
      acc = add(acc, mode ? mul(sub(v, m), sub(v, m)) : v);
    }
    PwVal leaf;
    leaf.v = acc;
    leaf.ok = len > 0;
    leaf = pw_xor_level(leaf, lane, 8);
    leaf = pw_xor_level(leaf, lane, 16);
    if (lane == 0) s_wp[warp] = leaf;
    __syncthreads();
    if (warp == 0) {
      PwVal v = s_wp[lane];
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) v = pw_xor_level(v, lane, k);
      if (lane == 0) s_chunk[c] = v;
    }
    __syncthreads();
  }
  if (tid == 0) {
    for (int64_t w = 1; w < chunks; w <<= 1)
      for (int64_t q = 0; q + w < chunks; q += 2 * w) s_chunk[q] = pw_combine(s_chunk[q], s_chunk[q + w]);
  }
  __syncthreads();
  const double r = s_chunk[0].v;
  __syncthreads();
  return r;
}

struct RestrictParams {
  mmpr_partition part;
  int n_ens;
  int64_t P;
  const double *x;
  int64_t pitch;
  double *stats;
  int64_t *counts;
  double *scratch;
};

__global__ void __launch_bounds__(RS_THREADS) restrict_kernel(const RestrictParams p) {
  __shared__ PwVal s_wp[32];
  __shared__ PwVal s_chunk[RS_MAX_CHUNKS];
  __shared__ int s_wcnt[MMPR_MAX_REGIONS][32];
  __shared__ int64_t s_total[MMPR_MAX_REGIONS];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int e = blockIdx.x;
  const int I = p.part.n_regions;
  const double *x = p.x + (int64_t)e * p.pitch;
  double *st = p.stats + (int64_t)e * 3 * I;

  int64_t count[MMPR_MAX_REGIONS];
  const double *members[MMPR_MAX_REGIONS];
  if (I == 1) {
    count[0] = p.P;
    members[0] = x;
  } else {
    double *scr = p.scratch + (int64_t)e * I * p.P;
    if (tid < MMPR_MAX_REGIONS) s_total[tid] = 0;
    __syncthreads();
    for (int64_t base = 0; base < p.P; base += RS_THREADS) {
      const int64_t i = base + tid;
      double v = 0.0;
      int r = -1;
      if (i < p.P) {
        v = x[i];
        r = region_of(p.part, v);
      }
      int myrank = 0;
      for (int q = 0; q < I; ++q) {
        const unsigned b = __ballot_sync(MMPR_FULL_MASK, r == q);
        if (r == q) myrank = __popc(b & ((1u << lane) - 1u));
        if (lane == 0) s_wcnt[q][warp] = __popc(b);
      }
      __syncthreads();
      if (r >= 0) {
        int64_t off = s_total[r];
        for (int w = 0; w < warp; ++w) off += s_wcnt[r][w];
        scr[(int64_t)r * p.P + off + myrank] = v;
      }
      __syncthreads();
      if (tid < I) {
        int64_t t = 0;
        for (int w = 0; w < 32; ++w) t += s_wcnt[tid][w];
        s_total[tid] += t;
      }
      __syncthreads();
    }
    for (int q = 0; q < I; ++q) {
      count[q] = s_total[q];
      members[q] = scr + (int64_t)q * p.P;
    }
    __syncthreads();
  }

  for (int q = 0; q < I; ++q) {
    const int64_t n = count[q];
    double mean, var;
    if (n == 0) {
      mean = p.part.centers[q];
      var = 0.0;
    } else if (n == 1) {
      mean = members[q][0];
      var = 0.0;
    } else {
      const double sum = cta_pairwise_sum(members[q], n, 0, 0.0, s_wp, s_chunk);
      mean = div(sum, (double)n);
      const double ss = cta_pairwise_sum(members[q], n, 1, mean, s_wp, s_chunk);
      var = div(ss, (double)n);
    }
    if (tid == 0) {
      st[q] = mean;
      st[I + q] = var;
      st[2 * I + q] = div((double)n, (double)p.P);
      if (p.counts) p.counts[(int64_t)e * I + q] = n;
    }
  }
}

// ---------------------------------------------------------------------------
// multi-region restriction spread over the whole GPU (I > 1)
// ---------------------------------------------------------------------------
// The one-CTA-per-ensemble kernel above compacts and reduces every ensemble
// serially; with 32 ensembles of 1e5 (config 3) or 2^20 (config 5) particles
// that leaves most SMs idle.  Same arithmetic, four stages:
//   count   : members per region in each 4096-particle chunk (many CTAs)
//   scatter : stable compaction of each chunk's members to the region arrays
//             at the chunk's exclusive offsets (index order kept)
//   partial : the pairwise tree of each region array cut into 128-slot
//             subtrees, one CTA each (sum, or sum of (x - mean)^2)
//   finish  : one warp per (ensemble, region) folds the subtree partials in
//             tree order -> mean, then variance
#define RM_CHUNK 4096
#define RM_THREADS 256
#define RM_SLOTS 128

__host__ __device__ inline int64_t rm_chunks(int64_t P) { return (P + RM_CHUNK - 1) / RM_CHUNK; }
__host__ __device__ inline int64_t rm_subtrees(int64_t n) {
  const int64_t nslots = int64_t(1) << pw_depth(n < 1 ? 1 : n);
  return nslots > RM_SLOTS ? nslots / RM_SLOTS : 1;
}

struct RmLayout {  // carved from the caller's scratch (doubles)
  double *members;       // [E][I][P]
  int64_t *blk_counts;   // [E][B][I]
  PwVal *partials;       // [E][I][maxsub]
  double *means;         // [E][I]
  int64_t B, maxsub;
};

__host__ __device__ inline int64_t rm_scratch_doubles(int64_t E, int64_t P, int I) {
  const int64_t B = rm_chunks(P), maxsub = rm_subtrees(P);
  return E * I * P + E * B * I + 2 * E * I * maxsub + E * I;
}

static RmLayout rm_layout(double *scratch, int64_t E, int64_t P, int I) {
  RmLayout L;
  L.B = rm_chunks(P);
  L.maxsub = rm_subtrees(P);
  L.members = scratch;
  L.blk_counts = reinterpret_cast<int64_t *>(scratch + E * I * P);
  L.partials = reinterpret_cast<PwVal *>(scratch + E * I * P + E * L.B * I);
  L.means = scratch + E * I * P + E * L.B * I + 2 * E * I * L.maxsub;
  return L;
}

__global__ void __launch_bounds__(RM_THREADS) rm_count_kernel(mmpr_partition part, int64_t P, const double *x,
                                                             int64_t pitch, RmLayout L) {
  __shared__ int s_cnt[MMPR_MAX_REGIONS];
  const int64_t b = blockIdx.x, e = blockIdx.y;
  const int I = part.n_regions;
  if (threadIdx.x < MMPR_MAX_REGIONS) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const double *xe = x + e * pitch;
  const int64_t lo = b * RM_CHUNK, hi = min(P, lo + RM_CHUNK);
  int c[MMPR_MAX_REGIONS] = {0, 0, 0, 0};
  for (int64_t i = lo + threadIdx.x; i < hi; i += RM_THREADS) {
    const int r = region_of(part, xe[i]);
#pragma unroll
    for (int q = 0; q < MMPR_MAX_REGIONS; ++q) c[q] += (r == q);
  }
  for (int q = 0; q < I; ++q) {
    int v = c[q];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(MMPR_FULL_MASK, v, m);
    if ((threadIdx.x & 31) == 0) atomicAdd(&s_cnt[q], v);
  }
  __syncthreads();
  if (threadIdx.x < I) L.blk_counts[(e * L.B + b) * I + threadIdx.x] = s_cnt[threadIdx.x];
}

__global__ void __launch_bounds__(RM_THREADS) rm_scatter_kernel(mmpr_partition part, int64_t P, const double *x,
                                                               int64_t pitch, RmLayout L, int64_t *counts_out) {
  __shared__ int64_t s_off[MMPR_MAX_REGIONS];
  __shared__ int s_wcnt[MMPR_MAX_REGIONS][RM_THREADS / 32];
  const int64_t b = blockIdx.x, e = blockIdx.y;
  const int I = part.n_regions;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < I) {  // exclusive offset of this chunk, and (last chunk) the totals
    int64_t off = 0, tot = 0;
    for (int64_t bb = 0; bb < L.B; ++bb) {
      const int64_t v = L.blk_counts[(e * L.B + bb) * I + threadIdx.x];
      if (bb < b) off += v;
      tot += v;
    }
    s_off[threadIdx.x] = off;
    if (b == 0 && counts_out) counts_out[e * I + threadIdx.x] = tot;
  }
  __syncthreads();
  const double *xe = x + e * pitch;
  const int64_t lo = b * RM_CHUNK, hi = min(P, lo + RM_CHUNK);
  for (int64_t base = lo; base < hi; base += RM_THREADS) {  // tiles in index order
    const int64_t i = base + threadIdx.x;
    double v = 0.0;
    int r = -1;
    if (i < hi) {
      v = xe[i];
      r = region_of(part, v);
    }
    int myrank = 0;
    for (int q = 0; q < I; ++q) {
      const unsigned bal = __ballot_sync(MMPR_FULL_MASK, r == q);
      if (r == q) myrank = __popc(bal & ((1u << lane) - 1u));
      if (lane == 0) s_wcnt[q][warp] = __popc(bal);
    }
    __syncthreads();
    if (r >= 0) {
      int64_t pos = s_off[r] + myrank;
      for (int w = 0; w < warp; ++w) pos += s_wcnt[r][w];
      L.members[(e * I + r) * P + pos] = v;
    }
    __syncthreads();
    if (threadIdx.x < I) {
      int64_t t = 0;
      for (int w = 0; w < RM_THREADS / 32; ++w) t += s_wcnt[threadIdx.x][w];
      s_off[threadIdx.x] += t;
    }
    __syncthreads();
  }
}

// subtree c (RM_SLOTS leaf slots) of the pairwise tree of region array (e, r)
__global__ void __launch_bounds__(1024) rm_partial_kernel(int I, int64_t P, const int64_t *counts, RmLayout L,
                                                          int squares) {
  __shared__ PwVal s_wp[32];
  const int64_t c = blockIdx.x;
  const int r = blockIdx.y;
  const int64_t e = blockIdx.z;
  const int64_t n = counts[e * I + r];
  if (n < 2 || c >= rm_subtrees(n)) return;  // n < 2: special-cased by the finisher
  const int D = pw_depth(n);
  const int64_t nslots = int64_t(1) << D;
  const double *a = L.members + (e * I + r) * P;
  const double m = squares ? L.means[e * I + r] : 0.0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t s = c * RM_SLOTS + (tid >> 3);
  const int j8 = tid & 7;
  int64_t off = 0, len = 0;
  if (s < nslots) pw_leaf(n, D, s, &off, &len);
  auto f = [&](double v) { return squares ? mul(sub(v, m), sub(v, m)) : v; };
  const int64_t cnt = len >> 3;
  double acc = 0.0;
  if (cnt > 0) {
    acc = f(a[off + j8]);
    for (int64_t k = 1; k < cnt; ++k) acc = add(acc, f(a[off + j8 + 8 * k]));
  }
  acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 1));
  acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 2));
  acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 4));
  if (cnt == 0) acc = 0.0;
  for (int64_t i = cnt * 8; i < len; ++i) acc = add(acc, f(a[off + i]));
  PwVal leaf;
  leaf.v = acc;
  leaf.ok = len > 0;
  leaf = pw_xor_level(leaf, lane, 8);
  leaf = pw_xor_level(leaf, lane, 16);
  if (lane == 0) s_wp[warp] = leaf;
  __syncthreads();
  if (warp == 0) {
    PwVal v = s_wp[lane];
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) v = pw_xor_level(v, lane, k);
    if (lane == 0) L.partials[(e * I + r) * L.maxsub + c] = v;
  }
}

// one thread per (ensemble, region): fold the subtree partials in tree order
__global__ void rm_finish_kernel(mmpr_partition part, int E, int64_t P, const int64_t *counts, RmLayout L,
                                 double *stats, int squares) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int I = part.n_regions;
  if (g >= (int64_t)E * I) return;
  const int64_t e = g / I;
  const int r = (int)(g - e * I);
  const int64_t n = counts[e * I + r];
  double *st = stats + e * 3 * I;
  const double *a = L.members + (e * I + r) * P;
  if (n < 2) {  // empty: center, 0; one member: x, 0 (particles.py:192-199)
    if (!squares) {
      st[r] = n == 0 ? part.centers[r] : a[0];
      st[2 * I + r] = div((double)n, (double)P);
      L.means[e * I + r] = st[r];
    } else {
      st[I + r] = 0.0;
    }
    return;
  }
  const int64_t k = rm_subtrees(n);
  const PwVal *pp = L.partials + (e * I + r) * L.maxsub;
  PwVal stk[17];
  PwVal cur = pp[0];
  for (int64_t i = 0; i < k; ++i) {  // binary-counter fold: ((p0+p1)+(p2+p3))+...
    cur = pp[i];
    int l = 0;
    for (; (i >> l) & 1; ++l) cur = pw_combine(stk[l], cur);
    stk[l] = cur;
  }
  int L2 = 0;
  while ((int64_t(1) << L2) < k) ++L2;
  const double total = stk[L2].v;
  if (!squares) {
    const double mean = div(total, (double)n);
    st[r] = mean;
    st[2 * I + r] = div((double)n, (double)P);
    L.means[e * I + r] = mean;
  } else {
    st[I + r] = div(total, (double)n);
  }
}

static int restrict_multi(const mmpr_partition &part, int32_t n_ens, int64_t P, const double *x, int64_t pitch,
                          double *stats, int64_t *counts, double *scratch, cudaStream_t st) {
  const int I = part.n_regions;
  RmLayout L = rm_layout(scratch, n_ens, P, I);
  int64_t *cnt = counts;  // the finisher needs the totals even when the caller passes none
  if (!cnt) return MMPR_ERR_ARG;
  const dim3 g1((unsigned)L.B, (unsigned)n_ens);
  rm_count_kernel<<<g1, RM_THREADS, 0, st>>>(part, P, x, pitch, L); mmpr_launched();
  rm_scatter_kernel<<<g1, RM_THREADS, 0, st>>>(part, P, x, pitch, L, cnt); mmpr_launched();
  const dim3 g3((unsigned)L.maxsub, (unsigned)I, (unsigned)n_ens);
  const int fin_blocks = (int)((n_ens * I + 127) / 128);
  for (int squares = 0; squares < 2; ++squares) {
    rm_partial_kernel<<<g3, 1024, 0, st>>>(I, P, cnt, L, squares); mmpr_launched();
    rm_finish_kernel<<<fin_blocks, 128, 0, st>>>(part, n_ens, P, cnt, L, stats, squares); mmpr_launched();
  }
  return mmpr_check_launch("restrict_multi");
}

// ---------------------------------------------------------------------------
// match
// ---------------------------------------------------------------------------
#define MT_THREADS 256
#define MT_PER_THREAD 8

struct MatchParams {
  mmpr_partition part;
  int n_ens;
  int64_t P;
  const double *targets;
  int64_t tgt_stride;
  const double *cur;
  int64_t cur_stride;
  const int64_t *counts;
  int64_t cnt_stride;
  const double *x_src;
  int64_t src_pitch;
  double *x_out;
  int64_t out_pitch;
  int policy;  // 0 raise, 1 collapse
  int32_t *status;
  int32_t *clamped;
  int chunks_per_ens;
};

enum { MATCH_KEEP = 0, MATCH_SET = 1, MATCH_AFFINE = 2 };

__global__ void __launch_bounds__(MT_THREADS) match_kernel(const MatchParams p) {
  __shared__ int s_mode[MMPR_MAX_REGIONS];
  __shared__ double s_scale[MMPR_MAX_REGIONS], s_m[MMPR_MAX_REGIONS], s_mu[MMPR_MAX_REGIONS];
  const int e = blockIdx.x / p.chunks_per_ens;
  const int chunk = blockIdx.x % p.chunks_per_ens;
  const int I = p.part.n_regions;
  if (threadIdx.x == 0) {
    const double *tg = p.targets + (int64_t)e * p.tgt_stride;
    const double *cs = p.cur + (int64_t)e * p.cur_stride;
    const int64_t *cn = p.counts + (int64_t)e * p.cnt_stride;
    int status = MMPR_STAT_OK, clamped = 0;
    for (int q = 0; q < I; ++q) {
      s_mode[q] = MATCH_KEEP;
      if (cn[q] == 0) continue;  // empty region: skipped
      const double mu_t = tg[q];
      double var_t = tg[I + q];
      if (var_t < 0.0) {
        clamped |= 1 << q;
        var_t = 0.0;
      }
      const double cur_mean = cs[q], cur_var = cs[I + q];
      if (cur_var == 0.0) {
        if (var_t > 0.0 && p.policy == 0 && status == MMPR_STAT_OK) status = q;
        s_mode[q] = MATCH_SET;
        s_mu[q] = mu_t;
        continue;
      }
      const double scale = __dsqrt_rn(div(var_t, cur_var));
      if (scale == 1.0 && mu_t == cur_mean) continue;  // exact identity keeps bits
      s_mode[q] = MATCH_AFFINE;
      s_scale[q] = scale;
      s_m[q] = cur_mean;
      s_mu[q] = mu_t;
    }
    if (chunk == 0) {
      p.status[e] = status;
      if (p.clamped) p.clamped[e] = clamped;
    }
  }
  __syncthreads();
  const double *src = p.x_src + (int64_t)e * p.src_pitch;
  double *dst = p.x_out + (int64_t)e * p.out_pitch;
  const int64_t base = (int64_t)chunk * MT_THREADS * MT_PER_THREAD;
#pragma unroll
  for (int k = 0; k < MT_PER_THREAD; ++k) {
    const int64_t i = base + (int64_t)k * MT_THREADS + threadIdx.x;
    if (i < p.P) {
      const double v = src[i];
      const int r = region_of(p.part, v);
      const int mode = s_mode[r];
      double o = v;
      if (mode == MATCH_SET) o = s_mu[r];
      else if (mode == MATCH_AFFINE) o = add(mul(s_scale[r], sub(v, s_m[r])), s_mu[r]);
      dst[i] = o;
    }
  }
}

}  // namespace mmpr

using namespace mmpr;

extern "C" int mmpr_restrict(const mmpr_partition *part, int32_t n_ens, int64_t particles, const double *x,
                             int64_t pitch, double *stats, int64_t *counts, double *scratch, void *stream) {
  if (!part || n_ens < 0 || particles < 1 || !x || !stats) return MMPR_ERR_ARG;
  if (part->n_regions < 1 || part->n_regions > MMPR_MAX_REGIONS) return MMPR_ERR_ARG;
  if (part->n_regions > 1 && !scratch) return MMPR_ERR_ARG;
  if (n_ens == 0) return MMPR_OK;
  if (part->n_regions == 1) {
    const int st = restrict_single_region(n_ens, particles, x, pitch, stats, counts, (cudaStream_t)stream);
    if (st != MMPR_ERR_UNSUPPORTED) return st;
  }
  // one cluster per ensemble (restrict_regions.cu) only on request: the
  // multi-kernel passes below are faster on the BASELINE bimodal shapes
  const char *cl_env = getenv("MMPR_RESTRICT_CLUSTER");
  if (part->n_regions > 1 && counts && cl_env && atoi(cl_env) == 1) {
    RegionsParams rp = {};
    rp.part = *part;
    rp.P = particles;
    rp.x = x;
    rp.pitch = pitch;
    rp.stats = stats;
    rp.counts = counts;
    rp.scratch = scratch;  // [n_ens][I][P] leads the multi-kernel scratch layout
    const int st = restrict_regions(rp, n_ens, false, (cudaStream_t)stream);
    if (st != MMPR_ERR_UNSUPPORTED) return st;
  }
  if (part->n_regions > 1 && counts && rm_chunks(particles) <= 65535 && rm_subtrees(particles) <= 65535)
    return restrict_multi(*part, n_ens, particles, x, pitch, stats, counts, scratch, (cudaStream_t)stream);
  const int D = pw_depth(particles);
  if (D > 7 && ((int64_t(1) << D) / 128) > RS_MAX_CHUNKS) return MMPR_ERR_UNSUPPORTED;
  RestrictParams p;
  p.part = *part;
  p.n_ens = n_ens;
  p.P = particles;
  p.x = x;
  p.pitch = pitch;
  p.stats = stats;
  p.counts = counts;
  p.scratch = scratch;
  restrict_kernel<<<n_ens, RS_THREADS, 0, (cudaStream_t)stream>>>(p); mmpr_launched();
  return mmpr_check_launch("restrict_kernel");
}

extern "C" int mmpr_match(const mmpr_partition *part, int32_t n_ens, int64_t particles, const double *targets,
                          int64_t tgt_stride, const double *cur_stats, int64_t cur_stride,
                          const int64_t *cur_counts, int64_t cnt_stride, const double *x_src, int64_t src_pitch,
                          double *x_out, int64_t out_pitch, int32_t policy, int32_t *status, int32_t *clamped,
                          void *stream) {
  if (!part || n_ens < 0 || particles < 1 || !targets || !cur_stats || !cur_counts || !x_src || !x_out ||
      !status || (policy != 0 && policy != 1))
    return MMPR_ERR_ARG;
  if (part->n_regions < 1 || part->n_regions > MMPR_MAX_REGIONS) return MMPR_ERR_ARG;
  if (n_ens == 0) return MMPR_OK;
  MatchParams p;
  p.part = *part;
  p.n_ens = n_ens;
  p.P = particles;
  p.targets = targets;
  p.tgt_stride = tgt_stride;
  p.cur = cur_stats;
  p.cur_stride = cur_stride;
  p.counts = cur_counts;
  p.cnt_stride = cnt_stride;
  p.x_src = x_src;
  p.src_pitch = src_pitch;
  p.x_out = x_out;
  p.out_pitch = out_pitch;
  p.policy = policy;
  p.status = status;
  p.clamped = clamped;
  const int64_t per_cta = (int64_t)MT_THREADS * MT_PER_THREAD;
  p.chunks_per_ens = (int)((particles + per_cta - 1) / per_cta);
  const int64_t grid = (int64_t)n_ens * p.chunks_per_ens;
  if (grid > 0x7fffffff) return MMPR_ERR_UNSUPPORTED;
  match_kernel<<<(unsigned)grid, MT_THREADS, 0, (cudaStream_t)stream>>>(p); mmpr_launched();
  return mmpr_check_launch("match_kernel");
}

extern "C" int64_t mmpr_restrict_scratch_doubles(int32_t n_ens, int64_t particles, int32_t n_regions) {
  if (n_regions <= 1) return 0;
  return mmpr::rm_scratch_doubles(n_ens, particles, n_regions);
}
