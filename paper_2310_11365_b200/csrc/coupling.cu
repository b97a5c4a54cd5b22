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
#include <stdint.h>

#include "mmpr_device.cuh"
#include "capi_internal.h"
#include "fine_common.cuh"

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
  restrict_kernel<<<n_ens, RS_THREADS, 0, (cudaStream_t)stream>>>(p);
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
  match_kernel<<<(unsigned)grid, MT_THREADS, 0, (cudaStream_t)stream>>>(p);
  return mmpr_check_launch("match_kernel");
}
