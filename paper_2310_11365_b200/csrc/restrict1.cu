// Single-region restriction (the unimodal configs): mean, population
// variance and fraction of every ensemble with one thread-block cluster per
// ensemble.
//
// Same arithmetic as restrict_kernel in coupling.cu -- np.mean and the
// two-pass np.var over numpy's pairwise tree (particles.py:176-205,
// coupling.py:26-29) -- but the ensemble is spread over up to 16 CTAs with
// the same leaf-slot layout as the fine sweep (fine.cu): every lane loads
// its leaf elements once into registers, the first pass yields the mean, the
// second pass folds (x - mean)^2 from the same registers, and the CTA
// partials of each pass meet in every CTA through distributed shared memory.
// One HBM read of the ensemble instead of two, and all SMs busy instead of
// one CTA per ensemble.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "capi_internal.h"
#include "fine_common.cuh"
#include "mmpr_device.cuh"

namespace mmpr {

struct Restrict1Params {
  int64_t P;
  const double *x;
  int64_t pitch;
  double *stats;    // [n_ens][3]: mean, var, fraction
  int64_t *counts;  // [n_ens] or NULL
  int D;
  int slots_per_cta;
  int ctas;
  // match prologue (MATCH kernels): x_out = match(target, x) then restrict(x_out)
  const double *targets;
  int64_t tgt_stride;
  const double *cur;
  int64_t cur_stride;
  const int64_t *cur_counts;
  int64_t cnt_stride;
  double *x_out;
  int64_t out_pitch;
  int policy;  // 0 raise, 1 collapse
  int32_t *status;
  int32_t *clamped;
};

enum { R1_KEEP = 0, R1_SET = 1, R1_AFFINE = 2 };

template <int PPT, bool HAS_TAIL, bool PADDED, bool MATCH>
__global__ void __launch_bounds__(1024, 1) restrict1_kernel(const Restrict1Params p) {
  using PartT = Part<PADDED>;
  __shared__ PartT s_wp[32];
  __shared__ __align__(16) ClusterSlot s_slot[2][FS_MAX_CLUSTER];
  __shared__ double s_total[2];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = (int)blockDim.x >> 5;
  const int rank = p.ctas > 1 ? (int)cluster_ctarank() : 0;
  const int e = (int)blockIdx.x / p.ctas;
  const int64_t nslots = int64_t(1) << p.D;
  const int64_t slot = (int64_t)rank * p.slots_per_cta + warp * 4 + (lane >> 3);
  const int j8 = lane & 7;
  int64_t off = 0, len = 0;
  if (slot < nslots) pw_leaf(p.P, p.D, slot, &off, &len);
  const int cnt = (int)(len >> 3);
  const int tail = (int)(len & 7);
  const bool slot_ok = len > 0;

  const double *xs = p.x + (int64_t)e * p.pitch;
  double x[PPT];
  double xt = 0.0;
#pragma unroll
  for (int m = 0; m < PPT; ++m) x[m] = (m < cnt) ? xs[off + j8 + 8 * m] : 0.0;
  if (HAS_TAIL && j8 < tail) xt = xs[off + 8 * cnt + j8];
  if constexpr (MATCH) {
    // single-region match (coupling.py:32-95; same rules as match_kernel in
    // coupling.cu), evaluated redundantly by every thread from broadcast loads
    const double *tg = p.targets + (int64_t)e * p.tgt_stride;
    const double *cs = p.cur + (int64_t)e * p.cur_stride;
    const int64_t cn = p.cur_counts[(int64_t)e * p.cnt_stride];
    int mode = R1_KEEP, status = MMPR_STAT_OK, clamped = 0;
    double scale = 1.0, mc = 0.0, mu = 0.0;
    if (cn != 0) {
      mu = tg[0];
      double var_t = tg[1];
      if (var_t < 0.0) {
        clamped = 1;
        var_t = 0.0;
      }
      mc = cs[0];
      const double cur_var = cs[1];
      if (cur_var == 0.0) {
        if (var_t > 0.0 && p.policy == 0) status = 0;
        mode = R1_SET;
      } else {
        scale = __dsqrt_rn(div(var_t, cur_var));
        if (!(scale == 1.0 && mu == mc)) mode = R1_AFFINE;  // exact identity keeps bits
      }
    }
    auto apply = [&](double v) {
      return mode == R1_SET ? mu : (mode == R1_AFFINE ? add(mul(scale, sub(v, mc)), mu) : v);
    };
#pragma unroll
    for (int m = 0; m < PPT; ++m) x[m] = apply(x[m]);
    if (HAS_TAIL) xt = apply(xt);
    double *xo = p.x_out + (int64_t)e * p.out_pitch;
#pragma unroll
    for (int m = 0; m < PPT; ++m)
      if (m < cnt) xo[off + j8 + 8 * m] = x[m];
    if (HAS_TAIL && j8 < tail) xo[off + 8 * cnt + j8] = xt;
    if (rank == 0 && tid == 0) {
      p.status[e] = status;
      if (p.clamped) p.clamped[e] = clamped;
    }
  }
  // peers' shared memory is written below: every CTA of the cluster must run
  if (p.ctas > 1) cluster_sync_all();

  // pass 0: sum(x); pass 1: sum((x - mean)^2), both in pairwise order
  double mean = 0.0;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    auto f = [&](double v) { return pass ? mul(sub(v, mean), sub(v, mean)) : v; };
    double acc = f(x[0]);
#pragma unroll
    for (int m = 1; m < PPT; ++m) {
      const double t = add(acc, f(x[m]));
      acc = (m < cnt) ? t : acc;
    }
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 1));
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 2));
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 4));
    if (cnt == 0) acc = 0.0;
    if (HAS_TAIL) {
      const double ft = f(xt);
#pragma unroll
      for (int i = 0; i < 7; ++i) {
        const double v = __shfl_sync(MMPR_FULL_MASK, ft, (lane & ~7) | i);
        if (i < tail) acc = add(acc, v);
      }
    }
    PartT leaf = PartT::make(acc, slot_ok);
    leaf = leaf.xor_level(lane, 8);
    leaf = leaf.xor_level(lane, 16);
    if (lane == 0) s_wp[warp] = leaf;
    __syncthreads();
    if (warp == 0) {
      PartT v = (lane < nwarps) ? s_wp[lane] : PartT::make(0.0, false);
#pragma unroll
      for (int m = 1; m < 32; m <<= 1)
        if (m < nwarps) v = v.xor_level(lane, m);
      if (p.ctas > 1) {
        if (lane < p.ctas) {
          int okv = 1;
          if constexpr (PADDED) okv = v.ok;
          st_cluster_v2(mapa_shared(smem_addr(&s_slot[pass][rank]), (uint32_t)lane),
                        (unsigned long long)__double_as_longlong(v.v), (unsigned long long)(uint32_t)okv);
        }
      } else if (lane == 0) {
        s_total[pass] = v.v;
      }
    }
    if (p.ctas > 1) {
      cluster_sync_all();
      if (warp == 0) {
        PartT c = (lane < p.ctas) ? PartT::make(s_slot[pass][lane].v, s_slot[pass][lane].ok != 0)
                                  : PartT::make(0.0, false);
#pragma unroll
        for (int m = 1; m < FS_MAX_CLUSTER; m <<= 1)
          if (m < p.ctas) c = c.xor_level(lane, m);
        if (lane == 0) s_total[pass] = c.v;
      }
    }
    __syncthreads();
    if (pass == 0) mean = div(s_total[0], (double)p.P);
  }
  if (tid == 0 && rank == 0) {
    double *st = p.stats + (int64_t)e * 3;
    double m = mean, var = div(s_total[1], (double)p.P);
    if (p.P == 1) {  // one member: M = x, S = 0 (particles.py:196-199); thread 0 holds it
      m = HAS_TAIL ? xt : x[0];
      var = 0.0;
    }
    st[0] = m;
    st[1] = var;
    st[2] = div((double)p.P, (double)p.P);
    if (p.counts) p.counts[e] = p.P;
  }
}

template <void (*KERN)(const Restrict1Params)>
static int launch_r1(const Restrict1Params &p, int n_ens, int threads, cudaStream_t stream);

// cluster geometry of one particle count (cached per host thread)
struct R1Geometry {
  int D, spc, ctas, ppt;
  bool padded;
};

static const R1Geometry &r1_geometry(int64_t P) {
  thread_local int64_t last_P = -1;
  thread_local R1Geometry g;
  if (P != last_P) {
    const int D = pw_depth(P);
    const int64_t nslots = int64_t(1) << D;
    int64_t max_leaf = 0;
    bool empty = false;
    for (int64_t s = 0; s < nslots; ++s) {
      int64_t o, l;
      pw_leaf(P, D, s, &o, &l);
      if (l > max_leaf) max_leaf = l;
      empty |= l == 0;
    }
    // 512-thread CTAs (two per SM, 16 per cluster) when the ensemble fills
    // exactly 1024 slots (P ~ 1e5), as in the fine sweep; else 1024 threads
    int spc = nslots < 128 ? (nslots < 4 ? 4 : (int)nslots) : 128;
    if (nslots == 1024) spc = 64;  // 51 vs 58 us per 64 x 1e5 fused match-restrict
    g.D = D;
    g.spc = spc;
    g.ctas = nslots <= spc ? 1 : (int)(nslots / spc);
    g.ppt = (int)((max_leaf + 7) / 8);
    g.padded = empty || nslots < spc;
    last_P = P;
  }
  return g;
}

template <bool MATCH>
static int launch_r1_shape(Restrict1Params p, int n_ens, cudaStream_t stream) {
  const R1Geometry &g = r1_geometry(p.P);
  if (g.ctas > FS_MAX_CLUSTER || g.ppt > 16) return MMPR_ERR_UNSUPPORTED;
  p.D = g.D;
  p.slots_per_cta = g.spc;
  p.ctas = g.ctas;
  const int threads = g.spc * 8;
  const bool tail = (p.P % 8) != 0;
  if (g.padded) {
    if (tail) return launch_r1<restrict1_kernel<16, true, true, MATCH>>(p, n_ens, threads, stream);
    return launch_r1<restrict1_kernel<16, false, true, MATCH>>(p, n_ens, threads, stream);
  }
  if (tail) return launch_r1<restrict1_kernel<16, true, false, MATCH>>(p, n_ens, threads, stream);
  return launch_r1<restrict1_kernel<16, false, false, MATCH>>(p, n_ens, threads, stream);
}

template <void (*KERN)(const Restrict1Params)>
static int launch_r1(const Restrict1Params &p, int n_ens, int threads, cudaStream_t stream) {
  static bool configured_dev[MMPR_MAX_DEVICES] = {};
  bool &configured = configured_dev[mmpr_current_device()];
  cudaError_t err;
  if (p.ctas > 8 && !configured) {
    err = cudaFuncSetAttribute(KERN, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return mmpr_check(err, "restrict1: non-portable cluster");
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_ens * p.ctas), 1, 1);
  cfg.blockDim = dim3((unsigned)threads, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)p.ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  err = cudaLaunchKernelEx(&cfg, KERN, p);
  if (err == cudaSuccess) mmpr_launched();
  return mmpr_check(err, "restrict1_kernel launch");
}

// Returns MMPR_ERR_UNSUPPORTED when the ensemble does not fit one cluster
// (the caller then uses the one-CTA-per-ensemble kernel).
int restrict_single_region(int n_ens, int64_t P, const double *x, int64_t pitch, double *stats, int64_t *counts,
                           cudaStream_t stream) {
  Restrict1Params p = {};
  p.P = P;
  p.x = x;
  p.pitch = pitch;
  p.stats = stats;
  p.counts = counts;
  return launch_r1_shape<false>(p, n_ens, stream);
}

}  // namespace mmpr

using namespace mmpr;

extern "C" int mmpr_match_restrict(int32_t n_ens, int64_t particles, const double *targets, int64_t tgt_stride,
                                   const double *cur_stats, int64_t cur_stride, const int64_t *cur_counts,
                                   int64_t cnt_stride, const double *x_src, int64_t src_pitch, double *x_out,
                                   int64_t out_pitch, int32_t policy, int32_t *status, int32_t *clamped,
                                   double *stats, int64_t *counts, void *stream) {
  if (n_ens < 0 || particles < 1 || !targets || !cur_stats || !cur_counts || !x_src || !x_out || !status ||
      !stats || (policy != 0 && policy != 1))
    return MMPR_ERR_ARG;
  if (n_ens == 0) return MMPR_OK;
  Restrict1Params p = {};
  p.P = particles;
  p.x = x_src;
  p.pitch = src_pitch;
  p.stats = stats;
  p.counts = counts;
  p.targets = targets;
  p.tgt_stride = tgt_stride;
  p.cur = cur_stats;
  p.cur_stride = cur_stride;
  p.cur_counts = cur_counts;
  p.cnt_stride = cnt_stride;
  p.x_out = x_out;
  p.out_pitch = out_pitch;
  p.policy = policy;
  p.status = status;
  p.clamped = clamped;
  const int st = launch_r1_shape<true>(p, n_ens, (cudaStream_t)stream);
  if (st != MMPR_ERR_UNSUPPORTED) return st;
  // beyond one cluster: the two separate passes
  mmpr_partition single = {};
  single.n_regions = 1;
  const int sm = mmpr_match(&single, n_ens, particles, targets, tgt_stride, cur_stats, cur_stride, cur_counts,
                            cnt_stride, x_src, src_pitch, x_out, out_pitch, policy, status, clamped, stream);
  if (sm != MMPR_OK) return sm;
  return mmpr_restrict(&single, n_ens, particles, x_out, out_pitch, stats, counts, nullptr, stream);
}
