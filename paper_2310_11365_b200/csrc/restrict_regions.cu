// Multi-region restriction (bimodal configs), optionally fused with the
// per-region match, with one thread-block cluster per ensemble.
//
// Replaces particles.region_statistics / coupling.restrict for I >= 2
// (/root/reference/pkg/src/mcparareal/particles.py:176-205,
// coupling.py:26-29) and coupling.match (coupling.py:32-95): per region
// i, members = x[assign == i] in index order, alpha_i = n_i / P,
// M_i = np.mean(members), S_i = np.var(members) (two-pass); numpy's pairwise
// sum runs over the COMPACTED member array, so its tree depends on n_i.
//
// One pass over the ensemble (instead of the six kernels of
// coupling.cu:restrict_multi plus a separate match pass):
//   load      every lane holds its leaf elements in registers (the fine
//             sweep's leaf-slot layout, restrict1.cu's cluster geometry);
//   match     (MATCH) per region an affine map onto the target moments,
//             membership from the PRE-transform positions (coupling.py:54),
//             the matched ensemble written out;
//   compact   per region, the index-order rank of every member: 8-lane
//             ballots per leaf row, slot -> warp -> CTA -> cluster prefix
//             (the CTA totals meet through DSMEM); members scattered to a
//             per-region scratch row (L2-resident);
//   reduce    per region the pairwise tree of its n_i members, its leaf slots
//             spread over the cluster's CTAs in tree order: leaf sums,
//             warp / CTA folds with validity flags, CTA partials through
//             DSMEM -> mean, then the same for (x - mean)^2 -> variance.
// Bit-identical to the multi-kernel path (tests/test_gpu_regions.py).
// Measured slower than that path on the BASELINE bimodal shapes (config 3:
// 12.2-12.5 vs 11.3-11.8 ms per run -- a cluster per ensemble runs 14
// ensembles at a time through latency-bound compaction and reduction
// phases), so the engine and mmpr_restrict use it only with
// MMPR_RESTRICT_CLUSTER=1; mmpr_match_restrict_regions always does.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "capi_internal.h"
#include "fine_common.cuh"
#include "mmpr_device.cuh"
#include "regions.cuh"
#include "regions_device.cuh"

namespace mmpr {

enum { RG_KEEP = 0, RG_SET = 1, RG_AFFINE = 2 };

template <int PPT, bool HAS_TAIL, bool MATCH>
__global__ void __launch_bounds__(1024, 1) restrict_regions_kernel(const RegionsParams p) {
  __shared__ RgSmem s_rg;
  __shared__ int s_mode[MMPR_MAX_REGIONS];
  __shared__ double s_scale[MMPR_MAX_REGIONS], s_m[MMPR_MAX_REGIONS], s_mu[MMPR_MAX_REGIONS];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = p.ctas > 1 ? (int)cluster_ctarank() : 0;
  const int e = (int)blockIdx.x / p.ctas;
  const int I = p.part.n_regions;
  const int64_t nslots = int64_t(1) << p.D;
  const int64_t slot = (int64_t)rank * p.slots_per_cta + warp * 4 + (lane >> 3);
  const int j8 = lane & 7;
  int64_t off = 0, len = 0;
  if (slot < nslots) pw_leaf(p.P, p.D, slot, &off, &len);
  const int cnt = (int)(len >> 3);
  const int tail = (int)(len & 7);

  const double *xs = p.x + (int64_t)e * p.pitch;
  double x[PPT];
  double xt = 0.0;
#pragma unroll
  for (int m = 0; m < PPT; ++m) x[m] = (m < cnt) ? xs[off + j8 + 8 * m] : 0.0;
  if (HAS_TAIL && j8 < tail) xt = xs[off + 8 * cnt + j8];

  if constexpr (MATCH) {
    // per-region parameters exactly as coupling.cu:match_kernel
    if (tid == 0) {
      const double *tg = p.targets + (int64_t)e * p.tgt_stride;
      const double *cs = p.cur + (int64_t)e * p.cur_stride;
      const int64_t *cn = p.cur_counts + (int64_t)e * p.cnt_stride;
      int status = MMPR_STAT_OK, clamped = 0;
      for (int q = 0; q < I; ++q) {
        s_mode[q] = RG_KEEP;
        if (cn[q] == 0) continue;  // empty region: skipped (coupling.py:57-60)
        const double mu_t = tg[q];
        double var_t = tg[I + q];
        if (var_t < 0.0) {
          clamped |= 1 << q;
          var_t = 0.0;
        }
        const double cur_mean = cs[q], cur_var = cs[I + q];
        if (cur_var == 0.0) {
          if (var_t > 0.0 && p.policy == 0 && status == MMPR_STAT_OK) status = q;
          s_mode[q] = RG_SET;
          s_mu[q] = mu_t;
          continue;
        }
        const double scale = __dsqrt_rn(div(var_t, cur_var));
        if (scale == 1.0 && mu_t == cur_mean) continue;  // exact identity keeps bits
        s_mode[q] = RG_AFFINE;
        s_scale[q] = scale;
        s_m[q] = cur_mean;
        s_mu[q] = mu_t;
      }
      if (rank == 0) {
        p.status[e] = status;
        if (p.clamped) p.clamped[e] = clamped;
      }
    }
    __syncthreads();
    auto apply = [&](double v) {
      const int r = rg_region(p.part, v);
      const int mode = s_mode[r];
      return mode == RG_SET ? s_mu[r] : (mode == RG_AFFINE ? add(mul(s_scale[r], sub(v, s_m[r])), s_mu[r]) : v);
    };
#pragma unroll
    for (int m = 0; m < PPT; ++m) x[m] = apply(x[m]);
    if (HAS_TAIL) xt = apply(xt);
    double *xo = p.x_out + (int64_t)e * p.out_pitch;
#pragma unroll
    for (int m = 0; m < PPT; ++m)
      if (m < cnt) xo[off + j8 + 8 * m] = x[m];
    if (HAS_TAIL && j8 < tail) xo[off + 8 * cnt + j8] = xt;
  }

  rg_restrict<PPT, HAS_TAIL>(s_rg, x, xt, cnt, tail, p.ctas, rank, p.part, p.P, p.scratch + (int64_t)e * I * p.P,
                             p.stats + (int64_t)e * 3 * I, p.counts ? p.counts + (int64_t)e * I : nullptr, true);
}

// ---------------------------------------------------------------------------
// host side: the cluster geometry of restrict1.cu (one cluster per ensemble)
// ---------------------------------------------------------------------------
struct RgGeometry {
  int D, spc, ctas, ppt;
};

static int rg_geometry_uncached(int64_t P, RgGeometry *g);

// cached per host thread (the worst-case depth scan below is not free)
static int rg_geometry(int64_t P, RgGeometry *g) {
  thread_local int64_t last_P = -1;
  thread_local int last_st = MMPR_ERR_ARG;
  thread_local RgGeometry last_g;
  if (P != last_P) {
    last_st = rg_geometry_uncached(P, &last_g);
    last_P = P;
  }
  *g = last_g;
  return last_st;
}

static int rg_geometry_uncached(int64_t P, RgGeometry *g) {
  const int D = pw_depth(P);
  const int64_t nslots = int64_t(1) << D;
  int64_t max_leaf = 0;
  for (int64_t s = 0; s < nslots; ++s) {
    int64_t o, l;
    pw_leaf(P, D, s, &o, &l);
    if (l > max_leaf) max_leaf = l;
  }
  int spc = nslots < 128 ? (nslots < 4 ? 4 : (int)nslots) : 128;
  if (nslots == 1024) spc = 64;  // 512-thread CTAs, 16 per cluster (as restrict1.cu)
  g->D = D;
  g->spc = spc;
  g->ctas = nslots <= spc ? 1 : (int)(nslots / spc);
  g->ppt = (int)((max_leaf + 7) / 8);
  if (g->ctas > FS_MAX_CLUSTER || g->ppt > 16) return MMPR_ERR_UNSUPPORTED;
  // the deepest member tree (n <= P) must fold in <= 32 chunks per CTA
  int dmax = 0;
  for (int64_t n = 2; n <= P; n = n < 4096 ? n + 1 : n + (n >> 6)) dmax = max(dmax, pw_depth(n));
  dmax = max(dmax, pw_depth(P));
  const int64_t cap_slots = (int64_t)g->spc * g->ctas;
  if ((int64_t(1) << dmax) > 32 * cap_slots) return MMPR_ERR_UNSUPPORTED;
  return MMPR_OK;
}

template <void (*KERN)(const RegionsParams)>
static int launch_rg(const RegionsParams &p, int n_ens, int threads, cudaStream_t stream) {
  static bool configured_dev[MMPR_MAX_DEVICES] = {};
  bool &configured = configured_dev[mmpr_current_device()];
  cudaError_t err;
  if (p.ctas > 8 && !configured) {
    err = cudaFuncSetAttribute(KERN, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return mmpr_check(err, "restrict_regions: non-portable cluster");
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_ens * p.ctas), 1, 1);
  cfg.blockDim = dim3((unsigned)threads, 1, 1);
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
  return mmpr_check(err, "restrict_regions_kernel launch");
}

int restrict_regions(RegionsParams p, int n_ens, bool match, cudaStream_t stream) {
  if (const char *env = getenv("MMPR_RESTRICT_CLUSTER"))
    if (atoi(env) == 0) return MMPR_ERR_UNSUPPORTED;  // the separate passes, for A/B and parity tests
  RgGeometry g;
  const int st = rg_geometry(p.P, &g);
  if (st != MMPR_OK) return st;
  p.D = g.D;
  p.slots_per_cta = g.spc;
  p.ctas = g.ctas;
  const int threads = g.spc * 8;
  const bool tail = (p.P % 8) != 0;
  if (match) {
    if (tail) return launch_rg<restrict_regions_kernel<16, true, true>>(p, n_ens, threads, stream);
    return launch_rg<restrict_regions_kernel<16, false, true>>(p, n_ens, threads, stream);
  }
  if (tail) return launch_rg<restrict_regions_kernel<16, true, false>>(p, n_ens, threads, stream);
  return launch_rg<restrict_regions_kernel<16, false, false>>(p, n_ens, threads, stream);
}

}  // namespace mmpr

using namespace mmpr;

extern "C" int mmpr_match_restrict_regions(const mmpr_partition *part, int32_t n_ens, int64_t particles,
                                           const double *targets, int64_t tgt_stride, const double *cur_stats,
                                           int64_t cur_stride, const int64_t *cur_counts, int64_t cnt_stride,
                                           const double *x_src, int64_t src_pitch, double *x_out,
                                           int64_t out_pitch, int32_t policy, int32_t *status, int32_t *clamped,
                                           double *stats, int64_t *counts, double *scratch, void *stream) {
  if (!part || part->n_regions < 1 || part->n_regions > MMPR_MAX_REGIONS || n_ens < 0 || particles < 1 ||
      !targets || !cur_stats || !cur_counts || !x_src || !x_out || !status || !stats || !counts || !scratch ||
      (policy != 0 && policy != 1))
    return MMPR_ERR_ARG;
  if (n_ens == 0) return MMPR_OK;
  RegionsParams p = {};
  p.part = *part;
  p.P = particles;
  p.x = x_src;
  p.pitch = src_pitch;
  p.stats = stats;
  p.counts = counts;
  p.scratch = scratch;
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
  const int st = restrict_regions(p, n_ens, true, (cudaStream_t)stream);
  if (st != MMPR_ERR_UNSUPPORTED) return st;
  // beyond one cluster: the separate passes
  const int sm = mmpr_match(part, n_ens, particles, targets, tgt_stride, cur_stats, cur_stride, cur_counts,
                            cnt_stride, x_src, src_pitch, x_out, out_pitch, policy, status, clamped, stream);
  if (sm != MMPR_OK) return sm;
  return mmpr_restrict(part, n_ens, particles, x_out, out_pitch, stats, counts, scratch, stream);
}
