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
};

template <int PPT, bool HAS_TAIL, bool PADDED>
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
static int launch_r1(const Restrict1Params &p, int n_ens, int threads, cudaStream_t stream) {
  static bool configured = false;
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
  return mmpr_check(err, "restrict1_kernel launch");
}

// Returns MMPR_ERR_UNSUPPORTED when the ensemble does not fit one cluster
// (the caller then uses the one-CTA-per-ensemble kernel).
int restrict_single_region(int n_ens, int64_t P, const double *x, int64_t pitch, double *stats, int64_t *counts,
                           cudaStream_t stream) {
  // geometry of the last particle count (fixed within a run)
  thread_local int64_t last_P = -1;
  thread_local int g_D, g_spc, g_ctas, g_ppt;
  thread_local bool g_padded;
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
    const int spc = nslots < 128 ? (nslots < 4 ? 4 : (int)nslots) : 128;
    g_D = D;
    g_spc = spc;
    g_ctas = nslots <= spc ? 1 : (int)(nslots / spc);
    g_ppt = (int)((max_leaf + 7) / 8);
    g_padded = empty || nslots < spc;
    last_P = P;
  }
  if (g_ctas > FS_MAX_CLUSTER || g_ppt > 16) return MMPR_ERR_UNSUPPORTED;
  Restrict1Params p;
  p.P = P;
  p.x = x;
  p.pitch = pitch;
  p.stats = stats;
  p.counts = counts;
  p.D = g_D;
  p.slots_per_cta = g_spc;
  p.ctas = g_ctas;
  const int threads = g_spc * 8;
  const bool tail = (P % 8) != 0;
  if (g_padded) {
    if (tail) return launch_r1<restrict1_kernel<16, true, true>>(p, n_ens, threads, stream);
    return launch_r1<restrict1_kernel<16, false, true>>(p, n_ens, threads, stream);
  }
  if (tail) return launch_r1<restrict1_kernel<16, true, false>>(p, n_ens, threads, stream);
  return launch_r1<restrict1_kernel<16, false, false>>(p, n_ens, threads, stream);
}

}  // namespace mmpr
