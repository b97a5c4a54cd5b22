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

namespace mmpr {

enum { RG_KEEP = 0, RG_SET = 1, RG_AFFINE = 2 };

__device__ __forceinline__ int rg_region(const mmpr_partition &part, double v) {
  // searchsorted(seps, v, side="right"); NaN sorts last (state.py:73-78)
  if (isnan(v)) return part.n_regions - 1;
  int r = 0;
#pragma unroll
  for (int i = 0; i < MMPR_MAX_REGIONS - 1; ++i)
    if (i < part.n_regions - 1 && part.seps[i] <= v) r = i + 1;
  return r;
}

struct __align__(16) RgSlot {
  double v;
  int ok;
  int pad;
};

template <int PPT, bool HAS_TAIL, bool MATCH>
__global__ void __launch_bounds__(1024, 1) restrict_regions_kernel(const RegionsParams p) {
  __shared__ PwVal s_wp[32];
  __shared__ PwVal s_chunk[32];  // per-chunk CTA partials of a member tree deeper than the ensemble's
  __shared__ __align__(16) RgSlot s_slot[FS_MAX_CLUSTER];
  __shared__ long long s_ccnt[FS_MAX_CLUSTER][MMPR_MAX_REGIONS];  // CTA member counts, written by peers
  __shared__ int s_wcnt[MMPR_MAX_REGIONS][32];                  // warp member counts -> exclusive offsets
  __shared__ int64_t s_off[MMPR_MAX_REGIONS], s_n[MMPR_MAX_REGIONS];
  __shared__ double s_mean;
  __shared__ int s_mode[MMPR_MAX_REGIONS];
  __shared__ double s_scale[MMPR_MAX_REGIONS], s_m[MMPR_MAX_REGIONS], s_mu[MMPR_MAX_REGIONS];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = (int)blockDim.x >> 5;
  const int rank = p.ctas > 1 ? (int)cluster_ctarank() : 0;
  const int e = (int)blockIdx.x / p.ctas;
  const int I = p.part.n_regions;
  const int64_t nslots = int64_t(1) << p.D;
  const int64_t slot = (int64_t)rank * p.slots_per_cta + warp * 4 + (lane >> 3);
  const int j8 = lane & 7;
  const int gbase = lane & 24;  // first lane of my leaf's 8-lane group
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

  // ---- compaction: index-order ranks of every region's members ---------------
  // leaf element (m, j8) has index off + 8m + j8, the trailing ones follow
  auto slot_bits = [&](bool pred) { return (__ballot_sync(MMPR_FULL_MASK, pred) >> gbase) & 0xffu; };
  int slot_cnt[MMPR_MAX_REGIONS] = {0, 0, 0, 0};
#pragma unroll
  for (int q = 0; q < MMPR_MAX_REGIONS; ++q) {
    if (q < I) {
      int c = 0;
#pragma unroll
      for (int m = 0; m < PPT; ++m) c += __popc(slot_bits(m < cnt && rg_region(p.part, x[m]) == q));
      if (HAS_TAIL) c += __popc(slot_bits(j8 < tail && rg_region(p.part, xt) == q));
      slot_cnt[q] = c;
    }
  }
  // exclusive prefix over the warp's four leaf groups, then over warps
  int pre_slot[MMPR_MAX_REGIONS] = {0, 0, 0, 0};
#pragma unroll
  for (int q = 0; q < MMPR_MAX_REGIONS; ++q) {
    if (q < I) {
      const int c = slot_cnt[q];
      const int c0 = __shfl_sync(MMPR_FULL_MASK, c, 0), c1 = __shfl_sync(MMPR_FULL_MASK, c, 8),
                c2 = __shfl_sync(MMPR_FULL_MASK, c, 16), c3 = __shfl_sync(MMPR_FULL_MASK, c, 24);
      const int g = lane >> 3;
      pre_slot[q] = (g > 0 ? c0 : 0) + (g > 1 ? c1 : 0) + (g > 2 ? c2 : 0);
      if (lane == 0) s_wcnt[q][warp] = c0 + c1 + c2 + c3;
    }
  }
  __syncthreads();
  if (warp == 0) {
    for (int q = 0; q < I; ++q) {
      const int v = lane < nwarps ? s_wcnt[q][lane] : 0;
      int incl = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(MMPR_FULL_MASK, incl, d);
        if (lane >= d) incl += u;
      }
      const int total = __shfl_sync(MMPR_FULL_MASK, incl, 31);
      if (lane < nwarps) s_wcnt[q][lane] = incl - v;  // exclusive
      // this CTA's total to every CTA of the cluster
      if (p.ctas > 1) {
        if (lane < p.ctas)
          asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(mapa_shared(smem_addr(&s_ccnt[rank][q]), (uint32_t)lane)),
                       "l"((long long)total)
                       : "memory");
      } else if (lane == 0) {
        s_ccnt[0][q] = total;
      }
    }
  }
  if (p.ctas > 1) cluster_sync_all();
  else __syncthreads();
  if (tid < I) {
    int64_t before = 0, all = 0;
    for (int c = 0; c < p.ctas; ++c) {
      const int64_t v = s_ccnt[c][tid];
      if (c < rank) before += v;
      all += v;
    }
    s_off[tid] = before;
    s_n[tid] = all;
  }
  __syncthreads();
  // scatter in index order
  double *scr = p.scratch + (int64_t)e * I * p.P;
#pragma unroll
  for (int q = 0; q < MMPR_MAX_REGIONS; ++q) {
    if (q < I) {
      int64_t pos = s_off[q] + s_wcnt[q][warp] + pre_slot[q];
      double *dst = scr + (int64_t)q * p.P;
#pragma unroll
      for (int m = 0; m < PPT; ++m) {
        const bool mine = m < cnt && rg_region(p.part, x[m]) == q;
        const unsigned bits = slot_bits(mine);
        if (mine) dst[pos + __popc(bits & ((1u << j8) - 1u))] = x[m];
        pos += __popc(bits);
      }
      if (HAS_TAIL) {
        const bool mine = j8 < tail && rg_region(p.part, xt) == q;
        const unsigned bits = slot_bits(mine);
        if (mine) dst[pos + __popc(bits & ((1u << j8) - 1u))] = xt;
      }
    }
  }
  // every CTA's members visible to the cluster (global memory, cluster scope)
  if (p.ctas > 1) cluster_sync_all();
  else __syncthreads();

  // ---- per region: pairwise tree over the n members, mean then variance -------
  double *st = p.stats + (int64_t)e * 3 * I;
  for (int q = 0; q < I; ++q) {
    const int64_t n = s_n[q];
    const double *a = scr + (int64_t)q * p.P;
    double mean = 0.0, var = 0.0;
    if (n >= 2) {
      // The member tree can be deeper than the ensemble's (an unaligned n
      // grows the right spine), so a CTA may own more slots than it has
      // 8-lane groups: it walks them in power-of-two chunks of `cap` slots
      // (consecutive subtrees) and folds the chunk partials as one more
      // tree level.
      const int Dq = pw_depth(n);
      const int64_t nsq = int64_t(1) << Dq;
      const int64_t spq = nsq >= p.ctas ? nsq / p.ctas : 1;
      const int64_t cap = (int64_t)nwarps * 4;
      const int64_t per = spq < cap ? spq : cap;
      const int nchunks = (int)(spq / per);
      const int64_t ls = warp * 4 + (lane >> 3);
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        auto f = [&](double v) { return pass ? mul(sub(v, mean), sub(v, mean)) : v; };
#pragma unroll 1
        for (int ch = 0; ch < nchunks; ++ch) {
          const bool valid = ls < per && (nsq >= p.ctas || rank < nsq);
          const int64_t sq = nsq >= p.ctas ? rank * spq + (int64_t)ch * per + ls : rank;
          int64_t qoff = 0, qlen = 0;
          if (valid) pw_leaf(n, Dq, sq, &qoff, &qlen);
          const int64_t qcnt = qlen >> 3;
          double acc = 0.0;
          if (qcnt > 0) {
            acc = f(a[qoff + j8]);
            for (int64_t k = 1; k < qcnt; ++k) acc = add(acc, f(a[qoff + j8 + 8 * k]));
          }
          acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 1));
          acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 2));
          acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 4));
          if (qcnt == 0) acc = 0.0;
          for (int64_t i = qcnt * 8; i < qlen; ++i) acc = add(acc, f(a[qoff + i]));
          PwVal leaf;
          leaf.v = acc;
          leaf.ok = qlen > 0;
          leaf = pw_xor_level(leaf, lane, 8);
          leaf = pw_xor_level(leaf, lane, 16);
          if (lane == 0) s_wp[warp] = leaf;
          __syncthreads();
          if (warp == 0) {
            PwVal v = lane < nwarps ? s_wp[lane] : PwVal{0.0, 0};
#pragma unroll
            for (int k = 1; k < 32; k <<= 1)
              if (k < nwarps) v = pw_xor_level(v, lane, k);
            if (lane == 0) s_chunk[ch] = v;
          }
          __syncthreads();  // s_wp is rewritten by the next chunk
        }
        if (warp == 0) {
          PwVal v = lane < nchunks ? s_chunk[lane] : PwVal{0.0, 0};
#pragma unroll
          for (int k = 1; k < 32; k <<= 1)
            if (k < nchunks) v = pw_xor_level(v, lane, k);
          v.v = __shfl_sync(MMPR_FULL_MASK, v.v, 0);  // every sending lane holds the CTA partial
          v.ok = __shfl_sync(MMPR_FULL_MASK, v.ok, 0);
          if (p.ctas > 1) {
            if (lane < p.ctas)
              st_cluster_v2(mapa_shared(smem_addr(&s_slot[rank]), (uint32_t)lane),
                            (unsigned long long)__double_as_longlong(v.v), (unsigned long long)(uint32_t)v.ok);
          } else if (lane == 0) {
            s_slot[0].v = v.v;
            s_slot[0].ok = v.ok;
          }
        }
        if (p.ctas > 1) cluster_sync_all();
        else __syncthreads();
        if (warp == 0) {
          PwVal c = lane < p.ctas ? PwVal{s_slot[lane].v, s_slot[lane].ok} : PwVal{0.0, 0};
#pragma unroll
          for (int k = 1; k < FS_MAX_CLUSTER; k <<= 1)
            if (k < p.ctas) c = pw_xor_level(c, lane, k);
          if (lane == 0) s_mean = div(c.v, (double)n);
        }
        // s_slot is rewritten by the next pass's peers only after they pass
        // this barrier, which needs every CTA's fold above to be done
        if (p.ctas > 1) cluster_sync_all();
        else __syncthreads();
        if (pass == 0) mean = s_mean;
        else var = s_mean;
      }
    } else {  // empty: the region's center, 0; one member: x, 0 (particles.py:192-199)
      mean = n == 0 ? p.part.centers[q] : a[0];
      var = 0.0;
    }
    if (rank == 0 && tid == 0) {
      st[q] = mean;
      st[I + q] = var;
      st[2 * I + q] = div((double)n, (double)p.P);
      if (p.counts) p.counts[(int64_t)e * I + q] = n;
    }
  }
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
