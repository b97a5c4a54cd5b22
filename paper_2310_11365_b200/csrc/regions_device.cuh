// Per-region restriction of an ensemble held in registers by one
// thread-block cluster (the fine sweep's leaf-slot layout), shared by the
// one-pass region kernel (restrict_regions.cu) and the iteration pipeline's
// bimodal units (pipeline.cu).
//
// particles.region_statistics (/root/reference/pkg/src/mcparareal/
// particles.py:176-205): per region i, members = x[assign == i] in index
// order, alpha_i = n_i / P, M_i = np.mean(members), S_i = np.var(members)
// (two-pass).  numpy's pairwise sum runs over the COMPACTED member array, so
// its tree depends on n_i:
//   compact  the index-order rank of every member: 8-lane ballots per leaf
//            row, slot -> warp -> CTA -> cluster prefix (CTA totals meet
//            through DSMEM); members scattered to a per-region scratch row
//            (L2-resident);
//   reduce   per region the pairwise tree of its n_i members, its leaf slots
//            spread over the cluster's CTAs in tree order: leaf sums, warp /
//            CTA folds with validity flags, CTA partials through DSMEM ->
//            mean, then the same over (x - mean)^2 -> variance.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mmpr.h"
#include "fine_common.cuh"
#include "mmpr_device.cuh"

namespace mmpr {

#ifdef MMPR_PIPE_PROFILE
// dev builds only: per-CTA cycle totals of rg_restrict's phases (thread 0)
__device__ unsigned long long g_rg_prof[1024][8];
#define RGPROF_START long long rgp_t = clock64()
#define RGPROF(k)                                                                 \
  if (threadIdx.x == 0) {                                                         \
    const long long rgp_now = clock64();                                          \
    g_rg_prof[blockIdx.x & 1023][k] += (unsigned long long)(rgp_now - rgp_t);     \
    rgp_t = rgp_now;                                                              \
  }
#else
#define RGPROF_START
#define RGPROF(k)
#endif

// NRG > 0: the region count at compile time
template <int NRG = 0>
__device__ __forceinline__ int rg_region(const mmpr_partition &part, double v) {
  // searchsorted(seps, v, side="right"); NaN sorts last (state.py:73-78)
  const int I = NRG > 0 ? NRG : part.n_regions;
  if (isnan(v)) return I - 1;
  int r = 0;
#pragma unroll
  for (int i = 0; i < (NRG > 0 ? NRG : MMPR_MAX_REGIONS) - 1; ++i)
    if (i < I - 1 && part.seps[i] <= v) r = i + 1;
  return r;
}

struct __align__(16) RgSlot {
  double v;
  int ok;
  int pad;
};

// shared memory of rg_restrict (one per CTA)
struct RgSmem {
  PwVal wp[32];
  PwVal chunk[32];  // per-chunk CTA partials of a member tree deeper than the ensemble's
  RgSlot slot[FS_MAX_CLUSTER];
  long long ccnt[FS_MAX_CLUSTER][MMPR_MAX_REGIONS];  // CTA member counts, written by peers
  int wcnt[MMPR_MAX_REGIONS][32];                  // warp member counts -> exclusive offsets
  int64_t off[MMPR_MAX_REGIONS], n[MMPR_MAX_REGIONS];
  double mean;
  // all-regions path (every member tree fits one chunk per CTA)
  PwVal wpr[MMPR_MAX_REGIONS][32];                // warp partials per region
  RgSlot slotr[2][MMPR_MAX_REGIONS][FS_MAX_CLUSTER];  // CTA partials per pass and region, written by peers
  double res[2][MMPR_MAX_REGIONS];                // means, variances
};

// Restriction of the cluster's ensemble (x[m] = element off + 8m + j8 of the
// lane's leaf for m < cnt, xt = trailing element off + 8cnt + j8 when
// j8 < tail).  scr: I rows of P doubles (this ensemble's scratch).  CTA 0's
// thread 0 writes st[3I] (means, variances, fractions) and counts[I] when
// `write`.  Every thread of every CTA of the cluster must call it.
// NRG > 0: the region count at compile time (== part.n_regions), so the
// per-region loops unroll for exactly that many regions.
template <int PPT, bool HAS_TAIL, int NRG = 0, bool CHUNKED = true>
__device__ __forceinline__ void rg_restrict(RgSmem &sm, const double (&x)[PPT], double xt, int cnt, int tail, int ctas, int rank,
                            const mmpr_partition &part, int64_t P, double *scr, double *st, int64_t *counts,
                            bool write) {
  constexpr int MAXR = NRG > 0 ? NRG : MMPR_MAX_REGIONS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = (int)blockDim.x >> 5;
  const int j8 = lane & 7;
  const int gbase = lane & 24;  // first lane of my leaf's 8-lane group
  const int I = NRG > 0 ? NRG : part.n_regions;
  RGPROF_START;

  // ---- compaction: index-order ranks of every region's members ---------------
  // leaf element (m, j8) has index off + 8m + j8, the trailing ones follow
  auto slot_bits = [&](bool pred) { return (__ballot_sync(MMPR_FULL_MASK, pred) >> gbase) & 0xffu; };
  int slot_cnt[MMPR_MAX_REGIONS] = {0, 0, 0, 0};
#pragma unroll
  for (int q = 0; q < MAXR; ++q) {
    if (q < I) {
      int c = 0;
#pragma unroll
      for (int m = 0; m < PPT; ++m) c += __popc(slot_bits(m < cnt && rg_region<NRG>(part, x[m]) == q));
      if (HAS_TAIL) c += __popc(slot_bits(j8 < tail && rg_region<NRG>(part, xt) == q));
      slot_cnt[q] = c;
    }
  }
  // exclusive prefix over the warp's four leaf groups, then over warps
  int pre_slot[MMPR_MAX_REGIONS] = {0, 0, 0, 0};
#pragma unroll
  for (int q = 0; q < MAXR; ++q) {
    if (q < I) {
      const int c = slot_cnt[q];
      const int c0 = __shfl_sync(MMPR_FULL_MASK, c, 0), c1 = __shfl_sync(MMPR_FULL_MASK, c, 8),
                c2 = __shfl_sync(MMPR_FULL_MASK, c, 16), c3 = __shfl_sync(MMPR_FULL_MASK, c, 24);
      const int g = lane >> 3;
      pre_slot[q] = (g > 0 ? c0 : 0) + (g > 1 ? c1 : 0) + (g > 2 ? c2 : 0);
      if (lane == 0) sm.wcnt[q][warp] = c0 + c1 + c2 + c3;
    }
  }
  __syncthreads();
  if (warp == 0) {
    for (int q = 0; q < I; ++q) {
      const int v = lane < nwarps ? sm.wcnt[q][lane] : 0;
      int incl = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(MMPR_FULL_MASK, incl, d);
        if (lane >= d) incl += u;
      }
      const int total = __shfl_sync(MMPR_FULL_MASK, incl, 31);
      if (lane < nwarps) sm.wcnt[q][lane] = incl - v;  // exclusive
      // this CTA's total to every CTA of the cluster
      if (ctas > 1) {
        if (lane < ctas)
          asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(mapa_shared(smem_addr(&sm.ccnt[rank][q]), (uint32_t)lane)),
                       "l"((long long)total)
                       : "memory");
      } else if (lane == 0) {
        sm.ccnt[0][q] = total;
      }
    }
  }
  RGPROF(0);
  if (ctas > 1) cluster_sync_all();
  else __syncthreads();
  RGPROF(1);
  if (tid < I) {
    int64_t before = 0, all = 0;
    for (int c = 0; c < ctas; ++c) {
      const int64_t v = sm.ccnt[c][tid];
      if (c < rank) before += v;
      all += v;
    }
    sm.off[tid] = before;
    sm.n[tid] = all;
  }
  __syncthreads();
  // scatter in index order
#pragma unroll
  for (int q = 0; q < MAXR; ++q) {
    if (q < I) {
      int64_t pos = sm.off[q] + sm.wcnt[q][warp] + pre_slot[q];
      double *dst = scr + (int64_t)q * P;
#pragma unroll
      for (int m = 0; m < PPT; ++m) {
        const bool mine = m < cnt && rg_region<NRG>(part, x[m]) == q;
        const unsigned bits = slot_bits(mine);
        if (mine) dst[pos + __popc(bits & ((1u << j8) - 1u))] = x[m];
        pos += __popc(bits);
      }
      if (HAS_TAIL) {
        const bool mine = j8 < tail && rg_region<NRG>(part, xt) == q;
        const unsigned bits = slot_bits(mine);
        if (mine) dst[pos + __popc(bits & ((1u << j8) - 1u))] = xt;
      }
    }
  }
  RGPROF(2);
  // every CTA's members visible to the cluster (global memory, cluster scope)
  if (ctas > 1) cluster_sync_all();
  else __syncthreads();
  RGPROF(3);

  // ---- per region: pairwise tree over the n members, mean then variance -------
  // When every region's member tree spreads over at most one 8-lane group
  // per leaf slot and CTA (the BASELINE shapes), all regions are reduced
  // together: one DSMEM exchange and cluster barrier per pass (mean, then
  // variance) for all regions, each lane group's members loaded with all
  // loads in flight at once.  Otherwise region by region, in chunks.
  bool together = true;
  for (int q = 0; q < I; ++q) {
    const int64_t n = sm.n[q];
    if (n < 2) continue;
    const int64_t nsq = int64_t(1) << pw_depth(n);
    if ((nsq >= ctas ? nsq / ctas : 1) > (int64_t)nwarps * 4) together = false;
  }
  if (!CHUNKED && !together) __trap();  // callers without the chunked path guarantee one chunk
  if (!CHUNKED || together) {
    const int64_t ls = warp * 4 + (lane >> 3);
    double mean_q[MMPR_MAX_REGIONS] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
      for (int q = 0; q < MAXR; ++q) {
        if (q >= I) continue;
        const int64_t n = sm.n[q];
        if (n < 2) continue;
        const double mu = mean_q[q];
        auto f = [&](double v) { return pass ? mul(sub(v, mu), sub(v, mu)) : v; };
        const double *a = scr + (int64_t)q * P;
        const int Dq = pw_depth(n);
        const int64_t nsq = int64_t(1) << Dq;
        const int64_t spq = nsq >= ctas ? nsq / ctas : 1;
        const bool valid = ls < spq && (nsq >= ctas || rank < nsq);
        const int64_t sq = nsq >= ctas ? rank * spq + ls : rank;
        int64_t qoff = 0, qlen = 0;
        if (valid) pw_leaf(n, Dq, sq, &qoff, &qlen);
        const int qcnt = (int)(qlen >> 3);
        const int qtail = (int)(qlen & 7);
        double v[16], t[7];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = k < qcnt ? __ldcg(a + qoff + j8 + 8 * k) : 0.0;
#pragma unroll
        for (int i = 0; i < 7; ++i) t[i] = i < qtail ? __ldcg(a + qoff + 8 * qcnt + i) : 0.0;
        double acc = f(v[0]);
#pragma unroll
        for (int k = 1; k < 16; ++k)
          if (k < qcnt) acc = add(acc, f(v[k]));
        acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 1));
        acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 2));
        acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 4));
        if (qcnt == 0) acc = 0.0;
#pragma unroll
        for (int i = 0; i < 7; ++i)
          if (i < qtail) acc = add(acc, f(t[i]));
        PwVal leaf;
        leaf.v = acc;
        leaf.ok = qlen > 0;
        leaf = pw_xor_level(leaf, lane, 8);
        leaf = pw_xor_level(leaf, lane, 16);
        if (lane == 0) sm.wpr[q][warp] = leaf;
      }
      RGPROF(4);
      __syncthreads();
      RGPROF(5);
      // warp q (mod nwarps) folds region q's warp partials and sends the CTA
      // partial to every CTA of the cluster
      for (int q = warp; q < I; q += nwarps) {
        if (sm.n[q] < 2) continue;
        PwVal v = lane < nwarps ? sm.wpr[q][lane] : PwVal{0.0, 0};
#pragma unroll
        for (int k = 1; k < 32; k <<= 1)
          if (k < nwarps) v = pw_xor_level(v, lane, k);
        if (ctas > 1) {
          if (lane < ctas)
            st_cluster_v2(mapa_shared(smem_addr(&sm.slotr[pass][q][rank]), (uint32_t)lane),
                          (unsigned long long)__double_as_longlong(v.v), (unsigned long long)(uint32_t)v.ok);
        } else if (lane == 0) {
          sm.slotr[pass][q][0].v = v.v;
          sm.slotr[pass][q][0].ok = v.ok;
        }
      }
      // (slotr[pass] is rewritten only by the next call's same pass, after
      // every CTA has passed that call's compaction barriers)
      RGPROF(6);
      if (ctas > 1) cluster_sync_all();
      else __syncthreads();
      RGPROF(7);
      for (int q = warp; q < I; q += nwarps) {
        if (sm.n[q] < 2) continue;
        PwVal c = lane < ctas ? PwVal{sm.slotr[pass][q][lane].v, sm.slotr[pass][q][lane].ok} : PwVal{0.0, 0};
#pragma unroll
        for (int k = 1; k < FS_MAX_CLUSTER; k <<= 1)
          if (k < ctas) c = pw_xor_level(c, lane, k);
        if (lane == 0) sm.res[pass][q] = div(c.v, (double)sm.n[q]);
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < MAXR; ++q)
        if (q < I) mean_q[q] = sm.res[0][q];
    }
    if (write && rank == 0 && tid == 0) {
      for (int q = 0; q < I; ++q) {
        const int64_t n = sm.n[q];
        // empty: the region's center, 0; one member: x, 0 (particles.py:192-199)
        st[q] = n >= 2 ? sm.res[0][q] : (n == 0 ? part.centers[q] : __ldcg(scr + (int64_t)q * P));
        st[I + q] = n >= 2 ? sm.res[1][q] : 0.0;
        st[2 * I + q] = div((double)n, (double)P);
        if (counts) counts[q] = n;
      }
    }
    return;
  }
  for (int q = 0; q < I; ++q) {
    const int64_t n = sm.n[q];
    const double *a = scr + (int64_t)q * P;
    double mean = 0.0, var = 0.0;
    if (n >= 2) {
      // The member tree can be deeper than the ensemble's (an unaligned n
      // grows the right spine), so a CTA may own more slots than it has
      // 8-lane groups: it walks them in power-of-two chunks of `cap` slots
      // (consecutive subtrees) and folds the chunk partials as one more
      // tree level.
      const int Dq = pw_depth(n);
      const int64_t nsq = int64_t(1) << Dq;
      const int64_t spq = nsq >= ctas ? nsq / ctas : 1;
      const int64_t cap = (int64_t)nwarps * 4;
      const int64_t per = spq < cap ? spq : cap;
      const int nchunks = (int)(spq / per);
      const int64_t ls = warp * 4 + (lane >> 3);
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        auto f = [&](double v) { return pass ? mul(sub(v, mean), sub(v, mean)) : v; };
#pragma unroll 1
        for (int ch = 0; ch < nchunks; ++ch) {
          const bool valid = ls < per && (nsq >= ctas || rank < nsq);
          const int64_t sq = nsq >= ctas ? rank * spq + (int64_t)ch * per + ls : rank;
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
          if (lane == 0) sm.wp[warp] = leaf;
          __syncthreads();
          if (warp == 0) {
            PwVal v = lane < nwarps ? sm.wp[lane] : PwVal{0.0, 0};
#pragma unroll
            for (int k = 1; k < 32; k <<= 1)
              if (k < nwarps) v = pw_xor_level(v, lane, k);
            if (lane == 0) sm.chunk[ch] = v;
          }
          __syncthreads();  // sm.wp is rewritten by the next chunk
        }
        if (warp == 0) {
          PwVal v = lane < nchunks ? sm.chunk[lane] : PwVal{0.0, 0};
#pragma unroll
          for (int k = 1; k < 32; k <<= 1)
            if (k < nchunks) v = pw_xor_level(v, lane, k);
          v.v = __shfl_sync(MMPR_FULL_MASK, v.v, 0);  // every sending lane holds the CTA partial
          v.ok = __shfl_sync(MMPR_FULL_MASK, v.ok, 0);
          if (ctas > 1) {
            if (lane < ctas)
              st_cluster_v2(mapa_shared(smem_addr(&sm.slot[rank]), (uint32_t)lane),
                            (unsigned long long)__double_as_longlong(v.v), (unsigned long long)(uint32_t)v.ok);
          } else if (lane == 0) {
            sm.slot[0].v = v.v;
            sm.slot[0].ok = v.ok;
          }
        }
        if (ctas > 1) cluster_sync_all();
        else __syncthreads();
        if (warp == 0) {
          PwVal c = lane < ctas ? PwVal{sm.slot[lane].v, sm.slot[lane].ok} : PwVal{0.0, 0};
#pragma unroll
          for (int k = 1; k < FS_MAX_CLUSTER; k <<= 1)
            if (k < ctas) c = pw_xor_level(c, lane, k);
          if (lane == 0) sm.mean = div(c.v, (double)n);
        }
        // sm.slot is rewritten by the next pass's peers only after they pass
        // this barrier, which needs every CTA's fold above to be done
        if (ctas > 1) cluster_sync_all();
        else __syncthreads();
        if (pass == 0) mean = sm.mean;
        else var = sm.mean;
      }
    } else {  // empty: the region's center, 0; one member: x, 0 (particles.py:192-199)
      mean = n == 0 ? part.centers[q] : a[0];
      var = 0.0;
    }
    if (write && rank == 0 && tid == 0) {
      st[q] = mean;
      st[I + q] = var;
      st[2 * I + q] = div((double)n, (double)P);
      if (counts) counts[q] = n;
    }
  }
}

// rg_restrict of an ensemble the calling threads have just written to
// (without the chunked path: every member tree of the pipeline's ensembles,
// P < 2^17 over 16 CTAs of 64 leaf slots, spreads over one chunk)
// global memory at src (each thread reloads exactly the elements it wrote,
// so no barrier is needed first).  Out of line: the restriction's working
// set does not share a register allocation with the caller's step loop.
template <int PPT, bool HAS_TAIL, int NRG>
__device__ __noinline__ void rg_restrict_reload(RgSmem &sm, const double *src, int off, int cnt, int tail, int ctas,
                                                int rank, const mmpr_partition &part, int64_t P, double *scr,
                                                double *st, int64_t *counts) {
  const int j8 = threadIdx.x & 7;
  double x[PPT];
  double xt = 0.0;
#pragma unroll
  for (int m = 0; m < PPT; ++m) x[m] = (m < cnt) ? src[off + j8 + 8 * m] : 0.0;
  if (HAS_TAIL && j8 < tail) xt = src[off + 8 * cnt + j8];
  rg_restrict<PPT, HAS_TAIL, NRG, false>(sm, x, xt, cnt, tail, ctas, rank, part, P, scr, st, counts, true);
}

}  // namespace mmpr
