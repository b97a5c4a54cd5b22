// Fine propagator: Euler-Maruyama over one Parareal slice for many slices.
//
// Replaces particles.propagate_fine + _em_step_raw + ensemble_statistic
// (/root/reference/pkg/src/mcparareal/particles.py:119-159,
//  /root/reference/pkg/src/mcparareal/models.py:61-67) and the slice loop of
// engine._fine_sweep (/root/reference/pkg/src/mcparareal/engine.py:110-124).
//
// Layout ("pairwise-leaf layout"): numpy's mean of P values is a fixed
// binary tree whose leaves are blocks of <= 128 consecutive particles summed
// by 8 interleaved accumulators.  Each leaf slot of the (padded) tree is
// owned by 8 lanes; lane j holds particles off+j, off+j+8, ... in registers
// for the whole slice, so
//   * the per-step mean is bit-identical to np.mean (lane-sequential sums,
//     xor-shuffle leaf combine, warp/CTA/cluster levels of the same tree);
//   * increments are read from a per-CTA contiguous range staged in shared
//     memory by 1-D bulk async copies (double-buffered, one step ahead);
//   * a slice larger than one CTA (P > ~12.8k) spans a thread-block cluster
//     and the tree's top levels are combined through DSMEM, one
//     barrier.cluster per step.
// Increments come from HBM: the numpy-exact FROZEN stream is materialised
// once per run by noise.cu (or injected by the caller).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "mmpr_device.cuh"
#include "fine_common.cuh"
#include "capi_internal.h"

namespace mmpr {

#ifdef MMPR_FINE_PROFILE
// dev builds only: per-CTA cycle totals of the step phases
__device__ long long g_fine_prof[4096][10];
#define PROF_MARK(var) long long var = clock64()
#define PROF_ADD(k, a, b) if (tid == 0) atomicAdd((unsigned long long *)&g_fine_prof[blockIdx.x & 4095][k], (unsigned long long)((b) - (a)))
#else
#define PROF_MARK(var)
#define PROF_ADD(k, a, b)
#endif

// Block-level barrier of one slice group: __syncthreads for one group per
// CTA, a named barrier (id 1 + group) when two groups share the CTA.
template <int GROUPS>
__device__ __forceinline__ void group_sync(int grp, int nthreads) {
  if (GROUPS == 1) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(nthreads) : "memory");
  }
}

// PPT: accumulator elements per lane (ceil(max leaf / 8) <= 16); HAS_TAIL:
// P % 8 != 0 (the last leaf adds its trailing elements one by one).
// GROUPS: slices per cluster.  With two groups each CTA holds particles of
// two different slices (one per half of its threads) that step
// independently, so one slice's FP64 update overlaps the other's reduction
// and exchange latency on the same SM.
// LO >= 0: every populated leaf has at least LO accumulator elements per
// lane (compile-time, so only elements LO..PPT-1 carry a predicate);
// LO < 0: the bound comes from p.cnt_min at run time.
// PHX: increments generated in registers by counter-based Philox
// (counter_noise.cuh) instead of read from HBM; the dynamic shared memory
// then holds the ziggurat tables and no copy pipeline runs.
template <int KIND, int PPT, bool HAS_TAIL, bool PADDED, int MAXT, int GROUPS, int LO = -1, bool PHX = false>
__global__ void __launch_bounds__(MAXT, PHX ? (MMPR_PHX_MINB * 512 / MAXT > 0 ? MMPR_PHX_MINB * 512 / MAXT : 1) : 1024 / MAXT) fine_sweep_kernel(const FineParams p) {
  using PartT = Part<PADDED>;
  extern __shared__ __align__(128) double s_dyn[];  // [GROUPS][nstages][stage_elems]
  __shared__ PartT s_wp_all[GROUPS][2][32];
  __shared__ __align__(16) ClusterSlot s_slot_all[GROUPS][2][FS_MAX_CLUSTER];
  __shared__ int s_bad_all[GROUPS][3];
  __shared__ __align__(8) uint64_t s_bar_all[GROUPS][FS_MAX_STAGES];
  __shared__ __align__(8) uint64_t s_red_bar_all[GROUPS][2];  // cluster partials of call parity 0/1

  const int lane = threadIdx.x & 31;
  const int gthreads = GROUPS == 1 ? (int)blockDim.x : (int)blockDim.x / GROUPS;
  const int grp = GROUPS == 1 ? 0 : (int)threadIdx.x / gthreads;
  const int tid = (int)threadIdx.x - grp * gthreads;  // thread index within the group
  const int warp = tid >> 5;
  const int nwarps = gthreads >> 5;
  const int rank = (p.ctas > 1) ? (int)cluster_ctarank() : 0;
  const int slice = (blockIdx.x / p.ctas) * GROUPS + grp;
  const bool active = slice < p.n_slices;  // an odd slice count leaves one group idle
  const int64_t nslots = int64_t(1) << p.D;

  const int ns = p.nstages;
  double *s_stage = s_dyn + (size_t)grp * ns * p.stage_elems;
  const cn::ZigTables *zt = reinterpret_cast<const cn::ZigTables *>(s_dyn);
  const uint32_t nkey = cn::slice_key(p.cn, (uint32_t)(p.cn.n_base + slice));
  if constexpr (PHX) cn::load_zig(reinterpret_cast<cn::ZigTables *>(s_dyn), (int)threadIdx.x, (int)blockDim.x);
  // PHX: this thread's increment column, generated one step ahead (cn::gen)
  double *zb = reinterpret_cast<double *>(reinterpret_cast<char *>(s_dyn) + sizeof(cn::ZigTables)) + threadIdx.x;
  const int zstride = (int)blockDim.x;
  PartT(*s_wp)[32] = s_wp_all[grp];
  ClusterSlot(*s_slot)[FS_MAX_CLUSTER] = s_slot_all[grp];
  int *s_bad = s_bad_all[grp];
  uint64_t *s_bar = s_bar_all[grp];
  uint64_t *s_red_bar = s_red_bar_all[grp];

  // ---- my leaf --------------------------------------------------------------
  const int64_t slot = (int64_t)rank * p.slots_per_cta + warp * 4 + (lane >> 3);
  const int j8 = lane & 7;
  int64_t off = 0, len = 0;
  if (slot < nslots) pw_leaf(p.P, p.D, slot, &off, &len);
  const int cnt = (int)(len >> 3);       // elements per lane in the 8-way part
  const int tail = (int)(len & 7);       // trailing elements added one by one
  // (trailing particles exist in the ensemble's last leaf only: the other warps skip their fold)
  const bool warp_tail = HAS_TAIL && __any_sync(MMPR_FULL_MASK, tail != 0);
  const int64_t tail_off = off + (len & ~int64_t(7));
  const bool slot_ok = len > 0;
  const int cmin = LO >= 0 ? LO : p.cnt_min;  // min cnt over the slice's populated slots

  int64_t lo, hi;
  {
    int64_t o2, l2;
    pw_leaf(p.P, p.D, (int64_t)rank * p.slots_per_cta, &lo, &l2);
    if (rank == p.ctas - 1) hi = p.P;
    else pw_leaf(p.P, p.D, (int64_t)(rank + 1) * p.slots_per_cta, &hi, &o2);
  }
  const uint32_t stage_bytes = (uint32_t)((((hi - lo) * 8) + 15) & ~int64_t(15));
  const int last_idx = (int)(hi - lo) - 1;
  const int my_idx = (int)(off - lo) + j8;  // smem index of my first element

  // ---- load positions --------------------------------------------------------
  double x[PPT];
  double xt = 0.0;
  const double *xin = p.x_in + (int64_t)slice * p.in_pitch;
#pragma unroll
  for (int m = 0; m < PPT; ++m) x[m] = (active && m < cnt) ? xin[off + j8 + 8 * m] : 0.0;
  if (HAS_TAIL && active && j8 < tail) xt = xin[tail_off + j8];

  // ---- increment pipeline -------------------------------------------------------
  const double *xi_slice = p.xi + (int64_t)slice * p.xi_slice_pitch;
  if (tid == 0) {
    for (int q = 0; q < ns; ++q) mbar_init(&s_bar[q], 1);
    mbar_init(&s_red_bar[0], 1);
    mbar_init(&s_red_bar[1], 1);
    fence_mbar_init();
    s_bad[0] = 0;
    s_bad[1] = 0;
    s_bad[2] = 0;
  }
  // every CTA's barriers must be initialised before any peer sends to them
  if (p.ctas > 1) cluster_sync_all();
  else __syncthreads();
  if (!PHX && tid == 0 && active) {
    for (int j = 0; j < ns && j < p.S; ++j) {
      mbar_arrive_expect_tx(&s_bar[j], stage_bytes);
      bulk_g2s(s_stage + j * p.stage_elems, xi_slice + j * p.xi_row_pitch + lo, stage_bytes, &s_bar[j]);
    }
    for (int j = ns; j < ns + p.l2_ahead && j < p.S; ++j)
      prefetch_l2(xi_slice + (int64_t)j * p.xi_row_pitch + lo, stage_bytes);
  }
  int issued = PHX ? 0 : ((p.S < ns) ? p.S : ns);

  // ---- sum(x) in numpy's pairwise order + non-finite flag --------------------
  // One group barrier per call (B1) and, in a cluster, one mbarrier wait for
  // the peers' partials.  Every warp reads all warp partials after B1, so
  // s_wp is double-buffered by call parity; the blow-up flag uses three
  // slots: slot r%3 is written before B1 of call r, read after it, and reset
  // by thread 0 after B1 of call r+1 (before it reaches B1 of r+2, after
  // which the slot's next writers run).  `refill` (>= 0) is the step whose
  // increments go into the stage this step just consumed.
  // PHX: `gen_step` >= 0 generates that step's increments while the
  // partials are in flight.
  auto gen = [&](int jg) {
    if constexpr (PHX)
      cn::gen<PPT, (LO > 0 ? LO : 0), HAS_TAIL>(nkey, (uint32_t)jg, zt, zb, zstride, (uint32_t)(off + j8), cnt,
                                                 (uint32_t)(tail_off + j8), j8 < tail);
  };
  auto reduce = [&](int r, int refill, double &mean_out, int &bad_out, int gen_step) {
    PROF_MARK(tr0);
    const int par = r & 1;
    const int bslot = r % 3;
    double acc = x[0];
#pragma unroll
    for (int m = 1; m < PPT; ++m) {
      if (m < cmin) {
        acc = add(acc, x[m]);
      } else {
        const double t = add(acc, x[m]);
        acc = (m < cnt) ? t : acc;
      }
    }
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 1));
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 2));
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 4));
    if (cnt == 0) acc = 0.0;  // a leaf shorter than 8 (P < 8) is summed from 0.0
    if (HAS_TAIL && warp_tail) {  // (warp-uniform: only the warp holding the ensemble's last leaf)
#pragma unroll
      for (int i = 0; i < 7; ++i) {
        const double v = __shfl_sync(MMPR_FULL_MASK, xt, (lane & ~7) | i);
        if (i < tail) acc = add(acc, v);
      }
    }
    // a finite leaf sum proves every element finite (inf/NaN propagate);
    // only a non-finite sum needs the exact per-element test
    int bad_local = 0;
    if (!finite(acc)) {
#pragma unroll
      for (int m = 0; m < PPT; ++m) bad_local |= (m < cnt && !finite(x[m])) ? 1 : 0;
      if (HAS_TAIL && j8 < tail) bad_local |= !finite(xt);
    }
    const int wbad = __any_sync(MMPR_FULL_MASK, bad_local);
    PartT leaf = PartT::make(acc, slot_ok);
    leaf = leaf.xor_level(lane, 8);
    leaf = leaf.xor_level(lane, 16);
    if (lane == 0) {
      s_wp[par][warp] = leaf;
      if (wbad) s_bad[bslot] = 1;
    }
    PROF_MARK(tb0);
    PROF_ADD(5, tr0, tb0);
    group_sync<GROUPS>(grp, gthreads);  // B1 (the only block-level barrier of a step)
    PROF_MARK(tb1);
    PROF_ADD(2, tb0, tb1);
    // the last warp issues the refill so warp 0's path to the cluster
    // exchange (the step's critical path) carries no TMA issue latency
    if (tid == gthreads - 32) {
      s_bad[(r + 2) % 3] = 0;
      if (refill >= 0) {
        const int st = refill % ns;
        mbar_arrive_expect_tx(&s_bar[st], stage_bytes);
        bulk_g2s(s_stage + st * p.stage_elems, xi_slice + (int64_t)refill * p.xi_row_pitch + lo, stage_bytes,
                 &s_bar[st]);
        ++issued;
        const int pf = refill + p.l2_ahead;  // pull a later step towards L2
        if (p.l2_ahead > 0 && pf < p.S) prefetch_l2(xi_slice + (int64_t)pf * p.xi_row_pitch + lo, stage_bytes);
      }
    }
    // every warp folds the group's warp partials with the same xor tree
    PartT v = (lane < nwarps) ? s_wp[par][lane] : PartT::make(0.0, false);
#pragma unroll
    for (int m = 1; m < 32; m <<= 1)
      if (m < nwarps) v = v.xor_level(lane, m);
    double total;
    int bad = s_bad[bslot];
    if (p.ctas > 1) {
      // Each CTA's partial goes to the same group of every CTA of the cluster
      // as one 16-byte st.async that completes tx bytes on the receiver's
      // mbarrier; a group waits only for its own barrier.
      if (tid == 0) mbar_arrive_expect_tx(&s_red_bar[par], 16u * (uint32_t)p.ctas);
      if (warp == 0 && lane < p.ctas) {
        const uint32_t remote = mapa_shared(smem_addr(&s_slot[par][rank]), (uint32_t)lane);
        const uint32_t rbar = mapa_shared(smem_addr(&s_red_bar[par]), (uint32_t)lane);
        int okv = 1;
        if constexpr (PADDED) okv = v.ok;
        st_async_v2(remote, __double_as_longlong(v.v),
                    (unsigned long long)(uint32_t)okv | ((unsigned long long)(uint32_t)bad << 32), rbar);
      }
      PROF_MARK(tc0);
      PROF_ADD(7, tb1, tc0);
      if (PHX && gen_step >= 0) gen(gen_step);
      mbar_wait_parity(&s_red_bar[par], (uint32_t)((r >> 1) & 1));
      PROF_MARK(tc1);
      PROF_ADD(3, tc0, tc1);
      PartT c = PartT::make(0.0, false);
      int b = 0;
      if (lane < p.ctas) {
        c = PartT::make(s_slot[par][lane].v, s_slot[par][lane].ok != 0);
        b = s_slot[par][lane].bad;
      }
#pragma unroll
      for (int m = 1; m < FS_MAX_CLUSTER; m <<= 1)
        if (m < p.ctas) c = c.xor_level(lane, m);
      total = __shfl_sync(MMPR_FULL_MASK, c.v, 0);
      bad = __any_sync(MMPR_FULL_MASK, b);
    } else {
      total = __shfl_sync(MMPR_FULL_MASK, v.v, 0);  // lanes >= nwarps folded empty slots
      if (PHX && gen_step >= 0) gen(gen_step);
    }
    mean_out = div(total, (double)p.P);
    bad_out = bad;
    PROF_MARK(tr9);
    PROF_ADD(8, tr0, tr9);
  };

  double s = 0.0;
  int bad = 0;
  int first_bad = MMPR_STAT_OK;
  if (p.t_slice && active && tid == 0 && rank == 0) p.t_slice[2 * slice] = globaltimer_ns();
  if (active) {
    reduce(0, -1, s, bad, p.S > 0 ? 0 : -1);
    for (int j = 0; j < p.S; ++j) {
      const int stage = j % ns;
      PROF_MARK(tw0);
      if constexpr (!PHX) mbar_wait_parity(&s_bar[stage], (uint32_t)((j / ns) & 1));
      PROF_MARK(tw1);
      PROF_ADD(0, tw0, tw1);
      const double *xb = s_stage + stage * p.stage_elems;
      if constexpr (PHX) {
        // this step's increments were generated during the previous reduction
#pragma unroll
        for (int m = 0; m < PPT; ++m)
          if (m < (LO > 0 ? LO : 0) || m < cnt) x[m] = em_update<KIND>(p, x[m], s, zb[m * zstride]);
        if (HAS_TAIL && j8 < tail) xt = em_update<KIND>(p, xt, s, zb[PPT * zstride]);
      } else {
#pragma unroll
        for (int m = 0; m < PPT; ++m) {
          if (m < cmin) {
            x[m] = em_update<KIND>(p, x[m], s, xb[my_idx + 8 * m]);
          } else {
            // past some lanes' leaves: clamped index, value kept only when live
            const int idx = max(0, min(my_idx + 8 * m, last_idx));
            const double nx = em_update<KIND>(p, x[m], s, xb[idx]);
            x[m] = (m < cnt) ? nx : x[m];
          }
        }
        if (HAS_TAIL && warp_tail && j8 < tail) xt = em_update<KIND>(p, xt, s, xb[(int)(tail_off - lo) + j8]);
      }
      PROF_MARK(tu1);
      PROF_ADD(1, tw1, tu1);
      // B1 inside reduce() orders every read of this stage before its refill
      reduce(j + 1, (!PHX && j + ns < p.S) ? j + ns : -1, s, bad, j + 1 < p.S ? j + 1 : -1);
      if (bad) {
        first_bad = j;
        break;
      }
    }
    // Drain copies still in flight after an early exit (the refill thread
    // owns the issued count).
    if (tid == gthreads - 32 && first_bad != MMPR_STAT_OK) {
      for (int j = first_bad + 1; j < issued; ++j) mbar_wait_parity(&s_bar[j % ns], (uint32_t)((j / ns) & 1));
    }
  }

  if (p.t_slice && active && tid == 0 && rank == 0) p.t_slice[2 * slice + 1] = globaltimer_ns();
  if (active) {
    double *xo = p.x_out + (int64_t)slice * p.out_pitch;
#pragma unroll
    for (int m = 0; m < PPT; ++m)
      if (m < cnt) xo[off + j8 + 8 * m] = x[m];
    if (HAS_TAIL && j8 < tail) xo[tail_off + j8] = xt;
  }
  // Fused restriction of the slice-end ensemble (restrict, coupling.py:26;
  // np.mean / two-pass np.var): the mean is the last step's statistic, the
  // variance one more pass of the same tree over (x - mean)^2 from registers.
  // first_bad is cluster-uniform, so every CTA of the cluster takes part.
  double var = 0.0;
  const bool want_stats = p.stats != nullptr && active && first_bad == MMPR_STAT_OK;
  if (want_stats) {
#pragma unroll
    for (int m = 0; m < PPT; ++m) {
      const double d = sub(x[m], s);
      x[m] = mul(d, d);
    }
    if (HAS_TAIL) {
      const double d = sub(xt, s);
      xt = mul(d, d);
    }
    int bad2 = 0;
    reduce(p.S + 1, -1, var, bad2, -1);
  }

  if (p.ctas > 1) cluster_sync_all();  // no peer may still be writing into this CTA
  if (!active) return;
  if (tid == 0 && rank == 0) {
    p.bad_step[slice] = first_bad;
    if (p.final_mean) p.final_mean[slice] = s;
    if (want_stats) {
      double *st = p.stats + 3 * (int64_t)slice;
      st[0] = s;
      st[1] = p.P == 1 ? 0.0 : var;  // one member: S = 0 (particles.py:196-199)
      st[2] = div((double)p.P, (double)p.P);
      if (p.counts) p.counts[slice] = p.P;
    }
  }
}

// ---------------------------------------------------------------------------
// host-side geometry
// ---------------------------------------------------------------------------
struct FineGeometry {
  int ppt;      // ceil(max leaf / 8)
  int cnt_min;  // min leaf / 8 over populated slots
  bool padded;  // some slot of a CTA is empty
  int groups;   // slices per cluster (two halves of every CTA when 2)
  int D;
  int slots_per_cta;  // per group
  int ctas;
  int threads;
  int stage_elems;
  int nstages;
  size_t smem_bytes;
};

static int fine_sm_count() {
  static int sms_dev[MMPR_MAX_DEVICES] = {};
  const int dev = mmpr_current_device();
  if (sms_dev[dev] == 0) {
    int v = 0;
    sms_dev[dev] = (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) ? v : 148;
  }
  return sms_dev[dev];
}

// n_slices > 0: the launch's slice count, for the small-launch rule below.
static int fine_geometry(int64_t P, FineGeometry *g, int n_slices = 0) {
  if (P < 1) return MMPR_ERR_ARG;
  g->D = pw_depth(P);
  const int64_t nslots = int64_t(1) << g->D;
  int64_t max_leaf = 0, min_leaf = INT64_MAX;
  bool empty = false;
  for (int64_t s = 0; s < nslots; ++s) {
    int64_t o, l;
    pw_leaf(P, g->D, s, &o, &l);
    if (l > max_leaf) max_leaf = l;
    if (l > 0 && l < min_leaf) min_leaf = l;
    empty |= l == 0;
  }
  g->cnt_min = (int)(min_leaf >> 3);
  // accumulator elements per lane: a leaf of 8 c + r particles holds c per lane and its r < 8 trailing
  // ones (only the last leaf of an ensemble whose size is not a multiple of 8 has any) in the tail element
  g->ppt = (int)((P % 8) ? (max_leaf >> 3) : (max_leaf + 7) / 8);
  if (g->ppt < 1) g->ppt = 1;
  // increment stages of the CTA's particle range(s) must fit next to the
  // ~2 KB of static shared memory (227 KB opt-in per CTA)
  const size_t smem_budget = 224 * 1024;
  // (two groups -- particles of two slices per CTA, stepping independently
  // -- measured slower than one on B200: they share the SM's FP64 pipe and
  // double the cluster fan-in; kept behind MMPR_FINE_GROUPS=2 for study)
  g->groups = 1;
  if (const char *env = getenv("MMPR_FINE_GROUPS")) {  // tuning override
    const int v = atoi(env);
    if (v == 1 || (v == 2 && nslots >= 128 && nslots / 64 <= FS_MAX_CLUSTER)) g->groups = v;
  }
  // Large ensembles: 512-thread CTAs (16 per cluster at P = 1e5) with two
  // increment stages, so two CTAs of different slices share an SM and one's
  // FP64 update overlaps the other's reduction latency (measured 8% faster
  // than one 1024-thread CTA per SM at config 4).
  int spc = g->groups == 2 ? 64 : ((nslots >= 1024 && nslots / 64 <= FS_MAX_CLUSTER) ? 64 : 128);
  // Few small ensembles (BASELINE config 1: 10 slices of 1e4 particles): one
  // 1024-thread CTA per slice pulls the whole step's increments through one
  // SM (80 KB per 2.6 us step, measured); 32 slots per CTA spread a slice
  // over a 4-CTA cluster while every CTA of the launch still has its own SM
  // (1.6 us per step; 16 and 8 slots per CTA measured no better).
  // (the cluster fold sends lane c's copy of the CTA total to CTA c, and the
  // warp butterfly leaves the total in the first `warps` lanes only: a
  // cluster must not have more CTAs than a CTA has warps -- 8 at 32 slots)
  if (spc == 128 && g->groups == 1 && n_slices > 0 && nslots >= 64 && nslots / 32 <= 8 &&
      n_slices * (nslots / 32) <= fine_sm_count())
    spc = 32;
  if (const char *env = getenv("MMPR_FINE_SLOTS_PER_CTA")) {  // tuning override (one group)
    const int v = atoi(env);
    if (g->groups == 1 && v >= 4 && v <= 128 && (v & (v - 1)) == 0 && nslots / v <= v / 4) spc = v;  // CTAs <= warps
  }
  while (spc > 4 && (size_t)spc * max_leaf * 8 * 2 * g->groups > smem_budget) spc >>= 1;
  if (nslots <= spc) {
    g->slots_per_cta = (int)(nslots < 4 ? 4 : nslots);
    g->ctas = 1;
  } else {
    g->slots_per_cta = spc;
    g->ctas = (int)(nslots / spc);
  }
  if (g->ctas > FS_MAX_CLUSTER) return MMPR_ERR_UNSUPPORTED;
  g->threads = g->slots_per_cta * 8 * g->groups;
  g->padded = empty || nslots < g->slots_per_cta;
  // largest per-CTA particle range
  int64_t max_range = 0;
  for (int c = 0; c < g->ctas; ++c) {
    int64_t lo, hi, l;
    pw_leaf(P, g->D, (int64_t)c * g->slots_per_cta, &lo, &l);
    if (c == g->ctas - 1) hi = P;
    else pw_leaf(P, g->D, (int64_t)(c + 1) * g->slots_per_cta, &hi, &l);
    if (hi - lo > max_range) max_range = hi - lo;
  }
  g->stage_elems = (int)((max_range + 1) & ~int64_t(1));
  const size_t stage = (size_t)g->stage_elems * 8;
  g->nstages = (int)(smem_budget / (stage * g->groups));
  if (g->threads <= 512 && g->groups == 1 && 2 * stage <= smem_budget / 2) g->nstages = 2;  // two CTAs per SM
  if (g->nstages > FS_MAX_STAGES) g->nstages = FS_MAX_STAGES;
  if (const char *env = getenv("MMPR_FINE_STAGES")) {  // tuning override
    const int v = atoi(env);
    if (v >= 2 && v <= FS_MAX_STAGES && (size_t)v * stage * g->groups <= smem_budget) g->nstages = v;
  }
  if (g->nstages < 2) g->nstages = 2;
  g->smem_bytes = stage * g->nstages * g->groups;
  return MMPR_OK;
}

template <void (*KERN)(const FineParams)>
static int launch_fine_t(const FineParams &p, const FineGeometry &g, cudaStream_t stream);

template <int KIND, int PPT, bool HAS_TAIL>
static int launch_fine(const FineParams &p, const FineGeometry &g, cudaStream_t stream, bool phx) {
  if (phx) {
    if (g.groups != 1) return MMPR_ERR_UNSUPPORTED;
    if (!g.padded && g.ppt <= PPT && g.cnt_min >= PPT - 1) {
      if (g.threads <= 512)
        return launch_fine_t<fine_sweep_kernel<KIND, PPT, HAS_TAIL, false, 512, 1, PPT - 1, true>>(p, g, stream);
      return launch_fine_t<fine_sweep_kernel<KIND, PPT, HAS_TAIL, false, 1024, 1, PPT - 1, true>>(p, g, stream);
    }
    if (g.padded) return launch_fine_t<fine_sweep_kernel<KIND, PPT, HAS_TAIL, true, 1024, 1, -1, true>>(p, g, stream);
    return launch_fine_t<fine_sweep_kernel<KIND, PPT, HAS_TAIL, false, 1024, 1, -1, true>>(p, g, stream);
  }
#ifdef MMPR_FINE_TWO_GROUPS
  if (g.groups == 2) {
    if (g.padded) return launch_fine_t<fine_sweep_kernel<KIND, PPT, HAS_TAIL, true, 1024, 2>>(p, g, stream);
    return launch_fine_t<fine_sweep_kernel<KIND, PPT, HAS_TAIL, false, 1024, 2>>(p, g, stream);
  }
#else
  if (g.groups != 1) return MMPR_ERR_UNSUPPORTED;
#endif
  // Every slot populated and every leaf within 8 elements of the longest
  // (P = 1e5: leaves of 96 and 104): only the last accumulator element is
  // predicated.  512-thread CTAs run two per SM (64 registers each).
  if (!g.padded && g.ppt <= PPT && g.cnt_min >= PPT - 1) {
    if (g.threads <= 512)
      return launch_fine_t<fine_sweep_kernel<KIND, PPT, HAS_TAIL, false, 512, 1, PPT - 1>>(p, g, stream);
    return launch_fine_t<fine_sweep_kernel<KIND, PPT, HAS_TAIL, false, 1024, 1, PPT - 1>>(p, g, stream);
  }
  if (g.padded) return launch_fine_t<fine_sweep_kernel<KIND, PPT, HAS_TAIL, true, 1024, 1>>(p, g, stream);
  return launch_fine_t<fine_sweep_kernel<KIND, PPT, HAS_TAIL, false, 1024, 1>>(p, g, stream);
}

template <void (*KERN)(const FineParams)>
static int launch_fine_t(const FineParams &p, const FineGeometry &g, cudaStream_t stream) {
  auto kern = KERN;
  // attributes are set once per instantiation (never during graph capture
  // of a repeated configuration)
  static int configured_smem_dev[MMPR_MAX_DEVICES] = {};
  static bool configured_nonportable_dev[MMPR_MAX_DEVICES] = {};
  const int dev = mmpr_current_device();
  int &configured_smem = configured_smem_dev[dev];
  bool &configured_nonportable = configured_nonportable_dev[dev];
  cudaError_t err;
  if ((int)g.smem_bytes > configured_smem) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem_bytes);
    if (err != cudaSuccess) return mmpr_check(err, "fine_sweep: smem attribute");
    configured_smem = (int)g.smem_bytes;
  }
  if (g.ctas > 8 && !configured_nonportable) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return mmpr_check(err, "fine_sweep: non-portable cluster");
    configured_nonportable = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(((p.n_slices + g.groups - 1) / g.groups) * g.ctas), 1, 1);
  cfg.blockDim = dim3((unsigned)g.threads, 1, 1);
  cfg.dynamicSmemBytes = g.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)g.ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  err = cudaLaunchKernelEx(&cfg, kern, p);
  if (err == cudaSuccess) mmpr_launched();
  return mmpr_check(err, "fine_sweep_kernel launch");
}

template <int PPT, bool HAS_TAIL>
static int dispatch_kind(const FineParams &p, const FineGeometry &g, cudaStream_t s, bool phx) {
  switch (p.model.kind) {
    case MMPR_MODEL_OU: return launch_fine<MMPR_MODEL_OU, PPT, HAS_TAIL>(p, g, s, phx);
    case MMPR_MODEL_LINEAR: return launch_fine<MMPR_MODEL_LINEAR, PPT, HAS_TAIL>(p, g, s, phx);
    case MMPR_MODEL_DOUBLE_WELL: return launch_fine<MMPR_MODEL_DOUBLE_WELL, PPT, HAS_TAIL>(p, g, s, phx);
    case MMPR_MODEL_CUBIC_MF: return launch_fine<MMPR_MODEL_CUBIC_MF, PPT, HAS_TAIL>(p, g, s, phx);
    case MMPR_MODEL_DW_MULT: return launch_fine<MMPR_MODEL_DW_MULT, PPT, HAS_TAIL>(p, g, s, phx);
    default: return MMPR_ERR_UNSUPPORTED;
  }
}

template <int PPT>
static int dispatch_tail(const FineParams &p, const FineGeometry &g, cudaStream_t s, bool phx) {
  if (p.P % 8) return dispatch_kind<PPT, true>(p, g, s, phx);
  return dispatch_kind<PPT, false>(p, g, s, phx);
}

}  // namespace mmpr

using namespace mmpr;

// per-slice timestamp sink of the next fine sweeps of this host thread
// (mmpr_set_fine_times); read when a launch is configured, so a captured
// graph keeps the pointer it was captured with
static thread_local int64_t *g_fine_times = nullptr;

extern "C" int mmpr_set_fine_times(int64_t *slice_times) {
  g_fine_times = slice_times;
  return MMPR_OK;
}

static int fine_sweep_impl(const mmpr_model *model, int32_t n_slices, int64_t particles, int32_t steps,
                           double dt, double sqrt_dt, const double *t0, const double *x_in, int64_t in_pitch,
                           double *x_out, int64_t out_pitch, const double *xi, int64_t xi_slice_pitch,
                           int64_t xi_row_pitch, int32_t *bad_step, double *final_mean, double *stats,
                           int64_t *counts, void *stream, const mmpr_counter_noise *cnoise = nullptr) {
  if (!model || n_slices < 0 || particles < 1 || steps < 0 || !x_in || !x_out || !bad_step || !t0)
    return MMPR_ERR_ARG;
  if (n_slices == 0) return MMPR_OK;
  const bool phx = cnoise != nullptr;
  if (phx && (particles > UINT32_MAX || cnoise->slice_offset < 0 || cnoise->kfield >= (1u << 12) ||
              (int64_t)cnoise->slice_offset + n_slices > (1 << 20) || steps > (1 << 24)))
    return MMPR_ERR_ARG;
  if (!phx && steps > 0 && (!xi || (xi_row_pitch & 1) || xi_row_pitch < particles ||
                    (reinterpret_cast<uintptr_t>(xi) & 15) || (steps > 1 && xi_slice_pitch < steps * xi_row_pitch)))
    return MMPR_ERR_ARG;
  if (model->stat_kind != 0) return MMPR_ERR_UNSUPPORTED;
  FineGeometry g;
  int st = fine_geometry(particles, &g, n_slices);
  // beyond one cluster (or on request, for testing) the grid variant runs
  const char *force = getenv("MMPR_FINE_FORCE_GRID");
  const bool use_grid = (st == MMPR_ERR_UNSUPPORTED && g.ctas > FS_MAX_CLUSTER) || (force && atoi(force) == 1);
  if (st != MMPR_OK && !use_grid) return st;
  FineParams p;
  p.model = *model;
  p.n_slices = n_slices;
  p.S = steps;
  p.P = particles;
  p.dt = dt;
  p.sqrt_dt = sqrt_dt;
  p.bsd = 0.0;
  switch (model->kind) {
    case MMPR_MODEL_OU: p.bsd = model->p[2] * sqrt_dt; break;
    case MMPR_MODEL_DOUBLE_WELL: p.bsd = model->p[4] * sqrt_dt; break;
    case MMPR_MODEL_CUBIC_MF: p.bsd = model->p[3] * sqrt_dt; break;
    default: break;
  }
  p.t0 = t0;
  p.x_in = x_in;
  p.in_pitch = in_pitch;
  p.x_out = x_out;
  p.out_pitch = out_pitch;
  p.xi = xi;
  p.xi_slice_pitch = xi_slice_pitch;
  p.xi_row_pitch = xi_row_pitch;
  p.bad_step = bad_step;
  p.final_mean = final_mean;
  p.stats = stats;
  p.counts = counts;
  p.cn = cn::CounterNoise{0u, 0u, 0u, 0};
  p.t_slice = reinterpret_cast<long long *>(g_fine_times);
  if (phx) p.cn = cn::CounterNoise{cnoise->key[0], 0u, cnoise->kfield, cnoise->slice_offset};
  cudaStream_t s = (cudaStream_t)stream;
  if (use_grid) return fine_grid_sweep(p, s, phx);
  p.D = g.D;
  p.slots_per_cta = g.slots_per_cta;
  p.ctas = g.ctas;
  p.stage_elems = g.stage_elems;
  p.nstages = g.nstages;
  p.cnt_min = g.cnt_min;
  p.l2_ahead = 3;
  if (const char *env = getenv("MMPR_FINE_L2_AHEAD")) p.l2_ahead = max(0, min(16, atoi(env)));
  if (phx) {
    g.smem_bytes = cn::gen_smem_bytes(g.ppt <= 8 ? 8 : (g.ppt <= 13 ? 13 : 16), g.threads);
    p.nstages = 2;
    p.l2_ahead = 0;
  }
  if (g.ppt <= 8) return dispatch_tail<8>(p, g, s, phx);
  if (g.ppt <= 13) return dispatch_tail<13>(p, g, s, phx);
  return dispatch_tail<16>(p, g, s, phx);
}

extern "C" int mmpr_fine_sweep(const mmpr_model *model, int32_t n_slices, int64_t particles, int32_t steps,
                               double dt, double sqrt_dt, const double *t0, const double *x_in,
                               int64_t in_pitch, double *x_out, int64_t out_pitch, const double *xi,
                               int64_t xi_slice_pitch, int64_t xi_row_pitch, int32_t *bad_step,
                               double *final_mean, void *stream) {
  return fine_sweep_impl(model, n_slices, particles, steps, dt, sqrt_dt, t0, x_in, in_pitch, x_out, out_pitch, xi,
                         xi_slice_pitch, xi_row_pitch, bad_step, final_mean, nullptr, nullptr, stream);
}

extern "C" int mmpr_fine_sweep_restrict(const mmpr_model *model, int32_t n_slices, int64_t particles,
                                        int32_t steps, double dt, double sqrt_dt, const double *t0,
                                        const double *x_in, int64_t in_pitch, double *x_out, int64_t out_pitch,
                                        const double *xi, int64_t xi_slice_pitch, int64_t xi_row_pitch,
                                        int32_t *bad_step, double *stats, int64_t *counts, void *stream) {
  if (!stats) return MMPR_ERR_ARG;
  return fine_sweep_impl(model, n_slices, particles, steps, dt, sqrt_dt, t0, x_in, in_pitch, x_out, out_pitch, xi,
                         xi_slice_pitch, xi_row_pitch, bad_step, nullptr, stats, counts, stream);
}

extern "C" int mmpr_fine_sweep_counter(const mmpr_model *model, int32_t n_slices, int64_t particles, int32_t steps,
                                       double dt, double sqrt_dt, const double *t0, const double *x_in,
                                       int64_t in_pitch, double *x_out, int64_t out_pitch,
                                       const mmpr_counter_noise *noise, int32_t *bad_step, double *stats,
                                       int64_t *counts, void *stream) {
  if (!noise) return MMPR_ERR_ARG;
  return fine_sweep_impl(model, n_slices, particles, steps, dt, sqrt_dt, t0, x_in, in_pitch, x_out, out_pitch,
                         nullptr, 0, 0, bad_step, nullptr, stats, counts, stream, noise);
}

extern "C" int mmpr_fine_sweep_occupancy(int64_t particles, int32_t *clusters_out, int32_t *ctas_out) {
  FineGeometry g;
  int st = fine_geometry(particles, &g);
  if (st == MMPR_ERR_UNSUPPORTED && g.ctas > FS_MAX_CLUSTER) {
    // grid variant: concurrent teams of co-resident CTAs per slice
    int teams = 0, c = 0;
    st = fine_grid_shape(particles, 1 << 30, &teams, &c);
    if (st != MMPR_OK) return st;
    if (clusters_out) *clusters_out = teams;
    if (ctas_out) *ctas_out = c;
    return MMPR_OK;
  }
  if (st != MMPR_OK) return st;
  if (ctas_out) *ctas_out = g.ctas;
  // note: reports the one-group, 1024-thread variant's cluster occupancy
  auto kern = fine_sweep_kernel<MMPR_MODEL_OU, 16, false, false, 1024, 1>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem_bytes);
  if (err != cudaSuccess) return mmpr_check(err, "occupancy: smem attribute");
  if (g.ctas > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)g.ctas, 1, 1);
  cfg.blockDim = dim3((unsigned)g.threads, 1, 1);
  cfg.dynamicSmemBytes = g.smem_bytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)g.ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  err = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
  if (err != cudaSuccess) return mmpr_check(err, "cudaOccupancyMaxActiveClusters");
  if (clusters_out) *clusters_out = n;
  return MMPR_OK;
}

#ifdef MMPR_FINE_PROFILE
// dev builds only: copy out (and reset) the per-CTA phase cycle totals
extern "C" int mmpr_dev_fine_prof(long long *host_out, int reset) {
  cudaDeviceSynchronize();
  if (host_out) cudaMemcpyFromSymbol(host_out, g_fine_prof, sizeof(g_fine_prof));
  if (reset) {
    static long long zeros[4096][10];
    cudaMemcpyToSymbol(g_fine_prof, zeros, sizeof(zeros));
  }
  return (int)cudaGetLastError();
}
#endif
