// Fine propagator for ensembles larger than one thread-block cluster
// (BASELINE config 5: P = 2^20 per subinterval).
//
// Same per-particle update and the same numpy pairwise order of the
// per-step sum(x) as fine.cu (reference: propagate_fine / em_step,
// /root/reference/pkg/src/mcparareal/particles.py:134-159; the mean is the
// np.mean of the empirical-law statistic, particles.py:116-131).  What
// changes is the second reduction level: a slice is held by a TEAM of C
// co-resident CTAs (C = leaf slots / slots per CTA, up to 256), and the C
// CTA partials of every step are exchanged through L2 instead of DSMEM:
//
//   B1   __syncthreads_or  (CTA fold of the warp partials + blow-up flag)
//   pub  thread 0 stores its 16-B partial, red.release.gpu on the team counter
//   spin thread 0 polls the counter with ld.acquire.gpu until all C arrived
//   B2   __syncthreads, then every warp folds the C partials (ld.cg) in the
//        tree order of the leaf slots -- bit-identical to the cluster kernel.
//
// The kernel is persistent: T teams (as many as fit co-resident, launched
// with the cooperative attribute so a too-large grid fails instead of
// dead-locking) loop over the slices.  The first reduction level runs in
// thread-block clusters of two CTAs through distributed shared memory, so
// only C/2 partials go through L2 (their co-residency is checked with the
// cluster occupancy query before launching).  Increments reach shared memory by
// TMA bulk copies, one per leaf and chunk; a step's increments are split
// into H chunks (H = 2 when two full steps of a CTA's range do not fit
// in its share of shared memory), so three half-step buffers keep the next
// chunks in flight while the current one is consumed.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "capi_internal.h"
#include "fine_common.cuh"
#include "mmpr_device.cuh"

namespace mmpr {

#ifdef MMPR_FINE_PROFILE
// dev builds only: per-CTA cycle totals of the step phases
__device__ long long g_grid_prof[2048][8];
#define GPROF_MARK(var) long long var = clock64()
#define GPROF_ADD(k, a, b) if (threadIdx.x == 0) g_grid_prof[blockIdx.x & 2047][k] += (b) - (a)
#else
#define GPROF_MARK(var)
#define GPROF_ADD(k, a, b)
#endif

#define FG_MAX_CTAS 2048   // teams * C
#define FG_MAX_TEAM 256    // C (8 partials per lane in the final fold)
#define FG_MAX_TEAMS 64
#define FG_MAX_SLOTS 128   // leaf slots per CTA (1024 threads)

struct __align__(16) GridPart {
  double v;
  int ok;
  int bad;
};

// exchange buffers (double-buffered by reduction parity) and one arrival
// counter per team on its own 128-B line; counters are zeroed by a memset
// node ahead of every launch
__device__ GridPart g_fg_parts[2][FG_MAX_CTAS];
__device__ unsigned int g_fg_count[FG_MAX_TEAMS * 32];

struct GridExtra {
  int cl;           // CTAs per thread-block cluster (first reduction level), 1 = none
  int teams;
  int leaf_stride;  // doubles per leaf in a chunk buffer (== 8 mod 16: conflict-free)
  int nbuf;         // chunk buffers in shared memory
  int chunk_elems;  // doubles per chunk buffer
};

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int *p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_gpu_add(unsigned int *p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Leaf-relative element range of chunk h: [8*h*MH, h == H-1 ? len : 8*(h+1)*MH).
template <int H, int MH>
__device__ __forceinline__ void chunk_range(int64_t len, int h, int64_t *a, int64_t *b) {
  *a = (int64_t)8 * h * MH;
  *b = (h == H - 1) ? len : min(len, (int64_t)8 * (h + 1) * MH);
  if (*b < *a) *b = *a;
}

// LO: compile-time lower bound on the accumulator elements per lane of every
// populated leaf (elements LO..PPT-1 carry a predicate); -1 = p.cnt_min.
// PHX: increments from counter-based Philox in registers (counter_noise.cuh);
// the dynamic shared memory holds the ziggurat tables, no copies run.
template <int KIND, int PPT, bool HAS_TAIL, bool PADDED, int H, int LO, bool PHX = false>
__global__ void __launch_bounds__(1024, 1) fine_grid_kernel(const FineParams p, const GridExtra e) {
  using PartT = Part<PADDED>;
  constexpr int MH = PPT / H;  // accumulator elements of chunk 0 (chunk H-1 takes the rest)
  extern __shared__ __align__(128) double s_buf[];  // [nbuf][chunk_elems]
  __shared__ PartT s_wp[32];
  __shared__ __align__(8) uint64_t s_bar[8];
  __shared__ int64_t s_leaf_off[FG_MAX_SLOTS];
  __shared__ int s_leaf_len[FG_MAX_SLOTS];
  __shared__ uint32_t s_chunk_bytes[H];
  __shared__ double s_mean;
  __shared__ int s_tbad;
  __shared__ __align__(16) ClusterSlot s_slot[2][FS_MAX_CLUSTER];
  __shared__ __align__(8) uint64_t s_red_bar[2];

  const int C = p.ctas;
  const int team = (int)blockIdx.x / C;
  const int rank = (int)blockIdx.x - team * C;
  const int tid = (int)threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nwarps = (int)blockDim.x >> 5;
  const int spc = p.slots_per_cta;
  const int64_t nslots = int64_t(1) << p.D;
  const bool issuer = warp == nwarps - 1;  // the last warp issues the copies
  const int NB = e.nbuf;
  const int LS = e.leaf_stride;
  const int K1 = e.cl;                        // cluster level: K1 CTAs exchange through DSMEM
  const int crank = K1 > 1 ? (int)cluster_ctarank() : 0;
  const int Cn = C / K1;                      // participants of the L2 level

  // ---- leaf geometry -----------------------------------------------------
  const int li = warp * 4 + (lane >> 3);  // local leaf index
  const int64_t slot = (int64_t)rank * spc + li;
  const int j8 = lane & 7;
  int64_t off = 0, len = 0;
  if (slot < nslots) pw_leaf(p.P, p.D, slot, &off, &len);
  const int cnt = (int)(len >> 3);
  const int tail = (int)(len & 7);
  const bool slot_ok = len > 0;
  const int cmin = LO >= 0 ? LO : p.cnt_min;
  if (j8 == 0) {
    s_leaf_off[li] = off;
    s_leaf_len[li] = (int)len;
  }
  // smem index (within a chunk buffer) of element m of this lane, and of the tail
  const int my_base = li * LS + j8;
  const int tail_idx = li * LS + (int)(8 * cnt - 8 * (H - 1) * MH) + j8;  // tail sits in chunk H-1

  const cn::ZigTables *zt = reinterpret_cast<const cn::ZigTables *>(s_buf);
  if constexpr (PHX) cn::load_zig(reinterpret_cast<cn::ZigTables *>(s_buf), tid, (int)blockDim.x);
  // PHX: this thread's increment column, generated one step ahead (cn::gen)
  double *zb = reinterpret_cast<double *>(reinterpret_cast<char *>(s_buf) + sizeof(cn::ZigTables)) + tid;
  const int zstride = (int)blockDim.x;
  if (tid == 0) {
    for (int q = 0; q < NB; ++q) mbar_init(&s_bar[q], 1);
    mbar_init(&s_red_bar[0], 1);
    mbar_init(&s_red_bar[1], 1);
    fence_mbar_init();
  }
  // peers' barriers must be initialised before any st.async reaches them
  if (K1 > 1) cluster_sync_all();
  else __syncthreads();
  if (issuer) {
#pragma unroll
    for (int h = 0; h < H; ++h) {
      uint32_t bytes = 0;
      for (int l = lane; l < spc; l += 32) {
        int64_t a, b;
        chunk_range<H, MH>(s_leaf_len[l], h, &a, &b);
        bytes += (uint32_t)((((b - a) * 8) + 15) & ~int64_t(15));
      }
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) bytes += __shfl_xor_sync(MMPR_FULL_MASK, bytes, m);
      if (lane == 0) s_chunk_bytes[h] = bytes;
    }
  }
  __syncthreads();

  unsigned int *counter = &g_fg_count[team * 32];
  GridPart *parts0 = &g_fg_parts[0][team * C];
  GridPart *parts1 = &g_fg_parts[1][team * C];
  uint32_t epoch = 0;    // reductions done by this team (all slices)
  uint32_t qbase = 0;    // chunks issued by this CTA before the current slice

  // issue chunk c (= step * H + h) of the current slice into buffer (qbase + c) % NB
  auto issue = [&](const double *xi_slice, int c) {
    const int h = c % H;
    const int j = c / H;
    const uint32_t q = qbase + (uint32_t)c;
    uint64_t *bar = &s_bar[q % NB];
    double *dst = s_buf + (size_t)(q % NB) * e.chunk_elems;
    if (lane == 0) mbar_arrive_expect_tx(bar, s_chunk_bytes[h]);
    __syncwarp();
    const double *row = xi_slice + (int64_t)j * p.xi_row_pitch;
    for (int l = lane; l < spc; l += 32) {
      int64_t a, b;
      chunk_range<H, MH>(s_leaf_len[l], h, &a, &b);
      const uint32_t bytes = (uint32_t)((((b - a) * 8) + 15) & ~int64_t(15));
      if (bytes) bulk_g2s(dst + l * LS, row + s_leaf_off[l] + a, bytes, bar);
    }
  };

  for (int slice = team; slice < p.n_slices; slice += e.teams) {
    const int total_chunks = p.S * H;
    const double *xi_slice = p.xi + (int64_t)slice * p.xi_slice_pitch;
    if (!PHX && issuer) {
      for (int c = 0; c < NB && c < total_chunks; ++c) issue(xi_slice, c);
    }
    const uint32_t nkey = cn::slice_key(p.cn, (uint32_t)(p.cn.n_base + slice));
    double x[PPT];
    double xt = 0.0;
    const double *xin = p.x_in + (int64_t)slice * p.in_pitch;
#pragma unroll
    for (int m = 0; m < PPT; ++m) x[m] = (m < cnt) ? xin[off + j8 + 8 * m] : 0.0;
    if (HAS_TAIL && j8 < tail) xt = xin[off + 8 * cnt + j8];

    // sum(x) in numpy's pairwise order + blow-up flag over the team
    // PHX: `gen_step` >= 0 generates that step's increments during the team
    // exchange (warps 1.. right after B1, warp 0 between publishing its
    // partial and polling for the team's)
    auto gen = [&](int jg) {
      if constexpr (PHX)
        cn::gen<PPT, (LO > 0 ? LO : 0), HAS_TAIL>(nkey, (uint32_t)jg, zt, zb, zstride, (uint32_t)(off + j8), cnt,
                                                   (uint32_t)(off + 8 * cnt + j8), j8 < tail);
    };
    auto reduce = [&](int refill_step, double &mean_out, int &bad_out, int gen_step) {
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
      if (cnt == 0) acc = 0.0;
      if (HAS_TAIL) {
#pragma unroll
        for (int i = 0; i < 7; ++i) {
          const double v = __shfl_sync(MMPR_FULL_MASK, xt, (lane & ~7) | i);
          if (i < tail) acc = add(acc, v);
        }
      }
      int bad_local = 0;
      if (!finite(acc)) {
#pragma unroll
        for (int m = 0; m < PPT; ++m) bad_local |= (m < cnt && !finite(x[m])) ? 1 : 0;
        if (HAS_TAIL && j8 < tail) bad_local |= !finite(xt);
      }
      PartT leaf = PartT::make(acc, slot_ok);
      leaf = leaf.xor_level(lane, 8);
      leaf = leaf.xor_level(lane, 16);
      if (lane == 0) s_wp[warp] = leaf;
      GPROF_MARK(pb0);
      const int cta_bad = __syncthreads_or(bad_local);  // B1
      GPROF_MARK(pb1);
      GPROF_ADD(1, pb0, pb1);
      // B1 orders every read of the consumed buffers before their refill; the
      // copies overlap the team exchange below
      if (!PHX && issuer && refill_step >= 0) {
        for (int h = 0; h < H; ++h) {
          const int c = refill_step * H + h + NB;
          if (c < total_chunks) issue(xi_slice, c);
        }
      }
      GridPart *parts = (epoch & 1) ? parts1 : parts0;
      if (PHX && warp != 0 && gen_step >= 0) gen(gen_step);
      if (warp == 0) {
        PartT v = (lane < nwarps) ? s_wp[lane] : PartT::make(0.0, false);
#pragma unroll
        for (int m = 1; m < 32; m <<= 1)
          if (m < nwarps) v = v.xor_level(lane, m);
        int okv = 1;
        if constexpr (PADDED) okv = v.ok;
        int vbad = cta_bad;
        bool publisher = true;
        if (K1 > 1) {
          // level 1: the K1 CTAs of the cluster exchange 16-byte partials
          // through DSMEM (st.async completing tx bytes on the receiver's
          // mbarrier) and fold them in slot order
          const int par = epoch & 1;
          if (lane == 0) mbar_arrive_expect_tx(&s_red_bar[par], 16u * (uint32_t)K1);
          __syncwarp();
          if (lane < K1) {
            const uint32_t remote = mapa_shared(smem_addr(&s_slot[par][crank]), (uint32_t)lane);
            const uint32_t rbar = mapa_shared(smem_addr(&s_red_bar[par]), (uint32_t)lane);
            st_async_v2(remote, __double_as_longlong(v.v),
                        (unsigned long long)(uint32_t)okv | ((unsigned long long)(uint32_t)cta_bad << 32), rbar);
          }
          mbar_wait_parity(&s_red_bar[par], (uint32_t)((epoch >> 1) & 1));
          PartT cv = PartT::make(0.0, false);
          int cb = 0;
          if (lane < K1) {
            cv = PartT::make(s_slot[par][lane].v, s_slot[par][lane].ok != 0);
            cb = s_slot[par][lane].bad;
          }
#pragma unroll
          for (int m = 1; m < FS_MAX_CLUSTER; m <<= 1)
            if (m < K1) cv = cv.xor_level(lane, m);
          v = cv;
          okv = 1;
          if constexpr (PADDED) okv = __shfl_sync(MMPR_FULL_MASK, (int)cv.ok, 0);
          vbad = __any_sync(MMPR_FULL_MASK, cb);
          publisher = crank == 0;
        }
        if (lane == 0) {
          if (publisher) {  // level 2: one partial per cluster (per CTA without clusters) through L2
            int4 w;
            w.x = __double2loint(v.v);
            w.y = __double2hiint(v.v);
            w.z = okv;
            w.w = vbad;
            __stcg(reinterpret_cast<int4 *>(&parts[rank / K1]), w);
            GPROF_MARK(pp0);
            red_release_gpu_add(counter, 1u);
            GPROF_MARK(pp1);
            GPROF_ADD(2, pp0, pp1);
          }
        }
        if (PHX && gen_step >= 0) {
          __syncwarp();
          gen(gen_step);
        }
        if (lane == 0) {
          const unsigned long long t0 = globaltimer();
          const unsigned int target = (epoch + 1) * (unsigned int)Cn;
          while (ld_acquire_gpu(counter) < target) {
            // a team member that never arrives (not co-resident) would hang
            // the device: fail the launch instead
            if (globaltimer() - t0 > 4000000000ull) __trap();
          }
        }
        __syncwarp();
        // warp 0 folds the C team partials in slot-tree order (L2 reads)
        PartT c = PartT::make(0.0, false);
        int b = 0;
        if (Cn <= 32) {
          if (lane < Cn) {
            const int4 w = __ldcg(reinterpret_cast<const int4 *>(&parts[lane]));
            c = PartT::make(__hiloint2double(w.y, w.x), w.z != 0);
            b = w.w;
          }
#pragma unroll
          for (int m = 1; m < 32; m <<= 1)
            if (m < Cn) c = c.xor_level(lane, m);
        } else {
          // k = Cn/32 consecutive partials per lane, folded as a binary counter
          const int k = Cn >> 5;
          PartT stk[3];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (i < k) {
              const int4 w = __ldcg(reinterpret_cast<const int4 *>(&parts[lane * k + i]));
              PartT cur = PartT::make(__hiloint2double(w.y, w.x), w.z != 0);
              b |= w.w;
#pragma unroll
              for (int l = 0; l < 3; ++l)
                if ((i >> l) & 1) cur = PartT::combine(stk[l], cur);
                else {
                  stk[l] = cur;
                  break;
                }
              if (i == 7) stk[0] = cur;  // k = 8: root of the lane's chunk
            }
          }
          c = (k == 2) ? stk[1] : (k == 4) ? stk[2] : stk[0];
#pragma unroll
          for (int m = 1; m < 32; m <<= 1) c = c.xor_level(lane, m);
        }
        const int any = __any_sync(MMPR_FULL_MASK, b);
        if (lane == 0) {
          s_mean = div(c.v, (double)p.P);
          s_tbad = any;
        }
      }
      GPROF_MARK(pb2);
      __syncthreads();  // B2
      GPROF_MARK(pb3);
      GPROF_ADD(4, pb1, pb2);
      GPROF_ADD(5, pb2, pb3);
      ++epoch;
      mean_out = s_mean;
      bad_out = s_tbad;
    };

    double s = 0.0;
    int bad = 0;
    int first_bad = MMPR_STAT_OK;
    int issued = PHX ? 0 : min(NB, total_chunks);
    if (p.t_slice && tid == 0 && rank == 0) p.t_slice[2 * slice] = globaltimer_ns();
    reduce(-1, s, bad, p.S > 0 ? 0 : -1);
    for (int j = 0; j < p.S; ++j) {
      GPROF_MARK(pu0);
      if constexpr (PHX) {
        // this step's increments were generated during the previous exchange
#pragma unroll
        for (int m = 0; m < PPT; ++m)
          if (m < (LO > 0 ? LO : 0) || m < cnt) x[m] = em_update<KIND>(p, x[m], s, zb[m * zstride]);
        if (HAS_TAIL && j8 < tail) xt = em_update<KIND>(p, xt, s, zb[PPT * zstride]);
      } else {
#pragma unroll
          for (int h = 0; h < H; ++h) {
            const uint32_t q = qbase + (uint32_t)(j * H + h);
            mbar_wait_parity(&s_bar[q % NB], (q / NB) & 1);
            const double *xb = s_buf + (size_t)(q % NB) * e.chunk_elems;
            const int m0 = h * MH;  // compile-time after unrolling
            const int m1 = (h == H - 1) ? PPT : (h + 1) * MH;
  #pragma unroll
            for (int m = 0; m < PPT; ++m) {
              if (m < m0 || m >= m1) continue;
              if (m < cmin) {
                x[m] = em_update<KIND>(p, x[m], s, xb[my_base + 8 * (m - m0)]);
              } else {
                const int idx = (m < cnt) ? my_base + 8 * (m - m0) : my_base;
                const double nx = em_update<KIND>(p, x[m], s, xb[idx]);
                x[m] = (m < cnt) ? nx : x[m];
              }
            }
            if (h == H - 1 && HAS_TAIL && j8 < tail) xt = em_update<KIND>(p, xt, s, xb[tail_idx]);
          }
      }
      GPROF_MARK(pu1);
      GPROF_ADD(0, pu0, pu1);
      reduce(j, s, bad, j + 1 < p.S ? j + 1 : -1);  // refills the buffers step j consumed
      GPROF_MARK(pu2);
      GPROF_ADD(6, pu1, pu2);
      if (!PHX) issued = min(total_chunks, NB + (j + 1) * H);
      if (bad) {
        first_bad = j;
        break;
      }
    }
    // every issued chunk is waited on exactly once so barrier phases stay in step
    const int consumed = (first_bad == MMPR_STAT_OK) ? total_chunks : (first_bad + 1) * H;
    if (issuer && lane == 0) {
      for (int c = consumed; c < issued; ++c) {
        const uint32_t q = qbase + (uint32_t)c;
        mbar_wait_parity(&s_bar[q % NB], (q / NB) & 1);
      }
    }
    qbase += (uint32_t)issued;
    if (p.t_slice && tid == 0 && rank == 0) p.t_slice[2 * slice + 1] = globaltimer_ns();
    __syncthreads();  // buffers free before the next slice's prologue
    double *xo = p.x_out + (int64_t)slice * p.out_pitch;
#pragma unroll
    for (int m = 0; m < PPT; ++m)
      if (m < cnt) xo[off + j8 + 8 * m] = x[m];
    if (HAS_TAIL && j8 < tail) xo[off + 8 * cnt + j8] = xt;
    // fused single-region restriction (see fine.cu): one more team reduction
    // of (x - mean)^2; first_bad is team-uniform
    double var = 0.0;
    const bool want_stats = p.stats != nullptr && first_bad == MMPR_STAT_OK;
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
      reduce(-1, var, bad2, -1);
    }
    if (tid == 0 && rank == 0) {
      p.bad_step[slice] = first_bad;
      if (p.final_mean) p.final_mean[slice] = s;
      if (want_stats) {
        double *st = p.stats + 3 * (int64_t)slice;
        st[0] = s;
        st[1] = p.P == 1 ? 0.0 : var;
        st[2] = div((double)p.P, (double)p.P);
        if (p.counts) p.counts[slice] = p.P;
      }
    }
  }
  if (K1 > 1) cluster_sync_all();  // no peer may still be writing into this CTA
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int leaf_stride_for(int64_t need) {
  int64_t ls = (need + 1) & ~int64_t(1);
  while (ls % 16 != 8) ls += 2;
  return (int)ls;
}

struct GridGeometry {
  int D, spc, C, H, ppt, cnt_min, threads, nbuf, leaf_stride, chunk_elems, teams, cl;
  bool padded;
  size_t smem;
};

static int grid_geometry(int64_t P, int n_slices, GridGeometry *g) {
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
  g->ppt = (int)((max_leaf + 7) / 8);
  g->cnt_min = (int)(min_leaf >> 3);
  if (g->ppt > 16) return MMPR_ERR_UNSUPPORTED;
  // 512-thread CTAs, two per SM: each SM holds CTAs of two teams, so one
  // team's exchange latency overlaps the other's update (measured 1.5x
  // faster than 1024-thread CTAs at P = 2^20)
  int spc = 64;
  if (const char *env = getenv("MMPR_FINE_GRID_SLOTS")) {  // tuning override
    const int v = atoi(env);
    if (v >= 32 && v <= 128 && (v & (v - 1)) == 0) spc = v;
  }
  while (spc > 32 && spc > nslots) spc >>= 1;
  if (nslots < spc) return MMPR_ERR_UNSUPPORTED;
  g->spc = spc;
  g->C = (int)(nslots / spc);
  if (g->C > FG_MAX_TEAM) return MMPR_ERR_UNSUPPORTED;
  g->threads = spc * 8;
  g->padded = empty;
  // CTAs per SM: register bound (64 per thread) first, fewer when the
  // increment buffers do not fit next to each other
  const char *chunks_env = getenv("MMPR_FINE_GRID_CHUNKS");  // testing override
  const bool force_two = chunks_env && atoi(chunks_env) == 2;
  int blocks_per_sm = 1024 / g->threads;
  for (;; --blocks_per_sm) {
    if (blocks_per_sm < 1) return MMPR_ERR_UNSUPPORTED;
    // 228 KB per SM, 1 KB reserved per CTA, ~2.5 KB static per CTA
    size_t budget = (size_t)(228 * 1024) / blocks_per_sm - 1024 - 2560;
    if (budget > 227 * 1024 - 2560) budget = 227 * 1024 - 2560;
    // one chunk per step when two full steps fit, else two chunks per step
    g->H = 1;
    g->leaf_stride = leaf_stride_for(max_leaf);
    if (force_two || (size_t)spc * g->leaf_stride * 8 * 2 > budget) {
      g->H = 2;
      const int MH = 16 / 2;  // kernels are instantiated with PPT = 16
      if (g->cnt_min < MH) continue;
      g->leaf_stride = leaf_stride_for(max_leaf - 8 * MH > 8 * MH ? max_leaf - 8 * MH : 8 * MH);
    }
    g->chunk_elems = spc * g->leaf_stride;
    const size_t chunk_bytes = (size_t)g->chunk_elems * 8;
    g->nbuf = (int)(budget / chunk_bytes);
    if (g->nbuf > 8) g->nbuf = 8;
    if (g->nbuf < g->H + 1) continue;
    g->smem = chunk_bytes * g->nbuf;
    break;
  }
  // First reduction level in clusters of two CTAs (pairs fold through DSMEM,
  // halving the L2 participants): measured 5.05 vs 5.80 ms at P = 2^20
  // (8 slices x 200 steps; clusters of 4/8 5.2-5.5 ms, 16 halve the teams).
  g->cl = (g->C % 2 == 0 && g->C >= 4) ? 2 : 1;
  if (const char *env = getenv("MMPR_FINE_GRID_CLUSTER")) {  // tuning override
    const int v = atoi(env);
    if (v >= 2 && v <= FS_MAX_CLUSTER && (v & (v - 1)) == 0 && g->C % v == 0) g->cl = v;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int resident = sms * blocks_per_sm;
  g->teams = resident / g->C;
  if (g->teams > n_slices) g->teams = n_slices;
  if (g->teams > FG_MAX_TEAMS) g->teams = FG_MAX_TEAMS;
  if (g->teams * g->C > FG_MAX_CTAS) g->teams = FG_MAX_CTAS / g->C;
  if (g->teams < 1) return MMPR_ERR_UNSUPPORTED;
  return MMPR_OK;
}

template <void (*KERN)(const FineParams, const GridExtra)>
static int launch_grid_t(const FineParams &p, const GridGeometry &g, cudaStream_t stream) {
  static int configured_smem_dev[MMPR_MAX_DEVICES] = {};
  int &configured_smem = configured_smem_dev[mmpr_current_device()];
  cudaError_t err;
  if ((int)g.smem > configured_smem) {
    err = cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
    if (err != cudaSuccess) return mmpr_check(err, "fine_grid: smem attribute");
    configured_smem = (int)g.smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3((unsigned)g.threads, 1, 1);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int teams = g.teams;
  if (g.cl > 1) {
    if (g.cl > 8) {
      err = cudaFuncSetAttribute(KERN, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (err != cudaSuccess) return mmpr_check(err, "fine_grid: non-portable cluster");
    }
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)g.cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3((unsigned)g.cl, 1, 1);
    int clusters = 0;  // every team's clusters must be co-resident
    err = cudaOccupancyMaxActiveClusters(&clusters, KERN, &cfg);
    if (err != cudaSuccess) return mmpr_check(err, "fine_grid: cluster occupancy");
    const int per_team = g.C / g.cl;
    if (clusters / per_team < teams) teams = clusters / per_team;
    if (teams < 1) {
      mmpr_set_error("fine_grid: team clusters do not fit co-resident", cudaErrorCooperativeLaunchTooLarge);
      return MMPR_ERR_UNSUPPORTED;
    }
  } else {
    // every team member must be resident: check before launching
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, KERN, g.threads, g.smem);
    if (err != cudaSuccess) return mmpr_check(err, "fine_grid: occupancy");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (per_sm * sms < g.teams * g.C) {
      mmpr_set_error("fine_grid: team does not fit co-resident", cudaErrorCooperativeLaunchTooLarge);
      return MMPR_ERR_UNSUPPORTED;
    }
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  void *counts = nullptr;
  err = cudaGetSymbolAddress(&counts, g_fg_count);
  if (err != cudaSuccess) return mmpr_check(err, "fine_grid: counter symbol");
  err = cudaMemsetAsync(counts, 0, sizeof(unsigned int) * 32 * g.teams, stream);
  if (err != cudaSuccess) return mmpr_check(err, "fine_grid: counter reset");
  GridExtra e;
  e.cl = g.cl;
  e.teams = teams;
  e.leaf_stride = g.leaf_stride;
  e.nbuf = g.nbuf;
  e.chunk_elems = g.chunk_elems;
  cfg.gridDim = dim3((unsigned)(teams * g.C), 1, 1);
  err = cudaLaunchKernelEx(&cfg, KERN, p, e);
  if (err == cudaSuccess) mmpr_launched();
  return mmpr_check(err, "fine_grid_kernel launch");
}

template <int KIND, bool HAS_TAIL>
static int grid_dispatch_shape(const FineParams &p, const GridGeometry &g, cudaStream_t s, bool phx) {
  // P = 2^20: every leaf holds 128 elements, no predicated accumulator element
  const bool full = !g.padded && g.cnt_min >= 16;
  if (phx) {  // no chunking: one PHX instantiation per leaf shape
    if (full) return launch_grid_t<fine_grid_kernel<KIND, 16, HAS_TAIL, false, 1, 16, true>>(p, g, s);
    if (g.padded) return launch_grid_t<fine_grid_kernel<KIND, 16, HAS_TAIL, true, 1, -1, true>>(p, g, s);
    return launch_grid_t<fine_grid_kernel<KIND, 16, HAS_TAIL, false, 1, -1, true>>(p, g, s);
  }
  if (g.H == 1) {
    if (full) return launch_grid_t<fine_grid_kernel<KIND, 16, HAS_TAIL, false, 1, 16>>(p, g, s);
    if (g.padded) return launch_grid_t<fine_grid_kernel<KIND, 16, HAS_TAIL, true, 1, -1>>(p, g, s);
    return launch_grid_t<fine_grid_kernel<KIND, 16, HAS_TAIL, false, 1, -1>>(p, g, s);
  }
  if (full) return launch_grid_t<fine_grid_kernel<KIND, 16, HAS_TAIL, false, 2, 16>>(p, g, s);
  if (g.padded) return launch_grid_t<fine_grid_kernel<KIND, 16, HAS_TAIL, true, 2, -1>>(p, g, s);
  return launch_grid_t<fine_grid_kernel<KIND, 16, HAS_TAIL, false, 2, -1>>(p, g, s);
}

template <bool HAS_TAIL>
static int grid_dispatch_kind(const FineParams &p, const GridGeometry &g, cudaStream_t s, bool phx) {
  switch (p.model.kind) {
    case MMPR_MODEL_OU: return grid_dispatch_shape<MMPR_MODEL_OU, HAS_TAIL>(p, g, s, phx);
    case MMPR_MODEL_LINEAR: return grid_dispatch_shape<MMPR_MODEL_LINEAR, HAS_TAIL>(p, g, s, phx);
    case MMPR_MODEL_DOUBLE_WELL: return grid_dispatch_shape<MMPR_MODEL_DOUBLE_WELL, HAS_TAIL>(p, g, s, phx);
    case MMPR_MODEL_CUBIC_MF: return grid_dispatch_shape<MMPR_MODEL_CUBIC_MF, HAS_TAIL>(p, g, s, phx);
    case MMPR_MODEL_DW_MULT: return grid_dispatch_shape<MMPR_MODEL_DW_MULT, HAS_TAIL>(p, g, s, phx);
    default: return MMPR_ERR_UNSUPPORTED;
  }
}

int fine_grid_shape(int64_t P, int n_slices, int *teams_out, int *ctas_out) {
  GridGeometry g;
  int st = grid_geometry(P, n_slices, &g);
  if (st != MMPR_OK) return st;
  if (teams_out) *teams_out = g.teams;
  if (ctas_out) *ctas_out = g.C;
  return MMPR_OK;
}

int fine_grid_sweep(FineParams p, cudaStream_t stream, bool phx) {
  GridGeometry g;
  int st = grid_geometry(p.P, p.n_slices, &g);
  if (st != MMPR_OK) return st;
  if (phx) {
    g.smem = cn::gen_smem_bytes(16, g.threads);
    g.H = 1;
  }
  p.D = g.D;
  p.slots_per_cta = g.spc;
  p.ctas = g.C;
  p.cnt_min = g.cnt_min;
  p.stage_elems = g.chunk_elems;
  p.nstages = g.nbuf;
  if (p.P % 8) return grid_dispatch_kind<true>(p, g, stream, phx);
  return grid_dispatch_kind<false>(p, g, stream, phx);
}

}  // namespace mmpr

#ifdef MMPR_FINE_PROFILE
extern "C" int mmpr_dev_grid_prof(long long *host_out, int reset) {
  cudaDeviceSynchronize();
  if (host_out) cudaMemcpyFromSymbol(host_out, mmpr::g_grid_prof, sizeof(mmpr::g_grid_prof));
  if (reset) {
    static long long zeros[2048][8];
    cudaMemcpyToSymbol(mmpr::g_grid_prof, zeros, sizeof(zeros));
  }
  return (int)cudaGetLastError();
}
#endif
