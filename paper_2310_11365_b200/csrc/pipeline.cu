// Iterations 1..K of mM-Parareal as one persistent, dependency-driven kernel.
//
// Replaces, for single-region MEAN_OF_F runs, the per-iteration launch
// sequence fine sweep -> coarse row -> match + micro restriction of
// engine.run_micro_macro (/root/reference/pkg/src/mcparareal/engine.py:
// 197-238; particles.propagate_fine particles.py:146-159; coupling.match /
// restrict coupling.py:26-95; the serial correction engine.py:210-236).
//
// Work unit (k, n), k = 0..K, n = 0..N, one thread-block cluster per unit
// (same leaf-slot layout and per-step cluster reduction as fine.cu):
//   match part (k >= 1, n >= 1): the serial correction of boundary n of row
//     k -- pred = C(macro[k][n-1]) (or the cached prediction of a converged
//     slice, n-1 < k), corrected = R(F^{k-1}_{n-1}) + (pred - cache[k-1][n-1]),
//     negative variance clamped -- then u^k_n = match(corrected, F^{k-1}_{n-1})
//     and micro[k][n] = R(u^k_n), from registers;
//   fine part (k < K, n < N): F^k_n = F(u^k_n) with the particles still in
//     registers, and R(F^k_n) fused as in fine.cu.
// Units are taken in ticket order (k-major) by whichever cluster is free, and
// a unit waits only on units with smaller tickets:
//   fine_done[k-1][n-1]  (F^{k-1}_{n-1} and its restriction),
//   chain_done[k][n-1]   (macro[k][n-1], the serial chain of row k),
//   chain_done[k-1][n]   (cache[k-1][n-1]),
//   consumed[k-1][n+1]   (the reader of the fine buffer slot this unit
//                          overwrites has loaded it).
// So row k+1 starts on the SMs that row k's last wave leaves idle, the serial
// coarse chain and the match run inside the units that need them, and no
// kernel boundary separates the iterations.  Every value is computed with
// the same operations in the same order as the per-iteration kernels, so the
// trace is bitwise identical to theirs (tests/test_gpu_pipeline.py).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <limits.h>

#include <type_traits>

#include "capi_internal.h"
#include "coarse_device.cuh"
#include "fine_common.cuh"
#include "mmpr_device.cuh"
#include "regions_device.cuh"

namespace mmpr {

#ifdef MMPR_PIPE_PROFILE
// dev builds only: per-CTA cycle totals of a unit's phases (thread 0)
__device__ unsigned long long g_pipe_prof[1024][8];
#define PPROF_START long long pprof_t = clock64()
#define PPROF(k)                                                        \
  if (threadIdx.x == 0) {                                               \
    const long long pprof_now = clock64();                              \
    g_pipe_prof[blockIdx.x & 1023][k] += (unsigned long long)(pprof_now - pprof_t); \
    pprof_t = pprof_now;                                                \
  }
#else
#define PPROF_START
#define PPROF(k)
#endif

#define PL_MAX_RANKS 8

// One launch processes the units of ranks [r0, r0 + nr): every unit (k, n)
// with owner(n) in that range, in k-major order.  io[r] are rank r's
// buffers -- this process's own, or another GPU's mapped through CUDA IPC
// (peer pointers), or, in the one-GPU emulation, another set of local
// buffers.  Flags accumulate over runs: run `epoch` (1, 2, ...) waits for
// epoch * count, so ranks never reset a word a peer may still be reading.
struct PipeParams {
  FineParams f;  // model, S, P, dt, sqrt_dt, bsd, increments, cluster geometry
  mmpr_moment_ode ode;
  mmpr_model ode_model;  // the model the moment ODE was built from
  mmpr_integrator integ;
  mmpr_pipeline_io io[PL_MAX_RANKS];
  int N, K, G, Ng;  // slices, iterations, ranks, slices per rank (N = G * Ng)
  int r0;           // first rank of this launch
  int lo_n;         // first boundary index of the launch's units
  int row_units;    // units per row for this launch
  int units;
  int rank_tickets;  // one-GPU emulation of multi-GPU scheduling: cluster c serves rank r0 + c % nranks
  int nranks;        // ranks of this launch
  int reuse;  // cached predictions for converged slices (engine skip_until)
  int retain;
  int epoch;
  int sys;  // ranks on several GPUs: system-scope ordering
  long long watchdog;  // pl_wait limit in cycles (see pl_wait)
  int *abort;          // this launch's abort word (last flag word of rank r0)
  int phx;             // increments from counter-based Philox (f.cn) instead of io.xi
  int phx_fresh;       // PHILOX_FRESH: unit (k, n)'s fine part draws iteration k's increments
  mmpr_partition part;  // NR > 1: the regions
  double *rg_scratch;   // NR > 1: [clusters][NR][P] compacted members of the unit's restrictions
  int rg_rows;          // NR > 1: clusters the scratch holds (the launch uses at most this many)
};

__device__ __forceinline__ int pl_ld_acquire(const int *p, bool sys) {
  int v;
  if (sys) asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Publish after this thread's (and, through the preceding block barrier,
// the CTA's) stores: fence at the consumers' scope, then a release add.
// fence=false for "consumed" signals, which order only loads whose values
// the CTA has already used (the release alone orders this thread's).
__device__ __forceinline__ void pl_publish(int *p, int v, bool sys, bool fence = true) {
  if (sys) {
    if (fence) __threadfence_system();
    asm volatile("red.release.sys.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  } else {
    if (fence) __threadfence();
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  }
}

// Publish a value (idempotent: several threads may publish the same chain
// step with the same value) after this thread's stores.
__device__ __forceinline__ void pl_publish_value(int *p, int v, bool sys) {
  if (sys) {
    __threadfence_system();
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  } else {
    __threadfence();
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  }
}

// Spin until *p >= target.  A dependency that never arrives is a bug; the
// watchdog turns it into a kernel fault instead of a hung device.  Its limit
// (PipeParams::watchdog, set by the host) scales with the launch's work --
// at least 2^34 cycles (~9 s), else one cycle per particle-step of the whole
// launch (~300x the launch's expected duration), 8x that for a peer GPU's
// flag, whose kernel a slow host may launch late -- so a legitimate wait on
// a long-slice configuration never trips it.
// On expiry the wait sets the launch's abort word and returns: every later
// wait returns at once, the units run to completion on whatever data is
// there, and every status they write is MMPR_STAT_WATCHDOG, so the host
// raises an error instead of the context dying on a sticky trap (and a
// multi-GPU driver can fall back collectively).
__device__ __forceinline__ void pl_wait(const int *p, int target, bool sys, long long watchdog, int *abort) {
  if (pl_ld_acquire(p, sys) >= target) return;
  const long long t0 = clock64();
  const long long limit = sys ? 8 * watchdog : watchdog;
  while (pl_ld_acquire(p, sys) < target) {
    if (*(volatile int *)abort) return;
    __nanosleep(64);
    if (clock64() - t0 > limit) {
      atomicExch(abort, 1);
      return;
    }
  }
}

// data another rank produced: L2 (same GPU) or uncached (peer GPU)
__device__ __forceinline__ double pl_ld(const double *p, bool remote) { return remote ? __ldcv(p) : __ldcg(p); }
__device__ __forceinline__ int64_t pl_ld64(const int64_t *p, bool remote) {
  return remote ? (int64_t)__ldcv((const long long *)p) : (int64_t)__ldcg((const long long *)p);
}

// flag words of one rank: [0] ticket, then fine_done[K][N], chain_done[K+1][N+1], consumed[K+1][N+1],
// chain_front[K+1]
struct PlFlags {
  int *base;
  int N, K;
  __device__ int *fine_done(int k, int n) const { return base + 1 + (int64_t)k * N + n; }
  __device__ int *chain_done(int k, int n) const {
    return base + 1 + (int64_t)K * N + (int64_t)k * (N + 1) + n;
  }
  __device__ int *consumed(int k, int n) const {
    return base + 1 + (int64_t)K * N + (int64_t)(K + 1) * (N + 1) + (int64_t)k * (N + 1) + n;
  }
  // hint: epoch * (N + 2) + first boundary of row k whose chain step this
  // rank has not yet published (atomicMax, monotone across epochs)
  __device__ int *chain_front(int k) const { return base + 1 + (int64_t)K * N + 2 * (int64_t)(K + 1) * (N + 1) + k; }
};

enum { PL_KEEP = 0, PL_SET = 1, PL_AFFINE = 2 };

__device__ __forceinline__ int pl_owner(const PipeParams &pp, int m) {
  const int o = m / pp.Ng;
  return o < pp.G ? o : pp.G - 1;
}

// One step of the serial correction (engine.py:210-236): boundary m of row
// k from macro[k][m-1] (rho0 for m = 1), R(F^{k-1}_{m-1}) and the previous
// row's prediction cache[k-1][m-1] (reused as the prediction itself for a
// converged slice, m-1 < k).  io: the rank owning boundary m; iop: the owner
// of slice m-1 (another rank's exchange arrays for a rank's first boundary).
// STORE: write macro[k][m], cache[k][m-1], raw[k-1][m-1],
// coarse_status[k][m-1] and publish chain_done(k, m); the corrected state
// also goes to s_chain for the calling CTA.
template <int OK, int MK, int NR, bool STORE = true>
__device__ __forceinline__ void pl_chain_step(const PipeParams &pp, const mmpr_pipeline_io &io,
                                              const mmpr_pipeline_io &iop, const PlFlags &fl, int k, int m,
                                              bool remote, double *s_out = nullptr) {
  constexpr int NV = 3 * NR;  // means, variances, fractions per region
  const int N = pp.N;
  const double *fs = iop.fine_stats + ((int64_t)(k - 1) * N + (m - 1)) * NV;
  const double *cin = io.cache + ((int64_t)(k - 1) * N + (m - 1)) * NV;
  double cur[NV], f[NV], c[NV], pred[NV], raw[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    cur[v] = (m - 1 == 0) ? io.rho0[v] : pl_ld(iop.macro + ((int64_t)k * (N + 1) + (m - 1)) * NV + v, remote);
    f[v] = pl_ld(fs + v, remote);
    c[v] = __ldcg(cin + v);
  }
  int st = MMPR_STAT_OK;
  if (pp.reuse && m - 1 < k) {
#pragma unroll
    for (int v = 0; v < NV; ++v) pred[v] = c[v];
  } else {
#pragma unroll
    for (int v = 0; v < NV; ++v) pred[v] = cur[v];
    long long steps;
    double h;
    const double t0 = __ldg(io.times + m - 1);
    euler_grid(pp.integ.dt, t0, __ldg(io.times + m), &steps, &h);
    st = integrate_euler_n<NV, OK, MK>(pp.ode, pp.ode_model, steps, h, t0, pred);
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) raw[v] = add(f[v], sub(pred[v], c[v]));
  // variance clamp when any region's corrected variance is negative; the
  // fractions stay the fine restriction's (engine.py:218-231)
  bool neg = false;
#pragma unroll
  for (int i = 0; i < NR; ++i) neg |= raw[NR + i] < 0.0;
  double nxt[NV];
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    nxt[i] = raw[i];
    nxt[NR + i] = (neg && raw[NR + i] < 0.0) ? 0.0 : raw[NR + i];
    nxt[2 * NR + i] = f[2 * NR + i];
  }
  if (s_out) {
#pragma unroll
    for (int v = 0; v < NV; ++v) s_out[v] = nxt[v];
  }
  if (STORE) {
    const int64_t e = (int64_t)(k - 1) * N + (m - 1);
    io.coarse_status[(int64_t)k * N + (m - 1)] = st;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      io.cache[((int64_t)k * N + (m - 1)) * NV + v] = pred[v];
      io.raw[e * NV + v] = raw[v];
      io.macro[((int64_t)k * (N + 1) + m) * NV + v] = nxt[v];
    }
    pl_publish_value(fl.chain_done(k, m), pp.epoch, pp.sys != 0);
  }
}

// Several ranks: advance rank r's chain of row k over its boundaries from
// the published frontier -- waiting for the inputs of boundaries up to
// n_must, stopping at the first boundary beyond it whose inputs are not yet
// there.  Called by the first CTA of every unit that needs a boundary, so a
// rank hands its last chain value to the next rank soon after its previous
// row is done instead of only when its last unit of the row starts.
// Steps evaluated twice (by two units racing) are identical and publish the
// same value.
template <int OK, int MK, int NR>
__device__ __forceinline__ void pl_advance_chain(const PipeParams &pp, int k, int r, int n_must) {
  const int N = pp.N, K = pp.K, ep = pp.epoch, cdone = pp.epoch * pp.f.ctas;
  const bool sys = pp.sys != 0;
  const mmpr_pipeline_io &io = pp.io[r];
  const PlFlags fl{io.flags, N, K};
  const int hi = (r == pp.G - 1) ? N : (r + 1) * pp.Ng - 1;
  const int lo = r * pp.Ng > 1 ? r * pp.Ng : 1;
  const int fr = *(volatile int *)fl.chain_front(k) - ep * (N + 2);
  for (int m = fr > lo ? fr : lo; m <= hi; ++m) {
    if (pl_ld_acquire(fl.chain_done(k, m), false) >= ep) continue;
    const int om = pl_owner(pp, m - 1);
    const mmpr_pipeline_io &iom = pp.io[om];
    const PlFlags flm{iom.flags, N, K};
    const bool rem = om != r;
    const bool msys = sys && rem;
    if (m > n_must) {
      if (pl_ld_acquire(flm.fine_done(k - 1, m - 1), msys) < cdone) return;
      if (m - 1 >= 1 && pl_ld_acquire(flm.chain_done(k, m - 1), msys) < ep) return;
      if (k - 1 >= 1 && pl_ld_acquire(fl.chain_done(k - 1, m), false) < ep) return;
    } else {
      pl_wait(flm.fine_done(k - 1, m - 1), cdone, msys, pp.watchdog, pp.abort);
      if (m - 1 >= 1) pl_wait(flm.chain_done(k, m - 1), ep, msys, pp.watchdog, pp.abort);
      if (k - 1 >= 1) pl_wait(fl.chain_done(k - 1, m), ep, false, pp.watchdog, pp.abort);
    }
    pl_chain_step<OK, MK, NR>(pp, io, iom, fl, k, m, rem);
    atomicMax(fl.chain_front(k), ep * (N + 2) + m + 1);
  }
}

// MULTI = false: one rank (the single-GPU engine); the rank table collapses
// to io[0] at compile time and the step loop keeps every value in registers.
// PHX: every unit's increments come from counter-based Philox in registers
// (counter_noise.cuh) -- the dynamic shared memory holds the ziggurat tables
// and the increment copies, their mbarriers and the L2 prefetch disappear.
// NR: regions of the partition (bimodal configs: 2) -- the match is per
// region with membership from the pre-transform positions, and R(u^k_n) /
// R(F^k_n) are region restrictions over compacted members (rg_restrict,
// regions_device.cuh) instead of the single-region tree passes.
// LOW >= 0 (the any-size form, PPT = 16): every leaf has at least LOW
// accumulator elements per lane (numpy's leaves hold 64..128 particles once
// an ensemble has more than one, so 8), the rest carry a predicate.
template <int KIND, int PPT, bool HAS_TAIL, int OK, int MK, bool MULTI, bool PHX = false, int NR = 1, int LOW = -1>
__global__ void __launch_bounds__(512, PHX ? MMPR_PHX_MINB : 2) pipeline_kernel(const PipeParams pp) {
  constexpr int LO = LOW >= 0 ? LOW : PPT - 1;  // LOW < 0: every leaf has PPT-1 or PPT elements per lane
  constexpr int NV = 3 * NR;   // macro state: means, variances, fractions per region
  using PartT = Part<false>;
  const FineParams &p = pp.f;
  extern __shared__ __align__(128) double s_stage[];  // [nstages][stage_elems]
  __shared__ PartT s_wp[2][32];
  __shared__ __align__(16) ClusterSlot s_slot[2][FS_MAX_CLUSTER];
  __shared__ int s_bad[3];
  __shared__ __align__(8) uint64_t s_bar[FS_MAX_STAGES];
  __shared__ __align__(8) uint64_t s_red_bar[2];
  __shared__ int s_ticket[2];
  __shared__ double s_mu[NR], s_scale[NR], s_mc[NR];  // per-region match maps
  __shared__ double s_chain[NV];  // this CTA's evaluation of the corrected state (one rank)
  __shared__ int s_mode[NR];
  __shared__ std::conditional_t<(NR > 1), RgSmem, char> s_rg;  // region restriction (NR > 1 only)
  // the partition in shared memory: the out-of-line restriction takes it by
  // reference, and a reference into the kernel parameters would make the
  // compiler copy the whole parameter block into the stack frame
  __shared__ std::conditional_t<(NR > 1), mmpr_partition, char> s_part;
  __shared__ const double *s_xi_base;  // this CTA's increments of the unit's slice, step 0
  __shared__ uint32_t s_stage_bytes;

  const int lane = threadIdx.x & 31;
  const int gthreads = (int)blockDim.x;
  const int tid = (int)threadIdx.x;
  const int warp = tid >> 5;
  const int nwarps = gthreads >> 5;
  const int rank = (p.ctas > 1) ? (int)cluster_ctarank() : 0;
  const int N = pp.N, K = pp.K;

  // ---- my leaf (fine.cu layout; P < 2^31 here, so 32-bit offsets) ------------
  const int64_t slot = (int64_t)rank * p.slots_per_cta + warp * 4 + (lane >> 3);
  const int j8 = lane & 7;
  int off, cnt, tail, tail_off, lo;
  {
    int64_t o64 = 0, l64 = 0, lo64, hi64, o2, l2;
    pw_leaf(p.P, p.D, slot, &o64, &l64);
    pw_leaf(p.P, p.D, (int64_t)rank * p.slots_per_cta, &lo64, &l2);
    if (rank == p.ctas - 1) hi64 = p.P;
    else pw_leaf(p.P, p.D, (int64_t)(rank + 1) * p.slots_per_cta, &hi64, &o2);
    off = (int)o64;
    cnt = (int)(l64 >> 3);
    tail = (int)(l64 & 7);
    tail_off = (int)(o64 + (l64 & ~int64_t(7)));
    lo = (int)lo64;
    if (tid == 0) s_stage_bytes = (uint32_t)((((hi64 - lo64) * 8) + 15) & ~int64_t(15));
  }
  const int my_idx = off - lo + j8;
  // trailing particles exist in the ensemble's last leaf only: the other warps skip their fold
  const bool warp_tail = HAS_TAIL && __any_sync(MMPR_FULL_MASK, tail != 0);
  const int ns = p.nstages;
  const cn::ZigTables *zt = reinterpret_cast<const cn::ZigTables *>(s_stage);
  if constexpr (PHX) cn::load_zig(reinterpret_cast<cn::ZigTables *>(s_stage), tid, gthreads);
  // PHX: this thread's increment column, generated one step ahead (cn::gen)
  double *zb = reinterpret_cast<double *>(reinterpret_cast<char *>(s_stage) + sizeof(cn::ZigTables)) + tid;

  if constexpr (NR > 1) {
    if (tid == 0) s_part = pp.part;
  }
  if (tid == 0) {
    for (int q = 0; q < ns; ++q) mbar_init(&s_bar[q], 1);
    mbar_init(&s_red_bar[0], 1);
    mbar_init(&s_red_bar[1], 1);
    fence_mbar_init();
    s_bad[0] = s_bad[1] = s_bad[2] = 0;
  }
  if (p.ctas > 1) cluster_sync_all();
  else __syncthreads();

  double x[PPT];
  double xt = 0.0;
  uint32_t ld = 0;  // increment loads issued (and completed) before this unit
  uint32_t r = 0;   // reduction calls made by this CTA (cluster-uniform sequence)

  // Pairwise-tree sum of x (or of (x - c)^2) over the ensemble, then / P;
  // as fine.cu's reduce (B1, warp fold, one st.async per peer CTA).
  // `refill` >= 0: the unit's step whose increments go into the stage freed
  // by the step just taken.
  // PHX: `gen_step` >= 0 generates that step's increments of slice `gen_n`
  // while the partials are in flight (cn::gen).
  auto reduce = [&](auto centered, double c, int refill, double &mean_out, int &bad_out, int gen_step = -1,
                    uint32_t gen_key = 0) {
    constexpr bool CEN = decltype(centered)::value;
    auto f = [&](double v) {
      if constexpr (CEN) {
        const double d = sub(v, c);
        return mul(d, d);
      } else {
        return v;
      }
    };
    const int par = r & 1;
    const int bslot = r % 3;
    double acc = f(x[0]);
#pragma unroll
    for (int m = 1; m < PPT; ++m) {
      if (m < LO) {
        acc = add(acc, f(x[m]));
      } else {
        const double t = add(acc, f(x[m]));
        acc = (m < cnt) ? t : acc;
      }
    }
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 1));
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 2));
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 4));
    if (HAS_TAIL && warp_tail) {  // (warp-uniform: only the warp holding the ensemble's last leaf)
      const double ft = f(xt);
#pragma unroll
      for (int i = 0; i < 7; ++i) {
        const double v = __shfl_sync(MMPR_FULL_MASK, ft, (lane & ~7) | i);
        if (i < tail) acc = add(acc, v);
      }
    }
    int bad_local = 0;
    if (!CEN && !finite(acc)) {
#pragma unroll
      for (int m = 0; m < PPT; ++m) bad_local |= (m < cnt && !finite(x[m])) ? 1 : 0;
      if (HAS_TAIL && j8 < tail) bad_local |= !finite(xt);
    }
    const int wbad = __any_sync(MMPR_FULL_MASK, bad_local);
    PartT leaf = PartT::make(acc, true);
    leaf = leaf.xor_level(lane, 8);
    leaf = leaf.xor_level(lane, 16);
    if (lane == 0) {
      s_wp[par][warp] = leaf;
      if (wbad) s_bad[bslot] = 1;
    }
    __syncthreads();  // B1
    if (tid == gthreads - 32) {
      s_bad[(r + 2) % 3] = 0;
      if (refill >= 0) {
        const uint32_t q = ld + (uint32_t)refill;
        const int st = (int)(q % (uint32_t)ns);
        const uint32_t bytes = s_stage_bytes;
        const double *base = s_xi_base;
        mbar_arrive_expect_tx(&s_bar[st], bytes);
        bulk_g2s(s_stage + st * p.stage_elems, base + (int64_t)refill * p.xi_row_pitch, bytes, &s_bar[st]);
        const int pf = refill + p.l2_ahead;
        if (p.l2_ahead > 0 && pf < p.S) prefetch_l2(base + (int64_t)pf * p.xi_row_pitch, bytes);
      }
    }
    PartT v = (lane < nwarps) ? s_wp[par][lane] : PartT::make(0.0, false);
#pragma unroll
    for (int m = 1; m < 32; m <<= 1)
      if (m < nwarps) v = v.xor_level(lane, m);
    double total;
    int bad = s_bad[bslot];
    if (p.ctas > 1) {
      if (tid == 0) mbar_arrive_expect_tx(&s_red_bar[par], 16u * (uint32_t)p.ctas);
      if (warp == 0 && lane < p.ctas) {
        const uint32_t remote = mapa_shared(smem_addr(&s_slot[par][rank]), (uint32_t)lane);
        const uint32_t rbar = mapa_shared(smem_addr(&s_red_bar[par]), (uint32_t)lane);
        st_async_v2(remote, __double_as_longlong(v.v),
                    (unsigned long long)1u | ((unsigned long long)(uint32_t)bad << 32), rbar);
      }
      if (PHX && gen_step >= 0)
        cn::gen<PPT, LO, HAS_TAIL>(gen_key, (uint32_t)gen_step, zt, zb, gthreads, (uint32_t)(off + j8), cnt,
                                   (uint32_t)(tail_off + j8), j8 < tail);
      mbar_wait_parity(&s_red_bar[par], (r >> 1) & 1u);
      PartT cc = PartT::make(0.0, false);
      int b = 0;
      if (lane < p.ctas) {
        cc = PartT::make(s_slot[par][lane].v, true);
        b = s_slot[par][lane].bad;
      }
#pragma unroll
      for (int m = 1; m < FS_MAX_CLUSTER; m <<= 1)
        if (m < p.ctas) cc = cc.xor_level(lane, m);
      total = __shfl_sync(MMPR_FULL_MASK, cc.v, 0);
      bad = __any_sync(MMPR_FULL_MASK, b);
    } else {
      total = __shfl_sync(MMPR_FULL_MASK, v.v, 0);
      if (PHX && gen_step >= 0)
        cn::gen<PPT, LO, HAS_TAIL>(gen_key, (uint32_t)gen_step, zt, zb, gthreads, (uint32_t)(off + j8), cnt,
                                   (uint32_t)(tail_off + j8), j8 < tail);
    }
    mean_out = div(total, (double)p.P);
    bad_out = bad;
    ++r;
  };
  using Plain = std::integral_constant<bool, false>;
  using Centered = std::integral_constant<bool, true>;

  // (read from the parameter bank at each use: nothing here stays live in
  // registers across the step loop)
#define sys (MULTI && pp.sys != 0)
#define ep (pp.epoch)
#define cdone (pp.epoch * p.ctas)  // a flag every CTA of a unit's cluster adds to
  auto owner = [&](int m) {
    if constexpr (!MULTI) return 0;
    const int o = m / pp.Ng;
    return o < pp.G ? o : pp.G - 1;
  };
  for (int it = 0;; ++it) {
    // ---- next ticket, broadcast to the cluster ---------------------------------
    if (rank == 0 && tid == 0) {
      int t;
      if (MULTI && pp.rank_tickets) {
        // rank rr's own units in (k, n) order, encoded as k * (N + 1) + n
        const int rr = pp.r0 + (int)(blockIdx.x / p.ctas) % pp.nranks;
        const int lo = rr * pp.Ng, hi = (rr == pp.G - 1) ? N : (rr + 1) * pp.Ng - 1;
        const int ru = hi - lo + 1;
        const int q = atomicAdd(pp.io[rr].flags, 1);
        t = q >= (K + 1) * ru ? INT_MAX : (q / ru) * (N + 1) + lo + q % ru;
      } else {
        t = atomicAdd(pp.io[pp.r0].flags, 1);
      }
      if (p.ctas > 1) {
        for (int c = 0; c < p.ctas; ++c) st_cluster_u32(mapa_shared(smem_addr(&s_ticket[it & 1]), (uint32_t)c), t);
      } else {
        s_ticket[it & 1] = t;
      }
    }
    if (p.ctas > 1) cluster_sync_all();
    else __syncthreads();
    const int t = s_ticket[it & 1];
    if (MULTI && pp.rank_tickets ? t == INT_MAX : t >= pp.units) break;
    const int k = (MULTI && pp.rank_tickets) ? t / (N + 1) : t / pp.row_units;
    const int n = (MULTI && pp.rank_tickets) ? t % (N + 1) : pp.lo_n + t % pp.row_units;
    const int r = owner(n);
    const mmpr_pipeline_io &io = pp.io[r];
    const PlFlags fl{io.flags, N, K};
    const bool has_match = k >= 1 && n >= 1;
    const bool has_fine = k < K && n < N;
    const int64_t srow = pp.retain ? k : (k & 1);
    double *snap_kn = io.snap + srow * io.snap_iter_stride + (int64_t)n * io.snap_slice_pitch;

    // the increments do not depend on anything: start their copies first
    if (!PHX && has_fine && tid == 0) {
      const double *base = io.xi + (int64_t)(n - r * pp.Ng) * io.xi_slice_pitch + lo;
      const uint32_t bytes = s_stage_bytes;
      s_xi_base = base;  // read by the refill thread after the next block barrier
      for (int j = 0; j < ns && j < p.S; ++j) {
        const int st = (int)((ld + (uint32_t)j) % (uint32_t)ns);
        mbar_arrive_expect_tx(&s_bar[st], bytes);
        bulk_g2s(s_stage + st * p.stage_elems, base + (int64_t)j * p.xi_row_pitch, bytes, &s_bar[st]);
      }
      for (int j = ns; j < ns + p.l2_ahead && j < p.S; ++j) prefetch_l2(base + (int64_t)j * p.xi_row_pitch, bytes);
    }

    double s = 0.0;
    bool mean_known = false;
    PPROF_START;
    if (has_match) {
      // F^{k-1}_{n-1}, its restriction and macro[k][n-1] belong to the owner
      // of slice n-1 (another rank for the first slice of a rank)
      const int rp = owner(n - 1);
      const mmpr_pipeline_io &iop = pp.io[rp];
      const PlFlags flp{iop.flags, N, K};
      const bool remote = rp != r;
      const bool rsys = sys && remote;
      // F^{k-1}_{n-1} complete: its loads go out first and land while thread 0
      // evaluates the serial correction
      if (tid == 0) pl_wait(flp.fine_done(k - 1, n - 1), cdone, rsys, pp.watchdog, pp.abort);
      __syncthreads();
      PPROF(0);
      const double *src = iop.fine + ((int64_t)((k - 1) & 1) * N + (n - 1)) * iop.fine_pitch;
#pragma unroll
      for (int m = 0; m < PPT; ++m) x[m] = (m < cnt) ? pl_ld(src + off + j8 + 8 * m, remote) : 0.0;
      if (HAS_TAIL && j8 < tail) xt = pl_ld(src + tail_off + j8, remote);
      // ---- serial correction of boundary n, then the match parameters ---------
      if (tid == 0) {
        if constexpr (MULTI) {
          // the chain of row k advances independently of unit order
          // (pl_advance_chain); other CTAs only wait for boundary n
          if (rank == 0) pl_advance_chain<OK, MK, NR>(pp, k, r, n);
          else pl_wait(fl.chain_done(k, n), ep, false, pp.watchdog, pp.abort);
        } else {
          // one rank: the chain follows the ticket order; every CTA evaluates
          // the step (identically) and the first CTA publishes it
          if (n - 1 >= 1) pl_wait(flp.chain_done(k, n - 1), ep, rsys, pp.watchdog, pp.abort);
          if (k - 1 >= 1) pl_wait(fl.chain_done(k - 1, n), ep, false, pp.watchdog, pp.abort);
          if (rank == 0) pl_chain_step<OK, MK, NR>(pp, io, iop, fl, k, n, remote, s_chain);
          else pl_chain_step<OK, MK, NR, false>(pp, io, iop, fl, k, n, remote, s_chain);
        }
        // row 0's reader of this snapshot slot (units (0, n < N) read it)
        if (!pp.retain && k == 2 && n < N) pl_wait(fl.consumed(0, n), cdone, false, pp.watchdog, pp.abort);
        double nxt[NV], f[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          nxt[v] = MULTI ? __ldcg(io.macro + ((int64_t)k * (N + 1) + n) * NV + v) : s_chain[v];
          f[v] = pl_ld(iop.fine_stats + ((int64_t)(k - 1) * N + (n - 1)) * NV + v, remote);
        }
        // match(corrected, F^{k-1}_{n-1}), raise policy (coupling.py:32-95):
        // per region an affine map onto the corrected moments; an empty
        // region is skipped, the first degenerate one is the status
        int status = MMPR_STAT_OK;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const int64_t cn = pl_ld64(iop.fine_counts + ((int64_t)(k - 1) * N + (n - 1)) * NR + q, remote);
          int mode = PL_KEEP;
          double scale = 1.0, mc = 0.0, mu = 0.0;
          if (cn != 0) {
            mu = nxt[q];
            double var_t = nxt[NR + q];
            if (var_t < 0.0) var_t = 0.0;
            mc = f[q];
            const double cur_var = f[NR + q];
            if (cur_var == 0.0) {
              if (var_t > 0.0 && status == MMPR_STAT_OK) status = q;
              mode = PL_SET;
            } else {
              scale = __dsqrt_rn(div(var_t, cur_var));
              if (!(scale == 1.0 && mu == mc)) mode = PL_AFFINE;
            }
          }
          s_mu[q] = mu;
          s_scale[q] = scale;
          s_mc[q] = mc;
          s_mode[q] = mode;
        }
        if (rank == 0)
          io.match_status[(int64_t)k * N + (n - 1)] = *(volatile int *)pp.abort ? MMPR_STAT_WATCHDOG : status;
      }
      __syncthreads();
      // membership from the pre-transform position (coupling.py:54)
      auto apply = [&](double v) {
        int q = 0;
        if constexpr (NR > 1) q = rg_region<NR>(s_part, v);
        const int mode = s_mode[q];
        const double mu = s_mu[q];
        return mode == PL_SET ? mu : (mode == PL_AFFINE ? add(mul(s_scale[q], sub(v, s_mc[q])), mu) : v);
      };
#pragma unroll
      for (int m = 0; m < PPT; ++m) x[m] = apply(x[m]);
      if (HAS_TAIL) xt = apply(xt);
      __syncthreads();  // every load of the source slot has returned
      if (tid == 0) pl_publish(flp.consumed(k, n), 1, sys, false);  // the slot's owner waits on it
#pragma unroll
      for (int m = 0; m < PPT; ++m)
        if (m < cnt) snap_kn[off + j8 + 8 * m] = x[m];
      if (HAS_TAIL && j8 < tail) snap_kn[tail_off + j8] = xt;
      PPROF(1);
      // micro restriction R(u^k_n) from registers (np.mean, two-pass np.var)
      if constexpr (NR == 1) {
        double var;
        int b0;
        reduce(Plain{}, 0.0, -1, s, b0);
        reduce(Centered{}, s, -1, var, b0, (PHX && has_fine && p.S > 0) ? 0 : -1,
               pp.phx_fresh ? p.cn.k0 ^ ((uint32_t)n | ((uint32_t)(k + 1) << 20)) : cn::slice_key(p.cn, (uint32_t)n));
        mean_known = true;
        if (rank == 0 && tid == 0) {
          double *mo = io.micro + ((int64_t)k * (N + 1) + n) * 3;
          mo[0] = s;
          mo[1] = var;
          mo[2] = div((double)p.P, (double)p.P);
          io.micro_counts[(int64_t)k * (N + 1) + n] = p.P;
        }
      } else {
        const int64_t e = (int64_t)k * (N + 1) + n;
        rg_restrict_reload<PPT, HAS_TAIL, NR>(s_rg, snap_kn, off, cnt, tail, p.ctas, rank, s_part, p.P,
                                          pp.rg_scratch + (int64_t)(blockIdx.x / p.ctas) * NR * p.P,
                                          io.micro + e * NV, io.micro_counts + e * NR);
        // the particles again from the snapshot this thread just wrote: no
        // value of x stays live across the call (which would keep the whole
        // array in the stack frame through the step loop)
#pragma unroll
        for (int m = 0; m < PPT; ++m) x[m] = (m < cnt) ? snap_kn[off + j8 + 8 * m] : 0.0;
        xt = (HAS_TAIL && j8 < tail) ? snap_kn[tail_off + j8] : 0.0;
      }
    } else if (k >= 1) {
      // n == 0: u^k_0 = ens0 (engine.py:208); boundary-0 rows of the trace
#pragma unroll
      for (int m = 0; m < PPT; ++m) x[m] = (m < cnt) ? io.x0[off + j8 + 8 * m] : 0.0;
      if (HAS_TAIL && j8 < tail) xt = io.x0[tail_off + j8];
#pragma unroll
      for (int m = 0; m < PPT; ++m)
        if (m < cnt) snap_kn[off + j8 + 8 * m] = x[m];
      if (HAS_TAIL && j8 < tail) snap_kn[tail_off + j8] = xt;
      if (rank == 0 && tid == 0) {
        const int64_t e = (int64_t)k * (N + 1);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          io.macro[e * NV + v] = io.rho0[v];
          io.micro[e * NV + v] = io.rho0[v];
        }
#pragma unroll
        for (int q = 0; q < NR; ++q) io.micro_counts[e * NR + q] = io.counts0[q];
      }
    } else if (has_fine) {
      // row 0: the lifted ensembles written by the prologue
#pragma unroll
      for (int m = 0; m < PPT; ++m) x[m] = (m < cnt) ? snap_kn[off + j8 + 8 * m] : 0.0;
      if (HAS_TAIL && j8 < tail) xt = snap_kn[tail_off + j8];
      if (!pp.retain) {
        __syncthreads();
        if (tid == 0) pl_publish(fl.consumed(0, n), 1, false, false);
      }
    }

    if (has_fine) {
      // ---- F(u^k_n): S Euler-Maruyama steps, particles in registers ------------
      PPROF(2);
      int bad = 0;
      // (fresh counter noise: iteration k's field, as the per-iteration sweep's
      // plan.counter_noise(k))
      const uint32_t nkey = pp.phx_fresh ? p.cn.k0 ^ ((uint32_t)n | ((uint32_t)(k + 1) << 20))
                                         : cn::slice_key(p.cn, (uint32_t)n);
      if (io.fine_times && rank == 0 && tid == 0) io.fine_times[((int64_t)k * N + n) * 2] = globaltimer_ns();
      if (!mean_known) reduce(Plain{}, 0.0, -1, s, bad, (PHX && p.S > 0) ? 0 : -1, nkey);
      int first_bad = MMPR_STAT_OK;
      for (int j = 0; j < p.S; ++j) {
        const uint32_t lj = ld + (uint32_t)j;
        const int stage = (int)(lj % (uint32_t)ns);
        if constexpr (PHX) {
          // this step's increments were generated during the previous reduction
#pragma unroll
          for (int m = 0; m < PPT; ++m)
            if (m < LO || m < cnt) x[m] = em_update<KIND>(p, x[m], s, zb[m * gthreads]);
          if (HAS_TAIL && j8 < tail) xt = em_update<KIND>(p, xt, s, zb[PPT * gthreads]);
        } else {
          mbar_wait_parity(&s_bar[stage], (lj / (uint32_t)ns) & 1u);
          const double *xb = s_stage + stage * p.stage_elems;
#pragma unroll
          for (int m = 0; m < PPT; ++m) {
            if (m < LO) {
              x[m] = em_update<KIND>(p, x[m], s, xb[my_idx + 8 * m]);
            } else {
              // past a shorter leaf this reads up to 8 (PPT - LO) doubles
              // beyond the CTA's range (into the next stage or the pad after
              // the last): the value is discarded, so no clamp is needed
              const double nx = em_update<KIND>(p, x[m], s, xb[my_idx + 8 * m]);
              x[m] = (m < cnt) ? nx : x[m];
            }
          }
          if (HAS_TAIL && warp_tail && j8 < tail) xt = em_update<KIND>(p, xt, s, xb[(int)(tail_off - lo) + j8]);
        }
        reduce(Plain{}, 0.0, (!PHX && j + ns < p.S) ? j + ns : -1, s, bad, (PHX && j + 1 < p.S) ? j + 1 : -1, nkey);
        if (bad) {
          first_bad = j;
          break;
        }
      }
      // loads issued for this unit: the first min(ns, S) plus one refill per
      // completed step while j + ns < S
      const int init = PHX ? 0 : (ns < p.S ? ns : p.S);
      const int done_steps = first_bad == MMPR_STAT_OK ? p.S : first_bad + 1;
      const int refills = PHX ? 0 : max(0, min(done_steps, p.S - ns));
      const int issued = init + refills;
      if (tid == gthreads - 32 && first_bad != MMPR_STAT_OK) {
        for (int j = first_bad + 1; j < issued; ++j) {
          const uint32_t lj = ld + (uint32_t)j;
          mbar_wait_parity(&s_bar[lj % (uint32_t)ns], (lj / (uint32_t)ns) & 1u);
        }
      }
      ld += (uint32_t)issued;
      // the unit's coordinates again from shared memory (not held in
      // registers across the step loop)
      const int tt = *(volatile int *)&s_ticket[it & 1];
      const int k = (MULTI && pp.rank_tickets) ? tt / (N + 1) : tt / pp.row_units;
      const int n = (MULTI && pp.rank_tickets) ? tt % (N + 1) : pp.lo_n + tt % pp.row_units;
      const int r = owner(n);
      const mmpr_pipeline_io &io = pp.io[r];
      const PlFlags fl{io.flags, N, K};
      if (io.fine_times && rank == 0 && tid == 0) io.fine_times[((int64_t)k * N + n) * 2 + 1] = globaltimer_ns();

      PPROF(3);
      // ---- write F^k_n into the parity buffer, restriction, publish -------------
      if (k >= 2) {
        // the reader of F^{k-2}_n (unit (k-1, n+1), owner of slice n+1) is done
        if (tid == 0) pl_wait(fl.consumed(k - 1, n + 1), cdone, sys && owner(n + 1) != r, pp.watchdog, pp.abort);
        __syncthreads();
      }
      double *xo = io.fine + ((int64_t)(k & 1) * N + n) * io.fine_pitch;
#pragma unroll
      for (int m = 0; m < PPT; ++m)
        if (m < cnt) xo[off + j8 + 8 * m] = x[m];
      if (HAS_TAIL && j8 < tail) xo[tail_off + j8] = xt;
      double var = 0.0;
      const bool ok = first_bad == MMPR_STAT_OK;
      if (ok) {
        if constexpr (NR == 1) {
          int b2;
          reduce(Centered{}, s, -1, var, b2);
        } else {
          const int64_t e = (int64_t)k * N + n;
          rg_restrict_reload<PPT, HAS_TAIL, NR>(s_rg, xo, off, cnt, tail, p.ctas, rank, s_part, p.P,
                                            pp.rg_scratch + (int64_t)(blockIdx.x / p.ctas) * NR * p.P,
                                            io.fine_stats + e * NV, io.fine_counts + e * NR);
        }
      }
      if (rank == 0 && tid == 0) {
        const int64_t e = (int64_t)k * N + n;
        io.bad[e] = *(volatile int *)pp.abort ? MMPR_STAT_WATCHDOG : first_bad;
        if (ok && NR == 1) {
          io.fine_stats[e * 3 + 0] = s;
          io.fine_stats[e * 3 + 1] = var;
          io.fine_stats[e * 3 + 2] = div((double)p.P, (double)p.P);
          io.fine_counts[e] = p.P;
        }
      }
      __syncthreads();
      if (tid == 0) pl_publish(fl.fine_done(k, n), 1, sys);
      PPROF(4);
      if (threadIdx.x == 0) {
#ifdef MMPR_PIPE_PROFILE
        g_pipe_prof[blockIdx.x & 1023][5] += 1;
#endif
      }
    }
  }
}
#undef sys
#undef ep
#undef cdone

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct PipeGeometry {
  int D, spc, ctas, threads, stage_elems, nstages, ppt;
  bool exact;  // every leaf has ppt-1 or ppt elements per lane and ppt is instantiated (else the any-size form)
  size_t smem;
  bool tail;
};

// The pipeline covers the cluster geometries of the fine sweep whose leaves
// hold PPT-1 or PPT accumulator elements per lane for an instantiated PPT:
// 13 (96..104-particle leaves: P = 1e5 and its binary fractions down to
// 6.25e3 -- BASELINE configs 2-4), 10 (72..80: P = 1e4, 2e4, 4e4, 8e4 --
// BASELINE config 1) and 16 (120..128: the powers of two from 2^13 to 2^17
// and sizes just below them), one cluster of up to 16 CTAs per unit -- 64
// leaf slots (512 threads) per CTA from 512 slots on, 32 (256 threads)
// below, where a launch has too few units to fill the SMs otherwise.  Any
// other size within one cluster (more than 4096 particles, at most 2^17)
// takes the any-size form: 16 elements per lane, the first 8 unconditional
// (numpy's leaves hold 64..128 particles), the rest predicated.
static int pipe_geometry(int64_t P, PipeGeometry *g) {
  if (P < 1) return MMPR_ERR_ARG;
  const int D = pw_depth(P);
  const int64_t nslots = int64_t(1) << D;
  if (nslots < 64 || nslots > 1024) return MMPR_ERR_UNSUPPORTED;
  int64_t max_leaf = 0, min_leaf = INT64_MAX;
  for (int64_t s = 0; s < nslots; ++s) {
    int64_t o, l;
    pw_leaf(P, D, s, &o, &l);
    if (l > max_leaf) max_leaf = l;
    if (l < min_leaf) min_leaf = l;
  }
  // accumulator elements per lane: a leaf of 8 c + r particles holds c per lane and its r < 8 trailing
  // ones (only the last leaf of an ensemble whose size is not a multiple of 8 has any) in the tail element
  int max_cnt = (int)((P % 8) ? (max_leaf >> 3) : (max_leaf + 7) / 8);
  if (max_cnt < 1) max_cnt = 1;
  const int min_cnt = (int)(min_leaf >> 3);
  // the smallest specialised element count every leaf fits (PPT-1 or PPT elements per lane), else the
  // any-size form
  g->exact = false;
  g->ppt = 16;
  for (int ppt : {10, 13, 16})
    if (!g->exact && max_cnt <= ppt && min_cnt >= ppt - 1) {
      g->exact = true;
      g->ppt = ppt;
    }
  if (!g->exact && (max_cnt > 16 || min_cnt < 8)) return MMPR_ERR_UNSUPPORTED;
  g->D = D;
  g->spc = nslots >= 512 ? 64 : 32;
  g->ctas = (int)(nslots / g->spc);
  g->threads = g->spc * 8;
  int64_t max_range = 0;
  for (int c = 0; c < g->ctas; ++c) {
    int64_t lo, hi, l;
    pw_leaf(P, D, (int64_t)c * g->spc, &lo, &l);
    if (c == g->ctas - 1) hi = P;
    else pw_leaf(P, D, (int64_t)(c + 1) * g->spc, &hi, &l);
    if (hi - lo > max_range) max_range = hi - lo;
  }
  g->stage_elems = (int)((max_range + 1) & ~int64_t(1));
  g->nstages = 2;
  // + pad for the unclamped elements past a short leaf (8 doubles per missing element)
  g->smem = (size_t)g->stage_elems * 8 * g->nstages + (g->exact ? 64 : 8 * 8 * 8);
  // two CTAs per SM where the stages allow it (P ~ 2^16 and 2^17 keep one: 64 KB per stage)
  if (g->smem > 226 * 1024) return MMPR_ERR_UNSUPPORTED;
  g->tail = (P % 8) != 0;
  return MMPR_OK;
}

template <void (*KERN)(const PipeParams)>
static int launch_pipe(const PipeParams &pp, const PipeGeometry &g, cudaStream_t stream) {
  static int configured_smem_dev[MMPR_MAX_DEVICES] = {};
  static int clusters_dev[MMPR_MAX_DEVICES] = {};
  const int dev = mmpr_current_device();
  cudaError_t err;
  if ((int)g.smem > configured_smem_dev[dev]) {
    err = cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
    if (err != cudaSuccess) return mmpr_check(err, "pipeline: smem attribute");
    err = cudaFuncSetAttribute(KERN, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return mmpr_check(err, "pipeline: non-portable cluster");
    configured_smem_dev[dev] = (int)g.smem;
    clusters_dev[dev] = 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3((unsigned)g.threads, 1, 1);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)g.ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (clusters_dev[dev] == 0) {
    // persistent grid: the clusters that can be co-resident (tickets are
    // taken at run time, so a cluster that is not resident never blocks one
    // that is)
    cfg.gridDim = dim3((unsigned)g.ctas, 1, 1);
    int n = 0;
    err = cudaOccupancyMaxActiveClusters(&n, KERN, &cfg);
    if (err != cudaSuccess) return mmpr_check(err, "pipeline: cudaOccupancyMaxActiveClusters");
    if (n < 1) return MMPR_ERR_UNSUPPORTED;
    clusters_dev[dev] = n;
  }
  int clusters = clusters_dev[dev];
  if (const char *env = getenv("MMPR_PIPELINE_CLUSTERS")) {  // tuning override
    const int v = atoi(env);
    if (v >= 1 && v < clusters) clusters = v;
  }
  if (clusters > pp.units) clusters = pp.units;
  if (pp.rg_rows > 0 && clusters > pp.rg_rows) clusters = pp.rg_rows;
  cfg.gridDim = dim3((unsigned)(clusters * g.ctas), 1, 1);
  err = cudaLaunchKernelEx(&cfg, KERN, pp);
  if (err == cudaSuccess) mmpr_launched();
  return mmpr_check(err, "pipeline_kernel launch");
}

// two regions: one rank, numpy-stream or injected increments
template <int KIND, int OK, int MK>
static int dispatch_pipe_regions(const PipeParams &pp, const PipeGeometry &g, cudaStream_t s) {
  if (pp.phx || pp.G > 1) return MMPR_ERR_UNSUPPORTED;
  if (g.tail) return launch_pipe<pipeline_kernel<KIND, 13, true, OK, MK, false, false, 2>>(pp, g, s);
  return launch_pipe<pipeline_kernel<KIND, 13, false, OK, MK, false, false, 2>>(pp, g, s);
}

template <int KIND, int OK, int MK>
static int dispatch_pipe_tail(const PipeParams &pp, const PipeGeometry &g, cudaStream_t s) {
  if (g.ppt != 13 || !g.exact) {  // the other geometries: one rank, numpy-stream or injected increments
    if (pp.phx || pp.G > 1) return MMPR_ERR_UNSUPPORTED;
    if (!g.exact) {  // any size within one cluster: 16 elements per lane, at least 8 of them populated
      if (g.tail) return launch_pipe<pipeline_kernel<KIND, 16, true, OK, MK, false, false, 1, 8>>(pp, g, s);
      return launch_pipe<pipeline_kernel<KIND, 16, false, OK, MK, false, false, 1, 8>>(pp, g, s);
    }
    if (g.ppt == 16) {
      if (g.tail) return launch_pipe<pipeline_kernel<KIND, 16, true, OK, MK, false>>(pp, g, s);
      return launch_pipe<pipeline_kernel<KIND, 16, false, OK, MK, false>>(pp, g, s);
    }
    if (g.tail) return launch_pipe<pipeline_kernel<KIND, 10, true, OK, MK, false>>(pp, g, s);
    return launch_pipe<pipeline_kernel<KIND, 10, false, OK, MK, false>>(pp, g, s);
  }
  if (pp.phx) {
    PipeGeometry gp = g;
    gp.smem = cn::gen_smem_bytes(13, g.threads);
    if (pp.G > 1) {
      if (g.tail) return launch_pipe<pipeline_kernel<KIND, 13, true, OK, MK, true, true>>(pp, gp, s);
      return launch_pipe<pipeline_kernel<KIND, 13, false, OK, MK, true, true>>(pp, gp, s);
    }
    if (g.tail) return launch_pipe<pipeline_kernel<KIND, 13, true, OK, MK, false, true>>(pp, gp, s);
    return launch_pipe<pipeline_kernel<KIND, 13, false, OK, MK, false, true>>(pp, gp, s);
  }
  if (pp.G > 1) {
    if (g.tail) return launch_pipe<pipeline_kernel<KIND, 13, true, OK, MK, true>>(pp, g, s);
    return launch_pipe<pipeline_kernel<KIND, 13, false, OK, MK, true>>(pp, g, s);
  }
  if (g.tail) return launch_pipe<pipeline_kernel<KIND, 13, true, OK, MK, false>>(pp, g, s);
  return launch_pipe<pipeline_kernel<KIND, 13, false, OK, MK, false>>(pp, g, s);
}

// (fine model kind, ODE kind, ODE model kind) combinations with a pipeline
// instantiation: the BASELINE unimodal configs and their close relatives,
// and config 3's bimodal double well with the two-region closure.
static int dispatch_pipe(const mmpr_model &model, const mmpr_moment_ode &ode, const mmpr_model &ode_model,
                         const PipeParams *pp, const PipeGeometry &g, cudaStream_t s, bool probe_phx = false,
                         int probe_ranks = 1) {
  const int fk = model.kind, ok = ode.kind, mk = ode_model.kind;
  const bool run = pp != nullptr;
  // instantiations that exist on one rank with numpy-stream / injected increments only
  if (!run && (probe_phx || probe_ranks > 1) && (ode.n_regions == 2 || g.ppt != 13 || !g.exact)) return MMPR_ERR_UNSUPPORTED;
  if (ode.n_regions == 2) {
    if (g.ppt != 13 || !g.exact) return MMPR_ERR_UNSUPPORTED;
    if (fk == MMPR_MODEL_DOUBLE_WELL && ok == MMPR_ODE_MULTIMODAL && mk == MMPR_MODEL_DOUBLE_WELL)
      return run ? dispatch_pipe_regions<MMPR_MODEL_DOUBLE_WELL, MMPR_ODE_MULTIMODAL, MMPR_MODEL_DOUBLE_WELL>(*pp, g, s)
                 : MMPR_OK;
    return MMPR_ERR_UNSUPPORTED;
  }
  if (ode.n_regions != 1) return MMPR_ERR_UNSUPPORTED;
  if (fk == MMPR_MODEL_OU && ok == MMPR_ODE_UNIMODAL && mk == MMPR_MODEL_OU)
    return run ? dispatch_pipe_tail<MMPR_MODEL_OU, MMPR_ODE_UNIMODAL, MMPR_MODEL_OU>(*pp, g, s) : MMPR_OK;
  if (fk == MMPR_MODEL_OU && ok == MMPR_ODE_PERTURBED_OU)
    return run ? dispatch_pipe_tail<MMPR_MODEL_OU, MMPR_ODE_PERTURBED_OU, 0>(*pp, g, s) : MMPR_OK;
  if (fk == MMPR_MODEL_LINEAR && ok == MMPR_ODE_UNIMODAL && mk == MMPR_MODEL_LINEAR)
    return run ? dispatch_pipe_tail<MMPR_MODEL_LINEAR, MMPR_ODE_UNIMODAL, MMPR_MODEL_LINEAR>(*pp, g, s) : MMPR_OK;
  if (fk == MMPR_MODEL_CUBIC_MF && ok == MMPR_ODE_GAUSSIAN_CUBIC)
    return run ? dispatch_pipe_tail<MMPR_MODEL_CUBIC_MF, MMPR_ODE_GAUSSIAN_CUBIC, 0>(*pp, g, s) : MMPR_OK;
  if (fk == MMPR_MODEL_CUBIC_MF && ok == MMPR_ODE_UNIMODAL && mk == MMPR_MODEL_CUBIC_MF)
    return run ? dispatch_pipe_tail<MMPR_MODEL_CUBIC_MF, MMPR_ODE_UNIMODAL, MMPR_MODEL_CUBIC_MF>(*pp, g, s)
               : MMPR_OK;
  return MMPR_ERR_UNSUPPORTED;
}

}  // namespace mmpr

using namespace mmpr;

#ifdef MMPR_PIPE_PROFILE
extern "C" int mmpr_dev_rg_prof(unsigned long long *host_out, int reset) {
  cudaDeviceSynchronize();
  if (host_out) cudaMemcpyFromSymbol(host_out, mmpr::g_rg_prof, sizeof(mmpr::g_rg_prof));
  if (reset) {
    static unsigned long long zeros[1024][8];
    cudaMemcpyToSymbol(mmpr::g_rg_prof, zeros, sizeof(zeros));
  }
  return (int)cudaGetLastError();
}

extern "C" int mmpr_dev_pipe_prof(unsigned long long *host_out, int reset) {
  cudaDeviceSynchronize();
  if (host_out) cudaMemcpyFromSymbol(host_out, mmpr::g_pipe_prof, sizeof(mmpr::g_pipe_prof));
  if (reset) {
    static unsigned long long zeros[1024][8];
    cudaMemcpyToSymbol(mmpr::g_pipe_prof, zeros, sizeof(zeros));
  }
  return (int)cudaGetLastError();
}
#endif

extern "C" int64_t mmpr_pipeline_flags_size(int32_t n_slices, int32_t iterations) {
  if (n_slices < 1 || iterations < 0) return 0;
  const int64_t N = n_slices, K = iterations;
  return 1 + K * N + 2 * (K + 1) * (N + 1) + (K + 1) + 1;  // ..., abort word
}

extern "C" int mmpr_pipeline_supported_ex(const mmpr_model *model, const mmpr_moment_ode *ode,
                                          const mmpr_model *ode_model, const mmpr_integrator *integ,
                                          int64_t particles, int32_t counter_noise, int32_t n_ranks) {
  if (!model || !ode || !ode_model || !integ || n_ranks < 1) return MMPR_ERR_ARG;
  if (model->stat_kind != MMPR_STAT_MEAN_OF_F || ode->n_regions < 1 || ode->n_regions > 2) return MMPR_ERR_UNSUPPORTED;
  if (integ->kind != MMPR_INTEG_EULER || !(integ->dt > 0.0)) return MMPR_ERR_UNSUPPORTED;
  PipeGeometry g;
  const int st = pipe_geometry(particles, &g);
  if (st != MMPR_OK) return st;
  return dispatch_pipe(*model, *ode, *ode_model, nullptr, g, nullptr, counter_noise != 0, n_ranks);
}

extern "C" int mmpr_pipeline_supported(const mmpr_model *model, const mmpr_moment_ode *ode,
                                       const mmpr_model *ode_model, const mmpr_integrator *integ,
                                       int64_t particles) {
  return mmpr_pipeline_supported_ex(model, ode, ode_model, integ, particles, 0, 1);
}

static int check_io(const mmpr_pipeline_io *io, int32_t n_slices, int32_t iterations, int64_t particles,
                    int32_t steps) {
  if (!io->times || !io->x0 || !io->rho0 || !io->counts0 || !io->snap || !io->fine || !io->macro || !io->micro ||
      !io->micro_counts || !io->fine_stats || !io->fine_counts || !io->raw || !io->cache || !io->bad ||
      !io->coarse_status || !io->match_status || !io->flags)
    return MMPR_ERR_ARG;
  if (io->snap_rows != iterations + 1 && io->snap_rows != 2) return MMPR_ERR_ARG;
  if (io->fine_pitch < particles || io->snap_slice_pitch < particles ||
      io->snap_iter_stride < (int64_t)(n_slices + 1) * io->snap_slice_pitch)
    return MMPR_ERR_ARG;
  if (io->counter_noise && ((io->counter_kfield >= (1u << 12) && io->counter_kfield != MMPR_COUNTER_FRESH) ||
                            n_slices > (1 << 20) || steps > (1 << 24) || (io->counter_kfield == MMPR_COUNTER_FRESH &&
                                                                          iterations >= (1 << 12))))
    return MMPR_ERR_ARG;
  if (steps > 0 && !io->counter_noise && (!io->xi || (io->xi_row_pitch & 1) || io->xi_row_pitch < particles ||
                    (reinterpret_cast<uintptr_t>(io->xi) & 15) ||
                    (steps > 1 && io->xi_slice_pitch < steps * io->xi_row_pitch)))
    return MMPR_ERR_ARG;
  return MMPR_OK;
}

extern "C" int mmpr_parareal_pipeline_ranks(const mmpr_model *model, const mmpr_moment_ode *ode,
                                            const mmpr_model *ode_model, const mmpr_integrator *integ,
                                            int32_t n_slices, int32_t iterations, int64_t particles,
                                            int32_t steps, double dt, double sqrt_dt, int32_t reuse_converged,
                                            int32_t n_ranks, const mmpr_pipeline_io *ios, int32_t first_rank,
                                            int32_t launch_ranks, int32_t epoch, int32_t reset_flags,
                                            int32_t multi_gpu, void *stream) {
  int st = mmpr_pipeline_supported_ex(model, ode, ode_model, integ, particles,
                                      (ios && n_ranks >= 1 && ios[0].counter_noise) ? 1 : 0, n_ranks >= 1 ? n_ranks : 1);
  if (st != MMPR_OK) return st;
  if (!ios || n_slices < 1 || iterations < 1 || steps < 0 || n_ranks < 1 || n_ranks > PL_MAX_RANKS ||
      n_slices % n_ranks != 0 || first_rank < 0 || launch_ranks < 1 || first_rank + launch_ranks > n_ranks ||
      epoch < 1 || (reset_flags && epoch != 1))
    return MMPR_ERR_ARG;
  const int retain = ios[first_rank].snap_rows == iterations + 1 || iterations == 1;
  for (int r = 0; r < n_ranks; ++r) {
    const mmpr_pipeline_io &io = ios[r];
    if (r >= first_rank && r < first_rank + launch_ranks) {  // ranks whose units run here: everything
      st = check_io(&io, n_slices, iterations, particles, steps);
      if (st != MMPR_OK) return st;
      if ((io.snap_rows == iterations + 1 || iterations == 1) != (retain != 0)) return MMPR_ERR_ARG;
    } else if (!io.flags || !io.macro || !io.fine_stats || !io.fine_counts || !io.fine ||
               io.fine_pitch < particles) {  // peers: their exchange arrays
      return MMPR_ERR_ARG;
    }
  }
  PipeGeometry g;
  pipe_geometry(particles, &g);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nflags = mmpr_pipeline_flags_size(n_slices, iterations);
  for (int r = first_rank; r < first_rank + launch_ranks; ++r) {
    // the ticket always; every flag only when the caller resets per run
    const size_t bytes = reset_flags ? (size_t)nflags * sizeof(int32_t) : sizeof(int32_t);
    cudaError_t err = cudaMemsetAsync(ios[r].flags, 0, bytes, s);
    if (err != cudaSuccess) return mmpr_check(err, "pipeline: flag reset");
    err = cudaMemsetAsync(ios[r].flags + nflags - 1, 0, sizeof(int32_t), s);  // abort word, every launch
    if (err != cudaSuccess) return mmpr_check(err, "pipeline: abort reset");
  }

  PipeParams pp = {};
  FineParams &p = pp.f;
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
  p.xi_slice_pitch = ios[first_rank].xi_slice_pitch;
  p.xi_row_pitch = ios[first_rank].xi_row_pitch;
  p.D = g.D;
  p.slots_per_cta = g.spc;
  p.ctas = g.ctas;
  p.stage_elems = g.stage_elems;
  p.nstages = g.nstages;
  p.cnt_min = 12;
  p.l2_ahead = 3;
  if (const char *env = getenv("MMPR_FINE_L2_AHEAD")) p.l2_ahead = max(0, min(16, atoi(env)));
  for (int r = 0; r < n_ranks; ++r) {
    const bool local = r >= first_rank && r < first_rank + launch_ranks;
    if (local && (ios[r].xi_row_pitch != p.xi_row_pitch || ios[r].xi_slice_pitch != p.xi_slice_pitch))
      return MMPR_ERR_ARG;
    pp.io[r] = ios[r];
  }
  pp.ode = *ode;
  pp.ode_model = *ode_model;
  pp.integ = *integ;
  pp.N = n_slices;
  pp.K = iterations;
  pp.G = n_ranks;
  pp.Ng = n_slices / n_ranks;
  pp.r0 = first_rank;
  pp.lo_n = first_rank * pp.Ng;
  const int hi_n = (first_rank + launch_ranks == n_ranks) ? n_slices : (first_rank + launch_ranks) * pp.Ng - 1;
  pp.row_units = hi_n - pp.lo_n + 1;
  pp.units = (iterations + 1) * pp.row_units;
  pp.reuse = reuse_converged ? 1 : 0;
  pp.retain = retain;
  pp.epoch = epoch;
  pp.sys = multi_gpu ? 1 : 0;
  {
    const long long work = (long long)iterations * n_slices * (long long)steps * (long long)particles;
    pp.watchdog = work > (1LL << 34) ? work : (1LL << 34);
    if (const char *env = getenv("MMPR_PIPELINE_WATCHDOG")) pp.watchdog = atoll(env);  // tests
  }
  pp.abort = ios[first_rank].flags + nflags - 1;
  pp.phx = ios[first_rank].counter_noise ? 1 : 0;
  pp.phx_fresh = pp.phx && ios[first_rank].counter_kfield == MMPR_COUNTER_FRESH;
  p.cn = cn::CounterNoise{ios[first_rank].counter_key[0], 0u, pp.phx_fresh ? 0u : ios[first_rank].counter_kfield, 0};
  pp.nranks = launch_ranks;
  if (ode->n_regions > 1) {
    // bimodal units restrict over compacted members in per-cluster scratch
    const mmpr_pipeline_io &io = ios[first_rank];
    if (n_ranks != 1 || io.partition.n_regions != ode->n_regions || !io.region_scratch ||
        io.region_scratch_rows < 1)
      return MMPR_ERR_ARG;
    pp.part = io.partition;
    pp.rg_scratch = io.region_scratch;
    pp.rg_rows = (int)(io.region_scratch_rows < INT_MAX ? io.region_scratch_rows : INT_MAX);
  }
  // one launch over several ranks normally takes one global ticket order;
  // MMPR_PIPELINE_RANK_TICKETS=1 gives every rank its own clusters and
  // ticket counter instead, the scheduling of one launch per GPU (the
  // clusters of a launch are co-resident, so every rank keeps at least one)
  pp.rank_tickets = 0;
  if (const char *env = getenv("MMPR_PIPELINE_RANK_TICKETS"))
    pp.rank_tickets = (atoi(env) == 1 && launch_ranks > 1) ? 1 : 0;
  return dispatch_pipe(*model, *ode, *ode_model, &pp, g, s);
}

extern "C" int mmpr_parareal_pipeline(const mmpr_model *model, const mmpr_moment_ode *ode,
                                      const mmpr_model *ode_model, const mmpr_integrator *integ,
                                      int32_t n_slices, int32_t iterations, int64_t particles, int32_t steps,
                                      double dt, double sqrt_dt, int32_t reuse_converged,
                                      const mmpr_pipeline_io *io, void *stream) {
  return mmpr_parareal_pipeline_ranks(model, ode, ode_model, integ, n_slices, iterations, particles, steps, dt,
                                      sqrt_dt, reuse_converged, 1, io, 0, 1, 1, 1, 0, stream);
}

// ---- exchange memory for the multi-GPU pipeline (CUDA IPC) -------------------
extern "C" int mmpr_exchange_alloc(int64_t bytes, void **dev_ptr) {
  if (bytes < 1 || !dev_ptr) return MMPR_ERR_ARG;
  return mmpr_check(cudaMalloc(dev_ptr, (size_t)bytes), "exchange: cudaMalloc");
}

extern "C" int mmpr_exchange_free(void *dev_ptr) {
  if (!dev_ptr) return MMPR_OK;
  return mmpr_check(cudaFree(dev_ptr), "exchange: cudaFree");
}

extern "C" int mmpr_ipc_handle(void *dev_ptr, unsigned char *handle_out) {
  if (!dev_ptr || !handle_out) return MMPR_ERR_ARG;
  cudaIpcMemHandle_t h;
  const int st = mmpr_check(cudaIpcGetMemHandle(&h, dev_ptr), "exchange: cudaIpcGetMemHandle");
  if (st != MMPR_OK) return st;
  memcpy(handle_out, &h, sizeof(h));
  return MMPR_OK;
}

extern "C" int mmpr_ipc_open(const unsigned char *handle, void **dev_ptr) {
  if (!handle || !dev_ptr) return MMPR_ERR_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return mmpr_check(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "exchange: cudaIpcOpenMemHandle");
}

extern "C" int mmpr_ipc_close(void *dev_ptr) {
  if (!dev_ptr) return MMPR_OK;
  return mmpr_check(cudaIpcCloseMemHandle(dev_ptr), "exchange: cudaIpcCloseMemHandle");
}

extern "C" int mmpr_device_can_access_peer(int32_t device, int32_t peer, int32_t *out) {
  if (!out) return MMPR_ERR_ARG;
  int v = 0;
  const int st = mmpr_check(cudaDeviceCanAccessPeer(&v, device, peer), "cudaDeviceCanAccessPeer");
  *out = v;
  return st;
}
