// Shared pieces of the fine-sweep kernels (cluster variant fine.cu, grid
// variant fine_grid.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mmpr_device.cuh"
#include "counter_noise.cuh"

namespace mmpr {

#define FS_MAX_CLUSTER 16
#define FS_MAX_STAGES 4

struct FineParams {
  mmpr_model model;
  int n_slices;
  int S;
  int64_t P;
  double dt, sqrt_dt, bsd;  // bsd = b*sqrt(dt) for constant-diffusion models
  const double *t0;
  const double *x_in;
  int64_t in_pitch;
  double *x_out;
  int64_t out_pitch;
  const double *xi;
  int64_t xi_slice_pitch, xi_row_pitch;
  int32_t *bad_step;
  double *final_mean;
  double *stats;      // optional single-region restriction of x_out: [mean, var, fraction] per slice
  int64_t *counts;    // optional member counts (= P) per slice
  int D;              // tree depth (2^D leaf slots)
  int slots_per_cta;  // 4 * warps per CTA
  int ctas;           // CTAs per slice (cluster size)
  int stage_elems;    // doubles per smem stage (16-B multiple)
  int nstages;        // increment stages in shared memory (2..FS_MAX_STAGES)
  int cnt_min;        // min elements per lane over populated slots
  int l2_ahead;       // steps of increments prefetched into L2 beyond the smem stages
  cn::CounterNoise cn;  // PHX kernels: increments from counter-based Philox (xi unused)
  long long *t_slice;   // optional [n_slices][2] globaltimer stamps (ns): slice start, slice end
};

// dynamic shared memory of a PHX kernel: the ziggurat tables
#define MMPR_PHX_SMEM ((size_t)sizeof(cn::ZigTables))

struct __align__(16) ClusterSlot {
  double v;
  int ok;
  int bad;
};

template <int KIND>
__device__ __forceinline__ double em_update(const FineParams &p, double x, double s, double xi) {
  // x + a(x,s)*dt + b(x,s)*sqrt(dt)*xi, left to right, each op rounded
  mmpr_model m = p.model;
  m.kind = KIND;  // folds the family switch at compile time
  const double a = drift(m, x, s);
  const double moved = add(x, mul(a, p.dt));
  double noise;
  if (constant_diffusion(KIND)) {
    noise = mul(p.bsd, xi);
  } else {
    noise = mul(mul(diffusion(m, x, s), p.sqrt_dt), xi);
  }
  return add(moved, noise);
}

// Partial sums of the pairwise tree.  With PADDED (an irregular tree, or
// fewer slots than lanes) a partial carries a validity flag so an empty right
// sibling passes its left sibling through unchanged; a perfect tree (every
// BASELINE size) uses plain adds.
template <bool PADDED>
struct Part;

template <>
struct Part<true> {
  double v;
  int ok;
  __device__ __forceinline__ static Part make(double v, bool ok) { return {v, ok ? 1 : 0}; }
  __device__ __forceinline__ Part xor_level(int lane, int m) const {
    PwVal a{v, ok};
    PwVal r = pw_xor_level(a, lane, m);
    return {r.v, r.ok};
  }
  __device__ __forceinline__ static Part combine(Part l, Part r) {
    PwVal c = pw_combine(PwVal{l.v, l.ok}, PwVal{r.v, r.ok});
    return {c.v, c.ok};
  }
  __device__ __forceinline__ bool valid() const { return ok != 0; }
};

template <>
struct Part<false> {
  double v;
  __device__ __forceinline__ static Part make(double v, bool) { return {v}; }
  __device__ __forceinline__ Part xor_level(int, int m) const {
    return {add(v, __shfl_xor_sync(MMPR_FULL_MASK, v, m))};  // IEEE add is commutative
  }
  __device__ __forceinline__ static Part combine(Part l, Part r) { return {add(l.v, r.v)}; }
  __device__ __forceinline__ bool valid() const { return true; }
};

// Grid (multi-team) variant for ensembles beyond one cluster, fine_grid.cu.
int fine_grid_sweep(FineParams p, cudaStream_t stream, bool phx = false);
int fine_grid_shape(int64_t P, int n_slices, int *teams_out, int *ctas_out);

// Single-region restriction with one cluster per ensemble, restrict1.cu
// (MMPR_ERR_UNSUPPORTED beyond one cluster).
int restrict_single_region(int n_ens, int64_t P, const double *x, int64_t pitch, double *stats, int64_t *counts,
                           cudaStream_t stream);

}  // namespace mmpr
