// Fine propagator for the interaction statistics beyond MEAN_OF_F:
//   ROTATOR_SUM   (S, C) = (np.mean(np.sin(x)), np.mean(np.cos(x)))
//                 plane rotator, models.py:286-314 (+ mod-2pi post_step)
//   EMPIRICAL_CDF s_i = (rank_i + 0.5) / P, rank from a stable argsort
//                 Burgers, models.py:317-334 / ensemble_statistic :61-83
// Reference step: particles._em_step_raw (particles.py:119-131), finiteness
// check per step as propagate_fine (particles.py:146-159).
//
// These models are not part of the BASELINE workloads, so the sweep is
// step-synchronous across launches instead of register-resident: per step
// one statistic pass over every slice (a CTA-per-slice pairwise reduction
// for ROTATOR_SUM, a stable segmented sort + rank scatter for EMPIRICAL_CDF)
// and one elementwise update pass.  All arithmetic keeps numpy's operation
// order; ranks are exact, so Burgers trajectories are bit-identical, and the
// rotator's sin/cos differ from numpy's only by libm ulps.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include <cub/device/device_segmented_sort.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "capi_internal.h"
#include "mmpr_device.cuh"

namespace mmpr {

#define SW_THREADS 1024
#define SW_MAX_CHUNKS 1024
#define SW_TWO_PI 6.283185307179586  // 2.0 * math.pi

struct DenseOffset {
  int64_t P, shift;
  __host__ __device__ __forceinline__ int64_t operator()(int64_t r) const { return r * P + shift; }
};

// (sum sin x, sum cos x) over numpy's pairwise tree, one CTA per slice
__global__ void __launch_bounds__(SW_THREADS) rotator_stat_kernel(int64_t P, const double *__restrict__ x_all,
                                                                  int64_t pitch, double *__restrict__ stat) {
  __shared__ PwVal s_wp[2][32];
  __shared__ PwVal s_chunk[2][SW_MAX_CHUNKS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double *x = x_all + (int64_t)blockIdx.x * pitch;
  const int D = pw_depth(P);
  const int64_t nslots = int64_t(1) << D;
  const int64_t chunks = nslots > 128 ? nslots / 128 : 1;
  for (int64_t c = 0; c < chunks; ++c) {
    const int64_t s = c * 128 + (tid >> 3);
    const int j8 = tid & 7;
    int64_t off = 0, len = 0;
    if (s < nslots) pw_leaf(P, D, s, &off, &len);
    const int64_t cnt = len >> 3;
    double as = 0.0, ac = 0.0;
    if (cnt > 0) {
      double sv, cv;
      sincos(x[off + j8], &sv, &cv);
      as = sv;
      ac = cv;
      for (int64_t k = 1; k < cnt; ++k) {
        sincos(x[off + j8 + 8 * k], &sv, &cv);
        as = add(as, sv);
        ac = add(ac, cv);
      }
    }
#pragma unroll
    for (int m = 1; m < 8; m <<= 1) {
      as = add(as, __shfl_xor_sync(MMPR_FULL_MASK, as, m));
      ac = add(ac, __shfl_xor_sync(MMPR_FULL_MASK, ac, m));
    }
    if (cnt == 0) as = ac = 0.0;
    for (int64_t i = cnt * 8; i < len; ++i) {
      double sv, cv;
      sincos(x[off + i], &sv, &cv);
      as = add(as, sv);
      ac = add(ac, cv);
    }
    PwVal ls{as, len > 0}, lc{ac, len > 0};
    ls = pw_xor_level(ls, lane, 8);
    ls = pw_xor_level(ls, lane, 16);
    lc = pw_xor_level(lc, lane, 8);
    lc = pw_xor_level(lc, lane, 16);
    if (lane == 0) {
      s_wp[0][warp] = ls;
      s_wp[1][warp] = lc;
    }
    __syncthreads();
    if (warp < 2) {
      PwVal v = s_wp[warp][lane];
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) v = pw_xor_level(v, lane, k);
      if (lane == 0) s_chunk[warp][c] = v;
    }
    __syncthreads();
  }
  if (tid < 2) {
    for (int64_t w = 1; w < chunks; w <<= 1)
      for (int64_t q = 0; q + w < chunks; q += 2 * w) s_chunk[tid][q] = pw_combine(s_chunk[tid][q], s_chunk[tid][q + w]);
    stat[2 * blockIdx.x + tid] = div(s_chunk[tid][0].v, (double)P);
  }
}

// keys = x with +-0 and NaNs canonicalised (numpy's argsort treats -0.0 == 0.0
// and sorts every NaN last, stable by index), values = particle index
__global__ void rank_prep_kernel(int n_slices, int64_t P, const double *__restrict__ x, int64_t pitch,
                                 double *__restrict__ keys, int32_t *__restrict__ idx) {
  const int64_t total = (int64_t)n_slices * P;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = g / P, i = g - n * P;
    double v = x[n * pitch + i];
    if (isnan(v)) v = __longlong_as_double(0x7ff8000000000000LL);
    keys[g] = add(v, 0.0);  // -0.0 + 0.0 = +0.0
    idx[g] = (int32_t)i;
  }
}

// s[order[i]] = (i + 0.5) / P
__global__ void rank_scatter_kernel(int n_slices, int64_t P, const int32_t *__restrict__ order,
                                    double *__restrict__ s) {
  const int64_t total = (int64_t)n_slices * P;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = g / P, i = g - n * P;
    s[n * P + order[g]] = div(add((double)i, 0.5), (double)P);
  }
}

// numpy's np.mod(x, 2 pi) for a positive modulus (npy_divmod)
__device__ __forceinline__ double np_mod_2pi(double x) {
  double m = fmod(x, SW_TWO_PI);
  if (m != 0.0) {
    if (m < 0.0) m = add(m, SW_TWO_PI);
  } else {
    m = 0.0;  // copysign(0.0, 2 pi)
  }
  return m;
}

struct StepwiseUpdate {
  int n_slices;
  int64_t P;
  int step;
  double dt, bsd;  // bsd = b * sqrt(dt) (constant diffusion)
  mmpr_model model;
  const double *x_in;
  int64_t in_pitch;
  double *x_out;
  int64_t out_pitch;
  const double *xi;  // row `step` of every slice
  int64_t xi_slice_pitch;
  const double *stat;  // rotator: [n][2]; Burgers: [n][P]
  int32_t *bad_step;
};

template <int KIND>
__global__ void stepwise_update_kernel(const StepwiseUpdate u) {
  const int64_t total = (int64_t)u.n_slices * u.P;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = g / u.P, i = g - n * u.P;
    const double x = u.x_in[n * u.in_pitch + i];
    const double xi = u.xi[n * u.xi_slice_pitch + i];
    double a;
    if (KIND == MMPR_MODEL_ROTATOR) {
      // K * (cos(x) * S - sin(x) * C) - sin(x)
      const double S = u.stat[2 * n], C = u.stat[2 * n + 1];
      double sv, cv;
      sincos(x, &sv, &cv);
      a = sub(mul(u.model.p[0], sub(mul(cv, S), mul(sv, C))), sv);
    } else {  // Burgers: 1 - s_i
      a = sub(1.0, u.stat[n * u.P + i]);
    }
    double y = add(add(x, mul(a, u.dt)), mul(u.bsd, xi));
    if (KIND == MMPR_MODEL_ROTATOR && u.model.p[2] != 0.0) y = np_mod_2pi(y);
    u.x_out[n * u.out_pitch + i] = y;
    if (!finite(y)) atomicCAS(&u.bad_step[n], MMPR_STAT_OK, u.step);
  }
}

__global__ void fill_status_kernel(int n, int32_t *bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) bad[i] = MMPR_STAT_OK;
}

static size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

}  // namespace mmpr

using namespace mmpr;

extern "C" int mmpr_fine_sweep_stepwise(const mmpr_model *model, int32_t n_slices, int64_t particles,
                                        int32_t steps, double dt, double sqrt_dt, const double *x_in,
                                        int64_t in_pitch, double *x_out, int64_t out_pitch, const double *xi,
                                        int64_t xi_slice_pitch, int64_t xi_row_pitch, int32_t *bad_step,
                                        void *workspace, uint64_t *workspace_bytes, void *stream) {
  if (!model || n_slices < 0 || particles < 1 || steps < 0 || !workspace_bytes) return MMPR_ERR_ARG;
  const bool rotator = model->kind == MMPR_MODEL_ROTATOR && model->stat_kind == MMPR_STAT_ROTATOR_SUM;
  const bool burgers = model->kind == MMPR_MODEL_BURGERS && model->stat_kind == MMPR_STAT_EMPIRICAL_CDF;
  if (!rotator && !burgers) return MMPR_ERR_UNSUPPORTED;
  const int64_t P = particles;
  const int64_t items = (int64_t)n_slices * P;
  if (burgers && items > INT32_MAX) return MMPR_ERR_UNSUPPORTED;
  if (rotator) {
    const int D = pw_depth(P);
    if (D > 7 && ((int64_t(1) << D) / 128) > SW_MAX_CHUNKS) return MMPR_ERR_UNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // workspace: stat | keys_in | keys_out | idx_in | idx_out | cub temp
  const size_t stat_bytes = align256(rotator ? (size_t)n_slices * 2 * 8 : (size_t)items * 8);
  const size_t key_bytes = burgers ? align256((size_t)items * 8) : 0;
  const size_t idx_bytes = burgers ? align256((size_t)items * 4) : 0;
  size_t cub_bytes = 0;
  cub::CountingInputIterator<int64_t> rows(0);
  cub::TransformInputIterator<int64_t, DenseOffset, cub::CountingInputIterator<int64_t>> seg_begin(rows,
                                                                                                 DenseOffset{P, 0});
  cub::TransformInputIterator<int64_t, DenseOffset, cub::CountingInputIterator<int64_t>> seg_end(rows,
                                                                                               DenseOffset{P, P});
  if (burgers) {
    cudaError_t err = cub::DeviceSegmentedSort::StableSortPairs(
        (void *)nullptr, cub_bytes, (const double *)nullptr, (double *)nullptr, (const int32_t *)nullptr,
        (int32_t *)nullptr, (int)items, n_slices, seg_begin, seg_end, st);
    if (err != cudaSuccess) return mmpr_check(err, "fine_sweep_stepwise: sort size query");
  }
  const size_t need = stat_bytes + 2 * key_bytes + 2 * idx_bytes + align256(cub_bytes);
  if (!workspace) {
    *workspace_bytes = (uint64_t)need;
    return MMPR_OK;
  }
  if (*workspace_bytes < need) return MMPR_ERR_ARG;
  if (!x_in || !x_out || !bad_step || (steps > 0 && !xi)) return MMPR_ERR_ARG;
  if (n_slices == 0) return MMPR_OK;
  char *w = (char *)workspace;
  double *stat = (double *)w;
  double *keys_in = (double *)(w + stat_bytes);
  double *keys_out = (double *)(w + stat_bytes + key_bytes);
  int32_t *idx_in = (int32_t *)(w + stat_bytes + 2 * key_bytes);
  int32_t *idx_out = (int32_t *)(w + stat_bytes + 2 * key_bytes + idx_bytes);
  void *cub_temp = (void *)(w + stat_bytes + 2 * key_bytes + 2 * idx_bytes);

  fill_status_kernel<<<(n_slices + 255) / 256, 256, 0, st>>>(n_slices, bad_step); mmpr_launched();
  int rc = mmpr_check_launch("fill_status_kernel");
  if (rc != MMPR_OK) return rc;
  if (steps == 0) {
    const cudaError_t err = cudaMemcpy2DAsync(x_out, out_pitch * 8, x_in, in_pitch * 8, P * 8, n_slices,
                                              cudaMemcpyDeviceToDevice, st);
    return mmpr_check(err, "fine_sweep_stepwise: copy");
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int eblocks = (int)std::min<int64_t>((items + 255) / 256, (int64_t)sms * 8);
  StepwiseUpdate u;
  u.n_slices = n_slices;
  u.P = P;
  u.dt = dt;
  u.bsd = model->p[1] * sqrt_dt;  // b * sqrt(dt), one IEEE product as numpy
  u.model = *model;
  u.x_out = x_out;
  u.out_pitch = out_pitch;
  u.xi_slice_pitch = xi_slice_pitch;
  u.stat = stat;
  u.bad_step = bad_step;
  for (int j = 0; j < steps; ++j) {
    const double *src = j == 0 ? x_in : x_out;
    const int64_t src_pitch = j == 0 ? in_pitch : out_pitch;
    if (rotator) {
      rotator_stat_kernel<<<n_slices, SW_THREADS, 0, st>>>(P, src, src_pitch, stat); mmpr_launched();
    } else {
      rank_prep_kernel<<<eblocks, 256, 0, st>>>(n_slices, P, src, src_pitch, keys_in, idx_in); mmpr_launched();
      size_t bytes = cub_bytes;
      cudaError_t err = cub::DeviceSegmentedSort::StableSortPairs(cub_temp, bytes, keys_in, keys_out, idx_in,
                                                                  idx_out, (int)items, n_slices, seg_begin,
                                                                  seg_end, st);
      if (err != cudaSuccess) return mmpr_check(err, "fine_sweep_stepwise: sort");
      rank_scatter_kernel<<<eblocks, 256, 0, st>>>(n_slices, P, idx_out, stat); mmpr_launched();
    }
    u.step = j;
    u.x_in = src;
    u.in_pitch = src_pitch;
    u.xi = xi + (int64_t)j * xi_row_pitch;
    if (rotator) stepwise_update_kernel<MMPR_MODEL_ROTATOR><<<eblocks, 256, 0, st>>>(u);
    else stepwise_update_kernel<MMPR_MODEL_BURGERS><<<eblocks, 256, 0, st>>>(u);
    mmpr_launched();
    rc = mmpr_check_launch("stepwise_update_kernel");
    if (rc != MMPR_OK) return rc;
  }
  return MMPR_OK;
}

// The interaction statistic alone (models.ensemble_statistic,
// /root/reference/pkg/src/mcparareal/models.py:61-83) for the ROTATOR_SUM
// and EMPIRICAL_CDF kinds: stat[2n..2n+1] = (np.mean(sin x), np.mean(cos x))
// per slice, or stat[n*P + i] = (rank_i + 0.5) / P with a stable argsort.
// Same kernels as the stepwise sweep; workspace queried with workspace = NULL.
extern "C" int mmpr_ensemble_statistic(const mmpr_model *model, int32_t n_slices, int64_t particles,
                                       const double *x, int64_t pitch, double *stat, void *workspace,
                                       uint64_t *workspace_bytes, void *stream) {
  if (!model || n_slices < 0 || particles < 1 || !workspace_bytes || (n_slices > 1 && pitch < particles))
    return MMPR_ERR_ARG;
  const bool rotator = model->stat_kind == MMPR_STAT_ROTATOR_SUM;
  const bool burgers = model->stat_kind == MMPR_STAT_EMPIRICAL_CDF;
  if (!rotator && !burgers) return MMPR_ERR_UNSUPPORTED;
  const int64_t P = particles;
  const int64_t items = (int64_t)n_slices * P;
  if (burgers && items > INT32_MAX) return MMPR_ERR_UNSUPPORTED;
  if (rotator) {
    const int D = pw_depth(P);
    if (D > 7 && ((int64_t(1) << D) / 128) > SW_MAX_CHUNKS) return MMPR_ERR_UNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t key_bytes = burgers ? align256((size_t)items * 8) : 0;
  const size_t idx_bytes = burgers ? align256((size_t)items * 4) : 0;
  size_t cub_bytes = 0;
  cub::CountingInputIterator<int64_t> rows(0);
  cub::TransformInputIterator<int64_t, DenseOffset, cub::CountingInputIterator<int64_t>> seg_begin(rows,
                                                                                                 DenseOffset{P, 0});
  cub::TransformInputIterator<int64_t, DenseOffset, cub::CountingInputIterator<int64_t>> seg_end(rows,
                                                                                               DenseOffset{P, P});
  if (burgers) {
    cudaError_t err = cub::DeviceSegmentedSort::StableSortPairs(
        (void *)nullptr, cub_bytes, (const double *)nullptr, (double *)nullptr, (const int32_t *)nullptr,
        (int32_t *)nullptr, (int)items, n_slices, seg_begin, seg_end, st);
    if (err != cudaSuccess) return mmpr_check(err, "ensemble_statistic: sort size query");
  }
  const size_t need = 2 * key_bytes + 2 * idx_bytes + align256(cub_bytes) + 256;
  if (!workspace) {
    *workspace_bytes = (uint64_t)need;
    return MMPR_OK;
  }
  if (*workspace_bytes < need || !x || !stat) return MMPR_ERR_ARG;
  if (n_slices == 0) return MMPR_OK;
  if (rotator) {
    rotator_stat_kernel<<<n_slices, SW_THREADS, 0, st>>>(P, x, n_slices > 1 ? pitch : P, stat); mmpr_launched();
    return mmpr_check_launch("rotator_stat_kernel");
  }
  char *w = (char *)workspace;
  double *keys_in = (double *)w;
  double *keys_out = (double *)(w + key_bytes);
  int32_t *idx_in = (int32_t *)(w + 2 * key_bytes);
  int32_t *idx_out = (int32_t *)(w + 2 * key_bytes + idx_bytes);
  void *cub_temp = (void *)(w + 2 * key_bytes + 2 * idx_bytes);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int eblocks = (int)std::min<int64_t>((items + 255) / 256, (int64_t)sms * 8);
  rank_prep_kernel<<<eblocks, 256, 0, st>>>(n_slices, P, x, n_slices > 1 ? pitch : P, keys_in, idx_in); mmpr_launched();
  size_t bytes = cub_bytes;
  cudaError_t err = cub::DeviceSegmentedSort::StableSortPairs(cub_temp, bytes, keys_in, keys_out, idx_in, idx_out,
                                                              (int)items, n_slices, seg_begin, seg_end, st);
  if (err != cudaSuccess) return mmpr_check(err, "ensemble_statistic: sort");
  rank_scatter_kernel<<<eblocks, 256, 0, st>>>(n_slices, P, idx_out, stat); mmpr_launched();
  return mmpr_check_launch("rank_scatter_kernel");
}
