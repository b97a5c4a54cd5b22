// Error metrics on the device: row sort and the W1 distance of two equally
// sized empirical measures.
//
// Replaces the hot loops of metrics.wasserstein_1d / relative_errors /
// statistical_floor / floor_from_references
// (/root/reference/pkg/src/mcparareal/metrics.py:35-47, 73-130, 133-218):
//   W1(a, b) = np.mean(np.abs(np.sort(a) - np.sort(b))).
// Sorting a multiset is deterministic, so the sorted rows equal numpy's (the
// order of +0.0 / -0.0 may differ, which |a - b| cannot see); the mean of
// |a - b| follows numpy's pairwise tree, so W1 is bit-identical.
//
// The row sort is CUB's segmented sort (a library primitive, used for the
// evaluation metrics only -- not on the fine-propagator path).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/device/device_segmented_sort.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "capi_internal.h"
#include "mmpr_device.cuh"

namespace mmpr {

struct RowOffset {
  int64_t pitch, shift;
  __host__ __device__ __forceinline__ int64_t operator()(int64_t r) const { return r * pitch + shift; }
};

#define MA_THREADS 1024
#define MA_MAX_CHUNKS 1024

// numpy pairwise sum of |a[i] - b[i]| for i < n by one CTA (thread 0 returns it)
__device__ double cta_pairwise_absdiff(const double *__restrict__ a, const double *__restrict__ b, int64_t n,
                                       PwVal *s_wp, PwVal *s_chunk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int D = pw_depth(n);
  const int64_t nslots = int64_t(1) << D;
  const int64_t chunks = nslots > 128 ? nslots / 128 : 1;
  auto f = [&](int64_t i) { return fabs(sub(a[i], b[i])); };
  for (int64_t c = 0; c < chunks; ++c) {
    const int64_t s = c * 128 + (tid >> 3);
    const int j8 = tid & 7;
    int64_t off = 0, len = 0;
    if (s < nslots) pw_leaf(n, D, s, &off, &len);
    const int64_t cnt = len >> 3;
    double acc = 0.0;
    if (cnt > 0) {
      acc = f(off + j8);
      for (int64_t k = 1; k < cnt; ++k) acc = add(acc, f(off + j8 + 8 * k));
    }
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 1));
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 2));
    acc = add(acc, __shfl_xor_sync(MMPR_FULL_MASK, acc, 4));
    if (cnt == 0) acc = 0.0;
    for (int64_t i = cnt * 8; i < len; ++i) acc = add(acc, f(off + i));
    PwVal leaf;
    leaf.v = acc;
    leaf.ok = len > 0;
    leaf = pw_xor_level(leaf, lane, 8);
    leaf = pw_xor_level(leaf, lane, 16);
    if (lane == 0) s_wp[warp] = leaf;
    __syncthreads();
    if (warp == 0) {
      PwVal v = s_wp[lane];
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) v = pw_xor_level(v, lane, k);
      if (lane == 0) s_chunk[c] = v;
    }
    __syncthreads();
  }
  double r = 0.0;
  if (tid == 0) {
    for (int64_t w = 1; w < chunks; w <<= 1)
      for (int64_t q = 0; q + w < chunks; q += 2 * w) s_chunk[q] = pw_combine(s_chunk[q], s_chunk[q + w]);
    r = s_chunk[0].v;
  }
  return r;
}

__global__ void __launch_bounds__(MA_THREADS) mean_absdiff_kernel(int64_t n, const double *a, int64_t pitch_a,
                                                                  const double *b, int64_t pitch_b, double *out) {
  __shared__ PwVal s_wp[32];
  __shared__ PwVal s_chunk[MA_MAX_CHUNKS];
  const int64_t r = blockIdx.x;
  const double s = cta_pairwise_absdiff(a + r * pitch_a, b + r * pitch_b, n, s_wp, s_chunk);
  if (threadIdx.x == 0) out[r] = div(s, (double)n);
}

// cum[r][e] = #{sorted_r < edge_e} (last edge: <=), one thread per (row, edge)
__global__ void hist_cum_kernel(int32_t n_rows, int64_t count, const double *__restrict__ sorted, int64_t pitch,
                                const double *__restrict__ edges, int32_t n_edges, int64_t *__restrict__ cum) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= (int64_t)n_rows * n_edges) return;
  const int64_t r = g / n_edges;
  const int e = (int)(g - r * n_edges);
  const double *a = sorted + r * pitch;
  const double v = edges[e];
  const bool right = e == n_edges - 1;
  int64_t lo = 0, hi = count;  // first index whose element is >= v (> v for the last edge)
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const double x = a[mid];
    if (right ? !(x > v) : (x < v)) lo = mid + 1;
    else hi = mid;
  }
  cum[g] = lo;
}

}  // namespace mmpr

using namespace mmpr;

extern "C" int mmpr_histogram_sorted(int32_t n_rows, int64_t count, const double *sorted, int64_t pitch,
                                     const double *edges, int32_t n_edges, int64_t *counts, void *stream) {
  if (n_rows < 0 || count < 0 || !sorted || !edges || n_edges < 2 || !counts) return MMPR_ERR_ARG;
  if (n_rows == 0) return MMPR_OK;
  // counts is used as the cumulative scratch: [n_rows][n_edges]; the host
  // differences it (n_edges - 1 bins per row)
  const int64_t total = (int64_t)n_rows * n_edges;
  hist_cum_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n_rows, count, sorted, pitch,
                                                                                    edges, n_edges, counts); mmpr_launched();
  return mmpr_check_launch("hist_cum_kernel");
}

extern "C" int mmpr_sort_rows(int32_t n_rows, int64_t count, const double *in, double *out, int64_t pitch,
                              void *temp, uint64_t *temp_bytes, void *stream) {
  if (n_rows < 0 || count < 0 || !temp_bytes || pitch < count) return MMPR_ERR_ARG;
  if (count > INT32_MAX || (int64_t)n_rows * pitch > INT32_MAX) return MMPR_ERR_UNSUPPORTED;
  cub::CountingInputIterator<int64_t> rows(0);
  cub::TransformInputIterator<int64_t, RowOffset, cub::CountingInputIterator<int64_t>> begin(rows,
                                                                                           RowOffset{pitch, 0});
  cub::TransformInputIterator<int64_t, RowOffset, cub::CountingInputIterator<int64_t>> end(rows,
                                                                                         RowOffset{pitch, count});
  size_t bytes = (size_t)*temp_bytes;
  const int num_items = (int)((int64_t)n_rows * pitch);
  if (!temp) {  // size query
    cudaError_t err = cub::DeviceSegmentedSort::SortKeys((void *)nullptr, bytes, (const double *)nullptr,
                                                         (double *)nullptr, num_items, n_rows, begin, end,
                                                         (cudaStream_t)stream);
    *temp_bytes = (uint64_t)bytes;
    return mmpr_check(err, "mmpr_sort_rows: size query");
  }
  if (!in || !out) return MMPR_ERR_ARG;
  if (n_rows == 0 || count == 0) return MMPR_OK;
  cudaError_t err = cub::DeviceSegmentedSort::SortKeys(temp, bytes, in, out, num_items, n_rows, begin, end,
                                                       (cudaStream_t)stream);
  return mmpr_check(err, "mmpr_sort_rows");
}

extern "C" int mmpr_mean_abs_diff(int32_t n_rows, int64_t count, const double *a, int64_t pitch_a,
                                  const double *b, int64_t pitch_b, double *out, void *stream) {
  if (n_rows < 0 || count < 1 || !a || !b || !out) return MMPR_ERR_ARG;
  if (n_rows == 0) return MMPR_OK;
  const int D = pw_depth(count);
  if (D > 7 && ((int64_t(1) << D) / 128) > MA_MAX_CHUNKS) return MMPR_ERR_UNSUPPORTED;
  mean_absdiff_kernel<<<n_rows, MA_THREADS, 0, (cudaStream_t)stream>>>(count, a, pitch_a, b, pitch_b, out); mmpr_launched();
  return mmpr_check_launch("mean_absdiff_kernel");
}
