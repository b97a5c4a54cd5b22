// Multi-region (cluster) restriction, restrict_regions.cu, shared with
// coupling.cu's mmpr_restrict.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mmpr.h"

namespace mmpr {

struct RegionsParams {
  mmpr_partition part;
  int64_t P;
  const double *x;
  int64_t pitch;
  double *stats;    // [n_ens][3I]
  int64_t *counts;  // [n_ens][I]
  double *scratch;  // [n_ens][I][P] compacted members
  int D, slots_per_cta, ctas;
  // match prologue (MATCH)
  const double *targets;
  int64_t tgt_stride;
  const double *cur;
  int64_t cur_stride;
  const int64_t *cur_counts;
  int64_t cnt_stride;
  double *x_out;
  int64_t out_pitch;
  int policy;  // 0 raise, 1 collapse
  int32_t *status;
  int32_t *clamped;
};

// One cluster per ensemble; MMPR_ERR_UNSUPPORTED when the ensemble does not
// fit one cluster (the caller keeps the multi-kernel path).
int restrict_regions(RegionsParams p, int n_ens, bool match, cudaStream_t stream);

}  // namespace mmpr
