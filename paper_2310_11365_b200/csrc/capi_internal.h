// Internal helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include "../../include/mmpr.h"

// Records `what: cudaGetErrorString(err)` for mmpr_last_error().
void mmpr_set_error(const char *what, cudaError_t err);

// Checks the last launch; returns MMPR_OK or MMPR_ERR_CUDA.
static inline int mmpr_check_launch(const char *what) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    mmpr_set_error(what, err);
    return MMPR_ERR_CUDA;
  }
  return MMPR_OK;
}

static inline int mmpr_check(cudaError_t err, const char *what) {
  if (err != cudaSuccess) {
    mmpr_set_error(what, err);
    return MMPR_ERR_CUDA;
  }
  return MMPR_OK;
}
