// Internal helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include "../../include/mmpr.h"

// Records `what: cudaGetErrorString(err)` for mmpr_last_error().
void mmpr_set_error(const char *what, cudaError_t err);

// Kernel launches issued by this library in this process (mmpr_kernel_launches):
// every launch site bumps it, so the host's launch claim counts kernels, not calls.
extern unsigned long long g_mmpr_kernel_launches;
static inline void mmpr_launched(int n = 1) { g_mmpr_kernel_launches += (unsigned long long)n; }

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

// Per-device memo of kernel attributes already applied (cudaFuncSetAttribute
// acts on the current device; attributes are set outside graph captures on
// the first launch of a configuration and only raised afterwards).
#define MMPR_MAX_DEVICES 64
static inline int mmpr_current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return (dev >= 0 && dev < MMPR_MAX_DEVICES) ? dev : 0;
}
