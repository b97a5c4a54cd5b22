// Library-level entry points of libmmpr: version and error reporting.
#include <cuda_runtime.h>
#include <stdio.h>

#include "capi_internal.h"

#ifndef MMPR_GIT_VERSION
#define MMPR_GIT_VERSION "dev"
#endif

static thread_local char g_last_error[512] = "";
unsigned long long g_mmpr_kernel_launches = 0;

void mmpr_set_error(const char *what, cudaError_t err) {
  snprintf(g_last_error, sizeof g_last_error, "%s: %s", what, cudaGetErrorString(err));
}

extern "C" const char *mmpr_version(void) { return "mmpr " MMPR_GIT_VERSION " sm_100a"; }

extern "C" const char *mmpr_last_error(void) { return g_last_error; }

extern "C" uint64_t mmpr_kernel_launches(void) { return (uint64_t)g_mmpr_kernel_launches; }
