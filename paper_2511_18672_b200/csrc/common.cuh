// common.cuh — shared host-side helpers of libsphinx (status plumbing, device checks).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/sphinx.h"

namespace sphinx {

// Records a CUDA error for sphinx_last_cuda_error() and maps it to SPHINX_ERR_CUDA.
sphinx_status cuda_fail(cudaError_t e);
// SPHINX_OK iff the current device is sm_100 (B200); caches per device.
sphinx_status check_device(int* sm_count = nullptr);
// True iff p is 16-byte aligned.
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline int cdiv(int a, int b) { return (a + b - 1) / b; }

}  // namespace sphinx

#define SPHINX_CHECK_LAUNCH()                          \
  do {                                                 \
    cudaError_t e_ = cudaGetLastError();               \
    if (e_ != cudaSuccess) return sphinx::cuda_fail(e_); \
  } while (0)
