// common.cuh — shared host-side helpers of libsphinx (status plumbing, device checks).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <utility>

#include "../../include/sphinx.h"

namespace sphinx {

// Records a CUDA error for sphinx_last_cuda_error() and maps it to SPHINX_ERR_CUDA.
sphinx_status cuda_fail(cudaError_t e);
// SPHINX_OK iff the current device is sm_100 (B200); caches per device.
sphinx_status check_device(int* sm_count = nullptr);
// True iff p is 16-byte aligned.
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline int cdiv(int a, int b) { return (a + b - 1) / b; }

// ---- programmatic dependent launch (PDL)
// Every sphinx kernel is launched with programmatic stream serialization: its CTAs may start
// while the previous kernel in the stream drains; each kernel runs its setup (smem carve-up,
// mbarrier init, TMEM alloc, tensor-map prefetch) first, then pdl_wait() before touching any
// data produced upstream.  pdl_trigger() lets the next kernel begin launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();  // SPHINX_PDL=0 disables (A/B measurement)

// A listed block of an NHWC map [N][h][w][c] (b x b pixels, hb x wb blocks per frame): element
// offset of its first pixel, valid rows, valid vectors per row (vpp vectors per pixel), frame.
struct BlockRef {
  size_t base;  // element offset of the block's first pixel
  int rows, colv, fr;
};

__device__ __forceinline__ BlockRef block_ref(int id, int h, int w, int c, int b, int hb, int wb,
                                              int vpp) {
  BlockRef r;
  r.fr = id / (hb * wb);
  const int rem = id - r.fr * hb * wb;
  const int by = rem / wb, bx = rem - by * wb;
  r.rows = min(b, h - by * b);
  r.colv = min(b, w - bx * b) * vpp;
  r.base = (((size_t)r.fr * h + by * b) * w + (size_t)bx * b) * c;
  return r;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace sphinx

#define SPHINX_CHECK_LAUNCH()                          \
  do {                                                 \
    cudaError_t e_ = cudaGetLastError();               \
    if (e_ != cudaSuccess) return sphinx::cuda_fail(e_); \
  } while (0)
