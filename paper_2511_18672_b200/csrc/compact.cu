// compact.cu — step (2): block mask (+ frame eligibility) -> ascending block-id list.
//
// P:352 "enables batched convolution over selected blocks"; Alg1 line 17 (A_u = 1[k <= u])
// and line 19 (inactive frames).  At paper sizes the whole list is <= N*115 entries
// (19 320 for 168 frames), so the step is latency-bound: ONE CTA of 1024 threads per list
// walks the flat ids in rounds of 16 384 (16 consecutive ids per thread).
#include "common.cuh"

namespace sphinx {

// Each thread owns kE consecutive flat ids per round (1024 x 16 = 16 384 ids: one round for
// every list of a 168-frame batch), takes them in order, and its output slot is an exclusive
// scan of the per-thread counts (warp shuffle scan + a 32-entry cross-warp scan).  The order is
// the flat id by construction (no atomics), so the list is bit-exact and deterministic.
constexpr int kE = 16;

__device__ __forceinline__ void compact_list(const uint8_t* __restrict__ mask, int n, int per_frame,
                                             const int32_t* __restrict__ k, int u, int select,
                                             int32_t* __restrict__ ids, int32_t* __restrict__ count) {
  __shared__ int warp_off[32];
  __shared__ int round_total;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int total = n * per_frame;
  int base = 0;
  for (int start = 0; start < total; start += blockDim.x * kE) {
    const int id0 = start + threadIdx.x * kE;
    uint32_t takes = 0;
    if (id0 < total) {
      int fr = id0 / per_frame, rem = id0 - fr * per_frame;
      int kf = k ? __ldg(k + fr) : 0;
#pragma unroll
      for (int e = 0; e < kE; ++e) {
        const int id = id0 + e;
        if (id < total) {
          bool take;
          if (select == SPHINX_SELECT_ACTIVE) take = mask[id] && (!k || (kf >= 0 && kf <= u));
          else if (select == SPHINX_SELECT_INACTIVE_FRAMES) take = kf > u;
          else if (select == SPHINX_SELECT_NOISE) take = (mask[id] && kf >= 0 && kf <= u) || kf > u;
          else take = !k || kf >= 0;
          takes |= (uint32_t)take << e;
        }
        if (++rem == per_frame) {  // next frame
          rem = 0;
          ++fr;
          if (k && id + 1 < total) kf = __ldg(k + fr);
        }
      }
    }
    const int c = __popc(takes);
    int incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    if (lane == 31) warp_off[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int v = lane < nwarps ? warp_off[lane] : 0;
      int wi = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, wi, d);
        if (lane >= d) wi += o;
      }
      if (lane < nwarps) warp_off[lane] = wi - v;
      if (lane == 31) round_total = wi;
    }
    __syncthreads();
    int slot = base + warp_off[warp] + incl - c;
    while (takes) {
      const int e = __ffs(takes) - 1;
      takes &= takes - 1;
      ids[slot++] = id0 + e;
    }
    base += round_total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = base;
}

__global__ void __launch_bounds__(1024) compact_kernel(const uint8_t* __restrict__ mask, int n,
                                                       int per_frame, const int32_t* __restrict__ k,
                                                       int u, int select,
                                                       int32_t* __restrict__ ids,
                                                       int32_t* __restrict__ count) {
  pdl_wait();
  pdl_trigger();
  compact_list(mask, n, per_frame, k, u, select, ids, count);
}

struct CompactJobs {
  sphinx_compact_job j[SPHINX_MAX_COMPACT_JOBS];
};

// Several independent lists (e.g. the UNet levels and the inactive-frame list of one step) in
// ONE launch: CTA b compacts job b (each list is still one CTA, order = flat id).
__global__ void __launch_bounds__(1024) compact_batch_kernel(const __grid_constant__ CompactJobs jobs) {
  pdl_wait();
  pdl_trigger();
  const sphinx_compact_job& jb = jobs.j[blockIdx.x];
  compact_list(jb.block_mask, jb.n, jb.hb * jb.wb, jb.start_step, jb.step_u, (int)jb.select, jb.block_ids,
               jb.count);
}

}  // namespace sphinx

using namespace sphinx;

extern "C" sphinx_status sphinx_compact_blocks(const uint8_t* block_mask, int32_t n, int32_t hb,
                                               int32_t wb, const int32_t* start_step,
                                               int32_t step_u, sphinx_select select,
                                               int32_t* block_ids, int32_t* count,
                                               sphinx_stream_t stream) {
  if (!block_ids || !count || n <= 0 || hb <= 0 || wb <= 0) return SPHINX_ERR_INVALID_ARGUMENT;
  if (select != SPHINX_SELECT_ACTIVE && select != SPHINX_SELECT_INACTIVE_FRAMES &&
      select != SPHINX_SELECT_ALL && select != SPHINX_SELECT_NOISE)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if ((select == SPHINX_SELECT_ACTIVE || select == SPHINX_SELECT_NOISE) && !block_mask)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if ((select == SPHINX_SELECT_INACTIVE_FRAMES || select == SPHINX_SELECT_NOISE) && !start_step)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if ((int64_t)n * hb * wb > (int64_t)1 << 30) return SPHINX_ERR_UNSUPPORTED;
  sphinx_status st = check_device();
  if (st != SPHINX_OK) return st;
  cudaError_t e = launch_k(compact_kernel, dim3(1), dim3(1024), 0,
                           reinterpret_cast<cudaStream_t>(stream), block_mask, (int)n, (int)(hb * wb),
                           start_step, (int)step_u, (int)select, block_ids, count);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

extern "C" sphinx_status sphinx_compact_blocks_batch(const sphinx_compact_job* jobs, int32_t n_jobs,
                                                     sphinx_stream_t stream) {
  if (!jobs || n_jobs <= 0 || n_jobs > SPHINX_MAX_COMPACT_JOBS) return SPHINX_ERR_INVALID_ARGUMENT;
  CompactJobs cj;
  for (int i = 0; i < n_jobs; ++i) {
    const sphinx_compact_job& jb = jobs[i];
    if (!jb.block_ids || !jb.count || jb.n <= 0 || jb.hb <= 0 || jb.wb <= 0) return SPHINX_ERR_INVALID_ARGUMENT;
    if (jb.select != SPHINX_SELECT_ACTIVE && jb.select != SPHINX_SELECT_INACTIVE_FRAMES &&
        jb.select != SPHINX_SELECT_ALL && jb.select != SPHINX_SELECT_NOISE)
      return SPHINX_ERR_INVALID_ARGUMENT;
    if ((jb.select == SPHINX_SELECT_ACTIVE || jb.select == SPHINX_SELECT_NOISE) && !jb.block_mask)
      return SPHINX_ERR_INVALID_ARGUMENT;
    if ((jb.select == SPHINX_SELECT_INACTIVE_FRAMES || jb.select == SPHINX_SELECT_NOISE) && !jb.start_step)
      return SPHINX_ERR_INVALID_ARGUMENT;
    if ((int64_t)jb.n * jb.hb * jb.wb > (int64_t)1 << 30) return SPHINX_ERR_UNSUPPORTED;
    cj.j[i] = jb;
  }
  sphinx_status st = check_device();
  if (st != SPHINX_OK) return st;
  cudaError_t e = launch_k(compact_batch_kernel, dim3(n_jobs), dim3(1024), 0,
                           reinterpret_cast<cudaStream_t>(stream), cj);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}
