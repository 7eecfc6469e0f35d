// compact.cu — step (2): block mask (+ frame eligibility) -> ascending block-id list.
//
// P:352 "enables batched convolution over selected blocks"; Alg1 line 17 (A_u = 1[k <= u])
// and line 19 (inactive frames).  At paper sizes the whole list is <= N*115 entries
// (19 320 for 168 frames), so the step is latency-bound: ONE CTA of 1024 threads walks
// the flat ids in rounds of 1024, each thread tests one block, and the output slot is
// a warp-ballot/popc prefix plus a 32-entry cross-warp scan.  The order is the flat
// id by construction (no atomics), so the list is bit-exact and deterministic.
#include "common.cuh"

namespace sphinx {

__device__ __forceinline__ void compact_list(const uint8_t* __restrict__ mask, int n, int per_frame,
                                             const int32_t* __restrict__ k, int u, int select,
                                             int32_t* __restrict__ ids, int32_t* __restrict__ count) {
  __shared__ int warp_off[32];
  __shared__ int round_total;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int total = n * per_frame;
  int base = 0;
  for (int start = 0; start < total; start += blockDim.x) {
    const int id = start + threadIdx.x;
    bool take = false;
    if (id < total) {
      const int fr = id / per_frame;
      if (select == SPHINX_SELECT_ACTIVE) {
        const int kf = k ? __ldg(k + fr) : 0;
        take = mask[id] && (!k || (kf >= 0 && kf <= u));
      } else if (select == SPHINX_SELECT_INACTIVE_FRAMES) {
        take = __ldg(k + fr) > u;
      } else {
        take = !k || __ldg(k + fr) >= 0;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    const int pre = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) warp_off[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      const int v = lane < nwarps ? warp_off[lane] : 0;
      int incl = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += o;
      }
      if (lane < nwarps) warp_off[lane] = incl - v;
      if (lane == 31) round_total = incl;
    }
    __syncthreads();
    if (take) ids[base + warp_off[warp] + pre] = id;
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
      select != SPHINX_SELECT_ALL)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (select == SPHINX_SELECT_ACTIVE && !block_mask) return SPHINX_ERR_INVALID_ARGUMENT;
  if (select == SPHINX_SELECT_INACTIVE_FRAMES && !start_step) return SPHINX_ERR_INVALID_ARGUMENT;
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
        jb.select != SPHINX_SELECT_ALL)
      return SPHINX_ERR_INVALID_ARGUMENT;
    if (jb.select == SPHINX_SELECT_ACTIVE && !jb.block_mask) return SPHINX_ERR_INVALID_ARGUMENT;
    if (jb.select == SPHINX_SELECT_INACTIVE_FRAMES && !jb.start_step) return SPHINX_ERR_INVALID_ARGUMENT;
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
