// shard_plan.cu — §8(e) multi-GPU data plane: the frame -> rank plan on the device.
//
// P:333 (spatial ResNet layers act per frame: frames are the independent units), north_star
// ("balanced by active-block count"): every rank computes the SAME deterministic
// longest-processing-time plan from the all-gathered masks and start steps --
//   cost[f]  = sum_l count_l[f] * C_l^2, count_l[f] = listed level-l blocks of frame f if
//              0 <= k[f] <= u (the frame runs this step), else 0   (executed MMA work);
//   order    = cost descending, frame id ascending on ties;
//   each frame in order goes to the least-loaded rank, lowest rank on ties --
// exactly the rule of paper_2511_18672_b200/dist.py lpt_assign (its host twin, which the tests
// compare bit for bit).  Outputs, all on the device: rank_of[f], the load per rank, k_mine (k of
// this rank's frames, -1 elsewhere: the compaction input), pair[l][s][o] = level-l blocks computed
// by rank s for frames owned by rank o (the owner-gather sizes), recv[l] = blocks this rank
// receives at level l.  Keeping the plan on the device removes the step's host round trip from the
// critical path: the host reads pair only when it issues the exchange, after the convs are queued.
//
// One CTA of 1024 threads: per-frame counts (a thread per frame), a bitonic sort of 64-bit keys
// ((2^39 - 1 - cost) << 24 | f) in shared memory, then the greedy pass in warp 0 (lane r holds
// rank r's load; a 64-bit (load << 8 | rank) shuffle-min per frame picks the rank).
#include "common.cuh"

namespace sphinx {

constexpr int kPlanMaxFrames = 4096;
constexpr int kPlanMaxWorld = 32;

struct PlanLevels {
  const uint8_t* mask[4];
  int per_frame[4];  // hb * wb
  long long c2[4];   // C_l^2
};

__global__ void __launch_bounds__(1024) shard_plan_kernel(PlanLevels lv, int n_levels, int n,
                                                          const int32_t* __restrict__ k, int u,
                                                          const int32_t* __restrict__ owner, int world,
                                                          int rank, int32_t* __restrict__ k_mine,
                                                          int32_t* __restrict__ rank_of,
                                                          long long* __restrict__ load_out,
                                                          int32_t* __restrict__ pair,
                                                          int32_t* __restrict__ recv) {
  extern __shared__ unsigned long long s_key[];  // [npow2]
  __shared__ int s_pair[4 * kPlanMaxWorld * kPlanMaxWorld];
  pdl_wait();
  pdl_trigger();
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  int* s_rank = reinterpret_cast<int*>(s_key + npow2);                 // [n]
  int* s_cnt = s_rank + n;                                             // [n_levels][n]
  for (int i = threadIdx.x; i < n_levels * world * world; i += blockDim.x) s_pair[i] = 0;
  // per-frame counts and the sort keys
  for (int f = threadIdx.x; f < npow2; f += blockDim.x) {
    if (f >= n) {
      s_key[f] = ~0ull;  // padding sorts last
      continue;
    }
    const int kf = __ldg(k + f);
    const bool act = kf >= 0 && kf <= u;
    long long cost = 0;
    for (int l = 0; l < n_levels; ++l) {
      int c = 0;
      if (act) {
        const uint8_t* m = lv.mask[l] + (size_t)f * lv.per_frame[l];
        for (int j = 0; j < lv.per_frame[l]; ++j) c += m[j] != 0;
      }
      s_cnt[l * n + f] = c;
      cost += (long long)c * lv.c2[l];
    }
    s_key[f] = ((unsigned long long)((1ll << 39) - 1 - cost) << 24) | (unsigned long long)f;
  }
  __syncthreads();
  // bitonic sort, ascending key = cost descending, frame ascending
  for (int size = 2; size <= npow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const unsigned long long a = s_key[i], b = s_key[j];
          if ((a > b) == up) {
            s_key[i] = b;
            s_key[j] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  // greedy LPT in warp 0: lane r < world holds rank r's load
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    long long ld = 0;
    for (int i = 0; i < n; ++i) {
      const unsigned long long key = s_key[i];
      const int f = (int)(key & 0xFFFFFFull);
      const long long cost = (1ll << 39) - 1 - (long long)(key >> 24);
      unsigned long long v = lane < world ? ((unsigned long long)ld << 8) | (unsigned long long)lane : ~0ull;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, d);
        v = o < v ? o : v;
      }
      const int r = (int)(v & 0xFF);
      if (lane == r) ld += cost;
      if (lane == 0) s_rank[f] = r;
    }
    if (lane < world) load_out[lane] = ld;
  }
  __syncthreads();
  for (int f = threadIdx.x; f < n; f += blockDim.x) {
    const int r = s_rank[f];
    rank_of[f] = r;
    k_mine[f] = r == rank ? __ldg(k + f) : -1;
    const int o = __ldg(owner + f);
    for (int l = 0; l < n_levels; ++l) {
      const int c = s_cnt[l * n + f];
      if (c) atomicAdd(&s_pair[(l * world + r) * world + o], c);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_levels * world * world; i += blockDim.x) pair[i] = s_pair[i];
  if (threadIdx.x < n_levels) {
    const int l = threadIdx.x;
    int s = 0;
    for (int src = 0; src < world; ++src)
      if (src != rank) s += s_pair[(l * world + src) * world + rank];
    recv[l] = s;
  }
}

}  // namespace sphinx

using namespace sphinx;

extern "C" sphinx_status sphinx_shard_plan(uint8_t* const* block_mask, const int32_t* blocks_per_frame,
                                           const int32_t* channels, int32_t n_levels, int32_t n,
                                           const int32_t* start_step, int32_t step_u, const int32_t* owner,
                                           int32_t world, int32_t rank, int32_t* k_mine, int32_t* rank_of,
                                           int64_t* load, int32_t* pair, int32_t* recv,
                                           sphinx_stream_t stream) {
  if (!block_mask || !blocks_per_frame || !channels || !start_step || !owner || !k_mine || !rank_of || !load ||
      !pair || !recv)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (n_levels < 1 || n_levels > 4 || n <= 0 || world < 1 || rank < 0 || rank >= world)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (n > kPlanMaxFrames || world > kPlanMaxWorld) return SPHINX_ERR_UNSUPPORTED;
  PlanLevels lv{};
  for (int l = 0; l < n_levels; ++l) {
    if (!block_mask[l] || blocks_per_frame[l] <= 0 || channels[l] <= 0) return SPHINX_ERR_INVALID_ARGUMENT;
    lv.mask[l] = block_mask[l];
    lv.per_frame[l] = blocks_per_frame[l];
    lv.c2[l] = (long long)channels[l] * channels[l];
    // cost < 2^39 keeps the sort key exact: n_blocks * C^2 per level, summed
    if ((long long)blocks_per_frame[l] * lv.c2[l] > (1ll << 36)) return SPHINX_ERR_UNSUPPORTED;
  }
  sphinx_status st = check_device();
  if (st != SPHINX_OK) return st;
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  const size_t smem = (size_t)npow2 * 8 + (size_t)n * 4 * (1 + n_levels);
  auto kern = shard_plan_kernel;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e != cudaSuccess) return cuda_fail(e);
    attr = true;
  }
  cudaError_t e = launch_k(kern, dim3(1), dim3(1024), smem, reinterpret_cast<cudaStream_t>(stream), lv,
                           (int)n_levels, (int)n, start_step, (int)step_u, owner, (int)world, (int)rank, k_mine,
                           rank_of, reinterpret_cast<long long*>(load), pair, recv);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}
