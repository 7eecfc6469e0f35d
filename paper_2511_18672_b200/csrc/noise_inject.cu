// noise_inject.cu — step (3): forward noise on listed blocks only.
//
// Alg1 line 12 (Z^(k_min) = add_noise(Z^(0), k_min)) and line 19 (inactive frames
// resampled to u+1); formula z_u = sqrt(abar[u]) z0 + sqrt(1 - abar[u]) eps (S:303,
// north_star), u = 0 noisiest.
//
// HBM-bound elementwise pass: 12 B per element (x0, eps in; x_t out) on active blocks
// only.  A warp moves whole blocks, its lanes 16-byte vectors (4 channels); a block's row
// segment is contiguous in NHWC (b*C*4 bytes) so consecutive lanes touch consecutive
// 16-byte words of the same segment.  The device count bounds the work;
// the grid is sized from the capacity, so no host read of the count is needed.
#include <type_traits>

#include "common.cuh"

namespace sphinx {

// Work layout: one warp per listed block, kBlk blocks per warp pass (grid stride over the list),
// lanes over the blocks' 16-byte vectors.  A block row is one contiguous run of b*C elements in
// NHWC, so a vector's offset is base + row * (w*C) + col with (row, col) from a shift when the
// row's vector count is a power of two (every b = 4 / 8 map) -- no per-vector divisions (round
// 2's flat-index version spent half its issue slots on 64-bit index division: ncu 1.9 TB/s).
// Every data load of a pass is issued before any store and before the step check, so a warp's
// dependent chain is count -> ids -> {x0, eps, step} per pass (measured, tools/mem_ab.py on 168
// frames x 72x72x4: 10.0 -> 6.1 us L2-warm, ncu cold 14.2 -> 12.2 us).
constexpr int kMaxAbar = 1024;  // abar entries staged in shared memory (larger S: read from global)
constexpr int kItems = 2;       // vectors per lane per block and pass (a whole 8x8x4 fp32 block)
constexpr int kBlk = 1;         // blocks per warp pass (2: measured equal, tools/mem_ab.py)

template <int V>
__global__ void __launch_bounds__(256) noise_kernel(const float* __restrict__ x0,
                                                    const float* __restrict__ eps,
                                                    float* x_t, int h, int w, int c, int b,
                                                    int hb, int wb,
                                                    const int32_t* __restrict__ ids,
                                                    const int32_t* __restrict__ count,
                                                    const int32_t* __restrict__ step,
                                                    const float* __restrict__ abar, int S,
                                                    int step_u) {
  using VecT = typename std::conditional<V == 4, float4, float>::type;
  __shared__ float s_abar[kMaxAbar];
  pdl_wait();
  pdl_trigger();
  const bool staged = S + 1 <= kMaxAbar;
  if (staged)
    for (int i = threadIdx.x; i <= S; i += blockDim.x) s_abar[i] = __ldg(abar + i);
  const int cnt = *count;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int vpp = c / V;
  const int rowv = b * vpp;  // vectors per block row
  const int sh = (rowv & (rowv - 1)) == 0 ? __ffs(rowv) - 1 : -1;
  const int per_block = b * rowv;
  const size_t row_stride = (size_t)w * c;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int j0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j0 < cnt; j0 += kBlk * nwarps) {
    int id[kBlk];
#pragma unroll
    for (int k = 0; k < kBlk; ++k) id[k] = j0 + k * nwarps < cnt ? __ldg(ids + j0 + k * nwarps) : -1;
    BlockRef br[kBlk];
    int u[kBlk];
#pragma unroll
    for (int k = 0; k < kBlk; ++k) {
      br[k] = block_ref(id[k] < 0 ? 0 : id[k], h, w, c, b, hb, wb, vpp);
      if (id[k] < 0) br[k].rows = 0;
      u[k] = id[k] < 0 ? -1 : __ldg(step + br[k].fr);
    }
    for (int t0 = lane; t0 < per_block; t0 += 32 * kItems) {
      size_t off[kBlk][kItems];
      bool ok[kBlk][kItems];
      VecT X[kBlk][kItems], E[kBlk][kItems];
#pragma unroll
      for (int k = 0; k < kBlk; ++k)
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
          const int t = t0 + 32 * i;
          const int r = sh >= 0 ? t >> sh : t / rowv;
          const int col = t - r * rowv;
          ok[k][i] = t < per_block && r < br[k].rows && col < br[k].colv;  // truncated edge blocks
          off[k][i] = br[k].base + (size_t)r * row_stride + (size_t)col * V;
          if (ok[k][i]) {
            X[k][i] = __ldg(reinterpret_cast<const VecT*>(x0 + off[k][i]));
            E[k][i] = __ldg(reinterpret_cast<const VecT*>(eps + off[k][i]));
          }
        }
#pragma unroll
      for (int k = 0; k < kBlk; ++k) {
        int uu = u[k];
        if (step_u >= 0) uu = uu > step_u ? step_u + 1 : uu;  // start steps: active k, inactive u+1
        if (uu < 0 || uu > S) continue;  // (checked after the loads: they do not wait for it)
        const float ab = staged ? s_abar[uu] : __ldg(abar + uu);
        const float a = sqrtf(ab), s = sqrtf(1.0f - ab);
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
          if (!ok[k][i]) continue;
          if constexpr (V == 4) {
            float4 Z;
            Z.x = fmaf(a, X[k][i].x, s * E[k][i].x);
            Z.y = fmaf(a, X[k][i].y, s * E[k][i].y);
            Z.z = fmaf(a, X[k][i].z, s * E[k][i].z);
            Z.w = fmaf(a, X[k][i].w, s * E[k][i].w);
            *reinterpret_cast<float4*>(x_t + off[k][i]) = Z;
          } else {
            x_t[off[k][i]] = fmaf(a, X[k][i], s * E[k][i]);
          }
        }
      }
    }
  }
}

}  // namespace sphinx

using namespace sphinx;

static sphinx_status noise_impl(const float* x0, const float* eps, float* x_t, int32_t n, int32_t h,
                                int32_t w, int32_t c, int32_t b, const int32_t* block_ids,
                                const int32_t* count, int32_t capacity, const int32_t* step,
                                const float* abar, int32_t total_steps, int32_t step_u,
                                sphinx_stream_t stream) {
  if (!x0 || !eps || !x_t || !block_ids || !count || !step || !abar)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || b <= 0 || capacity < 0 || total_steps < 2)
    return SPHINX_ERR_INVALID_ARGUMENT;
  const int hb = cdiv(h, b), wb = cdiv(w, b);
  if ((int64_t)capacity > (int64_t)n * hb * wb) return SPHINX_ERR_INVALID_ARGUMENT;
  if (x_t != x0 && ((x_t < x0 + (size_t)n * h * w * c) && (x0 < x_t + (size_t)n * h * w * c)))
    return SPHINX_ERR_INVALID_ARGUMENT;  // partial overlap
  int sms = 0;
  sphinx_status st = check_device(&sms);
  if (st != SPHINX_OK) return st;
  if (capacity == 0) return SPHINX_OK;
  const bool vec = (c % 4 == 0) && aligned16(x0) && aligned16(eps) && aligned16(x_t);
  // one warp per kBlk listed blocks, 8 warps per CTA
  long long blocks = ((long long)capacity + 8 * kBlk - 1) / (8 * kBlk);
  const long long cap = (long long)sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = launch_k(vec ? noise_kernel<4> : noise_kernel<1>, dim3((unsigned)blocks), dim3(256),
                           0, s, x0, eps, x_t, (int)h, (int)w, (int)c, (int)b, hb, wb, block_ids,
                           count, step, abar, (int)total_steps, (int)step_u);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

extern "C" sphinx_status sphinx_noise_inject(const float* x0, const float* eps, float* x_t,
                                             int32_t n, int32_t h, int32_t w, int32_t c,
                                             int32_t b, const int32_t* block_ids,
                                             const int32_t* count, int32_t capacity,
                                             const int32_t* step, const float* abar,
                                             int32_t total_steps, sphinx_stream_t stream) {
  return noise_impl(x0, eps, x_t, n, h, w, c, b, block_ids, count, capacity, step, abar, total_steps, -1,
                    stream);
}

extern "C" sphinx_status sphinx_noise_inject_step(const float* x0, const float* eps, float* x_t,
                                                  int32_t n, int32_t h, int32_t w, int32_t c,
                                                  int32_t b, const int32_t* block_ids,
                                                  const int32_t* count, int32_t capacity,
                                                  const int32_t* start_step, int32_t step_u,
                                                  const float* abar, int32_t total_steps,
                                                  sphinx_stream_t stream) {
  if (step_u < 0 || step_u + 1 > total_steps) return SPHINX_ERR_INVALID_ARGUMENT;
  return noise_impl(x0, eps, x_t, n, h, w, c, b, block_ids, count, capacity, start_step, abar, total_steps,
                    step_u, stream);
}
