// ddim_step.cu — NEXT-1: the partial step's latent update on listed blocks.
//
// Alg1 line 18 (Z^(u+1)_{A_u} = D.partial_step(...)): the denoiser's clean-latent estimate
// x0_hat turns into the next latent by the deterministic DDIM rule (eta = 0):
//   eps_hat = (z - sqrt(abar[u]) x0_hat) / sqrt(1 - abar[u])
//   z'      = sqrt(abar[u+1]) x0_hat + sqrt(1 - abar[u+1]) eps_hat
// HBM-bound elementwise pass over the listed blocks only (12 B per element: z, x0_hat in,
// z' out), same thread layout as noise_inject (one 16-byte vector per thread).  The
// inactive frames' resampling (Alg1 line 19) is sphinx_noise_inject at step u+1.
#include <type_traits>

#include "common.cuh"

namespace sphinx {

// Same work layout as noise_inject.cu: one warp per listed block (kDdimBlk blocks per pass),
// lanes over the blocks' 16-byte vectors (row, column from a shift: no per-vector division), all
// of a pass's loads issued before its stores (tools/mem_ab.py: 8.4 -> 4.9 us L2-warm, ncu cold
// 12.5 -> 10.2 us).
constexpr int kDdimItems = 2;
constexpr int kDdimBlk = 1;  // blocks per warp pass (2: measured equal)

template <int V>
__global__ void __launch_bounds__(256) ddim_kernel(const float* z, const float* __restrict__ x0h,
                                                   float* z_out, int h, int w, int c, int b, int hb,
                                                   int wb, const int32_t* __restrict__ ids,
                                                   const int32_t* __restrict__ count, float a0,
                                                   float inv_s0, float a1, float s1) {
  using VecT = typename std::conditional<V == 4, float4, float>::type;
  pdl_wait();
  pdl_trigger();
  const int cnt = *count;
  const int lane = threadIdx.x & 31;
  const int vpp = c / V;
  const int rowv = b * vpp;  // vectors per block row
  const int sh = (rowv & (rowv - 1)) == 0 ? __ffs(rowv) - 1 : -1;
  const int per_block = b * rowv;
  const size_t row_stride = (size_t)w * c;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int j0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j0 < cnt; j0 += kDdimBlk * nwarps) {
    BlockRef br[kDdimBlk];
#pragma unroll
    for (int k = 0; k < kDdimBlk; ++k) {
      const bool has = j0 + k * nwarps < cnt;
      br[k] = block_ref(has ? __ldg(ids + j0 + k * nwarps) : 0, h, w, c, b, hb, wb, vpp);
      if (!has) br[k].rows = 0;
    }
    for (int t0 = lane; t0 < per_block; t0 += 32 * kDdimItems) {
      size_t off[kDdimBlk][kDdimItems];
      bool ok[kDdimBlk][kDdimItems];
      VecT Z[kDdimBlk][kDdimItems], X[kDdimBlk][kDdimItems];
#pragma unroll
      for (int k = 0; k < kDdimBlk; ++k)
#pragma unroll
        for (int i = 0; i < kDdimItems; ++i) {
          const int t = t0 + 32 * i;
          const int r = sh >= 0 ? t >> sh : t / rowv;
          const int col = t - r * rowv;
          ok[k][i] = t < per_block && r < br[k].rows && col < br[k].colv;  // truncated edge blocks
          off[k][i] = br[k].base + (size_t)r * row_stride + (size_t)col * V;
          if (ok[k][i]) {
            Z[k][i] = *reinterpret_cast<const VecT*>(z + off[k][i]);
            X[k][i] = __ldg(reinterpret_cast<const VecT*>(x0h + off[k][i]));
          }
        }
#pragma unroll
      for (int k = 0; k < kDdimBlk; ++k)
#pragma unroll
        for (int i = 0; i < kDdimItems; ++i) {
          if (!ok[k][i]) continue;
          if constexpr (V == 4) {
            float4 o;
            o.x = fmaf(a1, X[k][i].x, s1 * ((Z[k][i].x - a0 * X[k][i].x) * inv_s0));
            o.y = fmaf(a1, X[k][i].y, s1 * ((Z[k][i].y - a0 * X[k][i].y) * inv_s0));
            o.z = fmaf(a1, X[k][i].z, s1 * ((Z[k][i].z - a0 * X[k][i].z) * inv_s0));
            o.w = fmaf(a1, X[k][i].w, s1 * ((Z[k][i].w - a0 * X[k][i].w) * inv_s0));
            *reinterpret_cast<float4*>(z_out + off[k][i]) = o;
          } else {
            z_out[off[k][i]] = fmaf(a1, X[k][i], s1 * ((Z[k][i] - a0 * X[k][i]) * inv_s0));
          }
        }
    }
  }
}

}  // namespace sphinx

using namespace sphinx;

extern "C" sphinx_status sphinx_ddim_step(const float* z, const float* x0_hat, float* z_out,
                                          int32_t n, int32_t h, int32_t w, int32_t c, int32_t b,
                                          const int32_t* block_ids, const int32_t* count,
                                          int32_t capacity, int32_t step_u, const float* abar_host,
                                          int32_t total_steps, sphinx_stream_t stream) {
  if (!z || !x0_hat || !z_out || !block_ids || !count || !abar_host)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || b <= 0 || capacity < 0 || total_steps < 2)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (step_u < 0 || step_u >= total_steps) return SPHINX_ERR_INVALID_ARGUMENT;
  const int hb = cdiv(h, b), wb = cdiv(w, b);
  if ((int64_t)capacity > (int64_t)n * hb * wb) return SPHINX_ERR_INVALID_ARGUMENT;
  const double ab0 = abar_host[step_u], ab1 = abar_host[step_u + 1];
  if (!(ab0 >= 0.0 && ab0 < 1.0 && ab1 >= 0.0 && ab1 <= 1.0)) return SPHINX_ERR_INVALID_ARGUMENT;
  int sms = 0;
  sphinx_status st = check_device(&sms);
  if (st != SPHINX_OK) return st;
  if (capacity == 0) return SPHINX_OK;
  // the step is a host scalar: the four coefficients are computed once, correctly rounded
  const float a0 = (float)sqrt(ab0), inv_s0 = (float)(1.0 / sqrt(1.0 - ab0));
  const float a1 = (float)sqrt(ab1), s1 = (float)sqrt(1.0 - ab1);
  const bool vec = (c % 4 == 0) && aligned16(z) && aligned16(x0_hat) && aligned16(z_out);
  long long blocks = ((long long)capacity + 8 * kDdimBlk - 1) / (8 * kDdimBlk);  // a warp per kDdimBlk blocks
  if (blocks > (long long)sms * 8) blocks = (long long)sms * 8;
  if (blocks < 1) blocks = 1;
  cudaError_t e = launch_k(vec ? ddim_kernel<4> : ddim_kernel<1>, dim3((unsigned)blocks), dim3(256), 0,
                           reinterpret_cast<cudaStream_t>(stream), z, x0_hat, z_out, (int)h, (int)w,
                           (int)c, (int)b, hb, wb, block_ids, count, a0, inv_s0, a1, s1);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}
