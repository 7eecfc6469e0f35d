// noise_inject.cu — step (3): forward noise on listed blocks only.
//
// Alg1 line 12 (Z^(k_min) = add_noise(Z^(0), k_min)) and line 19 (inactive frames
// resampled to u+1); formula z_u = sqrt(abar[u]) z0 + sqrt(1 - abar[u]) eps (S:303,
// north_star), u = 0 noisiest.
//
// HBM-bound elementwise pass: 12 B per element (x0, eps in; x_t out) on active blocks
// only.  One thread moves one 16-byte vector (4 channels) of one pixel; a block's row
// segment is contiguous in NHWC (b*C*4 bytes) so consecutive threads of a warp touch
// consecutive 16-byte words of the same segment.  The device count bounds the work;
// the grid is sized from the capacity, so no host read of the count is needed.
#include "common.cuh"

namespace sphinx {

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
  pdl_wait();
  pdl_trigger();
  const int cnt = *count;
  const int vpp = c / V;              // vectors per pixel
  const int per_block = b * b * vpp;  // vectors per (padded) block
  const long long total = (long long)cnt * per_block;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / per_block);
    const int r = (int)(e - (long long)j * per_block);
    const int p = r / vpp, v = r - p * vpp;
    const int id = __ldg(ids + j);
    const int fr = id / (hb * wb), rem = id - fr * hb * wb;
    const int by = rem / wb, bx = rem - by * wb;
    const int y = by * b + p / b, x = bx * b + p % b;
    if (y >= h || x >= w) continue;  // truncated edge block
    int u = __ldg(step + fr);
    if (step_u >= 0) u = u > step_u ? step_u + 1 : u;  // step = start steps: active k, inactive u+1
    if (u < 0 || u > S) continue;
    const float ab = __ldg(abar + u);
    const float a = sqrtf(ab), s = sqrtf(1.0f - ab);
    const size_t off = (((size_t)fr * h + y) * w + x) * c + (size_t)v * V;
    if constexpr (V == 4) {
      const float4 X = __ldg(reinterpret_cast<const float4*>(x0 + off));
      const float4 E = __ldg(reinterpret_cast<const float4*>(eps + off));
      float4 Z;
      Z.x = fmaf(a, X.x, s * E.x);
      Z.y = fmaf(a, X.y, s * E.y);
      Z.z = fmaf(a, X.z, s * E.z);
      Z.w = fmaf(a, X.w, s * E.w);
      *reinterpret_cast<float4*>(x_t + off) = Z;
    } else {
      x_t[off] = fmaf(a, __ldg(x0 + off), s * __ldg(eps + off));
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
  const int V = vec ? 4 : 1;
  const long long work = (long long)capacity * b * b * (c / V);
  long long blocks = (work + 255) / 256;
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
