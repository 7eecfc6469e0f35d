// ddim_step.cu — NEXT-1: the partial step's latent update on listed blocks.
//
// Alg1 line 18 (Z^(u+1)_{A_u} = D.partial_step(...)): the denoiser's clean-latent estimate
// x0_hat turns into the next latent by the deterministic DDIM rule (eta = 0):
//   eps_hat = (z - sqrt(abar[u]) x0_hat) / sqrt(1 - abar[u])
//   z'      = sqrt(abar[u+1]) x0_hat + sqrt(1 - abar[u+1]) eps_hat
// HBM-bound elementwise pass over the listed blocks only (12 B per element: z, x0_hat in,
// z' out), same thread layout as noise_inject (one 16-byte vector per thread).  The
// inactive frames' resampling (Alg1 line 19) is sphinx_noise_inject at step u+1.
#include "common.cuh"

namespace sphinx {

template <int V>
__global__ void __launch_bounds__(256) ddim_kernel(const float* z, const float* __restrict__ x0h,
                                                   float* z_out, int h, int w, int c, int b, int hb,
                                                   int wb, const int32_t* __restrict__ ids,
                                                   const int32_t* __restrict__ count, float a0,
                                                   float inv_s0, float a1, float s1) {
  pdl_wait();
  pdl_trigger();
  const int cnt = *count;
  const int vpp = c / V;
  const int per_block = b * b * vpp;
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
    if (y >= h || x >= w) continue;
    const size_t off = (((size_t)fr * h + y) * w + x) * c + (size_t)v * V;
    if constexpr (V == 4) {
      const float4 Z = *reinterpret_cast<const float4*>(z + off);
      const float4 X = __ldg(reinterpret_cast<const float4*>(x0h + off));
      float4 o;
      o.x = fmaf(a1, X.x, s1 * ((Z.x - a0 * X.x) * inv_s0));
      o.y = fmaf(a1, X.y, s1 * ((Z.y - a0 * X.y) * inv_s0));
      o.z = fmaf(a1, X.z, s1 * ((Z.z - a0 * X.z) * inv_s0));
      o.w = fmaf(a1, X.w, s1 * ((Z.w - a0 * X.w) * inv_s0));
      *reinterpret_cast<float4*>(z_out + off) = o;
    } else {
      const float X = __ldg(x0h + off);
      z_out[off] = fmaf(a1, X, s1 * ((z[off] - a0 * X) * inv_s0));
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
  const int V = vec ? 4 : 1;
  long long blocks = ((long long)capacity * b * b * (c / V) + 255) / 256;
  if (blocks > (long long)sms * 8) blocks = (long long)sms * 8;
  if (blocks < 1) blocks = 1;
  cudaError_t e = launch_k(vec ? ddim_kernel<4> : ddim_kernel<1>, dim3((unsigned)blocks), dim3(256), 0,
                           reinterpret_cast<cudaStream_t>(stream), z, x0_hat, z_out, (int)h, (int)w,
                           (int)c, (int)b, hb, wb, block_ids, count, a0, inv_s0, a1, s1);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}
