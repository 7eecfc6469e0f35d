// uncertainty_map.cu — NEXT-2: the blur/uncertainty producer feeding step (1).
//
// Alg1 lines 7-8 (B = laplacian_var(X); M_blur = otsu(norm(B))); "The resulting blur
// map is smoothed, normalized, and inverted, followed by Otsu thresholding to obtain a binary
// mask where 1 indicates blurry pixels"; constants per SPEC S:196-222 (reading R-24):
//   Y = 0.299 R + 0.587 G + 0.114 B;  L = 3x3 Laplacian (edge replication);
//   V = population variance of L over a window x window neighbourhood (edge replication);
//   S = smooth x smooth box mean of V (edge replication);
//   U = 1 - (S - min S) / (max S - min S)   per frame (constant S -> U = 1);
//   tau[n] = Otsu over a 256-bin histogram of U (bin i = (i/256, (i+1)/256]), exact argmax.
// U and tau are exactly the (uncertainty, tau_u) inputs of sphinx_block_mask (U > tau blurry).
//
// Kernels: (1) fused stencil per 32x32 tile: Y, L, V, S staged in shared memory over the
// tile + halo (radius 1 + window/2 + smooth/2), S written to the output buffer and per-frame
// min/max folded with integer atomics (S >= 0, so float bits order as ints); (2) normalise +
// invert in place and a per-CTA shared histogram folded into the per-frame histogram
// (integer atomics: deterministic); (3) one CTA per frame: the exact Otsu argmax.
#include "common.cuh"

namespace sphinx {

constexpr int kUT = 32;  // output tile edge

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__global__ void __launch_bounds__(256) lapvar_smooth_kernel(const float* __restrict__ rgb, int h, int w,
                                                            int rv, int rs, float* __restrict__ S_out,
                                                            int* __restrict__ minmax) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float sm[];
  const int n = blockIdx.z;
  const int y0 = blockIdx.y * kUT, x0 = blockIdx.x * kUT;
  const int R = rs + rv + 1;
  const int NY = kUT + 2 * R, NL = kUT + 2 * (rs + rv), NV = kUT + 2 * rs;
  float* Ys = sm;                 // Ys[a][b] = Y(clamp(y0-R+a), clamp(x0-R+b))
  float* Ls = Ys + NY * NY;       // Ls[a][b] = L(clamp(y0-rs-rv+a), clamp(x0-rs-rv+b))
  float* Vs = Ls + NL * NL;       // Vs[a][b] = V(clamp(y0-rs+a), clamp(x0-rs+b))
  const size_t plane = (size_t)h * w;
  const float* img = rgb + (size_t)n * plane * 3;
  for (int i = threadIdx.x; i < NY * NY; i += blockDim.x) {
    const int a = i / NY, b = i - (i / NY) * NY;
    const int yy = clampi(y0 - R + a, 0, h - 1), xx = clampi(x0 - R + b, 0, w - 1);
    const float* px = img + ((size_t)yy * w + xx) * 3;
    Ys[i] = 0.299f * __ldg(px) + 0.587f * __ldg(px + 1) + 0.114f * __ldg(px + 2);
  }
  __syncthreads();
  // L at the (clamped) image position p, from Y at clamp(p +- 1): index = image coord - (y0 - R)
  for (int i = threadIdx.x; i < NL * NL; i += blockDim.x) {
    const int a = i / NL, b = i - (i / NL) * NL;
    const int py = clampi(y0 - rs - rv + a, 0, h - 1), px = clampi(x0 - rs - rv + b, 0, w - 1);
    const int cy = py - (y0 - R), cx = px - (x0 - R);
    const int uy = clampi(py - 1, 0, h - 1) - (y0 - R), dy = clampi(py + 1, 0, h - 1) - (y0 - R);
    const int lx = clampi(px - 1, 0, w - 1) - (x0 - R), rx = clampi(px + 1, 0, w - 1) - (x0 - R);
    Ls[i] = Ys[uy * NY + cx] + Ys[dy * NY + cx] + Ys[cy * NY + lx] + Ys[cy * NY + rx] -
            4.0f * Ys[cy * NY + cx];
  }
  __syncthreads();
  // V at the (clamped) position p: two-pass variance of L(clamp(p + d)), d in [-rv, rv]^2
  const float inv_cnt = 1.0f / (float)((2 * rv + 1) * (2 * rv + 1));
  for (int i = threadIdx.x; i < NV * NV; i += blockDim.x) {
    const int a = i / NV, b = i - (i / NV) * NV;
    const int py = clampi(y0 - rs + a, 0, h - 1), px = clampi(x0 - rs + b, 0, w - 1);
    float mean = 0.0f;
    for (int ddy = -rv; ddy <= rv; ++ddy) {
      const int ly = clampi(py + ddy, 0, h - 1) - (y0 - rs - rv);
      for (int ddx = -rv; ddx <= rv; ++ddx)
        mean += Ls[ly * NL + clampi(px + ddx, 0, w - 1) - (x0 - rs - rv)];
    }
    mean *= inv_cnt;
    float var = 0.0f;
    for (int ddy = -rv; ddy <= rv; ++ddy) {
      const int ly = clampi(py + ddy, 0, h - 1) - (y0 - rs - rv);
      for (int ddx = -rv; ddx <= rv; ++ddx) {
        const float d = Ls[ly * NL + clampi(px + ddx, 0, w - 1) - (x0 - rs - rv)] - mean;
        var = fmaf(d, d, var);
      }
    }
    Vs[i] = var * inv_cnt;
  }
  __syncthreads();
  // S = box mean of V(clamp(y + d)); per-CTA min/max of S
  const float inv_box = 1.0f / (float)((2 * rs + 1) * (2 * rs + 1));
  float lo = 3.0e38f, hi = 0.0f;
  for (int i = threadIdx.x; i < kUT * kUT; i += blockDim.x) {
    const int y = y0 + i / kUT, x = x0 + (i % kUT);
    if (y >= h || x >= w) continue;
    float sacc = 0.0f;
    for (int ddy = -rs; ddy <= rs; ++ddy) {
      const int vy = clampi(y + ddy, 0, h - 1) - (y0 - rs);
      for (int ddx = -rs; ddx <= rs; ++ddx) sacc += Vs[vy * NV + clampi(x + ddx, 0, w - 1) - (x0 - rs)];
    }
    const float sv = sacc * inv_box;
    S_out[(size_t)n * plane + (size_t)y * w + x] = sv;
    lo = fminf(lo, sv);
    hi = fmaxf(hi, sv);
  }
  for (int d = 16; d > 0; d >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, d));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, d));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(minmax + 2 * n, __float_as_int(lo));  // S >= +0: float order == int order
    atomicMax(minmax + 2 * n + 1, __float_as_int(hi));
  }
}

__device__ __forceinline__ int u_bin(float v) {
  // bin i = (i/256, (i+1)/256]; v * 256 is exact
  int t = (int)ceilf(v * 256.0f) - 1;
  return t < 0 ? 0 : (t > 255 ? 255 : t);
}

__global__ void __launch_bounds__(256) normalize_hist_kernel(float* U, int plane, const int* __restrict__ minmax,
                                                             int* __restrict__ hist) {
  pdl_wait();
  pdl_trigger();
  __shared__ int sh[256];
  const int n = blockIdx.y;
  sh[threadIdx.x] = 0;
  __syncthreads();
  const float lo = __int_as_float(minmax[2 * n]), hi = __int_as_float(minmax[2 * n + 1]);
  const float range = hi - lo;
  float* u = U + (size_t)n * plane;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < plane; p += gridDim.x * blockDim.x) {
    const float v = range > 0.0f ? 1.0f - (u[p] - lo) / range : 1.0f;  // normalise + invert
    u[p] = v;
    atomicAdd(&sh[u_bin(v)], 1);
  }
  __syncthreads();
  if (sh[threadIdx.x]) atomicAdd(hist + 256 * n + threadIdx.x, sh[threadIdx.x]);
}

typedef unsigned __int128 u128;

// One CTA (256 threads) per frame: thread k scores the split after bin k exactly,
// sigma_b^2 N^2 = (n0 S - N S0)^2 / (n0 n1) as (quotient, remainder, denominator); thread 0
// takes the first maximum (ties -> smaller k).  tau = (k+1)/256; one non-empty bin -> 1 (= max U).
__global__ void __launch_bounds__(256) otsu_kernel(const int* __restrict__ hist, float* __restrict__ tau) {
  pdl_wait();
  pdl_trigger();
  __shared__ long long h[256];
  __shared__ u128 sq[256], sr[256], sd[256];
  const int n = blockIdx.x, k = threadIdx.x;
  h[k] = hist[256 * n + k];
  __syncthreads();
  long long N = 0, S = 0, n0 = 0, s0 = 0;
  int nonempty = 0;
  for (int i = 0; i < 256; ++i) {
    N += h[i];
    S += (long long)i * h[i];
    nonempty += h[i] > 0;
    if (i <= k) {
      n0 += h[i];
      s0 += (long long)i * h[i];
    }
  }
  const long long n1 = N - n0;
  if (k < 255 && n0 > 0 && n1 > 0) {
    const __int128 d = (__int128)n0 * S - (__int128)N * s0;
    u128 num = (u128)(d < 0 ? -d : d);
    num = num * num;
    const u128 den = (u128)n0 * (u128)n1;
    sq[k] = num / den;
    sr[k] = num % den;
    sd[k] = den;
  } else {
    sq[k] = 0;
    sr[k] = 0;
    sd[k] = 1;
  }
  __syncthreads();
  if (k == 0) {
    if (nonempty <= 1) {
      tau[n] = 1.0f;
      return;
    }
    int best = 0;
    for (int j = 1; j < 255; ++j)
      if (sq[j] > sq[best] || (sq[j] == sq[best] && sr[j] * sd[best] > sr[best] * sd[j])) best = j;
    tau[n] = (float)(best + 1) / 256.0f;
  }
}

}  // namespace sphinx

using namespace sphinx;

extern "C" size_t sphinx_uncertainty_workspace_size(int32_t n) {
  return n > 0 ? (size_t)n * 258 * sizeof(int32_t) : 0;
}

extern "C" sphinx_status sphinx_uncertainty_map(const float* rgb, int32_t n, int32_t h, int32_t w,
                                                int32_t window, int32_t smooth, float* uncertainty,
                                                float* tau_u, void* workspace,
                                                size_t workspace_bytes, sphinx_stream_t stream) {
  if (!rgb || !uncertainty || !tau_u || !workspace || n <= 0 || h <= 0 || w <= 0)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (window < 3 || window % 2 == 0 || smooth < 1 || smooth % 2 == 0)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < sphinx_uncertainty_workspace_size(n)) return SPHINX_ERR_INVALID_ARGUMENT;
  if (window > 15 || smooth > 15 || (int64_t)h * w > ((int64_t)1 << 26)) return SPHINX_ERR_UNSUPPORTED;
  sphinx_status st = check_device();
  if (st != SPHINX_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int* minmax = static_cast<int*>(workspace);
  int* hist = minmax + 2 * n;
  // min slots <- 0x7F7F7F7F (3.4e38, above any S), max slots and histograms <- 0
  cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)n * 256 * sizeof(int), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(minmax, 0x7F, (size_t)n * 2 * sizeof(int), s);
  if (e != cudaSuccess) return cuda_fail(e);
  // the max slots must start at 0: clear every second word with a strided 2-D memset
  e = cudaMemset2DAsync(minmax + 1, 2 * sizeof(int), 0, sizeof(int), (size_t)n, s);
  if (e != cudaSuccess) return cuda_fail(e);
  const int rv = window / 2, rs = smooth / 2, R = rs + rv + 1;
  const int NY = kUT + 2 * R, NL = kUT + 2 * (rs + rv), NV = kUT + 2 * rs;
  const size_t smem = (size_t)(NY * NY + NL * NL + NV * NV) * sizeof(float);
  static bool attr_set = false;
  if (!attr_set) {
    e = cudaFuncSetAttribute(lapvar_smooth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e != cudaSuccess) return cuda_fail(e);
    attr_set = true;
  }
  e = launch_k(lapvar_smooth_kernel, dim3(cdiv(w, kUT), cdiv(h, kUT), n), dim3(256), smem, s, rgb,
               (int)h, (int)w, rv, rs, uncertainty, minmax);
  if (e != cudaSuccess) return cuda_fail(e);
  const int plane = h * w;
  e = launch_k(normalize_hist_kernel, dim3(cdiv(plane, 256 * 8), n), dim3(256), 0, s, uncertainty, plane,
               static_cast<const int*>(minmax), hist);
  if (e != cudaSuccess) return cuda_fail(e);
  e = launch_k(otsu_kernel, dim3(n), dim3(256), 0, s, static_cast<const int*>(hist), tau_u);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}
