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
// Kernels: (1) fused stencil per 32x32 tile: Y, L, V (separable fp64 window sums), S
// (separable box) staged in shared memory over the tile + halo (radius 1 + window/2 +
// smooth/2), S written to the output buffer and per-frame min/max folded with integer
// atomics (S >= 0, so float bits order as ints); (2) normalise +
// invert in place and a per-CTA shared histogram folded into the per-frame histogram
// (integer atomics: deterministic); (3) one CTA per frame: the exact Otsu argmax.
#include "common.cuh"

namespace sphinx {

constexpr int kUT = 32;  // output tile edge

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Every stage works on the in-image rectangle its consumer needs and reads the previous stage
// with image-clamped coordinates (edge replication of each stage's input, exactly as defined):
//   S rows [sy0, sy1)  <- V rows [vy0, vy1) = [max(0, sy0-rs), min(h, sy1+rs))
//   V rows [vy0, vy1)  <- L rows [ly0, ly1) = [max(0, vy0-rv), min(h, vy1+rv))
//   L rows [ly0, ly1)  <- Y rows [yy0, yy1) = [max(0, ly0-1), min(h, ly1+1))      (same in x)
// The window variance uses separable fp32 row/column sums of L and L^2:
//   V = E[L^2] - E[L]^2 over the (2rv+1)^2 window.  The cancellation error is
//   ~ 2^-23 E[L^2]; for images in [0,1] the Laplacian of a window with small variance but a
//   large mean (constant curvature) is itself small, so after min-max normalisation the error
//   stays ~1e-6 (parity tolerance 1e-4 vs the fp64 two-pass oracle, tests/test_gpu_parity).
// RV, RS > 0: compile-time radii (the SPEC defaults 3 / 2): the window loops unroll and taps away
// from the image border skip the clamp (measured ncu: the generic version was issue-bound at 88%
// SM throughput on index arithmetic).  RV = RS = 0: runtime radii.
// INT: the tile's whole halo lies inside the image (about 79% of the 576x576 tiles), so no tap
// needs an edge-replication clamp or a per-element border test.
template <int RV, int RS, bool INT>
__device__ __forceinline__ void lapvar_body(const float* __restrict__ rgb, int h, int w, int rv_rt,
                                            int rs_rt, float* __restrict__ S_out, int* __restrict__ minmax,
                                            unsigned char* smraw) {
  const int rv = RV > 0 ? RV : rv_rt, rs = RS > 0 ? RS : rs_rt;
  const int n = blockIdx.z;
  const int sy0 = blockIdx.y * kUT, sx0 = blockIdx.x * kUT;
  const int sy1 = min(h, sy0 + kUT), sx1 = min(w, sx0 + kUT);
  const int vy0 = max(0, sy0 - rs), vy1 = min(h, sy1 + rs), vx0 = max(0, sx0 - rs), vx1 = min(w, sx1 + rs);
  const int ly0 = max(0, vy0 - rv), ly1 = min(h, vy1 + rv), lx0 = max(0, vx0 - rv), lx1 = min(w, vx1 + rv);
  const int yy0 = max(0, ly0 - 1), yy1 = min(h, ly1 + 1), yx0 = max(0, lx0 - 1), yx1 = min(w, lx1 + 1);
  const int YW = yx1 - yx0, LW = lx1 - lx0, VW = vx1 - vx0, SW = sx1 - sx0;
  const int YH = yy1 - yy0, LH = ly1 - ly0, VH = vy1 - vy0, SH = sy1 - sy0;
  // smem carve-up (max extents for T=32, r<=7: Y 62x62, L 60x60, rowsums 60x46 x2 fp64, V 46x46,
  // S-rowsums 46x32)
  float* R1 = reinterpret_cast<float*>(smraw);              // [LH][VW] sum_dx L
  float* R2 = R1 + LH * VW;                                 // [LH][VW] sum_dx L^2
  float* Ys = reinterpret_cast<float*>(R2 + LH * VW);       // [YH][YW]
  float* Ls = Ys + YH * YW;                                 // [LH][LW]
  float* Vs = Ls + LH * LW;                                 // [VH][VW]
  float* Ts = Vs + VH * VW;                                 // [VH][SW] sum_dx V (box rows)
  const size_t plane = (size_t)h * w;
  const float* img = rgb + (size_t)n * plane * 3;
  // luminance of the tile + halo: 8 pixels (24 independent loads) in flight per thread (one
  // pixel per iteration left each warp ~11 serial load latencies: ncu's top stall)
  {
    const int ny = YH * YW;
    for (int e0 = threadIdx.x; e0 < ny; e0 += 8 * 256) {
      float v[8][3];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int e = e0 + k * 256;
        if (e < ny) {
          const int a = e / YW, c = e - a * YW;
          const float* px = img + ((size_t)(yy0 + a) * w + (yx0 + c)) * 3;
          v[k][0] = __ldg(px);
          v[k][1] = __ldg(px + 1);
          v[k][2] = __ldg(px + 2);
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int e = e0 + k * 256;
        if (e < ny) Ys[e] = 0.299f * v[k][0] + 0.587f * v[k][1] + 0.114f * v[k][2];
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < LH * LW; e += blockDim.x) {
   const int a = __float2int_rz(((float)e + 0.5f) * (1.0f / (float)LW)), c = e - a * LW;
    const int i = a * LW + c;
    const int py = ly0 + a, px = lx0 + c;  // in-image position; neighbours clamped to the image
    const int cy = py - yy0, cx = px - yx0;
    const int uy = (INT ? py - 1 : max(py - 1, 0)) - yy0, dy = (INT ? py + 1 : min(py + 1, h - 1)) - yy0;
    const int lx = (INT ? px - 1 : max(px - 1, 0)) - yx0, rx = (INT ? px + 1 : min(px + 1, w - 1)) - yx0;
    Ls[i] = Ys[uy * YW + cx] + Ys[dy * YW + cx] + Ys[cy * YW + lx] + Ys[cy * YW + rx] - 4.0f * Ys[cy * YW + cx];
   }
  __syncthreads();
  for (int e = threadIdx.x; e < LH * VW; e += blockDim.x) {  // horizontal window sums of L and L^2
    const int a = __float2int_rz(((float)e + 0.5f) * (1.0f / (float)VW)), c = e - a * VW;
      const int px = vx0 + c;
      float s1 = 0.0f, s2 = 0.0f;
      if (INT || (px - rv >= 0 && px + rv < w)) {
        const float* lr = Ls + a * LW + (px - lx0);
        if constexpr (RV > 0) {
#pragma unroll
          for (int d = -RV; d <= RV; ++d) {
            const float l = lr[d];
            s1 += l;
            s2 = fmaf(l, l, s2);
          }
        } else {
          for (int d = -rv; d <= rv; ++d) {
            const float l = lr[d];
            s1 += l;
            s2 = fmaf(l, l, s2);
          }
        }
      } else {
        for (int d = -rv; d <= rv; ++d) {
          const float l = Ls[a * LW + min(max(px + d, 0), w - 1) - lx0];
          s1 += l;
          s2 = fmaf(l, l, s2);
        }
      }
      R1[a * VW + c] = s1;
      R2[a * VW + c] = s2;
    }
  __syncthreads();
  const float inv_cnt = 1.0f / (float)((2 * rv + 1) * (2 * rv + 1));
  for (int e = threadIdx.x; e < VH * VW; e += blockDim.x) {  // vertical window sums -> variance
    const int a = __float2int_rz(((float)e + 0.5f) * (1.0f / (float)VW)), c = e - a * VW;
      const int py = vy0 + a;
      float s1 = 0.0f, s2 = 0.0f;
      if (INT || (py - rv >= 0 && py + rv < h)) {
        const float* r1 = R1 + (py - ly0) * VW + c;
        const float* r2 = R2 + (py - ly0) * VW + c;
        if constexpr (RV > 0) {
#pragma unroll
          for (int d = -RV; d <= RV; ++d) {
            s1 += r1[d * VW];
            s2 += r2[d * VW];
          }
        } else {
          for (int d = -rv; d <= rv; ++d) {
            s1 += r1[d * VW];
            s2 += r2[d * VW];
          }
        }
      } else {
        for (int d = -rv; d <= rv; ++d) {
          const int r = min(max(py + d, 0), h - 1) - ly0;
          s1 += R1[r * VW + c];
          s2 += R2[r * VW + c];
        }
      }
      const float m = s1 * inv_cnt;
      Vs[a * VW + c] = fmaxf(fmaf(-m, m, s2 * inv_cnt), 0.0f);
    }
  __syncthreads();
  for (int e = threadIdx.x; e < VH * SW; e += blockDim.x) {  // box: horizontal sums of V
    const int a = __float2int_rz(((float)e + 0.5f) * (1.0f / (float)SW)), c = e - a * SW;
      const int px = sx0 + c;
      float s1 = 0.0f;
      if (INT || (px - rs >= 0 && px + rs < w)) {
        const float* vr = Vs + a * VW + (px - vx0);
        if constexpr (RS > 0) {
#pragma unroll
          for (int d = -RS; d <= RS; ++d) s1 += vr[d];
        } else {
          for (int d = -rs; d <= rs; ++d) s1 += vr[d];
        }
      } else {
        for (int d = -rs; d <= rs; ++d) s1 += Vs[a * VW + min(max(px + d, 0), w - 1) - vx0];
      }
      Ts[a * SW + c] = s1;
    }
  __syncthreads();
  const float inv_box = 1.0f / (float)((2 * rs + 1) * (2 * rs + 1));
  float lo = 3.0e38f, hi = 0.0f;
  for (int e = threadIdx.x; e < SH * SW; e += blockDim.x) {  // box: vertical sums -> S
   const int a = __float2int_rz(((float)e + 0.5f) * (1.0f / (float)SW)), c = e - a * SW;
    const int py = sy0 + a;
    float s1 = 0.0f;
    if (INT || (py - rs >= 0 && py + rs < h)) {
      const float* tr = Ts + (py - vy0) * SW + c;
      if constexpr (RS > 0) {
#pragma unroll
        for (int d = -RS; d <= RS; ++d) s1 += tr[d * SW];
      } else {
        for (int d = -rs; d <= rs; ++d) s1 += tr[d * SW];
      }
    } else {
      for (int d = -rs; d <= rs; ++d) s1 += Ts[(min(max(py + d, 0), h - 1) - vy0) * SW + c];
    }
    const float sv = s1 * inv_box;
    S_out[(size_t)n * plane + (size_t)py * w + sx0 + c] = sv;
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

template <int RV, int RS>
__global__ void __launch_bounds__(256) lapvar_smooth_kernel(const float* __restrict__ rgb, int h, int w,
                                                            int rv_rt, int rs_rt, float* __restrict__ S_out,
                                                            int* __restrict__ minmax) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smraw[];
  const int rv = RV > 0 ? RV : rv_rt, rs = RS > 0 ? RS : rs_rt, R = rv + rs + 1;
  const int sy0 = blockIdx.y * kUT, sx0 = blockIdx.x * kUT;
  const bool interior = sy0 - R >= 0 && sx0 - R >= 0 && sy0 + kUT + R <= h && sx0 + kUT + R <= w;
  if (interior) lapvar_body<RV, RS, true>(rgb, h, w, rv_rt, rs_rt, S_out, minmax, smraw);
  else lapvar_body<RV, RS, false>(rgb, h, w, rv_rt, rs_rt, S_out, minmax, smraw);
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
  // flat (blurry) regions put most pixels of a frame in a few bins: warp-aggregated increments
  // (one shared atomic per distinct bin of the warp) instead of up to 32-way same-address ones
  const int lane = threadIdx.x & 31;
  for (int p0 = blockIdx.x * blockDim.x; p0 < plane; p0 += gridDim.x * blockDim.x) {
    const int p = p0 + threadIdx.x;
    const bool in = p < plane;
    float v = 0.0f;
    if (in) {
      v = range > 0.0f ? 1.0f - (u[p] - lo) / range : 1.0f;  // normalise + invert
      u[p] = v;
    }
    const int bin = in ? u_bin(v) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    if (in && lane == __ffs(peers) - 1) atomicAdd(&sh[bin], __popc(peers));
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
  __shared__ int sk[256];
  sk[k] = k;
  __syncthreads();
  // tree argmax; a candidate with the larger score wins, on ties the smaller split index
  for (int off = 128; off > 0; off >>= 1) {
    if (k < off) {
      const int a = sk[k], b = sk[k + off];
      const bool b_better = sq[b] > sq[a] || (sq[b] == sq[a] && sr[b] * sd[a] > sr[a] * sd[b]) ||
                            (sq[b] == sq[a] && sr[b] * sd[a] == sr[a] * sd[b] && b < a);
      if (b_better) sk[k] = b;
    }
    __syncthreads();
  }
  if (k == 0) tau[n] = nonempty <= 1 ? 1.0f : (float)(sk[0] + 1) / 256.0f;
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
  const size_t smem = (size_t)NL * NV * 2 * sizeof(float) +
                      (size_t)(NY * NY + NL * NL + NV * NV + NV * kUT) * sizeof(float);
  static bool attr_set = false;
  if (!attr_set) {
    e = cudaFuncSetAttribute(lapvar_smooth_kernel<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(lapvar_smooth_kernel<3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e != cudaSuccess) return cuda_fail(e);
    attr_set = true;
  }
  e = launch_k((rv == 3 && rs == 2) ? lapvar_smooth_kernel<3, 2> : lapvar_smooth_kernel<0, 0>,
               dim3(cdiv(w, kUT), cdiv(h, kUT), n), dim3(256), smem, s, rgb, (int)h, (int)w, rv, rs,
               uncertainty, minmax);
  if (e != cudaSuccess) return cuda_fail(e);
  const int plane = h * w;
  e = launch_k(normalize_hist_kernel, dim3(cdiv(plane, 256 * 8), n), dim3(256), 0, s, uncertainty, plane,
               static_cast<const int*>(minmax), hist);
  if (e != cudaSuccess) return cuda_fail(e);
  e = launch_k(otsu_kernel, dim3(n), dim3(256), 0, s, static_cast<const int*>(hist), tau_u);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}
