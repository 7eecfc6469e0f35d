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
// Kernels: (1) fused stencil, one column-sweep CTA per 116-column x 64-row strip: Y, L, the
// window sums of L and L^2 -> V, the box sums -> S, each stage one row behind the previous (see
// below); S written to the output buffer and per-frame min/max folded with integer atomics
// (S >= 0, so float bits order as ints); (2) normalise + invert in place and a per-CTA shared
// histogram (run-length + warp-aggregated increments) folded into the per-frame histogram (integer
// atomics: deterministic); (3) one CTA per frame: scans of the histogram and the exact Otsu argmax.
#include "common.cuh"

namespace sphinx {

// ---------------------------------------------------------------- (1) fused stencil
// Column sweep: a CTA of kSW threads owns a strip of kSW image columns (thread i = column
// x0 - R + i, R = rv + rs + 1 halo columns each side, kSW - 2R output columns) and walks its
// kSH output rows (+ R halo rows above and below) top to bottom; per row, four stages behind one
// another, each one row behind the stage it reads:
//   Y (row yY)         luminance of the row (shared ring of 4 rows)
//   L (row yY - 1)     3x3 Laplacian from the Y ring (shared row, double-buffered)
//   H, V (rows yL, yL - rv)  horizontal window sums of L and L^2 (thread-private ring of 16 rows
//                      in shared memory), then the vertical window sums -> V (shared row)
//   T, S (rows yV, yV - rs)  horizontal box sums of V (thread-private ring), vertical -> S
// Every stage's input is edge-replicated: reads use image-clamped rows and columns (a stage's
// rows outside the image are never produced; the clamped row always is, and is still in its
// ring).  Three barriers per row; the window sums are plain sums in a fixed order.
constexpr int kSW = 128;   // threads = strip columns
#ifndef SPHINX_UNC_KSH
#define SPHINX_UNC_KSH 32
#endif
constexpr int kSH = SPHINX_UNC_KSH;  // output rows per CTA
constexpr int kRing = 16;  // thread-private row rings (radius <= 7)

template <bool RINGS>  // shared row rings only for runtime radii (compile-time radii: registers)
struct SweepSmem {
  static constexpr int kR = RINGS ? kRing : 1;
  float Ys[4][kSW];
  float Ls[2][kSW];
  float Vs[2][kSW];
  float H1[kR][kSW], H2[kR][kSW], Ts[kR][kSW];
};

template <int RV, int RS, bool INT>
__device__ __forceinline__ void lapvar_sweep_body(const float* __restrict__ rgb, int h, int w, int rv_rt,
                                                  int rs_rt, float* __restrict__ S_out,
                                                  int* __restrict__ minmax, SweepSmem<RV == 0>& sm) {
  auto& Ys = sm.Ys;
  auto& Ls = sm.Ls;
  auto& Vs = sm.Vs;
  auto& H1 = sm.H1;
  auto& H2 = sm.H2;
  auto& Ts = sm.Ts;
  const int rv = RV > 0 ? RV : rv_rt, rs = RS > 0 ? RS : rs_rt, R = rv + rs + 1;
  const int TW = kSW - 2 * R;
  const int n = blockIdx.z, i = threadIdx.x;
  const int x0 = blockIdx.x * TW, x1 = min(w, x0 + TW);
  const int y0 = blockIdx.y * kSH, y1 = min(h, y0 + kSH);
  const int xb = x0 - R;  // image column of smem column 0
  const int g = xb + i;   // this thread's column
  // image-clamped column -> smem column (interior strips: no clamp)
  auto cix = [&](int x) { return (INT ? x : min(max(x, 0), w - 1)) - xb; };
  auto crow = [&](int y) { return INT ? y : min(max(y, 0), h - 1); };
  const bool in_img = g >= 0 && g < w;
  const bool l_ok = in_img && g >= x0 - rs - rv && g < x1 + rs + rv;
  const bool h_ok = in_img && g >= x0 - rs && g < x1 + rs;
  const bool t_ok = g >= x0 && g < x1;
  const int yY_lo = max(0, y0 - R), yY_hi = min(h, y1 + R);
  const int yL_lo = max(0, y0 - rs - rv), yL_hi = min(h, y1 + rs + rv);
  const int yV_lo = max(0, y0 - rs), yV_hi = min(h, y1 + rs);
  const size_t plane = (size_t)h * w;
  const float* img = rgb + (size_t)n * plane * 3;
  const float inv_cnt = 1.0f / (float)((2 * rv + 1) * (2 * rv + 1));
  const float inv_box = 1.0f / (float)((2 * rs + 1) * (2 * rs + 1));
  float lo = 3.0e38f, hi = 0.0f;
  // compile-time radii: the vertical windows live in registers (virtual rows, oldest first)
  float rh1[2 * (RV > 0 ? RV : 0) + 1], rh2[2 * (RV > 0 ? RV : 0) + 1], rt[2 * (RS > 0 ? RS : 0) + 1];
  // the next Y row's pixel, loaded one iteration ahead
  float pr = 0.f, pg = 0.f, pb = 0.f;
  auto load_px = [&](int y) {
    if (in_img && y >= yY_lo && y < yY_hi) {
      const float* px = img + ((size_t)y * w + g) * 3;
      pr = __ldg(px);
      pg = __ldg(px + 1);
      pb = __ldg(px + 2);
    }
  };
  load_px(y0 - R);
  const int T = (y1 - y0) + 2 * R;
  for (int t = 0; t < T; ++t) {
    const int yY = y0 - R + t, yL = yY - 1, yV = yL - rv, yS = yV - rs;
    // ---- Y
    if (in_img && yY >= yY_lo && yY < yY_hi) Ys[yY & 3][i] = 0.299f * pr + 0.587f * pg + 0.114f * pb;
    load_px(yY + 1);
    __syncthreads();
    // ---- L (same operation order as the oracle: up + down + left + right - 4 centre)
    if (l_ok && yL >= yL_lo && yL < yL_hi) {
      const float* yc = Ys[yL & 3];
      const float up = Ys[crow(yL - 1) & 3][i], dn = Ys[crow(yL + 1) & 3][i];
      Ls[yL & 1][i] = up + dn + yc[cix(g - 1)] + yc[cix(g + 1)] - 4.0f * yc[i];
    }
    __syncthreads();
    // ---- H (row yL) and V (row yV)
    if (h_ok) {
      if (yL >= yL_lo && yL < yL_hi) {
        const float* lr = Ls[yL & 1];
        float s1 = 0.0f, s2 = 0.0f;
        if constexpr (RV > 0) {
#pragma unroll
          for (int d = -RV; d <= RV; ++d) {
            const float l = lr[cix(g + d)];
            s1 += l;
            s2 = fmaf(l, l, s2);
          }
          // register ring of the last 2RV+1 virtual rows; the image's first row also stands for
          // the rows above it (edge replication)
          const bool fill = yL == 0 && y0 - rs - rv < 0;
#pragma unroll
          for (int k = 0; k < 2 * RV; ++k) {
            rh1[k] = fill ? s1 : rh1[k + 1];
            rh2[k] = fill ? s2 : rh2[k + 1];
          }
          rh1[2 * RV] = s1;
          rh2[2 * RV] = s2;
        } else {
          for (int d = -rv; d <= rv; ++d) {
            const float l = lr[cix(g + d)];
            s1 += l;
            s2 = fmaf(l, l, s2);
          }
          H1[yL & (kRing - 1)][i] = s1;
          H2[yL & (kRing - 1)][i] = s2;
        }
      } else if constexpr (RV > 0) {
        if (yL >= h) {  // below the image: the last row stands for the rows below it
#pragma unroll
          for (int k = 0; k < 2 * RV; ++k) {
            rh1[k] = rh1[k + 1];
            rh2[k] = rh2[k + 1];
          }
        }
      }
      if (yV >= yV_lo && yV < yV_hi) {
        float a = 0.0f, b = 0.0f;
        if constexpr (RV > 0) {
#pragma unroll
          for (int k = 0; k <= 2 * RV; ++k) {
            a += rh1[k];
            b += rh2[k];
          }
        } else {
          for (int d = -rv; d <= rv; ++d) {
            const int r = crow(yV + d) & (kRing - 1);
            a += H1[r][i];
            b += H2[r][i];
          }
        }
        const float m = a * inv_cnt;
        Vs[yV & 1][i] = fmaxf(fmaf(-m, m, b * inv_cnt), 0.0f);
      }
    }
    __syncthreads();
    // ---- T (row yV) and S (row yS)
    if (t_ok) {
      if (yV >= yV_lo && yV < yV_hi) {
        const float* vr = Vs[yV & 1];
        float s1 = 0.0f;
        if constexpr (RS > 0) {
#pragma unroll
          for (int d = -RS; d <= RS; ++d) s1 += vr[cix(g + d)];
          const bool fill = yV == 0 && y0 - rs < 0;
#pragma unroll
          for (int k = 0; k < 2 * RS; ++k) rt[k] = fill ? s1 : rt[k + 1];
          rt[2 * RS] = s1;
        } else {
          for (int d = -rs; d <= rs; ++d) s1 += vr[cix(g + d)];
          Ts[yV & (kRing - 1)][i] = s1;
        }
      } else if constexpr (RS > 0) {
        if (yV >= h) {
#pragma unroll
          for (int k = 0; k < 2 * RS; ++k) rt[k] = rt[k + 1];
        }
      }
      if (yS >= y0 && yS < y1) {
        float s1 = 0.0f;
        if constexpr (RS > 0) {
#pragma unroll
          for (int k = 0; k <= 2 * RS; ++k) s1 += rt[k];
        } else {
          for (int d = -rs; d <= rs; ++d) s1 += Ts[crow(yS + d) & (kRing - 1)][i];
        }
        const float sv = s1 * inv_box;
        S_out[(size_t)n * plane + (size_t)yS * w + g] = sv;
        lo = fminf(lo, sv);
        hi = fmaxf(hi, sv);
      }
    }
  }
  for (int d = 16; d > 0; d >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, d));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, d));
  }
  if ((threadIdx.x & 31) == 0 && hi >= lo) {
    atomicMin(minmax + 2 * n, __float_as_int(lo));  // S >= +0: float order == int order
    atomicMax(minmax + 2 * n + 1, __float_as_int(hi));
  }
}

template <int RV, int RS>
__global__ void __launch_bounds__(kSW) lapvar_sweep_kernel(const float* __restrict__ rgb, int h, int w,
                                                           int rv_rt, int rs_rt, float* __restrict__ S_out,
                                                           int* __restrict__ minmax) {
  pdl_wait();
  pdl_trigger();
  const int rv = RV > 0 ? RV : rv_rt, rs = RS > 0 ? RS : rs_rt, R = rv + rs + 1;
  const int x0 = blockIdx.x * (kSW - 2 * R), y0 = blockIdx.y * kSH;
  // every column and row the strip touches (with its halo) lies inside the image: no clamps
  const bool interior = x0 - R >= 0 && x0 - R + kSW <= w && y0 - R >= 0 && y0 + kSH + R <= h;
  __shared__ SweepSmem<RV == 0> sm;
  if (interior) lapvar_sweep_body<RV, RS, true>(rgb, h, w, rv_rt, rs_rt, S_out, minmax, sm);
  else lapvar_sweep_body<RV, RS, false>(rgb, h, w, rv_rt, rs_rt, S_out, minmax, sm);
}

__device__ __forceinline__ int u_bin(float v) {
  // bin i = (i/256, (i+1)/256]; v * 256 is exact
  int t = (int)ceilf(v * 256.0f) - 1;
  return t < 0 ? 0 : (t > 255 ? 255 : t);
}

// ---------------------------------------------------------------- (2) normalise + histogram
// Each thread normalises 8 consecutive pixels (two 16-byte loads and stores when the frame is
// 16-byte aligned) and counts runs of equal bins in a register: flat, blurry regions put long runs
// in one bin, so a shared increment is issued only when the bin changes (and once at the end).
// The CTA histogram is folded into the frame's with integer atomics (deterministic).
constexpr int kNormPx = 8;

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
  // 16-byte vectors when every frame starts 16-byte aligned
  const bool vec = (plane & 3) == 0 && (reinterpret_cast<uintptr_t>(U) & 15) == 0;
  const int step = gridDim.x * blockDim.x * kNormPx;
  for (int pb = (blockIdx.x * blockDim.x + threadIdx.x) * kNormPx; pb < plane; pb += step) {
    float v[kNormPx];
    const int np = min(kNormPx, plane - pb);
    if (vec && np == kNormPx) {
      const float4 a = *reinterpret_cast<const float4*>(u + pb), b = *reinterpret_cast<const float4*>(u + pb + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < kNormPx; ++k) v[k] = k < np ? u[pb + k] : 0.0f;
    }
#pragma unroll
    for (int k = 0; k < kNormPx; ++k) v[k] = range > 0.0f ? 1.0f - (v[k] - lo) / range : 1.0f;  // normalise + invert
    if (vec && np == kNormPx) {
      *reinterpret_cast<float4*>(u + pb) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(u + pb + 4) = make_float4(v[4], v[5], v[6], v[7]);
    } else {
      for (int k = 0; k < np; ++k) u[pb + k] = v[k];
    }
    int run_bin = u_bin(v[0]), run = 1;
#pragma unroll
    for (int k = 1; k < kNormPx; ++k) {
      if (k >= np) break;
      const int bin = u_bin(v[k]);
      if (bin == run_bin) {
        ++run;
      } else {
        atomicAdd(&sh[run_bin], run);
        run_bin = bin;
        run = 1;
      }
    }
    atomicAdd(&sh[run_bin], run);
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
  __shared__ long long h[256], hs[256];
  __shared__ u128 sq[256], sr[256], sd[256];
  const int n = blockIdx.x, k = threadIdx.x;
  const long long hk = hist[256 * n + k];
  h[k] = hk;
  hs[k] = (long long)k * hk;
  const int nonempty = __syncthreads_count(hk > 0);
  // inclusive scans of the counts and of the bin-index sums (Hillis-Steele, 8 steps)
  for (int off = 1; off < 256; off <<= 1) {
    const long long a = k >= off ? h[k - off] : 0, b = k >= off ? hs[k - off] : 0;
    __syncthreads();
    h[k] += a;
    hs[k] += b;
    __syncthreads();
  }
  const long long n0 = h[k], s0 = hs[k], N = h[255], S = hs[255];
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
  const int TW = kSW - 2 * R;  // output columns per strip
  e = launch_k((rv == 3 && rs == 2) ? lapvar_sweep_kernel<3, 2> : lapvar_sweep_kernel<0, 0>,
               dim3(cdiv(w, TW), cdiv(h, kSH), n), dim3(kSW), 0, s, rgb, (int)h, (int)w, rv, rs,
               uncertainty, minmax);
  if (e != cudaSuccess) return cuda_fail(e);
  const int plane = h * w;
  e = launch_k(normalize_hist_kernel, dim3(cdiv(plane, 256 * kNormPx), n), dim3(256), 0, s, uncertainty, plane,
               static_cast<const int*>(minmax), hist);
  if (e != cudaSuccess) return cuda_fail(e);
  e = launch_k(otsu_kernel, dim3(n), dim3(256), 0, s, static_cast<const int*>(hist), tau_u);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}
