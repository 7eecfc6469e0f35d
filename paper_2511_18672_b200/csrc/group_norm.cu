// group_norm.cu — NEXT-3: GroupNorm statistics and GroupNorm+SiLU for the block-sparse
// UNet ResNet block ("ResNet layers ... can be safely applied only to frames selected
// for refinement"; P:352 latent reuse for unrefined regions; readings R-26, R-27).
//
// GroupNorm needs per-(frame, group) statistics of the FULL current map, but on a partial
// step only the listed blocks change (inactive blocks hold cached values).  So the
// statistics are kept per BLOCK in a persistent buffer: stats[(id * G + g)] = (mean, M2) of
// the block's real pixels x the group's C/G channels.  A partial step rewrites the entries of
// listed blocks only (they read active bytes only), and the frame statistics are combined
// from all Hb*Wb entries of the frame (Chan's pairwise update, a few KB from L2).  Equal to the
// full-map definition up to rounding.
//
//  gn_block_stats_kernel  one CTA per listed block: 16-byte loads (8 channels) per thread,
//                         per-channel shifted sums (shift = the block's first pixel, so no
//                         cancellation for |mean| >> std), per-channel (mean, M2), then
//                         per-group Chan combination.  HBM-bound on the active bytes.
//  gn_silu_kernel         contiguous chunk of the list per CTA (frames change rarely along the
//                         ascending list): frame statistics -> per-channel (mean, gamma*rstd,
//                         beta) in shared memory, then a = bf16(SiLU(gamma (x-mean) rstd +
//                         beta)) for every pixel of the block AND its 1-pixel ring clipped to
//                         the image: exactly the pixels a 3x3 conv over the listed blocks reads
//                         (ring pixels of unlisted neighbours = normalised cached values with the
//                         current statistics).  Two CTAs may write the same ring pixel: both
//                         write identical bits (same inputs, same instruction sequence).
#include <cuda_bf16.h>

#include "common.cuh"

namespace sphinx {

constexpr int kGnThreads = 256;

__device__ __forceinline__ void unpack8(const uint4 r, float (&f)[8]) {
  const uint32_t w4[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    f[2 * k] = __uint_as_float(w4[k] << 16);
    f[2 * k + 1] = __uint_as_float(w4[k] & 0xffff0000u);
  }
}

__global__ void __launch_bounds__(kGnThreads) gn_block_stats_kernel(
    const __nv_bfloat16* __restrict__ x, int h, int w, int c, int G, int b, int hb, int wb,
    const int32_t* __restrict__ ids, const int32_t* __restrict__ count, float2* stats) {
  extern __shared__ float sm[];
  const int V = c >> 3;               // 16-byte vectors per pixel
  const int R = kGnThreads / V;       // pixel lanes
  float* s1 = sm;                     // [R][c]
  float* s2 = sm + R * c;             // [R][c]
  float* cmean = sm + 2 * R * c;      // [c]
  float* cm2 = cmean + c;             // [c]
  pdl_wait();
  pdl_trigger();
  const int cnt = *count;
  const int t = threadIdx.x, v = t % V, r0 = t / V;
  const int cg = c / G;
  for (int j = blockIdx.x; j < cnt; j += gridDim.x) {
    const int id = __ldg(ids + j);
    const int n = id / (hb * wb), rem = id - n * hb * wb;
    const int by = rem / wb, bx = rem - by * wb;
    const int rows = min(b, h - by * b), cols = min(b, w - bx * b), np = rows * cols;
    const __nv_bfloat16* base = x + (((size_t)n * h + by * b) * w + bx * b) * c;
    if (r0 < R) {
      float K[8], a1[8], a2[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(base) + v), K);
#pragma unroll
      for (int i = 0; i < 8; ++i) a1[i] = a2[i] = 0.f;
#pragma unroll 4
      for (int p = r0; p < np; p += R) {
        const int py = p / cols, px = p - py * cols;
        float f[8];
        unpack8(__ldg(reinterpret_cast<const uint4*>(base + ((size_t)py * w + px) * c) + v), f);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float d = f[i] - K[i];
          a1[i] += d;
          a2[i] = fmaf(d, d, a2[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        s1[r0 * c + v * 8 + i] = a1[i];
        s2[r0 * c + v * 8 + i] = a2[i];
      }
    }
    __syncthreads();
    const float inv_np = 1.f / (float)np;
    for (int ch = t; ch < c; ch += kGnThreads) {
      float S1 = 0.f, S2 = 0.f;
      for (int r = 0; r < R; ++r) {
        S1 += s1[r * c + ch];
        S2 += s2[r * c + ch];
      }
      const float K = __bfloat162float(base[ch]);
      cmean[ch] = K + S1 * inv_np;
      cm2[ch] = fmaxf(S2 - S1 * S1 * inv_np, 0.f);
    }
    __syncthreads();
    for (int g = t; g < G; g += kGnThreads) {
      float m = 0.f;
      for (int k = 0; k < cg; ++k) m += cmean[g * cg + k];
      m /= (float)cg;
      float M2 = 0.f, dev = 0.f;
      for (int k = 0; k < cg; ++k) {
        const float d = cmean[g * cg + k] - m;
        M2 += cm2[g * cg + k];
        dev = fmaf(d, d, dev);
      }
      stats[(size_t)id * G + g] = make_float2(m, fmaf((float)np, dev, M2));
    }
    __syncthreads();
  }
}

// Chan et al. pairwise update of (count, mean, M2).
__device__ __forceinline__ void chan_merge(float& na, float& ma, float& qa, float nb, float mb, float qb) {
  const float n = na + nb;
  if (nb == 0.f) return;
  const float d = mb - ma, f = nb / n;
  ma = fmaf(d, f, ma);
  qa = qa + qb + d * d * na * f;
  na = n;
}

__global__ void __launch_bounds__(kGnThreads) gn_silu_kernel(
    const __nv_bfloat16* __restrict__ x, const float2* __restrict__ stats,
    const float* __restrict__ gamma, const float* __restrict__ beta, float eps, int h, int w,
    int c, int G, int b, int hb, int wb, const int32_t* __restrict__ ids,
    const int32_t* __restrict__ count, __nv_bfloat16* a) {
  extern __shared__ float sm[];
  float* s_mean = sm;          // [c] group mean per channel
  float* s_scale = sm + c;     // [c] gamma * rstd
  float* s_beta = sm + 2 * c;  // [c]
  float* g_mean = sm + 3 * c;  // [G]
  float* g_rstd = g_mean + G;  // [G]
  pdl_wait();
  pdl_trigger();
  const int cnt = *count;
  const int j0 = (int)((long long)blockIdx.x * cnt / gridDim.x);
  const int j1 = (int)((long long)(blockIdx.x + 1) * cnt / gridDim.x);
  const int t = threadIdx.x, V = c >> 3, cg = c / G;
  // threads per group for the frame reduction: a power of two <= 32 dividing the warp
  int tpg = 32;
  while (tpg > 1 && tpg * G > kGnThreads) tpg >>= 1;
  const int nblk = hb * wb;
  const int rb = h - (hb - 1) * b, cb = w - (wb - 1) * b;  // rows / cols of edge blocks
  int cur = -1;
  for (int j = j0; j < j1; ++j) {
    const int id = __ldg(ids + j);
    const int n = id / nblk, rem = id - n * nblk;
    const int by = rem / wb, bx = rem - by * wb;
    if (n != cur) {
      __syncthreads();  // previous frame's tables no longer read
      for (int g0 = 0; g0 < G; g0 += kGnThreads / tpg) {
        const int g = g0 + t / tpg, sub = t % tpg;
        float na = 0.f, ma = 0.f, qa = 0.f;
        if (g < G) {
          for (int i = sub; i < nblk; i += tpg) {
            const int iy = i / wb, ix = i - iy * wb;
            const float npx = (float)((iy == hb - 1 ? rb : b) * (ix == wb - 1 ? cb : b) * cg);
            const float2 st = __ldg(stats + ((size_t)n * nblk + i) * G + g);
            chan_merge(na, ma, qa, npx, st.x, st.y);
          }
        }
        // butterfly over the tpg lanes of the group (fixed order: deterministic)
        for (int o = 1; o < tpg; o <<= 1) {
          const float nb2 = __shfl_xor_sync(0xffffffffu, na, o);
          const float mb2 = __shfl_xor_sync(0xffffffffu, ma, o);
          const float qb2 = __shfl_xor_sync(0xffffffffu, qa, o);
          // merge in a lane-independent order so both partners hold identical bits
          if ((t & o) == 0) {
            chan_merge(na, ma, qa, nb2, mb2, qb2);
          } else {
            float nn = nb2, mm = mb2, qq = qb2;
            chan_merge(nn, mm, qq, na, ma, qa);
            na = nn; ma = mm; qa = qq;
          }
        }
        if (g < G && sub == 0) {
          g_mean[g] = ma;
          g_rstd[g] = 1.f / sqrtf(qa / na + eps);
        }
      }
      __syncthreads();
      for (int ch = t; ch < c; ch += kGnThreads) {
        const int g = ch / cg;
        s_mean[ch] = g_mean[g];
        s_scale[ch] = __ldg(gamma + ch) * g_rstd[g];
        s_beta[ch] = __ldg(beta + ch);
      }
      __syncthreads();
      cur = n;
    }
    const int y0 = max(by * b - 1, 0), y1 = min(by * b + b + 1, h);
    const int x0 = max(bx * b - 1, 0), x1 = min(bx * b + b + 1, w);
    const int rw = x1 - x0, total = (y1 - y0) * rw * V;
    for (int e = t; e < total; e += kGnThreads) {
      const int p = e / V, vv = e - p * V;
      const int yy = y0 + p / rw, xx = x0 + p % rw;
      const size_t off = (((size_t)n * h + yy) * w + xx) * c + vv * 8;
      float f[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(x + off)), f);
      uint32_t o4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float r2[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int ch = vv * 8 + 2 * k + q;
          const float tt = fmaf(f[2 * k + q] - s_mean[ch], s_scale[ch], s_beta[ch]);
          r2[q] = tt / (1.f + expf(-tt));
        }
        const __nv_bfloat162 pk = __floats2bfloat162_rn(r2[0], r2[1]);
        o4[k] = *reinterpret_cast<const uint32_t*>(&pk);
      }
      *reinterpret_cast<uint4*>(a + off) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
    }
  }
}

static int gn_grid(int capacity, int sms) {
  const int cap = sms * 8;
  return capacity < cap ? (capacity > 0 ? capacity : 1) : cap;
}

}  // namespace sphinx

using namespace sphinx;

static sphinx_status gn_check(const void* x, int32_t n, int32_t h, int32_t w, int32_t c,
                              int32_t groups, int32_t block, const int32_t* ids, const int32_t* count,
                              int32_t capacity) {
  if (!x || !ids || !count) return SPHINX_ERR_INVALID_ARGUMENT;
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || block <= 0 || groups <= 0 || capacity < 0)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (c % groups) return SPHINX_ERR_INVALID_ARGUMENT;
  if ((int64_t)capacity > (int64_t)n * cdiv(h, block) * cdiv(w, block)) return SPHINX_ERR_INVALID_ARGUMENT;
  if (c % 8 || c > 8 * kGnThreads || groups > kGnThreads || block > 64) return SPHINX_ERR_UNSUPPORTED;
  if (!aligned16(x)) return SPHINX_ERR_UNSUPPORTED;
  return SPHINX_OK;
}

extern "C" size_t sphinx_gn_stats_size(int32_t n, int32_t h, int32_t w, int32_t groups,
                                       int32_t block) {
  if (n <= 0 || h <= 0 || w <= 0 || groups <= 0 || block <= 0) return 0;
  return (size_t)n * cdiv(h, block) * cdiv(w, block) * groups * sizeof(float2);
}

extern "C" sphinx_status sphinx_gn_block_stats(const void* x, int32_t n, int32_t h, int32_t w,
                                               int32_t c, int32_t groups, int32_t block,
                                               const int32_t* block_ids, const int32_t* count,
                                               int32_t capacity, float* stats,
                                               sphinx_stream_t stream) {
  sphinx_status st = gn_check(x, n, h, w, c, groups, block, block_ids, count, capacity);
  if (st != SPHINX_OK) return st;
  if (!stats || (reinterpret_cast<uintptr_t>(stats) & 7u)) return SPHINX_ERR_INVALID_ARGUMENT;
  int sms = 0;
  if ((st = check_device(&sms)) != SPHINX_OK) return st;
  if (capacity == 0) return SPHINX_OK;
  const int V = c / 8, R = kGnThreads / V;
  const size_t smem = (size_t)(2 * R * c + 2 * c) * sizeof(float);
  cudaError_t e = launch_k(gn_block_stats_kernel, dim3(gn_grid(capacity, sms)), dim3(kGnThreads), smem,
                           reinterpret_cast<cudaStream_t>(stream),
                           static_cast<const __nv_bfloat16*>(x), (int)h, (int)w, (int)c, (int)groups,
                           (int)block, cdiv(h, block), cdiv(w, block), block_ids, count,
                           reinterpret_cast<float2*>(stats));
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

extern "C" sphinx_status sphinx_gn_silu(const void* x, const float* stats, const float* gamma,
                                        const float* beta, float eps, int32_t n, int32_t h,
                                        int32_t w, int32_t c, int32_t groups, int32_t block,
                                        const int32_t* block_ids, const int32_t* count,
                                        int32_t capacity, void* a, sphinx_stream_t stream) {
  sphinx_status st = gn_check(x, n, h, w, c, groups, block, block_ids, count, capacity);
  if (st != SPHINX_OK) return st;
  if (!stats || !gamma || !beta || !a || a == x || !(eps >= 0.f)) return SPHINX_ERR_INVALID_ARGUMENT;
  if (!aligned16(a)) return SPHINX_ERR_UNSUPPORTED;
  int sms = 0;
  if ((st = check_device(&sms)) != SPHINX_OK) return st;
  if (capacity == 0) return SPHINX_OK;
  const size_t smem = (size_t)(3 * c + 2 * groups) * sizeof(float);
  cudaError_t e = launch_k(gn_silu_kernel, dim3(gn_grid(capacity, sms)), dim3(kGnThreads), smem,
                           reinterpret_cast<cudaStream_t>(stream),
                           static_cast<const __nv_bfloat16*>(x), reinterpret_cast<const float2*>(stats),
                           gamma, beta, eps, (int)h, (int)w, (int)c, (int)groups, (int)block,
                           cdiv(h, block), cdiv(w, block), block_ids, count,
                           static_cast<__nv_bfloat16*>(a));
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

extern "C" sphinx_status sphinx_sparse_resblock(
    const void* x, const void* w1, const float* b1, const void* w2, const float* b2,
    const float* gn1_gamma, const float* gn1_beta, const float* gn2_gamma, const float* gn2_beta,
    int32_t groups, float eps, void* h_buf, float* x_stats, float* h_stats, void* y,
    sphinx_dtype y_dtype, void* a_scratch, int32_t n, int32_t h, int32_t w, int32_t c,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity,
    void* workspace, size_t workspace_bytes, sphinx_stream_t stream) {
  if (!h_buf || !y || !a_scratch || !x_stats || !h_stats) return SPHINX_ERR_INVALID_ARGUMENT;
  if (h_buf == x || y == x || y == h_buf || a_scratch == x || a_scratch == h_buf || a_scratch == y ||
      x_stats == h_stats)
    return SPHINX_ERR_INVALID_ARGUMENT;
  sphinx_status st;
  // (1) statistics of x on the listed blocks; (2) a = SiLU(GN1(x)) on listed blocks + ring
  if ((st = sphinx_gn_block_stats(x, n, h, w, c, groups, block, block_ids, count, capacity, x_stats,
                                  stream)) != SPHINX_OK)
    return st;
  if ((st = sphinx_gn_silu(x, x_stats, gn1_gamma, gn1_beta, eps, n, h, w, c, groups, block, block_ids,
                           count, capacity, a_scratch, stream)) != SPHINX_OK)
    return st;
  // (3) h = conv1(a) + b1 on listed pixels (bf16, persistent: cached elsewhere)
  if ((st = sphinx_sparse_conv3x3(a_scratch, w1, b1, h_buf, SPHINX_BF16, n, h, w, c, c, block,
                                  block_ids, count, capacity, workspace, workspace_bytes, stream)) !=
      SPHINX_OK)
    return st;
  // (4) statistics of h on the listed blocks; (5) a = SiLU(GN2(h))
  if ((st = sphinx_gn_block_stats(h_buf, n, h, w, c, groups, block, block_ids, count, capacity,
                                  h_stats, stream)) != SPHINX_OK)
    return st;
  if ((st = sphinx_gn_silu(h_buf, h_stats, gn2_gamma, gn2_beta, eps, n, h, w, c, groups, block,
                           block_ids, count, capacity, a_scratch, stream)) != SPHINX_OK)
    return st;
  // (6) y = x + conv2(a) + b2 on listed pixels (identity skip fused in the epilogue)
  return sphinx_sparse_conv3x3_residual(a_scratch, w2, b2, x, y, y_dtype, n, h, w, c, c, block,
                                        block_ids, count, capacity, workspace, workspace_bytes,
                                        stream);
}
