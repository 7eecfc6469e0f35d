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
// Stats buffer = [N][Hb][Wb][G] float2 block entries + [N][G] float2 frame entries (mean, rstd).
// Work unit = (listed block, channel slice of whole groups); thread t owns one 16-byte vector
// (8 channels) of the slice for the whole unit and walks pixel lanes, 4 loads in flight.
//  gn_block_stats_kernel  per unit: per-channel shifted sums (shift = the block's first pixel,
//                         so no cancellation for |mean| >> std) -> per-channel (mean, M2) ->
//                         per-group Chan combination.  HBM-bound on the active bytes.
//  gn_finalize_kernel     one warp per (frame, group): the frame's Hb*Wb entries -> (mean, rstd).
//  gn_silu_kernel         per unit over the block AND its 1-pixel ring clipped to the image
//                         (exactly the pixels a 3x3 conv over the listed blocks reads; ring pixels
//                         of unlisted neighbours = normalised cached values with the current
//                         statistics): a = bf16(SiLU((x - mean) gamma rstd + beta)).  Two units
//                         may write the same ring pixel: identical bits (same inputs, same code).
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

// Work unit = (listed block, channel slice).  A slice holds S channels, S | c and S a
// multiple of lcm(c/G, 8), so it contains whole groups and whole 16-byte vectors; thread t
// owns vector v = t % (S/8) of the slice for the whole unit and walks pixel lanes t / (S/8).
struct GnGeom {
  int h, w, c, G, b, hb, wb;
  int S, V, R, nslice;  // slice channels, vectors per slice pixel, pixel lanes, slices per pixel
  int rg, nrg;          // gn_silu: ring rows per unit, units per (block, slice)
};

__global__ void __launch_bounds__(kGnThreads, 4) gn_block_stats_kernel(
    const __nv_bfloat16* __restrict__ x, const GnGeom g, const int32_t* __restrict__ ids,
    const int32_t* __restrict__ count, float2* stats) {
  __shared__ float s1[2 * kGnThreads * 8];  // [R][S] shifted sums, then [R][S] squares
  __shared__ float cmean[kGnThreads * 8], cm2[kGnThreads * 8];
  pdl_wait();
  pdl_trigger();
  const int cnt = *count;
  const int t = threadIdx.x, V = g.V, R = g.R, S = g.S;
  const int v = t % V, r0 = t / V;
  const int cg = g.c / g.G;
  float* s2 = s1 + R * S;
  const long long units = (long long)cnt * g.nslice;
  for (long long u = blockIdx.x; u < units; u += gridDim.x) {
    const int j = (int)(u / g.nslice), sl = (int)(u - (long long)j * g.nslice);
    const int id = __ldg(ids + j);
    const int n = id / (g.hb * g.wb), rem = id - n * g.hb * g.wb;
    const int by = rem / g.wb, bx = rem - by * g.wb;
    const int rows = min(g.b, g.h - by * g.b), cols = min(g.b, g.w - bx * g.b), np = rows * cols;
    const __nv_bfloat16* base = x + (((size_t)n * g.h + by * g.b) * g.w + bx * g.b) * g.c + sl * S;
    if (r0 < R) {
      float K[8], a1[8], a2[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(base) + v), K);
#pragma unroll
      for (int i = 0; i < 8; ++i) a1[i] = a2[i] = 0.f;
      const float inv_cols = 1.f / (float)cols;  // exact floor((pp + 0.5) / cols) for pp < 2^20
      const uint32_t row_stride = (uint32_t)g.w * g.c;
      // 4 independent (predicated) 16-byte loads in flight per thread
      for (int p0 = r0; p0 < np; p0 += 4 * R) {
        uint4 raw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int pp = p0 + q * R;
          const int py = __float2int_rz(((float)pp + 0.5f) * inv_cols), px = pp - py * cols;
          if (pp < np)
            raw[q] = __ldg(reinterpret_cast<const uint4*>(base + (uint32_t)py * row_stride + (uint32_t)px * g.c) + v);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (p0 + q * R < np) {
            float f[8];
            unpack8(raw[q], f);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float d = f[i] - K[i];
              a1[i] += d;
              a2[i] = fmaf(d, d, a2[i]);
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        s1[r0 * S + v * 8 + i] = a1[i];
        s2[r0 * S + v * 8 + i] = a2[i];
      }
    }
    __syncthreads();
    const float inv_np = 1.f / (float)np;
    for (int ch = t; ch < S; ch += kGnThreads) {
      float A = 0.f, B2 = 0.f;
      for (int r = 0; r < R; ++r) {
        A += s1[r * S + ch];
        B2 += s2[r * S + ch];
      }
      const float K = __bfloat162float(base[ch]);
      cmean[ch] = K + A * inv_np;
      cm2[ch] = fmaxf(B2 - A * A * inv_np, 0.f);
    }
    __syncthreads();
    for (int q = t; q < S / cg; q += kGnThreads) {
      float m = 0.f;
      for (int k = 0; k < cg; ++k) m += cmean[q * cg + k];
      m /= (float)cg;
      float M2 = 0.f, dev = 0.f;
      for (int k = 0; k < cg; ++k) {
        const float d = cmean[q * cg + k] - m;
        M2 += cm2[q * cg + k];
        dev = fmaf(d, d, dev);
      }
      stats[(size_t)id * g.G + sl * (S / cg) + q] = make_float2(m, fmaf((float)np, dev, M2));
    }
    __syncthreads();
  }
}

// Chan et al. pairwise update of (count, mean, M2).
__device__ __forceinline__ void chan_merge(float& na, float& ma, float& qa, float nb, float mb, float qb) {
  if (nb == 0.f) return;
  const float n = na + nb;
  const float d = mb - ma, f = nb / n;
  ma = fmaf(d, f, ma);
  qa = qa + qb + d * d * na * f;
  na = n;
}

// Frame statistics: one warp per (frame, group) combines the frame's Hb*Wb block entries
// (lane-strided, then a fixed butterfly: deterministic, both partners hold identical bits) into
// (mean, rstd) = (mean, 1/sqrt(M2/count + eps)) at fstats[n * G + g].
// With `tab` != NULL the warp also writes, for the group's channels, the fused-conv table
// tab[n][ch] = (gamma*rstd, beta - mean*gamma*rstd), i.e. a = SiLU(x * scale + shift).
__global__ void __launch_bounds__(kGnThreads) gn_finalize_kernel(const float2* __restrict__ stats,
                                                                  float2* fstats, const GnGeom g,
                                                                  int n_frames, float eps,
                                                                  const float* __restrict__ gamma,
                                                                  const float* __restrict__ beta,
                                                                  float2* tab) {
  pdl_wait();
  pdl_trigger();
  const int warp = (blockIdx.x * kGnThreads + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n_frames * g.G) return;
  const int n = warp / g.G, gi = warp - n * g.G;
  const int nblk = g.hb * g.wb, cg = g.c / g.G;
  const int rb = g.h - (g.hb - 1) * g.b, cb = g.w - (g.wb - 1) * g.b;
  float na = 0.f, ma = 0.f, qa = 0.f;
  for (int i = lane; i < nblk; i += 32) {
    const int iy = i / g.wb, ix = i - iy * g.wb;
    const float npx = (float)((iy == g.hb - 1 ? rb : g.b) * (ix == g.wb - 1 ? cb : g.b) * cg);
    const float2 st = __ldg(stats + ((size_t)n * nblk + i) * g.G + gi);
    chan_merge(na, ma, qa, npx, st.x, st.y);
  }
  for (int o = 1; o < 32; o <<= 1) {
    const float nb2 = __shfl_xor_sync(0xffffffffu, na, o);
    const float mb2 = __shfl_xor_sync(0xffffffffu, ma, o);
    const float qb2 = __shfl_xor_sync(0xffffffffu, qa, o);
    if ((lane & o) == 0) {
      chan_merge(na, ma, qa, nb2, mb2, qb2);
    } else {
      float nn = nb2, mm = mb2, qq = qb2;
      chan_merge(nn, mm, qq, na, ma, qa);
      na = nn; ma = mm; qa = qq;
    }
  }
  const float rstd = 1.f / sqrtf(qa / na + eps);
  if (lane == 0) fstats[warp] = make_float2(ma, rstd);
  if (tab != nullptr) {
    for (int k = lane; k < cg; k += 32) {
      const int ch = gi * cg + k;
      const float sc = __ldg(gamma + ch) * rstd;
      tab[(size_t)n * g.c + ch] = make_float2(sc, fmaf(-ma, sc, __ldg(beta + ch)));
    }
  }
}

// a = bf16(SiLU((x - mean_g) * gamma_c * rstd_g + beta_c)) over (listed block + 1-px ring,
// channel slice, group of ring rows) units: each thread's 8 channels' parameters are loaded
// once per unit into registers, then up to 8 predicated 16-byte loads are in flight.
// (Measured: a flat one-vector-per-thread variant is 1.4-2x slower here: per-element
// parameter loads and empty CTAs past the device count.)
__global__ void __launch_bounds__(kGnThreads, 4) gn_silu_kernel(
    const __nv_bfloat16* __restrict__ x, const float2* __restrict__ fstats,
    const float* __restrict__ gamma, const float* __restrict__ beta, const GnGeom g,
    const int32_t* __restrict__ ids, const int32_t* __restrict__ count, __nv_bfloat16* a) {
  pdl_wait();
  pdl_trigger();
  const int cnt = *count;
  const int t = threadIdx.x, V = g.V, R = g.R, S = g.S;
  const int v = t % V, r0 = t / V;
  if (r0 >= R) return;
  const int cg = g.c / g.G;
  const int per_blk = g.nslice * g.nrg;
  const long long units = (long long)cnt * per_blk;
  for (long long u = blockIdx.x; u < units; u += gridDim.x) {
    const int j = (int)(u / per_blk), r = (int)(u - (long long)j * per_blk);
    const int sl = r / g.nrg, rgi = r - sl * g.nrg;
    const int id = __ldg(ids + j);
    const int n = id / (g.hb * g.wb), rem = id - n * g.hb * g.wb;
    const int by = rem / g.wb, bx = rem - by * g.wb;
    const int c0 = sl * S + v * 8;
    float mu[8], sc[8], be[8];
    {
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + c0));
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + c0 + 4));
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(beta + c0));
      const float4 b1 = __ldg(reinterpret_cast<const float4*>(beta + c0 + 4));
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      const int q0 = c0 / cg, rq = c0 - q0 * cg;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        int gi = q0, rr = rq + i;
        while (rr >= cg) {
          rr -= cg;
          ++gi;
        }
        const float2 fs = __ldg(fstats + (size_t)n * g.G + gi);
        mu[i] = fs.x;
        sc[i] = gg[i] * fs.y;
        be[i] = bb[i];
      }
    }
    // this unit's ring rows: [by*b - 1 + rgi*rg, ... + rg) clipped to the image
    const int ya = by * g.b - 1 + rgi * g.rg;
    const int y0 = max(ya, 0), y1 = min(min(ya + g.rg, by * g.b + g.b + 1), g.h);
    if (y0 >= y1) continue;
    const int x0 = max(bx * g.b - 1, 0), x1 = min(bx * g.b + g.b + 1, g.w);
    const int rw = x1 - x0, np = (y1 - y0) * rw;
    const __nv_bfloat16* xb = x + (((size_t)n * g.h + y0) * g.w + x0) * g.c + c0;
    __nv_bfloat16* ab = a + (((size_t)n * g.h + y0) * g.w + x0) * g.c + c0;
    const float inv_rw = 1.f / (float)rw;  // exact floor((pp + 0.5) / rw) for pp < 2^20
    const uint32_t row_stride = (uint32_t)g.w * g.c;
    for (int p0 = r0; p0 < np; p0 += 4 * R) {
      uint4 raw[4];
      uint32_t off[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int pp = p0 + q * R;
        const int py = __float2int_rz(((float)pp + 0.5f) * inv_rw), px = pp - py * rw;
        off[q] = (uint32_t)py * row_stride + (uint32_t)px * g.c;
        if (pp < np) raw[q] = __ldg(reinterpret_cast<const uint4*>(xb + off[q]));
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (p0 + q * R >= np) continue;
        float f[8];
        unpack8(raw[q], f);
        uint32_t o4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float r2[2];
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int i = 2 * k + h2;
            const float tt = fmaf(f[i] - mu[i], sc[i], be[i]);
            // SiLU with the SFU exponential: relative error ~1e-6 (inside the bar of R-27)
            r2[h2] = __fdividef(tt, 1.f + __expf(-tt));
          }
          const __nv_bfloat162 pk = __floats2bfloat162_rn(r2[0], r2[1]);
          o4[k] = *reinterpret_cast<const uint32_t*>(&pk);
        }
        *reinterpret_cast<uint4*>(ab + off[q]) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
      }
    }
  }
}

static int gcd_i(int a, int b) { return b ? gcd_i(b, a % b) : a; }

// Slice: the largest S | c, S a multiple of lcm(c/G, 8), with S/8 <= 64 vectors (>= 4 pixel
// lanes per CTA); else the smallest such S (S/8 <= 256 guaranteed by the host checks).
static GnGeom gn_geom(int h, int w, int c, int G, int b) {
  GnGeom g;
  g.h = h; g.w = w; g.c = c; g.G = G; g.b = b;
  g.hb = cdiv(h, b); g.wb = cdiv(w, b);
  const int cg = c / G, L = cg / gcd_i(cg, 8) * 8;
  int best = 0;
  for (int S = L; S <= c; S += L)
    if (c % S == 0 && S / 8 <= 64) best = S;
  g.S = best ? best : L;
  g.V = g.S / 8;
  g.R = kGnThreads / g.V;
  g.nslice = c / g.S;
  // ring rows per gn_silu unit: about 8 16-byte loads per thread in one batch, but at least half
  // the ring (each unit's parameter and id loads are amortised over more pixels: at the UNet levels
  // 5 rows instead of 2 measured 7% faster per GN stage, tools/gn_ab.py)
  g.rg = max(1, min(b + 2, max((4 * g.R) / (b + 2), cdiv(b + 2, 2))));
#ifdef SPHINX_DEV_KNOBS
  if (const char* env = getenv("SPHINX_GN_RG")) g.rg = max(1, min(b + 2, atoi(env)));  // dev A/B
#endif
  g.nrg = cdiv(b + 2, g.rg);
  return g;
}

static int gn_grid(long long units, int sms) {
  const long long cap = (long long)sms * 8;
  return (int)(units < cap ? (units > 0 ? units : 1) : cap);
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
  if (c % 8 || block > 64) return SPHINX_ERR_UNSUPPORTED;
  const int cg = c / groups;
  if (cg / gcd_i(cg, 8) * 8 > 8 * kGnThreads) return SPHINX_ERR_UNSUPPORTED;  // slice > 256 vectors
  if (!aligned16(x)) return SPHINX_ERR_UNSUPPORTED;
  return SPHINX_OK;
}

static size_t gn_block_bytes(int32_t n, int32_t h, int32_t w, int32_t groups, int32_t block) {
  return (size_t)n * cdiv(h, block) * cdiv(w, block) * groups * sizeof(float2);
}

extern "C" size_t sphinx_gn_stats_size(int32_t n, int32_t h, int32_t w, int32_t groups,
                                       int32_t block) {
  if (n <= 0 || h <= 0 || w <= 0 || groups <= 0 || block <= 0) return 0;
  return gn_block_bytes(n, h, w, groups, block) + (size_t)n * groups * sizeof(float2);
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
  const GnGeom g = gn_geom(h, w, c, groups, block);
  cudaError_t e = launch_k(gn_block_stats_kernel, dim3(gn_grid((long long)capacity * g.nslice, sms)),
                           dim3(kGnThreads), 0, reinterpret_cast<cudaStream_t>(stream),
                           static_cast<const __nv_bfloat16*>(x), g, block_ids, count,
                           reinterpret_cast<float2*>(stats));
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

extern "C" sphinx_status sphinx_gn_silu(const void* x, float* stats, const float* gamma,
                                        const float* beta, float eps, int32_t n, int32_t h,
                                        int32_t w, int32_t c, int32_t groups, int32_t block,
                                        const int32_t* block_ids, const int32_t* count,
                                        int32_t capacity, void* a, sphinx_stream_t stream) {
  sphinx_status st = gn_check(x, n, h, w, c, groups, block, block_ids, count, capacity);
  if (st != SPHINX_OK) return st;
  if (!stats || !gamma || !beta || !a || a == x || !(eps >= 0.f)) return SPHINX_ERR_INVALID_ARGUMENT;
  if (!aligned16(a) || !aligned16(gamma) || !aligned16(beta) ||
      (reinterpret_cast<uintptr_t>(stats) & 7u))
    return SPHINX_ERR_UNSUPPORTED;
  int sms = 0;
  if ((st = check_device(&sms)) != SPHINX_OK) return st;
  if (capacity == 0) return SPHINX_OK;
  const GnGeom g = gn_geom(h, w, c, groups, block);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const float2* blk = reinterpret_cast<const float2*>(stats);
  float2* fst = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(stats) + gn_block_bytes(n, h, w, groups, block));
  const int warps = n * groups;
  cudaError_t e = launch_k(gn_finalize_kernel, dim3(cdiv(warps, kGnThreads / 32)), dim3(kGnThreads), 0, s,
                           blk, fst, g, (int)n, eps, static_cast<const float*>(nullptr),
                           static_cast<const float*>(nullptr), static_cast<float2*>(nullptr));
  if (e != cudaSuccess) return cuda_fail(e);
  e = launch_k(gn_silu_kernel, dim3(gn_grid((long long)capacity * g.nslice * g.nrg, sms)), dim3(kGnThreads), 0, s,
               static_cast<const __nv_bfloat16*>(x), static_cast<const float2*>(fst), gamma, beta, g,
               block_ids, count, static_cast<__nv_bfloat16*>(a));
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

extern "C" sphinx_status sphinx_gn_scale_shift(float* stats, const float* gamma, const float* beta,
                                               float eps, int32_t n, int32_t h, int32_t w, int32_t c,
                                               int32_t groups, int32_t block, float* table,
                                               sphinx_stream_t stream) {
  if (!stats || !gamma || !beta || !table || !(eps >= 0.f) || n <= 0 || h <= 0 || w <= 0 || c <= 0 ||
      groups <= 0 || block <= 0 || c % groups)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(stats) & 7u) || (reinterpret_cast<uintptr_t>(table) & 7u))
    return SPHINX_ERR_INVALID_ARGUMENT;
  int sms = 0;
  sphinx_status st = check_device(&sms);
  if (st != SPHINX_OK) return st;
  const GnGeom g = gn_geom(h, w, c, groups, block);
  float2* fst = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(stats) + gn_block_bytes(n, h, w, groups, block));
  cudaError_t e = launch_k(gn_finalize_kernel, dim3(cdiv(n * groups, kGnThreads / 32)), dim3(kGnThreads), 0,
                           reinterpret_cast<cudaStream_t>(stream), static_cast<const float2*>(
                               reinterpret_cast<float2*>(stats)), fst, g, (int)n, eps, gamma, beta,
                           reinterpret_cast<float2*>(table));
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

static sphinx_status resblock_impl(
    const void* x, const void* w1, const float* b1, const void* w2, const float* b2,
    const float* gn1_gamma, const float* gn1_beta, const float* gn2_gamma, const float* gn2_beta,
    int32_t groups, float eps, void* h_buf, float* x_stats, float* h_stats, void* y,
    sphinx_dtype y_dtype, void* a_scratch, int32_t n, int32_t h, int32_t w, int32_t c,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity,
    void* workspace, size_t workspace_bytes, bool fused, sphinx_stream_t stream) {
  if (!h_buf || !y || !a_scratch || !x_stats || !h_stats) return SPHINX_ERR_INVALID_ARGUMENT;
  if (h_buf == x || y == x || y == h_buf || a_scratch == x || a_scratch == h_buf || a_scratch == y ||
      x_stats == h_stats)
    return SPHINX_ERR_INVALID_ARGUMENT;
  sphinx_status st;
  if (fused) {
    if (block != 8 || c % 8) return SPHINX_ERR_UNSUPPORTED;
    // Fused path (opt-in, measured slower than the separate pass: DESIGN.md 6.8): GN+SiLU is applied inside the conv (transform warps between the halo
    // TMA and the MMA), so the activation never round-trips through HBM; a_scratch holds the
    // per-(frame, channel) (scale, shift) table ([N][c] float2 <= N*h*w*c*2 bytes).
    float* tab = static_cast<float*>(a_scratch);
    if ((st = sphinx_gn_block_stats(x, n, h, w, c, groups, block, block_ids, count, capacity, x_stats,
                                    stream)) != SPHINX_OK)
      return st;
    if ((st = sphinx_gn_scale_shift(x_stats, gn1_gamma, gn1_beta, eps, n, h, w, c, groups, block, tab,
                                    stream)) != SPHINX_OK)
      return st;
    if ((st = sphinx_sparse_conv3x3_gn_silu(x, tab, w1, b1, nullptr, h_buf, SPHINX_BF16, n, h, w, c, c,
                                            block, block_ids, count, capacity, workspace, workspace_bytes,
                                            stream)) != SPHINX_OK)
      return st;
    if ((st = sphinx_gn_block_stats(h_buf, n, h, w, c, groups, block, block_ids, count, capacity, h_stats,
                                    stream)) != SPHINX_OK)
      return st;
    if ((st = sphinx_gn_scale_shift(h_stats, gn2_gamma, gn2_beta, eps, n, h, w, c, groups, block, tab,
                                    stream)) != SPHINX_OK)
      return st;
    return sphinx_sparse_conv3x3_gn_silu(h_buf, tab, w2, b2, x, y, y_dtype, n, h, w, c, c, block, block_ids,
                                         count, capacity, workspace, workspace_bytes, stream);
  }
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
  // (6) y = x + conv2(a) + b2 on listed pixels (identity skip fused in the epilogue); same list
  // and workspace as conv1, so its edge plan is reused
  return sphinx_sparse_conv3x3_ex(a_scratch, w2, b2, x, y, y_dtype, n, h, w, c, c, block, block_ids,
                                  count, capacity, workspace, workspace_bytes, SPHINX_CONV_REUSE_PLAN,
                                  stream);
}

extern "C" sphinx_status sphinx_sparse_resblock(
    const void* x, const void* w1, const float* b1, const void* w2, const float* b2,
    const float* gn1_gamma, const float* gn1_beta, const float* gn2_gamma, const float* gn2_beta,
    int32_t groups, float eps, void* h_buf, float* x_stats, float* h_stats, void* y,
    sphinx_dtype y_dtype, void* a_scratch, int32_t n, int32_t h, int32_t w, int32_t c,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity,
    void* workspace, size_t workspace_bytes, sphinx_stream_t stream) {
  return resblock_impl(x, w1, b1, w2, b2, gn1_gamma, gn1_beta, gn2_gamma, gn2_beta, groups, eps, h_buf,
                       x_stats, h_stats, y, y_dtype, a_scratch, n, h, w, c, block, block_ids, count,
                       capacity, workspace, workspace_bytes, false, stream);
}

extern "C" sphinx_status sphinx_sparse_resblock_ex(
    const void* x, const void* w1, const float* b1, const void* w2, const float* b2,
    const float* gn1_gamma, const float* gn1_beta, const float* gn2_gamma, const float* gn2_beta,
    int32_t groups, float eps, void* h_buf, float* x_stats, float* h_stats, void* y,
    sphinx_dtype y_dtype, void* a_scratch, int32_t n, int32_t h, int32_t w, int32_t c,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity,
    void* workspace, size_t workspace_bytes, int32_t flags, sphinx_stream_t stream) {
  if (flags & ~SPHINX_RB_FUSED_GN) return SPHINX_ERR_INVALID_ARGUMENT;
  return resblock_impl(x, w1, b1, w2, b2, gn1_gamma, gn1_beta, gn2_gamma, gn2_beta, groups, eps, h_buf,
                       x_stats, h_stats, y, y_dtype, a_scratch, n, h, w, c, block, block_ids, count,
                       capacity, workspace, workspace_bytes, (flags & SPHINX_RB_FUSED_GN) != 0, stream);
}
