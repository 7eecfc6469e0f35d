// temporal_attn.cu — NEXT-4: frame-sparse temporal attention with the latent (K/V) cache
// ("Every T steps, the model performs a full denoising pass over all input and
// target frames, during which the intermediate latent representations from each temporal
// attention layer are cached.  In the subsequent (T-1) partial denoising steps, frames that are
// not actively refined simply retrieve and reuse these cached latents"; reading R-28).
//
// Temporal attention mixes, at every pixel, the frames of one sequence (T frames).  The q|k|v
// projections live in a persistent NHWC buffer [N][H][W][3C]: the full step writes every token,
// a partial step rewrites only listed (frame, block) tokens (sphinx_sparse_pointwise), so
// unlisted tokens ARE the cache.  This kernel computes the attention output of listed tokens
// only, reading each pixel's T tokens once:
//   ta_plan_kernel   one CTA: per (sequence, block position) a bitmask of listed frames
//                    (atomicOr of bits: order-free, deterministic).
//   ta_attn_kernel   unit = (sequence, block position, pixel) with a non-zero mask: the pixel's
//                    T x 3C bf16 tokens are staged in shared memory by one thread with T bulk
//                    async copies (cp.async.bulk + mbarrier), double-buffered so the next
//                    pixel's tokens land while this one computes (row stride 6C+16 bytes, an odd
//                    number of 16-byte units: the per-key 16-byte reads are conflict-free);
//                    one warp per (listed frame, head): lane m < T computes the score q.k_m
//                    (head dim 64, fp32), warp-shuffle softmax (SFU exponential), lane l then
//                    accumulates output dims (2l, 2l+1) over the T values; bf16 store.
// CUDA cores, not tensor cores: per (query, head) the work is T x 64 x 2 MACs against T x 256 B
// of staged tokens — an L2/latency-bound gather-reduce, not a dense contraction.
#include <cuda_bf16.h>

#include "common.cuh"
#include "ptx.cuh"

namespace sphinx {

constexpr int kTaThreads = 256;
constexpr int kHeadDim = 64;

__global__ void __launch_bounds__(1024) ta_plan_kernel(const int32_t* __restrict__ ids,
                                                       const int32_t* __restrict__ count, int T,
                                                       int nblk, int n_units, uint32_t* posmask) {
  pdl_wait();
  pdl_trigger();
  for (int i = threadIdx.x; i < n_units; i += blockDim.x) posmask[i] = 0u;
  __syncthreads();
  const int cnt = *count;
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
    const int id = __ldg(ids + j);
    const int n = id / nblk, pos = id - n * nblk;
    atomicOr(posmask + (n / T) * nblk + pos, 1u << (n % T));
  }
}

struct TaGeom {
  int h, w, c, heads, T, b, hb, wb, n_seq, nbuf;
  uint32_t rs;  // staged token row stride in bytes: 6c + 16 (an odd number of 16-byte units)
  float scale;
};

// Next unit (sequence, block position, pixel) at or after u, stepping by `step`, whose pixel is
// inside the image and whose position has a listed frame; -1 if none.
__device__ __forceinline__ long long ta_next(long long u, long long step, long long units,
                                             const uint32_t* __restrict__ posmask, const TaGeom& g,
                                             uint32_t& M, size_t& pix, int& s) {
  const int nblk = g.hb * g.wb, bb = g.b * g.b;
  for (; u < units; u += step) {
    s = (int)(u / ((long long)nblk * bb));
    const int r = (int)(u - (long long)s * nblk * bb);
    const int pos = r / bb, px = r - pos * bb;
    M = __ldg(posmask + s * nblk + pos);
    if (M == 0u) continue;
    const int by = pos / g.wb, bx = pos - by * g.wb;
    const int yy = by * g.b + px / g.b, xx = bx * g.b + px % g.b;
    if (yy >= g.h || xx >= g.w) continue;
    pix = (size_t)yy * g.w + xx;
    return u;
  }
  return -1;
}

__global__ void __launch_bounds__(kTaThreads) ta_attn_kernel(
    const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* o, const uint32_t* __restrict__ posmask,
    const TaGeom g) {
  extern __shared__ __align__(128) uint8_t ta_sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(ta_sm);
  uint8_t* rows = ta_sm + 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const int c = g.c, c3 = 3 * c, T = g.T;
  const size_t plane = (size_t)g.h * g.w;
  const long long units = (long long)g.n_seq * g.hb * g.wb * g.b * g.b;
  const uint32_t tok_bytes = (uint32_t)c3 * 2;
  // one elected thread stages the pixel's T tokens with bulk async copies (one per frame)
  auto stage = [&](int buf, int s, size_t pix) {
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&bars[buf], tok_bytes * (uint32_t)T);
      uint8_t* dst = rows + (size_t)buf * T * g.rs;
      for (int m = 0; m < T; ++m)
        bulk_g2s(dst + (size_t)m * g.rs, qkv + (((size_t)s * T + m) * plane + pix) * c3, tok_bytes, &bars[buf]);
    }
  };
  uint32_t M;
  size_t pix;
  int s;
  long long u = ta_next(blockIdx.x, gridDim.x, units, posmask, g, M, pix, s);
  if (u >= 0) stage(0, s, pix);
  uint32_t phase = 0u;  // bit k = parity of buffer k
  int buf = 0;
  while (u >= 0) {
    uint32_t Mn;
    size_t pixn;
    int sn;
    const long long un = ta_next(u + gridDim.x, gridDim.x, units, posmask, g, Mn, pixn, sn);
    if (un >= 0 && g.nbuf == 2) stage(buf ^ 1, sn, pixn);  // prefetch (that buffer is free)
    mbar_wait(&bars[buf], (phase >> buf) & 1u);
    phase ^= 1u << buf;
    const uint8_t* tk = rows + (size_t)buf * T * g.rs;
    const int nq = __popc(M);
    for (int task = warp; task < nq * g.heads; task += kTaThreads / 32) {
      const int qi = task / g.heads, hd = task - qi * g.heads;
      uint32_t mm = M;
      for (int k = 0; k < qi; ++k) mm &= mm - 1;
      const int f = __ffs(mm) - 1;
      float sc = -INFINITY;
      if (lane < T) {
        // 16-byte reads: the row stride is an odd number of 16-byte units, so the 8 lanes of each
        // quarter-warp phase hit distinct bank quads (conflict-free); q is a broadcast
        const uint4* q4 = reinterpret_cast<const uint4*>(tk + (size_t)f * g.rs + hd * kHeadDim * 2);
        const uint4* k4 = reinterpret_cast<const uint4*>(tk + (size_t)lane * g.rs + (c + hd * kHeadDim) * 2);
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int k = 0; k < kHeadDim / 8; ++k) {
          const uint4 qa = q4[k], ka = k4[k];
          const uint32_t qw[4] = {qa.x, qa.y, qa.z, qa.w}, kw[4] = {ka.x, ka.y, ka.z, ka.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            a0 = fmaf(__uint_as_float(qw[i] << 16), __uint_as_float(kw[i] << 16), a0);
            a1 = fmaf(__uint_as_float(qw[i] & 0xffff0000u), __uint_as_float(kw[i] & 0xffff0000u), a1);
          }
        }
        sc = (a0 + a1) * g.scale;
      }
      float mx = sc;
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
      const float pr = lane < T ? __expf(sc - mx) : 0.f;
      float den = pr;
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o2);
      float o0 = 0.f, o1 = 0.f;
      const uint32_t* vcol = reinterpret_cast<const uint32_t*>(tk + (2 * c + hd * kHeadDim) * 2) + lane;
      const uint32_t rsw = g.rs / 4;
      for (int m = 0; m < T; ++m) {
        const float pm = __shfl_sync(0xffffffffu, pr, m);
        const uint32_t vw = vcol[m * rsw];
        o0 = fmaf(pm, __uint_as_float(vw << 16), o0);
        o1 = fmaf(pm, __uint_as_float(vw & 0xffff0000u), o1);
      }
      const float inv = 1.f / den;
      const __nv_bfloat162 pk = __floats2bfloat162_rn(o0 * inv, o1 * inv);
      *reinterpret_cast<__nv_bfloat162*>(o + (((size_t)s * T + f) * plane + pix) * c + hd * kHeadDim +
                                         2 * lane) = pk;
    }
    __syncthreads();  // every warp is done with this buffer before it is staged again
    if (un >= 0 && g.nbuf == 1) stage(0, sn, pixn);
    if (g.nbuf == 2) buf ^= 1;
    u = un; M = Mn; pix = pixn; s = sn;
  }
}

static size_t ta_row(int c) { return (size_t)6 * c + 16; }
static size_t ta_smem(int c, int T, int nbuf) { return 128 + (size_t)nbuf * T * ta_row(c); }

}  // namespace sphinx

using namespace sphinx;

extern "C" size_t sphinx_temporal_attention_workspace_size(int32_t n, int32_t h, int32_t w,
                                                            int32_t frames_per_seq, int32_t block) {
  if (n <= 0 || h <= 0 || w <= 0 || block <= 0 || frames_per_seq <= 0 || n % frames_per_seq) return 0;
  return (size_t)(n / frames_per_seq) * cdiv(h, block) * cdiv(w, block) * sizeof(uint32_t);
}

extern "C" sphinx_status sphinx_temporal_attention(const void* qkv, void* o, int32_t n, int32_t h,
                                                   int32_t w, int32_t c, int32_t heads,
                                                   int32_t frames_per_seq, int32_t block,
                                                   const int32_t* block_ids, const int32_t* count,
                                                   int32_t capacity, void* workspace,
                                                   size_t workspace_bytes, sphinx_stream_t stream) {
  if (!qkv || !o || !block_ids || !count || !workspace || qkv == o) return SPHINX_ERR_INVALID_ARGUMENT;
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || heads <= 0 || block <= 0 || capacity < 0 ||
      frames_per_seq <= 0 || n % frames_per_seq || c % heads)
    return SPHINX_ERR_INVALID_ARGUMENT;
  const int T = frames_per_seq;
  if ((int64_t)capacity > (int64_t)n * cdiv(h, block) * cdiv(w, block)) return SPHINX_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < sphinx_temporal_attention_workspace_size(n, h, w, T, block))
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (c / heads != kHeadDim || T > 32 || block > 64 || ta_smem(c, T, 1) > 227 * 1024)
    return SPHINX_ERR_UNSUPPORTED;
  if (!aligned16(qkv) || !aligned16(o) || (reinterpret_cast<uintptr_t>(workspace) & 3u))
    return SPHINX_ERR_UNSUPPORTED;
  int sms = 0;
  sphinx_status st = check_device(&sms);
  if (st != SPHINX_OK) return st;
  if (capacity == 0) return SPHINX_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int hb = cdiv(h, block), wb = cdiv(w, block), n_seq = n / T;
  uint32_t* posmask = static_cast<uint32_t*>(workspace);
  cudaError_t e = launch_k(ta_plan_kernel, dim3(1), dim3(1024), 0, s, block_ids, count, T, hb * wb,
                           n_seq * hb * wb, posmask);
  if (e != cudaSuccess) return cuda_fail(e);
  TaGeom g;
  g.h = h; g.w = w; g.c = c; g.heads = heads; g.T = T; g.b = block; g.hb = hb; g.wb = wb;
  g.n_seq = n_seq;
  g.rs = (uint32_t)ta_row(c);
  g.scale = 1.f / sqrtf((float)kHeadDim);
  // double-buffer the staged tokens (prefetch the next pixel during this one) when two fit
  g.nbuf = ta_smem(c, T, 2) <= 200 * 1024 ? 2 : 1;
  const size_t smem = ta_smem(c, T, g.nbuf);
  e = cudaFuncSetAttribute(ta_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return cuda_fail(e);
  const long long units = (long long)n_seq * hb * wb * block * block;
  int per_sm = (int)((228 * 1024) / (smem + 1024));
  per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
  const long long cap = (long long)sms * per_sm;
  const int grid = (int)(units < cap ? units : cap);
  e = launch_k(ta_attn_kernel, dim3(grid), dim3(kTaThreads), smem, s, static_cast<const __nv_bfloat16*>(qkv),
               static_cast<__nv_bfloat16*>(o), static_cast<const uint32_t*>(posmask), g);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

extern "C" sphinx_status sphinx_temporal_block(
    const void* x, const void* wqkv, const float* bqkv, const void* wo, const float* bo,
    int32_t heads, int32_t frames_per_seq, void* qkv_buf, void* o_scratch, void* y,
    sphinx_dtype y_dtype, int32_t n, int32_t h, int32_t w, int32_t c, int32_t block,
    const int32_t* block_ids, const int32_t* count, int32_t capacity, void* workspace,
    size_t workspace_bytes, void* attn_workspace, size_t attn_workspace_bytes,
    sphinx_stream_t stream) {
  if (!qkv_buf || !o_scratch || !y || qkv_buf == x || o_scratch == x || y == x || y == qkv_buf ||
      o_scratch == qkv_buf || o_scratch == y)
    return SPHINX_ERR_INVALID_ARGUMENT;
  sphinx_status st;
  // (1) q|k|v of the listed tokens into the persistent buffer (unlisted tokens = the cache)
  if ((st = sphinx_sparse_pointwise(x, wqkv, bqkv, nullptr, qkv_buf, SPHINX_BF16, n, h, w, c, 3 * c,
                                    block, block_ids, count, capacity, workspace, workspace_bytes,
                                    stream)) != SPHINX_OK)
    return st;
  // (2) attention of the listed tokens over their sequence's frames (fresh + cached K/V)
  if ((st = sphinx_temporal_attention(qkv_buf, o_scratch, n, h, w, c, heads, frames_per_seq, block,
                                      block_ids, count, capacity, attn_workspace, attn_workspace_bytes,
                                      stream)) != SPHINX_OK)
    return st;
  // (3) output projection + identity residual on listed pixels (persistent y)
  return sphinx_sparse_pointwise(o_scratch, wo, bo, x, y, y_dtype, n, h, w, c, c, block, block_ids,
                                 count, capacity, workspace, workspace_bytes, stream);
}
