// scatter_cached.cu — step (5): out = active(block) ? src : latent cache (bit copy).
//
// P:352 "reuses cached latents from the last full denoising step for unrefined
// regions".  HBM-bound copy, 2 x map bytes (read src-or-cache, write out).
// FULL layout: CTAs of 256 threads over (pixel rows x 16-byte words of a row), coalesced for
// any C; COMPACT layout: one CTA per (frame, pixel row), each block's row segment taken from
// its compact slot (binary search of the ascending list) or from the cache.  The element
// type never passes through a float conversion (NaN payloads, -0 kept).
#include "common.cuh"

namespace sphinx {

// One CTA row (blockIdx.y) per pixel row of one frame, threads over the row's 16-byte words (4
// per thread in flight): consecutive threads cover consecutive words, so each warp's accesses
// are coalesced whatever C is (4 fp32 latent channels or 640 bf16 feature channels), and the
// frame / block-row lookups are per CTA (the flat-index version spent its issue slots on 64-bit
// divisions: 57% of HBM).
__global__ void __launch_bounds__(256) scatter_full_kernel(
    const int4* src, const int4* __restrict__ cache, int4* out, int h, int w, int px_vec, int b,
    int hb, int wb, const uint8_t* __restrict__ mask, const int32_t* __restrict__ k, int u,
    int in_place, int rows) {
  pdl_wait();
  pdl_trigger();
  const int row_vec = w * px_vec;
  const float inv_pv = 1.0f / (float)px_vec;  // exact floor((xv + 0.5) / px_vec) for xv < 2^20
  // blockDim.y pixel rows per CTA: short rows (the 4-channel fp32 latent is 72 words) still
  // give every warp a full row segment
  for (int row = blockIdx.y * blockDim.y + threadIdx.y; row < rows; row += gridDim.y * blockDim.y) {
    const int n = row / h, y = row - n * h;
    const int kf = k ? __ldg(k + n) : 0;
    const bool frame_ok = !k || (kf >= 0 && kf <= u);
    const uint8_t* mrow = mask + ((size_t)n * hb + y / b) * wb;
    const size_t base = (size_t)row * row_vec;
    for (int x0 = blockIdx.x * blockDim.x * 4 + threadIdx.x; x0 < row_vec; x0 += gridDim.x * blockDim.x * 4) {
      int4 v[4];
      bool act[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int xv = x0 + q * blockDim.x;
        act[q] = false;
        if (xv < row_vec) {
          const int x = __float2int_rz(((float)xv + 0.5f) * inv_pv);
          act[q] = frame_ok && mrow[x / b];
          if (!(in_place && act[q])) v[q] = act[q] ? src[base + xv] : __ldg(cache + base + xv);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int xv = x0 + q * blockDim.x;
        if (xv < row_vec && !(in_place && act[q])) out[base + xv] = v[q];
      }
    }
  }
}

__global__ void __launch_bounds__(256) scatter_compact_kernel(
    const int4* __restrict__ src, const int4* __restrict__ cache, int4* __restrict__ out, int h,
    int w, int px_vec, int b, int hb, int wb, const int32_t* __restrict__ ids,
    const int32_t* __restrict__ count) {
  pdl_wait();
  pdl_trigger();
  const int n = blockIdx.x / h, y = blockIdx.x - (blockIdx.x / h) * h;
  const int by = y / b, py = y - by * b;
  const int cnt = *count;
  const size_t row = ((size_t)n * h + y) * w;
  for (int bx = 0; bx < wb; ++bx) {
    // position of this block in the ascending list (binary search), -1 if unlisted
    const int id = (n * hb + by) * wb + bx;
    int lo = 0, hi = cnt - 1, j = -1;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      const int v = __ldg(ids + mid);
      if (v == id) { j = mid; break; }
      if (v < id) lo = mid + 1; else hi = mid - 1;
    }
    const int x0 = bx * b, npx = min(b, w - x0);
    const size_t base = (row + x0) * px_vec;
    const int nv = npx * px_vec;
    if (j >= 0) {
      const size_t sb = ((size_t)j * b + py) * b * px_vec;
      for (int i = threadIdx.x; i < nv; i += blockDim.x) out[base + i] = src[sb + i];
    } else {
      for (int i = threadIdx.x; i < nv; i += blockDim.x) out[base + i] = cache[base + i];
    }
  }
}

}  // namespace sphinx

using namespace sphinx;

extern "C" sphinx_status sphinx_scatter_cached(const void* src, sphinx_src_layout src_layout,
                                               const void* cache, void* out, sphinx_dtype dtype,
                                               int32_t n, int32_t h, int32_t w, int32_t c,
                                               int32_t b, const uint8_t* block_mask,
                                               const int32_t* start_step, int32_t step_u,
                                               const int32_t* block_ids, const int32_t* count,
                                               sphinx_stream_t stream) {
  if (!src || !cache || !out || n <= 0 || h <= 0 || w <= 0 || c <= 0 || b <= 0)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (dtype != SPHINX_BF16 && dtype != SPHINX_F32) return SPHINX_ERR_INVALID_ARGUMENT;
  if (src_layout == SPHINX_SRC_FULL && !block_mask) return SPHINX_ERR_INVALID_ARGUMENT;
  if (src_layout == SPHINX_SRC_COMPACT && (!block_ids || !count))
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (src_layout != SPHINX_SRC_FULL && src_layout != SPHINX_SRC_COMPACT)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (out == cache) return SPHINX_ERR_INVALID_ARGUMENT;
  if (src_layout == SPHINX_SRC_COMPACT && out == src) return SPHINX_ERR_INVALID_ARGUMENT;
  const int elem = dtype == SPHINX_BF16 ? 2 : 4;
  if (((int64_t)c * elem) % 16 != 0 || !aligned16(src) || !aligned16(cache) || !aligned16(out))
    return SPHINX_ERR_UNSUPPORTED;
  sphinx_status st = check_device();
  if (st != SPHINX_OK) return st;
  const int px_vec = (int)((int64_t)c * elem / 16);
  const int hb = cdiv(h, b), wb = cdiv(w, b);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int grid = n * h;
  if (src_layout == SPHINX_SRC_FULL) {
    int sms = 148;
    check_device(&sms);
    if ((long long)w * px_vec >= (1 << 20)) return SPHINX_ERR_UNSUPPORTED;  // row index math
    const int rows = n * h, row_vec = w * px_vec;
    // threads along the row's 16-byte words, 4 words in flight each (a multiple of 32, <= 256);
    // the rest of the 256 threads over rows
    int bdx = (cdiv(row_vec, 4) + 31) / 32 * 32;
    bdx = bdx < 32 ? 32 : (bdx > 256 ? 256 : bdx);
    while (256 % bdx) bdx += 32;
    const int bdy = 256 / bdx;
    const int gx = cdiv(row_vec, bdx * 4);
    const int gyr = cdiv(rows, bdy);
    const int gy = gyr < 65535 ? gyr : 65535;
    cudaError_t e = launch_k(scatter_full_kernel, dim3(gx, gy), dim3(bdx, bdy), 0, s,
                             static_cast<const int4*>(src), static_cast<const int4*>(cache),
                             static_cast<int4*>(out), (int)h, (int)w, px_vec, (int)b, hb, wb,
                             block_mask, start_step, (int)step_u, out == src ? 1 : 0, rows);
    if (e != cudaSuccess) return cuda_fail(e);
  } else {
    cudaError_t e = launch_k(scatter_compact_kernel, dim3(grid), dim3(256), 0, s,
                             static_cast<const int4*>(src), static_cast<const int4*>(cache),
                             static_cast<int4*>(out), (int)h, (int)w, px_vec, (int)b, hb, wb,
                             block_ids, count);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  return SPHINX_OK;
}
