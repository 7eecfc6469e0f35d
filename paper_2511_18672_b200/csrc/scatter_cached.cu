// scatter_cached.cu — step (5): out = active(block) ? src : latent cache (bit copy).
//
// P:352 "reuses cached latents from the last full denoising step for unrefined
// regions".  HBM-bound copy.  One CTA per (frame, pixel row): in NHWC the b
// pixels of one block on one row are a contiguous b*C*elem-byte segment, so each
// segment is a coalesced run of 16-byte words taken wholesale from src or cache.
// The element type never passes through a float conversion (NaN payloads, -0 kept).
#include "common.cuh"

namespace sphinx {

__global__ void __launch_bounds__(256) scatter_full_kernel(
    const int4* src, const int4* __restrict__ cache, int4* out, int h, int w, int px_vec, int b,
    int hb, int wb, const uint8_t* __restrict__ mask, const int32_t* __restrict__ k, int u,
    int in_place) {
  const int n = blockIdx.x / h, y = blockIdx.x - (blockIdx.x / h) * h, by = y / b;
  const int kf = k ? __ldg(k + n) : 0;
  const bool frame_ok = !k || (kf >= 0 && kf <= u);
  const size_t row = ((size_t)n * h + y) * w;
  for (int bx = 0; bx < wb; ++bx) {
    const bool act = frame_ok && mask[((size_t)n * hb + by) * wb + bx];
    if (in_place && act) continue;
    const int x0 = bx * b, npx = min(b, w - x0);
    const size_t base = (row + x0) * px_vec;
    const int nv = npx * px_vec;
    const int4* sp = act ? src : cache;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) out[base + i] = sp[base + i];
  }
}

__global__ void __launch_bounds__(256) scatter_compact_kernel(
    const int4* __restrict__ src, const int4* __restrict__ cache, int4* __restrict__ out, int h,
    int w, int px_vec, int b, int hb, int wb, const int32_t* __restrict__ ids,
    const int32_t* __restrict__ count) {
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
  if (src_layout == SPHINX_SRC_FULL)
    scatter_full_kernel<<<grid, 256, 0, s>>>(
        static_cast<const int4*>(src), static_cast<const int4*>(cache), static_cast<int4*>(out), h,
        w, px_vec, b, hb, wb, block_mask, start_step, step_u, out == src ? 1 : 0);
  else
    scatter_compact_kernel<<<grid, 256, 0, s>>>(
        static_cast<const int4*>(src), static_cast<const int4*>(cache), static_cast<int4*>(out), h,
        w, px_vec, b, hb, wb, block_ids, count);
  SPHINX_CHECK_LAUNCH();
  return SPHINX_OK;
}
