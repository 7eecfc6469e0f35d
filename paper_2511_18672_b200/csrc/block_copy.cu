// block_copy.cu — the multi-GPU data plane's pack / unpack of listed blocks.
//
// P:352 ("batched convolution over selected blocks") and P:489 ("latent scatter-gather
// operations"): the refined blocks of a frame computed on one GPU travel to the GPU that owns
// the frame's request as a COMPACT array of blocks in list order, [count][b][b][C], and land at
// their NHWC positions there.  Both directions are pure bit copies (no float conversion: NaN
// payloads and -0 survive), HBM-bound: 2 x the listed bytes.
//
// One CTA per listed block (grid-stride over the device count), threads over the block's
// 16-byte words in (row, pixel, channel-vector) order, so each warp touches contiguous NHWC
// row segments (b*C*elem bytes) on the map side and one contiguous run on the compact side.
#include "common.cuh"

namespace sphinx {

template <bool kPack>
__global__ void __launch_bounds__(256) block_copy_kernel(const int4* __restrict__ src,
                                                         int4* __restrict__ dst, int h, int w,
                                                         int px_vec, int b, int hb, int wb,
                                                         const int32_t* __restrict__ ids,
                                                         const int32_t* __restrict__ count) {
  pdl_wait();
  pdl_trigger();
  const int cnt = *count;
  const int row_words = b * px_vec;       // one block row in the compact slot
  const int blk_words = b * row_words;    // one compact slot
  for (int j = blockIdx.x; j < cnt; j += gridDim.x) {
    const int id = __ldg(ids + j);
    const int n = id / (hb * wb), r = id - n * (hb * wb);
    const int by = r / wb, bx = r - by * wb;
    const int y0 = by * b, x0 = bx * b;
    const int nr = min(b, h - y0), ncol = min(b, w - x0);  // truncated edge blocks (R-2)
    const int seg = ncol * px_vec;                        // real words of one block row
    const size_t slot = (size_t)j * blk_words;
    for (int i = threadIdx.x; i < nr * seg; i += blockDim.x) {
      const int py = i / seg, q = i - py * seg;
      const size_t m = (((size_t)n * h + y0 + py) * w + x0) * px_vec + q;
      const size_t c = slot + (size_t)py * row_words + q;
      if constexpr (kPack) dst[c] = __ldg(src + m);
      else dst[m] = __ldg(src + c);
    }
  }
}

static sphinx_status block_copy(bool pack, const void* src, void* dst, sphinx_dtype dtype, int32_t n,
                                int32_t h, int32_t w, int32_t c, int32_t b, const int32_t* ids,
                                const int32_t* count, int32_t capacity, sphinx_stream_t stream) {
  if (!src || !dst || !ids || !count || src == dst) return SPHINX_ERR_INVALID_ARGUMENT;
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || b <= 0 || capacity < 0) return SPHINX_ERR_INVALID_ARGUMENT;
  if (dtype != SPHINX_BF16 && dtype != SPHINX_F32) return SPHINX_ERR_INVALID_ARGUMENT;
  const int hb = cdiv(h, b), wb = cdiv(w, b);
  if ((int64_t)capacity > (int64_t)n * hb * wb) return SPHINX_ERR_INVALID_ARGUMENT;
  const int elem = dtype == SPHINX_BF16 ? 2 : 4;
  if (((int64_t)c * elem) % 16 != 0 || !aligned16(src) || !aligned16(dst)) return SPHINX_ERR_UNSUPPORTED;
  int sms = 148;
  sphinx_status st = check_device(&sms);
  if (st != SPHINX_OK) return st;
  if (capacity == 0) return SPHINX_OK;
  const int px_vec = (int)((int64_t)c * elem / 16);
  const int grid = capacity < sms * 8 ? capacity : sms * 8;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = pack ? launch_k(block_copy_kernel<true>, dim3(grid), dim3(256), 0, s,
                                  static_cast<const int4*>(src), static_cast<int4*>(dst), (int)h,
                                  (int)w, px_vec, (int)b, hb, wb, ids, count)
                       : launch_k(block_copy_kernel<false>, dim3(grid), dim3(256), 0, s,
                                  static_cast<const int4*>(src), static_cast<int4*>(dst), (int)h,
                                  (int)w, px_vec, (int)b, hb, wb, ids, count);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

// Halo windows of listed blocks, map to map (same NHWC geometry): for every listed block, the pixels
// a 3x3 conv over it reads -- rows [by*b - 1, by*b + b + 1) x columns [bx*b - 1, bx*b + b + 1),
// clipped to the image -- end up copied from src to dst.  src may be pinned host memory (read by the
// GPU over PCIe through unified addressing): a serving loop then moves only the features its convs
// read instead of whole maps.  Each block copies its own pixels and the parts of its 1-pixel ring that
// belong to UNLISTED neighbours (a listed neighbour copies those pixels as its own), so every needed
// pixel crosses once (a binary search of the ascending list tells listed from unlisted).  One CTA
// task per (block, window row); each thread keeps 4 16-byte loads in flight.
__device__ __forceinline__ bool listed(const int32_t* __restrict__ ids, int cnt, int id) {
  int lo = 0, hi = cnt - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int v = __ldg(ids + mid);
    if (v == id) return true;
    if (v < id) lo = mid + 1;
    else hi = mid - 1;
  }
  return false;
}

__device__ __forceinline__ void copy_run(const int4* __restrict__ src, int4* __restrict__ dst, size_t base,
                                         int words) {
  for (int i0 = threadIdx.x; i0 < words; i0 += 4 * blockDim.x) {
    int4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + q * blockDim.x;
      if (i < words) v[q] = src[base + i];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + q * blockDim.x;
      if (i < words) dst[base + i] = v[q];
    }
  }
}

__global__ void __launch_bounds__(256) halo_window_kernel(const int4* __restrict__ src, int4* __restrict__ dst,
                                                          int h, int w, int px_vec, int b, int hb, int wb,
                                                          const int32_t* __restrict__ ids,
                                                          const int32_t* __restrict__ count) {
  pdl_wait();
  pdl_trigger();
  const int cnt = *count;
  const long long tasks = (long long)cnt * (b + 2);
  __shared__ int s_keep[3];  // this row's left ring pixel / middle run / right ring pixel: copy?
  for (long long t = blockIdx.x; t < tasks; t += gridDim.x) {
    const int j = (int)(t / (b + 2)), r = (int)(t - (long long)j * (b + 2));
    const int id = __ldg(ids + j);
    const int n = id / (hb * wb), rem = id - n * (hb * wb);
    const int by = rem / wb, bx = rem - by * wb;
    const int y = by * b - 1 + r;
    if (y < 0 || y >= h) continue;  // (uniform across the CTA)
    // the block row owning pixel row y: by - 1 (top ring), by, or by + 1 (bottom ring)
    const int oy = r == 0 ? by - 1 : (r == b + 1 ? by + 1 : by);
    if (threadIdx.x < 3) {
      const int ox = bx - 1 + (int)threadIdx.x;
      bool keep;
      if (ox < 0 || ox >= wb) keep = false;  // outside the image (clipped anyway)
      else if (oy == by && ox == bx) keep = true;  // the block's own pixels
      else keep = !listed(ids, cnt, (n * hb + oy) * wb + ox);
      s_keep[threadIdx.x] = keep;
    }
    __syncthreads();
    const size_t row = ((size_t)n * h + y) * w;
    // left ring pixel, middle run (b pixels, clipped), right ring pixel
    const int xs[3] = {bx * b - 1, bx * b, bx * b + b};
    const int xe[3] = {bx * b, min(bx * b + b, w), bx * b + b + 1};
    for (int part = 0; part < 3; ++part) {
      const int x0 = max(xs[part], 0), x1 = min(xe[part], w);
      if (s_keep[part] && x1 > x0) copy_run(src, dst, (row + x0) * px_vec, (x1 - x0) * px_vec);
    }
    __syncthreads();  // s_keep is rewritten by the next task
  }
}

}  // namespace sphinx

extern "C" sphinx_status sphinx_gather_halo_windows(const void* src, void* dst, sphinx_dtype dtype, int32_t n,
                                                    int32_t h, int32_t w, int32_t c, int32_t block,
                                                    const int32_t* block_ids, const int32_t* count,
                                                    int32_t capacity, sphinx_stream_t stream) {
  using namespace sphinx;
  if (!src || !dst || !block_ids || !count || src == dst) return SPHINX_ERR_INVALID_ARGUMENT;
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || block <= 0 || capacity < 0) return SPHINX_ERR_INVALID_ARGUMENT;
  if (dtype != SPHINX_BF16 && dtype != SPHINX_F32) return SPHINX_ERR_INVALID_ARGUMENT;
  const int hb = cdiv(h, block), wb = cdiv(w, block);
  if ((int64_t)capacity > (int64_t)n * hb * wb) return SPHINX_ERR_INVALID_ARGUMENT;
  const int elem = dtype == SPHINX_BF16 ? 2 : 4;
  if (((int64_t)c * elem) % 16 != 0 || !aligned16(src) || !aligned16(dst)) return SPHINX_ERR_UNSUPPORTED;
  int sms = 148;
  sphinx_status st = check_device(&sms);
  if (st != SPHINX_OK) return st;
  if (capacity == 0) return SPHINX_OK;
  const int px_vec = (int)((int64_t)c * elem / 16);
  const long long tasks = (long long)capacity * (block + 2);
  const int grid = (int)(tasks < (long long)sms * 16 ? tasks : (long long)sms * 16);
  cudaError_t e = launch_k(halo_window_kernel, dim3(grid), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream),
                           static_cast<const int4*>(src), static_cast<int4*>(dst), (int)h, (int)w, px_vec,
                           (int)block, hb, wb, block_ids, count);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

extern "C" sphinx_status sphinx_gather_blocks(const void* src, void* dst, sphinx_dtype dtype, int32_t n,
                                              int32_t h, int32_t w, int32_t c, int32_t block,
                                              const int32_t* block_ids, const int32_t* count,
                                              int32_t capacity, sphinx_stream_t stream) {
  return sphinx::block_copy(true, src, dst, dtype, n, h, w, c, block, block_ids, count, capacity, stream);
}

extern "C" sphinx_status sphinx_scatter_blocks(const void* src, void* out, sphinx_dtype dtype, int32_t n,
                                               int32_t h, int32_t w, int32_t c, int32_t block,
                                               const int32_t* block_ids, const int32_t* count,
                                               int32_t capacity, sphinx_stream_t stream) {
  return sphinx::block_copy(false, src, out, dtype, n, h, w, c, block, block_ids, count, capacity, stream);
}
