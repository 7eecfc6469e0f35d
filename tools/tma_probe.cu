// TMA throughput probe (dev tool, not part of the product): one producer thread per CTA keeps
// `slots` boxes of {64 ch, bw px, 1} in flight from a [rows][W][C] bf16 tensor; 1 CTA per SM.
// Reports chip GB/s for box widths / channel strides / footprints (L2-resident vs HBM stream).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../paper_2511_18672_b200/csrc/ptx.cuh"
using namespace sphinx;

__global__ void __launch_bounds__(128) probe(const __grid_constant__ CUtensorMap tm, int iters, int slots,
                                            int slot_bytes, int C, int W, int bw, int rows) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // each producer warp (lane 0) owns slots/nw of the ring and its barriers
  const int nw = blockDim.x / 32, wid = threadIdx.x / 32;
  if ((threadIdx.x & 31) != 0) return;
  slots /= nw;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 200 * 1024) + wid * 64;
  uint8_t* ring = smem + wid * slots * slot_bytes;
  iters /= nw;
  for (int i = 0; i < slots; ++i) mbar_init(&bar[i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t ph = 0;
  const uint64_t pol = policy_evict_normal();
  uint64_t st = 0x9E3779B97F4A7C15ull * (blockIdx.x * 4 + wid + 1);
  for (int i = 0; i < iters; ++i) {
    const int s = i & (slots - 1);
    if (i >= slots) {
      mbar_wait(&bar[s], (uint32_t)((ph >> s) & 1));
      ph ^= 1ull << s;
    }
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    const uint32_t r = (uint32_t)(st >> 33);
    const int c0 = (int)((i & 1) * 64);
    const int x = (int)(r & 15);
    const int row = (int)((r >> 7) & (uint32_t)(rows - 1));
    mbar_arrive_expect_tx(&bar[s], slot_bytes);
    tma_load_3d(&tm, &bar[s], ring + s * slot_bytes, c0, x, row, pol);
  }
  for (int s = 0; s < slots && s < iters; ++s) mbar_wait(&bar[s], (uint32_t)((ph >> s) & 1));
}

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                        CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  PFN enc = (PFN)fp;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = (size_t)4 << 30;
  void* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  printf("nw,C,bw,box_B,inflight_KB,footprint_MB,GBps,ops_per_us_per_SM\n");
  const int Cs[1] = {320};
  const int bws[5] = {8, 10, 20, 40, 80};
  const int infl[2] = {64, 128};
  const size_t foot[2] = {(size_t)16 << 20, (size_t)4 << 30};
  for (int nw = 1; nw <= 4; nw *= 2)
  for (int ci = 0; ci < 1; ++ci)
    for (int fi = 0; fi < 2; ++fi)
      for (int bi = 0; bi < 5; ++bi)
        for (int ii = 0; ii < 2; ++ii) {
          const int C = Cs[ci], W = 96, bw = bws[bi];
          int rows = 1;
          while ((size_t)rows * 2 * W * C * 2 <= foot[fi]) rows *= 2;
          CUtensorMap tm;
          cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)rows};
          cuuint64_t strides[2] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2};
          cuuint32_t box[3] = {64, (cuuint32_t)bw, 1}, es[3] = {1, 1, 1};
          if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode fail\n");
            return 1;
          }
          const int slot = bw * 128;
          int slots = infl[ii] * 1024 / slot;
          int sl = 1;
          while (sl * 2 <= slots && sl * 2 <= 64) sl *= 2;
          slots = sl;
          const int iters = (int)((size_t)64 << 20) / sms / slot;  // ~64 MB moved per launch... per SM share
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            probe<<<sms, 32 * nw, 210 * 1024>>>(tm, iters, slots, slot, C, W, bw, rows);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
          }
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          const double bytes = (double)iters * slot * sms;
          printf("%d,%d,%d,%d,%d,%zu,%.0f,%.1f\n", nw, C, bw, slot, infl[ii], foot[fi] >> 20, bytes / ms / 1e6,
                 (double)iters / (ms * 1e3));
          if (cudaGetLastError() != cudaSuccess) { printf("cuda error\n"); return 1; }
        }
  return 0;
}
