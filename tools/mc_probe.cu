// TMA multicast probe (dev tool, not part of the product): is the ~55 GB/s per-SM TMA ingress the
// conv kernels sit at (DESIGN 6.4) a limit of the receiving SM, or of the requests each SM issues?
// Clusters of 2 CTAs, one CTA per SM, each with a ring of 16 KB boxes from an L2-resident bf16
// tensor.  unicast: each CTA issues and receives its own boxes.  multicast: every box lands in BOTH
// CTAs of the cluster, the two CTAs issuing alternate boxes (mask 0b11), so each SM issues half of
// what it receives.  Reports the bytes landed in shared memory per second, chip-wide.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2511_18672_b200/csrc/ptx.cuh"
using namespace sphinx;

constexpr int kBox = 16384;

__device__ __forceinline__ void tma_load_3d_mc(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1,
                                               int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32) probe(const __grid_constant__ CUtensorMap tm,
                                                                       int rounds, int slots, int rows, int mc,
                                                                       int box, int strided) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + slots * kBox);  // slots hold up to kBox bytes
  uint64_t* empty = bar + slots;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < slots; ++s) {
      mbar_init(&bar[s], 1);
      mbar_init(&empty[s], 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < slots; ++s) mbar_arrive_expect_tx(&bar[s], box);
  }
  __syncwarp();
  cluster_sync();
  uint64_t st = 0x9E3779B97F4A7C15ull * (blockIdx.x + 1);
  for (int k = 0; k < rounds && threadIdx.x == 0; ++k) {
    for (int s = 0; s < slots; ++s) {
      st = st * 6364136223846793005ull + 1442695040888963407ull;
      const int row = (int)((st >> 33) & (uint64_t)(rows - 1));
      if (strided) {  // weight tile: (tap, chunk) index and a block of 80 output channels
        tma_load_3d(&tm, &bar[s], smem + s * kBox, 0, (int)((st >> 40) % 45), 80 * (int)((st >> 50) & 3),
                    policy_evict_normal());
      } else if (!mc) {
        tma_load_3d(&tm, &bar[s], smem + s * kBox, 0, 0, row, policy_evict_normal());
      } else if ((uint32_t)(s & 1) == rank) {
        if (k > 0) mbar_wait(&empty[s], (uint32_t)((k - 1) & 1));
        tma_load_3d_mc(&tm, &bar[s], smem + s * kBox, 0, 0, row, (uint16_t)0x3);
      }
    }
    for (int s = 0; s < slots; ++s) {
      mbar_wait(&bar[s], (uint32_t)(k & 1));
      if (k + 1 < rounds) mbar_arrive_expect_tx(&bar[s], box);
      if (mc) {
        uint32_t r;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(&empty[s])), "r"((uint32_t)(s & 1)));
        mbar_arrive_cluster(r);
      }
    }
  }
  __syncwarp();
  cluster_sync();  // no CTA leaves while its peer may still write into it
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
  const int rows = 1024;  // 1024 x 16 KB = 16 MB: L2-resident, like the weights
  void* buf;
  cudaMalloc(&buf, (size_t)rows * kBox);
  cudaMemset(buf, 1, (size_t)rows * kBox);
  CUtensorMap tm;
  cuuint64_t dims[3] = {64, 128, (cuuint64_t)rows};
  cuuint64_t strides[2] = {128, 128 * 128};
  cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    printf("encode fail\n");
    return 1;
  }
  // strided variant: the conv's weight tiles, 80 rows of 128 B (64 channels of one output channel
  // and tap) with a row stride of 9 * 320 * 2 = 5760 B (OHWI weights, C_in = 320), 10 KB per box
  CUtensorMap tms;
  {
    cuuint64_t d2[3] = {64, 45, 320};  // [C_out = 320][45 (tap, chunk)][64 ch]
    cuuint64_t s2[2] = {128, 5760};
    cuuint32_t b2[3] = {64, 1, 80};
    if (enc(&tms, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, d2, s2, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
      printf("encode fail (strided)\n");
      return 1;
    }
  }
  const int slots = 8;  // 128 KB in flight per CTA
  const int smem = slots * kBox + 2 * slots * 8 + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("mode,ctas,GBps_landed,GBps_per_SM_landed,GBps_per_SM_issued\n");
  for (int ctas = 16; ctas <= sms; ctas *= 2) {
    const int g = ctas > sms ? sms : ctas;
    for (int mode = 0; mode < 3; ++mode) {  // 0 unicast, 1 multicast (16 KB contiguous), 2 unicast strided
      const int rounds = 400, mc = mode == 1, strided = mode == 2, box = strided ? 10240 : kBox;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        probe<<<g - (g & 1), 32, smem>>>(strided ? tms : tm, rounds, slots, rows, mc, box, strided);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      if (cudaGetLastError() != cudaSuccess) {
        printf("cuda error\n");
        return 1;
      }
      const int n = g - (g & 1);
      const double landed = (double)rounds * slots * box * n;  // every CTA receives every slot each round
      const char* nm = mode == 0 ? "unicast" : (mode == 1 ? "multicast" : "unicast_weight_tiles");
      printf("%s,%d,%.0f,%.1f,%.1f\n", nm, n, landed / ms / 1e6, landed / ms / 1e6 / n,
             landed / ms / 1e6 / n / (mc ? 2 : 1));
    }
    if (ctas * 2 > sms && ctas < sms) ctas = sms / 2;
  }
  return 0;
}
