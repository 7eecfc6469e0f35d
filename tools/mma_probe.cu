// Dev microbenchmark (not part of the library): tcgen05.mma issue rate of one vs two issuing
// threads on one SM, cta_group::1, M = 128, bf16 -> fp32, operands in shared memory (SW128,
// content irrelevant).  Floor per instruction: 128 * N / 256 cycles (B300_MICROARCH "tcgen05
// floor").  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_18672_b200/csrc \
//        -o /tmp/mma_probe tools/mma_probe.cu -lcuda && /tmp/mma_probe
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace sphinx;

constexpr int ITER = 2048;

// WAIT (bits): every 4 MMAs also 1 = wait on an already-complete mbarrier phase, 2 = fence,
// 4 = the wait uses mbarrier.test_wait (non-blocking probe) in a spin instead of try_wait
// 8 = descriptors precomputed once (per-MMA: add the K offset >> 4 to the start-address field)
// (the shape of the conv kernels' per-(tap, chunk) loop: wait operands, fence, 4 MMAs, commit)
__device__ __forceinline__ void mbar_wait_test(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "TW_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra TW_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
template <int N, int ISSUERS, int COMMIT_EVERY, int WAIT = 0>
__global__ void __launch_bounds__(128, 1) probe(unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;             // 128 rows x 128 B
  uint8_t* sB = smem + 16384;     // N rows x 128 B
  __shared__ uint64_t bars[6];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 6; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    mbar_arrive(&bars[4]);  // phase 0 of bars[4] complete: waits on parity 0 return at once
    mbar_arrive(&bars[5]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  constexpr uint32_t idesc = idesc_bf16_f32(128, N);
  if (lane == 0 && warp < ISSUERS) {
    const uint32_t d = tbase + (uint32_t)(warp * 256);
    const uint32_t a = smem_u32(sA), b = smem_u32(sB);
    uint32_t ph = 0;
    const uint64_t ad0 = umma_desc_sw128(a, 1024, 0), bd0 = umma_desc_sw128(b, 1024, 0);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < ITER; ++i) {
      const int k = i & 3;
      if (WAIT && k == 0) {
        if (WAIT & 1) {
          if (WAIT & 4) mbar_wait_test(&bars[4 + warp], 0);
          else mbar_wait(&bars[4 + warp], 0);
        }
        if (WAIT & 2) tc_fence_after();
      }
      if (WAIT & 8) {
        tc_mma_bf16(d, ad0 + (uint64_t)(k * 2), bd0 + (uint64_t)(k * 2), idesc, i ? 1u : 0u);
      } else {
        tc_mma_bf16(d, umma_desc_sw128(a + k * 32, 1024, 0), umma_desc_sw128(b + k * 32, 1024, 0), idesc,
                    i ? 1u : 0u);
      }
      if (COMMIT_EVERY && (i % COMMIT_EVERY) == COMMIT_EVERY - 1) tc_commit(&bars[2 + warp]);
    }
    tc_commit(&bars[warp]);
    mbar_wait(&bars[warp], 0);
    const unsigned long long t1 = clock64();
    out[blockIdx.x * 2 + warp] = t1 - t0;
    (void)ph;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

// cta_group::2 variant (cluster of 2, M = 256, the conv kernels' configuration): the leader issues,
// commits multicast to both CTAs; WAIT as above (bit 1: completed-phase wait every MPW MMAs).
template <int N, int WAIT, int MPW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe2(unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + 16384;  // N/2 rows x 128 B
  __shared__ uint64_t bars[4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < (16384 + N * 64) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    mbar_arrive(&bars[3]);  // completed phase 0
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc_cg2<512>(&tslot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tslot;
  constexpr uint32_t idesc = idesc_bf16_f32(256, N);
  if (rank == 0 && warp == 0 && lane == 0) {
    const uint32_t a = smem_u32(sA), b = smem_u32(sB);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < ITER; ++i) {
      const int k = i & 3;
      if (WAIT && (i % MPW) == 0) {
        mbar_wait(&bars[3], 0);
        tc_fence_after();
      }
      tc_mma_bf16_cg2(tbase, umma_desc_sw128(a + k * 32, 1024, 0), umma_desc_sw128(b + k * 32, 1024, 0), idesc,
                      i ? 1u : 0u);
      if ((i % MPW) == MPW - 1) tc_commit_cg2_mc(&bars[1]);
    }
    tc_commit_cg2_mc(&bars[0]);
    mbar_wait(&bars[0], 0);
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 0) tmem_dealloc_cg2<512>(tbase);
}

template <int N, int WAIT, int MPW>
void run2() {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * 2);
  cudaMemset(d, 0, sizeof(unsigned long long) * 2);
  const int smem = 16384 + N * 64 + 1024;
  cudaFuncSetAttribute(probe2<N, WAIT, MPW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe2<N, WAIT, MPW><<<2, 128, smem>>>(d);
  probe2<N, WAIT, MPW><<<2, 128, smem>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"cta_group\": 2, \"N\": %d, \"wait\": %d, \"mma_per_wait\": %d, \"cyc_per_mma\": %.1f, \"floor\": %d, "
         "\"err\": \"%s\"}\n", N, WAIT, MPW, (double)h[0] / ITER, 256 * N / 512, cudaGetErrorString(e));
  cudaFree(d);
}

template <int N, int ISSUERS, int COMMIT_EVERY, int WAIT = 0>
void run(int ctas) {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * 2 * ctas);
  cudaMemset(d, 0, sizeof(unsigned long long) * 2 * ctas);
  const int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(probe<N, ISSUERS, COMMIT_EVERY, WAIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N, ISSUERS, COMMIT_EVERY, WAIT><<<ctas, 128, smem>>>(d);
  probe<N, ISSUERS, COMMIT_EVERY, WAIT><<<ctas, 128, smem>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2 * 148];
  cudaMemcpy(h, d, sizeof(unsigned long long) * 2 * ctas, cudaMemcpyDeviceToHost);
  double c0 = (double)h[0] / ITER, c1 = ISSUERS > 1 ? (double)h[1] / ITER : 0;
  printf("{\"N\": %d, \"wait_every_4\": %d, \"issuers\": %d, \"commit_every\": %d, \"ctas\": %d, \"cyc_per_mma_issuer0\": %.1f, "
         "\"cyc_per_mma_issuer1\": %.1f, \"floor\": %d, \"err\": \"%s\"}\n",
         N, WAIT, ISSUERS, COMMIT_EVERY, ctas, c0, c1, 128 * N / 256, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<64, 1, 0>(1);
  run<64, 2, 0>(1);
  run<128, 1, 0>(1);
  run<128, 2, 0>(1);
  run<160, 1, 0>(1);
  run<160, 1, 4>(1);
  run<160, 2, 0>(1);
  run<160, 2, 4>(1);
  run<256, 1, 0>(1);
  run<256, 2, 0>(1);
  run<160, 1, 4>(148);
  run<160, 2, 4>(148);
  run<160, 1, 4, 3>(1);
  run<160, 1, 4, 1>(1);
  run<160, 1, 4, 2>(1);
  run<160, 1, 4, 11>(1);
  run<160, 1, 4, 8>(1);
  run<64, 1, 0, 8>(1);
  run<128, 1, 4, 11>(1);
  run2<160, 0, 4>();
  run2<160, 1, 4>();
  run2<160, 1, 8>();
  run2<256, 1, 4>();
  run2<160, 1, 36>();
  return 0;
}
