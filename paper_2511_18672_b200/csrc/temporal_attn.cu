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
//                    q|k|v tokens of all T frames are staged in shared memory -- one 4-D TMA
//                    tensor copy (128-B swizzled rows) with the double-buffered ring (on wide
//                    levels a unit is a (pixel, head group) so that ring fits twice), else T
//                    bulk async copies (cp.async.bulk + mbarrier) -- into a ring of nbuf buffers (the next
//                    pixels' tokens land while this one computes); row stride 6C+16 bytes (an odd
//                    number of 16-byte units: conflict-free ldmatrix rows).  With the ring
//                    double-buffered the warps run a task stream: no CTA barrier per unit, warp w
//                    takes tasks w, w+nw, ... of the concatenated (unit, head, query tile)
//                    sequence and the last warp done with a buffer restages it.
//                    One warp per (head, 16 listed queries): S = Q K^T with mma.sync m16n8k16
//                    (bf16 in, fp32 accumulate), register softmax (quad shuffles, SFU exp), then
//                    O = P V with P split into bf16 hi + lo parts (|P - hi - lo| <= 2^-17 P) and
//                    V^T fragments from ldmatrix.trans; bf16 output of listed queries only.
// Per (pixel, head) the contraction is tiny (<= 32 x 32 x 64): warp-level mma.sync is the right
// tensor-core granularity (a CTA-wide tcgen05 tile would be >90% padding); the kernel is bound by
// staging the T tokens of every pixel with a listed frame (HBM/L2), not by the math.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstring>

#include "common.cuh"
#include "ptx.cuh"

namespace sphinx {

constexpr int kTaThreads = 256;     // default CTA size (SPHINX_TA_THREADS=512: 16 warps)
constexpr int kTaMaxThreads = 512;
constexpr int kTaMaxBuf = 5;        // staging ring depth limit (bars at offset 0..39)
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

// ---- warp-level tensor-core helpers (mma.sync m16n8k16 bf16 -> fp32, ldmatrix)
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

struct TaGeom {
  int h, w, c, heads, T, b, hb, wb, n_seq, nbuf;
  int ppu;      // pixels per unit: 2 = two x-adjacent pixels share one bulk copy per frame
  int kv_only;  // stage k|v of every frame + q of listed frames only (one-pixel units)
  int tmode;    // one TMA tensor copy per unit (4-D map: 64-element rows x 3C/64 x pixels x
                // frames, 128-B swizzle); staged rows are then swizzled, stride 6C
  uint32_t bstride;  // bytes per staging buffer
  int ngrp, hpg;     // tensor mode: head groups per pixel (one unit each), heads per group
  int pm_smem;  // the per-position frame masks are copied to shared memory (after the ring)
  int stream;   // task stream: no CTA barrier per unit; warp w takes tasks w, w+nw, ... of the
                // concatenated (unit, head, query tile) sequence; the last warp done with a
                // buffer restages it
  uint32_t rs;  // staged frame row stride in bytes: ppu*6c + 16 (an odd number of 16-byte units)
  float scale;
};

// Next unit (sequence, block position, group of ppu x-adjacent pixels) at or after u, stepping
// by `step`, whose first pixel is inside the image and whose position has a listed frame; -1 if
// none.  npx = pixels of the group inside the image.
__device__ __forceinline__ int ta_next(int u, int step, int units,
                                       const uint32_t* __restrict__ posmask, const TaGeom& g,
                                       uint32_t& M, size_t& pix, int& s, int& npx) {
  const int nblk = g.hb * g.wb, bbu = g.b * g.b / g.ppu;
  for (; u < units; u += step) {
    const int u0 = u / g.ngrp;  // unit = (pixel unit, head group), group fastest
    s = u0 / (nblk * bbu);
    const int r = u0 - s * nblk * bbu;
    const int pos = r / bbu, px = (r - pos * bbu) * g.ppu;
    M = posmask[s * nblk + pos];  // shared (pm_smem) or global
    if (M == 0u) continue;
    const int by = pos / g.wb, bx = pos - by * g.wb;
    const int yy = by * g.b + px / g.b, xx = bx * g.b + px % g.b;
    if (yy >= g.h || xx >= g.w) continue;
    pix = (size_t)yy * g.w + xx;
    npx = (g.ppu == 2 && xx + 1 < g.w) ? 2 : 1;
    return u;
  }
  return -1;
}

__global__ void __launch_bounds__(kTaMaxThreads) ta_attn_kernel(
    const __grid_constant__ CUtensorMap tm, const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* o,
    const uint32_t* __restrict__ posmask, const TaGeom g) {
  extern __shared__ __align__(128) uint8_t ta_sm[];
  // staging buffers start at the first 1024-byte boundary past the 128-byte header (the 128-B
  // swizzle of tensor mode repeats every 1024 B of shared address space)
  const uint32_t sm0 = smem_u32(ta_sm);
  uint8_t* rows = ta_sm + (g.tmode ? (((sm0 + 128u + 1023u) & ~1023u) - sm0) : 128u);
  auto swz = [&](uint32_t a) { return g.tmode ? (a ^ (((a >> 7) & 7u) << 4)) : a; };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ta_sm);
  // a 16-byte zero row at offset 64: ldmatrix rows of padded keys (>= T) point here
  const uint32_t zero_row = smem_u32(ta_sm + 64);
  if (threadIdx.x < 4) reinterpret_cast<uint32_t*>(ta_sm + 64)[threadIdx.x] = 0u;
  // per-buffer count of warps done with the unit it holds (offsets 80..99)
  int* done = reinterpret_cast<int*>(ta_sm + 80);
  if (threadIdx.x < kTaMaxBuf) done[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < g.nbuf; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  pdl_wait();
  pdl_trigger();
  // the unit walk reads one frame mask per unit on its serial path: from shared memory, not L2
  const uint32_t* pm = posmask;
  if (g.pm_smem) {
    uint32_t* pm_s = reinterpret_cast<uint32_t*>(rows + (size_t)g.nbuf * g.bstride);
    const int npos = g.n_seq * g.hb * g.wb;
    for (int i = threadIdx.x; i < npos; i += blockDim.x) pm_s[i] = __ldg(posmask + i);
    pm = pm_s;
  }
  __syncthreads();
  const int c = g.c, c3 = 3 * c, T = g.T;
  const size_t plane = (size_t)g.h * g.w;
  const int units = g.n_seq * g.hb * g.wb * g.b * g.b / g.ppu * g.ngrp;
  const int cs = g.hpg * kHeadDim;  // channels of one staged q (k, v) part
  // warp 0 stages the pixel's T tokens (q|k|v rows, contiguous per frame) with T bulk async copies
  // onto an mbarrier, lane m issuing frame m's copy (one issuing thread was TMA-op-rate bound:
  // ~T ops back to back per pixel).  Lane 0 posts the expected bytes before any copy is issued.
  // (Measured alternatives: k|v of all frames + q of listed frames only -- more, smaller copies
  // -- and 16-byte cp.async by all threads were both 1.3x slower.)
  const uint32_t tok_bytes = (uint32_t)c3 * 2;
  const bool kv_only = g.kv_only && g.ppu == 1;
  auto stage = [&](int buf, int s, size_t pix, int npx, uint32_t Mq, bool me, int grp) {
    if (me) {
      uint8_t* dst0 = rows + (size_t)buf * g.bstride;
      if (g.tmode) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&bars[buf], (uint32_t)(6 * cs) * (uint32_t)T);
          asm volatile(
              "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst0)),
              "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&bars[buf])), "r"(0), "r"(grp * g.hpg),
              "r"(0), "r"((int)pix), "r"(s * T)
              : "memory");
        }
      } else if (!kv_only) {
        if (lane == 0) mbar_arrive_expect_tx(&bars[buf], tok_bytes * (uint32_t)(T * npx));
        __syncwarp();
        if (lane < T)
          bulk_g2s(dst0 + (size_t)lane * g.rs, qkv + (((size_t)s * T + lane) * plane + pix) * c3,
                   tok_bytes * (uint32_t)npx, &bars[buf]);
      } else {
        // k|v of every frame (the cache of unlisted ones) + q of the listed frames only: a third
        // fewer bytes; op i < T is frame i's k|v, op T + j the j-th listed frame's q
        const uint32_t kvb = (uint32_t)c * 4, qb = (uint32_t)c * 2;
        const int nq = __popc(Mq);
        if (lane == 0) mbar_arrive_expect_tx(&bars[buf], kvb * (uint32_t)T + qb * (uint32_t)nq);
        __syncwarp();
        for (int i = lane; i < T + nq; i += 32) {
          const int m = i < T ? i : __fns(Mq, 0, i - T + 1);
          const __nv_bfloat16* src = qkv + (((size_t)s * T + m) * plane + pix) * c3;
          if (i < T) bulk_g2s(dst0 + (size_t)m * g.rs + qb, src + c, kvb, &bars[buf]);
          else bulk_g2s(dst0 + (size_t)m * g.rs, src, qb, &bars[buf]);
        }
      }
    }
  };
  // staging ring of g.nbuf buffers: unit i of this CTA lives in buffer i % nbuf; after unit i is
  // computed its buffer is refilled with unit i + nbuf (nbuf - 1 units land while one computes)
  int uq[kTaMaxBuf], sq[kTaMaxBuf], npq[kTaMaxBuf];
  uint32_t Mq[kTaMaxBuf];
  size_t pq[kTaMaxBuf];
  uint32_t Mn;
  size_t pixn;
  int sn, npxn;
  int un = ta_next(blockIdx.x, gridDim.x, units, pm, g, Mn, pixn, sn, npxn);
  for (int i = 0; i < g.nbuf; ++i) {
    uq[i] = un;
    if (un >= 0) {
      Mq[i] = Mn; pq[i] = pixn; sq[i] = sn; npq[i] = npxn;
      stage(i, sn, pixn, npxn, Mn, warp == 0, un % g.ngrp);
      un = ta_next(un + gridDim.x, gridDim.x, units, pm, g, Mn, pixn, sn, npxn);
    }
  }
  uint32_t phase = 0u;  // bit k = parity of buffer k
  int buf = 0;
  const int nwarps = blockDim.x >> 5;
  int tbase = 0;  // stream mode: index (mod nwarps) of the current unit's first task
  while (uq[buf] >= 0) {
    const uint32_t M = Mq[buf];
    const size_t pix = pq[buf];
    const int s = sq[buf], npx = npq[buf];
    mbar_wait(&bars[buf], (phase >> buf) & 1u);
    phase ^= 1u << buf;
    const uint32_t tk0 = smem_u32(rows + (size_t)buf * g.bstride);
    const int nq = __popc(M);
    const int mtiles = (nq + 15) >> 4;
    const int gq = lane >> 2, tq = lane & 3;        // mma fragment row group / thread-in-group
    const int mi = lane >> 3, ri = lane & 7;        // ldmatrix: matrix index / row within it
    const int NT = (T + 7) >> 3;                    // key tiles of 8 (<= 4)
    // frame of the lane-th listed query (one find-nth-set per lane per unit, shuffled below)
    const int lfr = lane < nq ? __fns(M, 0, lane + 1) : 0;
    const int ntask = g.hpg * mtiles;
    const int grp = uq[buf] % g.ngrp;
    int first = warp;
    if (g.stream) {
      first = warp - tbase;
      if (first < 0) first += nwarps;
      tbase = (tbase + npx * ntask) % nwarps;
    }
    for (int task2 = first; task2 < npx * ntask; task2 += nwarps) {
      const int pp = task2 / ntask, task = task2 - pp * ntask;  // pixel of the group, (head, m-tile)
      const uint32_t tk = tk0 + (uint32_t)(pp * 6 * cs);
      const int hd = task % g.hpg, mt = task / g.hpg;
      // ---- S = Q K^T on the tensor cores (bf16 products exact, fp32 accumulation)
      float S[4][4];
#pragma unroll
      for (int j = 0; j < 4; ++j) S[j][0] = S[j][1] = S[j][2] = S[j][3] = 0.f;
      // this lane's ldmatrix row for the Q tile: query (mi & 1) * 8 + ri of the m-tile
      const int qidx = mt * 16 + (mi & 1) * 8 + ri;
      const int qf = __shfl_sync(0xffffffffu, lfr, qidx < nq ? qidx : 0);
      const uint32_t qrow = tk + (uint32_t)qf * g.rs + (uint32_t)(hd * kHeadDim + (mi >> 1) * 8) * 2;
#pragma unroll
      for (int kk = 0; kk < kHeadDim / 16; ++kk) {
        uint32_t a[4];
        ldsm_x4(swz(qrow + kk * 32), a);
#pragma unroll
        for (int j = 0; j < 4; j += 2) {
          if (j >= NT) break;
          // matrices: (keys 8j.., dims lo), (keys 8j.., dims hi), (keys 8j+8.., lo), (.., hi)
          const int key = 8 * (j + (mi >> 1)) + ri;
          const uint32_t addr = key < T ? swz(tk + (uint32_t)key * g.rs + (uint32_t)(cs + hd * kHeadDim + kk * 16 +
                                                                                   (mi & 1) * 8) * 2)
                                        : zero_row;
          uint32_t bm[4];
          ldsm_x4(addr, bm);
          mma16816(S[j], a, bm[0], bm[1]);
          if (j + 1 < NT) mma16816(S[j + 1], a, bm[2], bm[3]);
        }
      }
      // ---- softmax over keys (row gq: S[j][0..1], row gq+8: S[j][2..3]); masked keys -> 0
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool ok = j < NT && 8 * j + 2 * tq + e < T;
          S[j][e] = ok ? S[j][e] * g.scale : -INFINITY;
          S[j][2 + e] = ok ? S[j][2 + e] * g.scale : -INFINITY;
          mx0 = fmaxf(mx0, S[j][e]);
          mx1 = fmaxf(mx1, S[j][2 + e]);
        }
      }
#pragma unroll
      for (int o2 = 1; o2 < 4; o2 <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o2));
      }
      float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          S[j][e] = __expf(S[j][e] - mx0);          // exp(-inf) = 0 for masked keys
          S[j][2 + e] = __expf(S[j][2 + e] - mx1);
          sum0 += S[j][e];
          sum1 += S[j][2 + e];
        }
      }
#pragma unroll
      for (int o2 = 1; o2 < 4; o2 <<= 1) {
        sum0 += __shfl_xor_sync(0xffffffffu, sum0, o2);
        sum1 += __shfl_xor_sync(0xffffffffu, sum1, o2);
      }
      // ---- O = P V: P (fp32) split into bf16 hi + lo parts (P - hi - lo ~ 2^-17 P), V bf16 exact
      float O[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) O[j][0] = O[j][1] = O[j][2] = O[j][3] = 0.f;
#pragma unroll
      for (int k2 = 0; k2 < 2; ++k2) {
        if (16 * k2 >= T) break;
        uint32_t ph[4], pl[4];
        const int t0 = 2 * k2, t1 = 2 * k2 + 1;
        const float p00 = S[t0][0], p01 = S[t0][1], p02 = S[t0][2], p03 = S[t0][3];
        const float p10 = t1 < 4 ? S[t1][0] : 0.f, p11 = t1 < 4 ? S[t1][1] : 0.f;
        const float p12 = t1 < 4 ? S[t1][2] : 0.f, p13 = t1 < 4 ? S[t1][3] : 0.f;
        ph[0] = pack_bf16(p00, p01); ph[1] = pack_bf16(p02, p03);
        ph[2] = pack_bf16(p10, p11); ph[3] = pack_bf16(p12, p13);
        pl[0] = pack_bf16(p00 - bf16_lo(ph[0]), p01 - bf16_hi(ph[0]));
        pl[1] = pack_bf16(p02 - bf16_lo(ph[1]), p03 - bf16_hi(ph[1]));
        pl[2] = pack_bf16(p10 - bf16_lo(ph[2]), p11 - bf16_hi(ph[2]));
        pl[3] = pack_bf16(p12 - bf16_lo(ph[3]), p13 - bf16_hi(ph[3]));
        // V^T fragments via ldmatrix.trans: matrices (keys lo 8, dims lo), (keys hi 8, dims lo),
        // (keys lo, dims hi), (keys hi, dims hi) of a 16-key x 16-dim slab
        const int key = 16 * k2 + (mi & 1) * 8 + ri;
#pragma unroll
        for (int jn = 0; jn < 4; ++jn) {
          const uint32_t addr = key < T ? swz(tk + (uint32_t)key * g.rs +
                                                  (uint32_t)(2 * cs + hd * kHeadDim + jn * 16 + (mi >> 1) * 8) * 2)
                                        : zero_row;
          uint32_t bv[4];
          ldsm_x4_t(addr, bv);
          mma16816(O[2 * jn], ph, bv[0], bv[1]);
          mma16816(O[2 * jn], pl, bv[0], bv[1]);
          mma16816(O[2 * jn + 1], ph, bv[2], bv[3]);
          mma16816(O[2 * jn + 1], pl, bv[2], bv[3]);
        }
      }
      const float inv0 = 1.f / sum0, inv1 = 1.f / sum1;
      const int q0 = mt * 16 + gq, q1 = q0 + 8;
      const int f0 = __shfl_sync(0xffffffffu, lfr, q0 & 31), f1 = __shfl_sync(0xffffffffu, lfr, q1 & 31);
      if (q0 < nq) {
        __nv_bfloat16* dst = o + (((size_t)s * T + f0) * plane + pix + pp) * c + (grp * g.hpg + hd) * kHeadDim + 2 * tq;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint32_t*>(dst + 8 * j) = pack_bf16(O[j][0] * inv0, O[j][1] * inv0);
      }
      if (q1 < nq) {
        __nv_bfloat16* dst = o + (((size_t)s * T + f1) * plane + pix + pp) * c + (grp * g.hpg + hd) * kHeadDim + 2 * tq;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint32_t*>(dst + 8 * j) = pack_bf16(O[j][2] * inv1, O[j][3] * inv1);
      }
    }
    bool me = warp == 0;
    if (g.stream) {
      // every warp passes every unit (waiting for it to land even without a task in it, so no
      // warp runs a ring lap ahead of the loads); the last one out restages the buffer
      __syncwarp();
      int last = 0;
      if (lane == 0) {
        __threadfence_block();  // this warp's reads of the buffer precede its arrival
        last = atomicAdd(&done[buf], 1) == nwarps - 1;
        if (last) {
          done[buf] = 0;
          __threadfence_block();
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
      }
      me = __shfl_sync(0xffffffffu, last, 0) != 0;
    } else {
      __syncthreads();  // every warp is done with this buffer before it is staged again
    }
    uq[buf] = un;
    if (un >= 0) {
      Mq[buf] = Mn; pq[buf] = pixn; sq[buf] = sn; npq[buf] = npxn;
      stage(buf, sn, pixn, npxn, Mn, me, un % g.ngrp);
      un = ta_next(un + gridDim.x, gridDim.x, units, pm, g, Mn, pixn, sn, npxn);
    }
    buf = buf + 1 == g.nbuf ? 0 : buf + 1;
  }
}

static size_t ta_row(int c, int ppu = 1) { return (size_t)ppu * 6 * c + 16; }
static size_t ta_smem(int c, int T, int nbuf, int ppu = 1) { return 128 + (size_t)nbuf * T * ta_row(c, ppu); }
// tensor mode: 1024-aligned buffers of T unpadded 6C-byte rows (+1024 alignment slack)
static size_t ta_tbuf(int c, int T) { return ((size_t)T * 6 * c + 1023) / 1024 * 1024; }
static size_t ta_smem_t(int c, int T, int nbuf) { return 128 + 1024 + (size_t)nbuf * ta_tbuf(c, T); }

typedef CUresult (*PFN_taEncodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                        const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                        const cuuint32_t*, CUtensorMapInterleave,
                                        CUtensorMapSwizzle, CUtensorMapL2promotion,
                                        CUtensorMapFloatOOBfill);
static PFN_taEncodeTiled_t ta_encode_tiled() {
  static PFN_taEncodeTiled_t fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_taEncodeTiled_t>(ptr);
  }
  return fn;
}

}  // namespace sphinx

using namespace sphinx;

extern "C" size_t sphinx_temporal_attention_workspace_size(int32_t n, int32_t h, int32_t w,
                                                            int32_t frames_per_seq, int32_t block) {
  if (n <= 0 || h <= 0 || w <= 0 || block <= 0 || frames_per_seq <= 0 || n % frames_per_seq) return 0;
  return (size_t)(n / frames_per_seq) * cdiv(h, block) * cdiv(w, block) * sizeof(uint32_t);
}

static sphinx_status temporal_attention_impl(const void* qkv, void* o, int32_t n, int32_t h, int32_t w,
                                             int32_t c, int32_t heads, int32_t frames_per_seq,
                                             int32_t block, const int32_t* block_ids,
                                             const int32_t* count, int32_t capacity, void* workspace,
                                             size_t workspace_bytes, int32_t head_group,
                                             sphinx_stream_t stream) {
  if (!qkv || !o || !block_ids || !count || !workspace || qkv == o) return SPHINX_ERR_INVALID_ARGUMENT;
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || heads <= 0 || block <= 0 || capacity < 0 ||
      frames_per_seq <= 0 || n % frames_per_seq || c % heads)
    return SPHINX_ERR_INVALID_ARGUMENT;
  const int T = frames_per_seq;
  if ((int64_t)capacity > (int64_t)n * cdiv(h, block) * cdiv(w, block)) return SPHINX_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < sphinx_temporal_attention_workspace_size(n, h, w, T, block))
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (c / heads != kHeadDim || T > 32 || block > 64 || ta_smem(c, T, 1) > 227 * 1024 ||
      (long long)n * cdiv(h, block) * cdiv(w, block) * block * block >= (1ll << 31))
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
  g.scale = 1.f / sqrtf((float)kHeadDim);
  // One pixel per unit.  Staging (tools/ta_ab.py, 21 frames at 25% clustered density):
  //  * the double-buffered ring fits twice per SM (level 0): two CTAs of 8 warps, task stream
  //    (62 us; 66 with a CTA barrier per unit; 84 single-buffered; one CTA with a 3-5 deep ring
  //    93-122 us: two CTAs interleaving units beat a deeper ring);
  //  * it fits once (level 1): one CTA of 16 warps, task stream (39 us; 42 for two single-buffered
  //    CTAs of 8 warps);
  //  * it does not fit (level 2): one single-buffered CTA of 16 warps with a barrier per unit
  //    (26.7 us; 27.4 as a task stream, 28.7 with 8 warps).
  // SPHINX_TA_PPU=2 stages two x-adjacent pixels per unit with one bulk copy per frame:
  // measured slower at level 0 (90 vs 65 us: the larger buffers halve the resident CTAs).
  g.ppu = 1;
  g.nbuf = ta_smem(c, T, 2) <= 227 * 1024 ? 2 : 1;
  g.stream = g.nbuf == 2 ? 1 : 0;
#ifdef SPHINX_DEV_KNOBS  // measured-slower staging variants: dev builds only
  if (const char* env = getenv("SPHINX_TA_NBUF")) {
    const int nb = atoi(env);
    if (nb >= 1 && nb <= kTaMaxBuf && ta_smem(c, T, nb) <= 227 * 1024) g.nbuf = nb;
  }
  if (const char* env = getenv("SPHINX_TA_PPU"))
    if (atoi(env) == 2 && block % 2 == 0 && ta_smem(c, T, g.nbuf, 2) <= 227 * 1024) g.ppu = 2;
  g.kv_only = 0;
  if (const char* env = getenv("SPHINX_TA_KVONLY")) g.kv_only = atoi(env) != 0;
  if (const char* env = getenv("SPHINX_TA_STREAM")) g.stream = atoi(env) != 0;
#else
  g.kv_only = 0;
#endif
  g.rs = (uint32_t)ta_row(c, g.ppu);
  g.bstride = (uint32_t)((size_t)T * g.rs);
  // tensor mode: one 4-D TMA copy per unit instead of T bulk copies (the staging is bulk-op-rate
  // bound).  Default with the double-buffered ring (levels 0/1: 65.5 -> 55.5 and 40.1 -> 35.5 us
  // same-box); single-buffered (level 2) it measured slower (27.3 -> 29.7 us).
  // SPHINX_TA_TMAP=0/1 overrides.
  bool want_t = g.nbuf == 2;
#ifdef SPHINX_DEV_KNOBS
  if (const char* env = getenv("SPHINX_TA_TMAP")) want_t = atoi(env) != 0;
#endif
  g.tmode = want_t && g.ppu == 1 && !g.kv_only && (3 * c) % 64 == 0 && 3 * c / 64 <= 256 &&
            ta_smem_t(c, T, g.nbuf) <= 227 * 1024;
  // head groups (SPHINX_TA_HGROUP=k heads per unit, tensor mode): a unit stages the q|k|v slices of
  // k heads only, so wide levels get the small double-buffered ring of level 0
  // Default: when even the double-buffered ring of all heads does not fit (level 2), the largest
  // group whose ring fits twice per SM (same box, level 2: 27.9 -> 21.2 us with 5-head groups;
  // 10-head groups 22.1, 4-head 24.4; level 1 unchanged within noise, so it keeps all heads).
  g.hpg = heads;
  g.ngrp = 1;
  int want_k = 0;
  if (g.nbuf == 1 && g.ppu == 1 && !g.kv_only)
    for (int k = heads - 1; k >= 1; --k)
      if (heads % k == 0 && ta_smem_t(k * kHeadDim, T, 2) <= 113 * 1024) {
        want_k = k;
        break;
      }
  if (head_group > 0) want_k = head_group;  // caller override (tests); heads = no grouping
  {
    const int k = want_k;
    if (k >= 1 && k < heads && heads % k == 0 && g.ppu == 1 && !g.kv_only &&
        (long long)n_seq * hb * wb * block * block * (heads / k) < (1ll << 31)) {
      g.hpg = k;
      g.ngrp = heads / k;
      g.nbuf = ta_smem_t(k * kHeadDim, T, 2) <= 227 * 1024 ? 2 : 1;
      g.stream = g.nbuf == 2 ? 1 : 0;
      g.tmode = 1;
    }
  }
  const int cs = g.hpg * kHeadDim;
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  if (g.tmode) {
    g.rs = (uint32_t)(6 * cs);
    g.bstride = (uint32_t)ta_tbuf(cs, T);
    PFN_taEncodeTiled_t enc = ta_encode_tiled();
    if (!enc) return SPHINX_ERR_CUDA;
    // 5-D: 64-element rows x C/64 x {q, k, v} x pixels x frames; box = one head group's rows
    const cuuint64_t dims[5] = {64, (cuuint64_t)(c / 64), 3, (cuuint64_t)h * w, (cuuint64_t)n};
    const cuuint64_t strides[4] = {128, (cuuint64_t)c * 2, (cuuint64_t)(3 * c) * 2,
                                   (cuuint64_t)h * w * 3 * c * 2};
    const cuuint32_t box[5] = {64, (cuuint32_t)g.hpg, 3, 1, (cuuint32_t)T};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(qkv), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return SPHINX_ERR_UNSUPPORTED;
  }
  // resident CTAs per SM by shared memory; the frame masks go to shared memory when that does
  // not lower it
  auto fit = [](size_t bytes) {
    const int k = (int)((228 * 1024) / (bytes + 1024));
    return k < 1 ? 1 : (k > 8 ? 8 : k);
  };
  const size_t pm_bytes = (size_t)n_seq * hb * wb * sizeof(uint32_t);
  const size_t ring = g.tmode ? ta_smem_t(cs, T, g.nbuf) : ta_smem(c, T, g.nbuf, g.ppu);
  g.pm_smem = pm_bytes <= 8192 && ring + pm_bytes <= 227 * 1024 && fit(ring + pm_bytes) == fit(ring);
#ifdef SPHINX_DEV_KNOBS
  if (const char* env = getenv("SPHINX_TA_PMSMEM")) g.pm_smem = g.pm_smem && atoi(env) != 0;
#endif
  const size_t smem = ring + (g.pm_smem ? pm_bytes : 0);
  int per_sm = fit(smem);
  // one resident CTA per SM (the ring does not fit twice): 16 warps; two CTAs of 8 otherwise
  int threads = per_sm == 1 ? kTaMaxThreads : kTaThreads;
#ifdef SPHINX_DEV_KNOBS
  if (const char* env = getenv("SPHINX_TA_THREADS")) threads = atoi(env) == 512 ? 512 : kTaThreads;
#endif
  if (per_sm > 65536 / (threads * 128)) per_sm = 65536 / (threads * 128);  // <= 128 regs/thread
  e = cudaFuncSetAttribute(ta_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return cuda_fail(e);
  const long long units = (long long)n_seq * hb * wb * block * block / g.ppu * g.ngrp;
  const long long cap = (long long)sms * per_sm;
  const int grid = (int)(units < cap ? units : cap);
  e = launch_k(ta_attn_kernel, dim3(grid), dim3(threads), smem, s, tm, static_cast<const __nv_bfloat16*>(qkv),
               static_cast<__nv_bfloat16*>(o), static_cast<const uint32_t*>(posmask), g);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

extern "C" sphinx_status sphinx_temporal_attention(const void* qkv, void* o, int32_t n, int32_t h,
                                                   int32_t w, int32_t c, int32_t heads,
                                                   int32_t frames_per_seq, int32_t block,
                                                   const int32_t* block_ids, const int32_t* count,
                                                   int32_t capacity, void* workspace,
                                                   size_t workspace_bytes, sphinx_stream_t stream) {
  return temporal_attention_impl(qkv, o, n, h, w, c, heads, frames_per_seq, block, block_ids, count,
                                 capacity, workspace, workspace_bytes, 0, stream);
}

extern "C" sphinx_status sphinx_temporal_attention_ex(const void* qkv, void* o, int32_t n, int32_t h,
                                                      int32_t w, int32_t c, int32_t heads,
                                                      int32_t frames_per_seq, int32_t block,
                                                      const int32_t* block_ids, const int32_t* count,
                                                      int32_t capacity, void* workspace,
                                                      size_t workspace_bytes, int32_t head_group,
                                                      sphinx_stream_t stream) {
  if (head_group < 0 || (head_group > 0 && (heads % head_group))) return SPHINX_ERR_INVALID_ARGUMENT;
  return temporal_attention_impl(qkv, o, n, h, w, c, heads, frames_per_seq, block, block_ids, count,
                                 capacity, workspace, workspace_bytes, head_group, stream);
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
