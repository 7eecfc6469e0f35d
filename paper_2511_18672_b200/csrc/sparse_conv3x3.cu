// sparse_conv3x3.cu — step (4): halo gather + 3x3 implicit GEMM on listed blocks,
// tcgen05 tensor cores with TMEM accumulators, TMA operand staging (sm_100a).
//
// "tiles the feature maps into blocks ... enables batched convolution over
// selected blocks, amortizing memory and compute overhead while preserving spatial
// correlation across boundaries"; P:333 spatial ResNet layers act per frame.
//
// GEMM view:  M = pixels of listed blocks (b*b per block),
// N = C_out, K = 9 * C_in ordered (tap, channel) to match the OHWI weights.
//  - A tile (128 x 64): 128 / b^2 blocks; for every (tap, 64-channel chunk) each
//    block's rows are ONE 4-D TMA box {64 ch, b, b, 1} of the NHWC map at the
//    tap-shifted origin (bx*b+dx-1, by*b+dy-1).  The box lands as b^2 rows of
//    128 B in the canonical K-major SWIZZLE_128B layout, and TMA's out-of-bound
//    zero fill IS the conv's zero padding (image borders) and the ragged edge.
//  - B tile (BN x 64): 3-D TMA box {64 ch, 1 tap, BN} of W viewed as [C_out][9][C_in].
//  - One elected thread issues tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN,
//    K=16) x 4 per stage into a TMEM accumulator; tcgen05.commit releases the smem
//    stage (empty barrier) and, after the last K step, hands the accumulator to the
//    epilogue.  Two TMEM accumulators (2*BN columns) let the epilogue of tile i
//    overlap the main loop of tile i+1.
//  - Epilogue: 8 warps (two per TMEM lane quarter, alternate 32-column chunks) tcgen05.ld
//    their 32 TMEM lanes (= 32 pixels), add bias (+ residual), and store straight into the
//    full-resolution NHWC output at each pixel's own position (the scatter of computed
//    blocks is fused; unlisted pixels untouched).
//  - Persistent CTAs (grid = #SMs) walk the tile list in a static stride; the tile
//    count comes from the device-side block count, so no host synchronisation.
//  Warp roles (352 threads): w0 weight (B) TMA producer, w6 halo (A) TMA producer (halo
//  mode), w1 TMEM allocator + MMA issuer, w2..w5 + w7..w10 epilogue.  The fused-GN variant
//  (NORM) keeps w2..w5 as epilogue and uses w7..w14 as GroupNorm+SiLU transform warps.
//  (The per-tap / halo / split-K / stream-K / edge-class details are documented inline and in
//  DESIGN.md section 6.4.)
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace sphinx {

constexpr int kBM = 128;          // MMA M: pixels per tile
constexpr int kBK = 64;           // channels per K chunk: 128 B rows, SWIZZLE_128B
constexpr int kStageA = kBM * kBK * 2;  // 16 KB
constexpr int kThreads = 224;
constexpr int kAWarp = 6;  // halo mode: the halo (A) producer warp when the producers are split
constexpr int kXWarp = 7;   // NORM (fused GroupNorm+SiLU) kernels: first transform warp
constexpr int kXThreads = 256;  // transform threads (8 warps)
constexpr int kThreadsNorm = kThreads + kXThreads;
// non-NORM kernels: 4 more epilogue warps (7..10) split the accumulator columns with warps 2..5
// (same TMEM lane quarters, warp & 3), halving the TMEM drain and the split-K park / reduce
constexpr int kThreadsEpi8 = kThreads + 128;

#ifdef SPHINX_TRACE
// Dev-only timeline trace (libsphinx_trace.so): globaltimer stamps per CTA of one launch.
// slots: 0 entry, 1 after pdl_wait, 2 first MMA, 3 last MMA commit, 4 epilogue done, 5 exit,
//        6 chunks issued by the MMA warp, 7 B producer done, 8 first A issued, 9 first B issued,
//        10 first A full (MMA), 11 last accumulator ready (epilogue), 12 epilogue tiles,
//        13 sum of TMEM-drain durations, 14 last TMEM-drain duration (ns), 15 setup done,
//        16 split partial parked, 17 split rendezvous done, 18 split reduction done, 19 ns.
__device__ unsigned long long g_conv_trace[1024 * 24];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define CONV_TRACE(k, v) \
  do {                   \
    if (p.trace) g_conv_trace[blockIdx.x * 24 + (k)] = (v); \
  } while (0)
// accumulate the time spent in `stmt` (a barrier wait) into slot k (20: operand full, 21: accumulator
// empty, 22: A-resident region full, 23: epilogue waiting for the accumulator)
// (only with dbg bit 8: the global read-modify-write per wait perturbs the loop it measures)
#define TWAIT(k, stmt)                                                                \
  do {                                                                                \
    const bool _on = p.trace && (p.dbg & 8);                                          \
    const unsigned long long _t0 = _on ? gtimer() : 0ull;                             \
    stmt;                                                                             \
    if (_on) g_conv_trace[blockIdx.x * 24 + (k)] += gtimer() - _t0;                   \
  } while (0)
#else
#define CONV_TRACE(k, v) \
  do {                   \
  } while (0)
#define TWAIT(k, stmt) \
  do {                 \
    stmt;              \
  } while (0)
#endif

struct ConvParams {
  const int32_t* ids;
  const int32_t* count;
  const float* bias;
  void* y;
  const __nv_bfloat16* res;  // NEXT-3: bf16 NHWC residual added in the epilogue (identity skip), or NULL
  const float2* norm_tab;    // NEXT-3 fused GN+SiLU: [N][c_in] (scale, shift), a = SiLU(x*scale+shift)
  int cin;
  int y_f32;
  int h, w, cout, b, hb, wb;
  int kc;         // 64-channel chunks per tap
  int taps;       // 9 = 3x3 conv; 1 = pointwise (1x1) projection (NEXT-4), per-tap path only
  int n_tiles_n;  // tiles along C_out
  int n_last;     // width of the last C_out tile (== BN: C_out is tiled in equal widths)
  int ring_bytes; // operand-ring bytes of the launched configuration (split-K staging bound)
  int tma_y;      // per-tap mode, bf16 y: the epilogue stages each 32-column chunk in shared memory
                  // and writes it with one TMA tensor store per block (tmY)
  int bpt;        // blocks per 128-row tile = 128 / b^2
  // split-K workspace (NULL = never split): per-(tile, split) fp32 partial tiles and one
  // arrival counter per (tile, CTA of the pair); counters are zero between launches.
  float* ws_part;
  int32_t* ws_cnt;
  int ws_slots;    // partial-tile slots available
  int ws_tiles;    // counter capacity in tiles
  int halo;        // 1: halo-staged A operand (b = 8)
  // edge-class packing (halo mode, H % 8 or W % 8 != 0): the plan kernel writes the list
  // partitioned into full / bottom-edge / right-edge blocks (each ascending) and the counts
  const int32_t* plan_ids;   // [capacity] or NULL (no plan: every block is "full")
  const int32_t* plan_meta;  // [3] = {n_full, n_bottom, n_right}
  int rb, cr;                // valid rows of bottom-edge blocks, valid cols of right-edge blocks
  int bpt_b, bpt_r;          // blocks per CTA tile of the two edge classes
  int trace;         // SPHINX_TRACE builds: record this launch's timeline
  int early_input;   // x (and the list) predate the preceding kernel: the halo producer does not
                     // wait either -- only the epilogue does (its stores, and kernel completion
                     // after the predecessor's, keep the stream order)
  int early_list;    // ids/count/plan were written before the immediately preceding kernel: read
                     // them (and start the weight loads) before griddepcontrol.wait; only the
                     // halo producer and the epilogue wait for the predecessor
  int dbg;           // SPHINX_TRACE builds: 1 = skip epilogue global stores, 2 = skip bias
  int allow_streamk; // halo mode may use stream-K when it shortens the makespan
};

// Split-K factor chosen ON THE DEVICE from the device-side tile count (CUDA-graph safe).
// Splitting is used only when all (tile, split) units fit in ONE round of the co-resident
// persistent grid (units <= clusters), which makes the split CTAs' rendezvous safe; among
// those S, minimise ksteps/S + kRedCost (the fixed cost of the partial-tile exchange).
// Every CTA evaluates the same pure function of the count.
__device__ __forceinline__ int choose_split(int tiles, int n_clusters, int ksteps, int max_split,
                                           const ConvParams& p) {
  constexpr int kMinSteps = 4, kRedCost = 6;
  const int kMaxSplit = max_split < 16 ? max_split : 16;
  if (p.ws_part == nullptr || tiles <= 0 || tiles > p.ws_tiles || tiles * 2 > n_clusters) return 1;
  int best = 1, best_cost = ksteps * 1000;
  for (int sk = 2; sk <= kMaxSplit; ++sk) {
    if (ksteps / sk < kMinSteps || tiles * sk > n_clusters || tiles * sk > p.ws_slots) break;
    // the reducing unit stages sk column slices of every part in the operand ring
    if ((long long)sk * ((p.n_last / 8 + sk - 1) / sk) * 8 * kBM * 4 > p.ring_bytes) break;
    const int cost = ksteps * 1000 / sk + kRedCost * 1000;
    if (cost < best_cost) {
      best_cost = cost;
      best = sk;
    }
  }
  return best;
}

// Shared-memory plan.  Per-tap mode (HALO = false): a ring of kStages stages, each the A tile
// of one (tap, 64-ch chunk) [128 rows x 128 B] plus its B tile [BN/CG rows x 128 B].
// Halo mode (HALO = true, b = 8): an A ring of kANum slots, each holding the (b+2)^2 halos of
// the CTA's blocks for one 64-ch chunk, stored densely as halo lines of 10 px x 128 B
// (1280 B) ordered [line][block]; the 8-row UMMA core groups sit at stride 1280 B and a tap
// (dy,dx) is the start shift dy*bpt*1280 + dx*128.  Valid because the SW128 XOR phase is
// derived from absolute smem address bits (measured: base-offset field 0), exactly as TMA
// writes it.  Plus a B ring of kBNum (tap, chunk) weight tiles.
template <int BN, int CG, bool HALO, bool EDGE = false, bool NORM = false>
struct ConvCfg {
  static constexpr int kBNc = BN / CG;  // B rows (output channels) held by this CTA
  static constexpr int kStageB = kBNc * kBK * 2;
  static constexpr int kStageBytes = kStageA + kStageB;
  // barriers + split-K pixel table + per-accumulator bias slices (2 x 256 fp32)
  // NORM: + the per-chunk (scale, shift) table [8 blocks][8 groups][20 floats] + halo row info
  static constexpr int kBarBytes = 512 + kBM * 8 + 2 * 256 * 4 + (NORM ? 8 * 8 * 20 * 4 + 512 : 0);
  static constexpr int kMaxSmem = 232448;          // 227 KB opt-in per CTA
  static constexpr int kAvail = kMaxSmem - 1024 - kBarBytes;
  // per-tap mode: + the TMA-store staging of the epilogue (8 warps x 2 buffers x 32 rows x 64 B)
  static constexpr int kStoreBytes = HALO ? 0 : 2 * 2 * kBM * 64;
  static constexpr int kStagesFit = (kAvail - kStoreBytes) / kStageBytes;
  static constexpr int kStages = kStagesFit > 8 ? 8 : kStagesFit;
  // halo mode (BPT = 2 blocks of 8x8)
  static constexpr int kHaloRow = 1280;
  // full-block tiles: 10 lines x 2 blocks (+ the UMMA over-read of padding groups stays inside);
  // edge tiles up to 8 blocks: 32 line slots
  static constexpr int kASlot = (EDGE ? 32 : 20) * kHaloRow;
  // edge kernels at >= 128 B rows per CTA keep 2 halo slots so the weight ring stays deep
  static constexpr int kANum = (EDGE && kBNc >= 128) ? 2 : 3;
  static constexpr int kBNumFit = (kAvail - kANum * kASlot - 1024) / kStageB;
  static constexpr int kBNum = kBNumFit > 16 ? 16 : kBNumFit;
  // halo A ring padded to 1 KB so the B ring (SW128, 1024-B atoms) stays aligned
  static constexpr int kARing = (kANum * kASlot + 1023) / 1024 * 1024;
  static constexpr int kRingBytes = HALO ? kARing + kBNum * kStageB : kStages * kStageBytes;
  static constexpr int kNumBars = HALO ? kANum + kBNum : kStages;
  static constexpr uint32_t kTmemCols = (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                        : (2 * BN <= 256) ? 256 : 512;
  static constexpr int kSmem = 1024 + kRingBytes + kStoreBytes + kBarBytes;
  static_assert(HALO ? kBNum >= 3 : kStages >= 3, "pipeline too shallow");
  static_assert((2 * kNumBars + 5 + 3) * 8 <= 512, "barrier area");
  // stream-K owner staging: 2 buffers x kMaxParts parts x (32 cols x 128 rows fp32)
  static constexpr int kMaxParts = (kRingBytes / (2 * 32 * kBM * 4)) < 6 ? (kRingBytes / (2 * 32 * kBM * 4)) : 6;
  static_assert(kRingBytes >= (kBM + 16) * BN * 4, "split-K staging must fit the ring");
};

__device__ __forceinline__ void decode_block(int id, int hb, int wb, int& n, int& by, int& bx) {
  n = id / (hb * wb);
  const int r = id - n * hb * wb;
  by = r / wb;
  bx = r - by * wb;
}

// NORM hand-off: transform threads publish their generic-proxy smem writes to the tensor core
// (async proxy) and to the leader CTA's MMA thread (cluster scope).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_release_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Explicit shared-space accesses for the transform warps (pointers derived from the aligned
// dynamic-smem base otherwise compile to generic LD.E/ST.E).
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, const uint4& v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void sts64f(uint32_t a, float x, float y) {
  asm volatile("st.shared.v2.f32 [%0], {%1,%2};" ::"r"(a), "f"(x), "f"(y) : "memory");
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// + residual[pix + co + i] for i < NV (bf16, same NHWC layout as y), 16-byte loads.
template <int NV>
__device__ __forceinline__ void add_residual(const ConvParams& p, size_t pix, int co, float* v) {
  const __nv_bfloat16* rp = p.res + pix + co;
#pragma unroll
  for (int g = 0; g < NV; g += 8) {
    if (co + g < p.cout) {
      const uint4 r = __ldg(reinterpret_cast<const uint4*>(rp + g));
      const uint32_t w4[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[g + 2 * k] += __uint_as_float(w4[k] << 16);
        v[g + 2 * k + 1] += __uint_as_float(w4[k] & 0xffff0000u);
      }
    }
  }
}

// 32 consecutive output channels [co, co+32) of one pixel: + bias (+ residual), fp32 or bf16 store.
__device__ __forceinline__ void store_row_chunk(const ConvParams& p, size_t pix, int co, float (&v)[32],
                                                const float* sb) {
  // sb: this chunk's 32 bias values in shared memory (zero-padded): broadcast LDS.128, no
  // predicated global loads queued behind the previous chunk's stores
  if (sb) {  // (nullptr: bias already added)
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      const float4 b4 = *reinterpret_cast<const float4*>(sb + i);
      v[i] += b4.x;
      v[i + 1] += b4.y;
      v[i + 2] += b4.z;
      v[i + 3] += b4.w;
    }
  }
  if (p.res) add_residual<32>(p, pix, co, v);
#ifdef SPHINX_TRACE
  if (p.dbg & 1) {
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += v[i];
    if (acc == 12345.678f) static_cast<float*>(p.y)[pix] = acc;  // keep the values live
    return;
  }
#endif
  if (p.y_f32) {
    float* yp = static_cast<float*>(p.y) + pix + co;
#pragma unroll
    for (int g = 0; g < 32; g += 4)
      if (co + g < p.cout)
        *reinterpret_cast<float4*>(yp + g) = make_float4(v[g], v[g + 1], v[g + 2], v[g + 3]);
  } else {
    __nv_bfloat16* yp = static_cast<__nv_bfloat16*>(p.y) + pix + co;
#pragma unroll
    for (int g = 0; g < 32; g += 8) {
      if (co + g < p.cout) {
        uint4 pk;
        __nv_bfloat162 t0 = __floats2bfloat162_rn(v[g + 0], v[g + 1]);
        __nv_bfloat162 t1 = __floats2bfloat162_rn(v[g + 2], v[g + 3]);
        __nv_bfloat162 t2 = __floats2bfloat162_rn(v[g + 4], v[g + 5]);
        __nv_bfloat162 t3 = __floats2bfloat162_rn(v[g + 6], v[g + 7]);
        pk.x = *reinterpret_cast<uint32_t*>(&t0);
        pk.y = *reinterpret_cast<uint32_t*>(&t1);
        pk.z = *reinterpret_cast<uint32_t*>(&t2);
        pk.w = *reinterpret_cast<uint32_t*>(&t3);
        *reinterpret_cast<uint4*>(yp + g) = pk;
      }
    }
  }
}

// Work unit u -> (tile, k-split index, splits of that tile, split-tile slot).
struct Unit {
  int t, sk, ns, slot;
};
__device__ __forceinline__ Unit decode_unit(int u, int n_full, int nsplit) {
  Unit r;
  if (u < n_full) {
    r.t = u; r.sk = 0; r.ns = 1; r.slot = 0;
  } else {
    const int v = u - n_full;
    r.slot = v / nsplit;
    r.t = n_full + r.slot;
    r.sk = v - r.slot * nsplit;
    r.ns = nsplit;
  }
  return r;
}

// A CTA's work as a sequence of segments (tile, chunk range [k0, k1), role).
//  mode 0: units u = cluster + i * clusters: unsplit tiles (FULL) then the tail split units
//          (SPLIT: co-resident rendezvous, distributed fixed-order reduction).
//  mode 1: stream-K (halo mode): cluster c owns the contiguous range [c*W/C, (c+1)*W/C) of
//          the flattened (tile, chunk) space, W = tiles * KC.  A tile cut by range boundaries
//          has one OWNER (the cluster holding its chunk 0; that segment is the LAST of the
//          owner's range) and PART contributors (each such segment is the FIRST of its range):
//          parts park fp32 partials and signal, never wait; the owner waits at its very end,
//          adds the parts in cluster order (deterministic) and stores.
enum SegRole { kFull = 0, kSplit = 1, kPart = 2, kOwner = 3 };
struct Seg {
  int t, k0, k1, role, sk, ns, slot;
};
struct SegIter {
  int mode, cluster, C, total, n_full, nsplit, kc;
  long long x, hi, W;
  __device__ __forceinline__ bool get(Seg& g) {
    if (mode == 0) {
      if (x >= total) return false;
      const Unit U = decode_unit((int)x, n_full, nsplit);
      g.t = U.t; g.sk = U.sk; g.ns = U.ns; g.slot = U.slot;
      g.k0 = U.sk * kc / U.ns;
      g.k1 = (U.sk + 1) * kc / U.ns;
      g.role = U.ns > 1 ? kSplit : kFull;
      return true;
    }
    if (x >= hi) return false;
    g.t = (int)(x / kc);
    g.k0 = (int)(x - (long long)g.t * kc);
    g.k1 = (int)min((long long)kc, g.k0 + (hi - x));
    g.role = (g.k0 == 0 && g.k1 == kc) ? kFull : (g.k0 == 0 ? kOwner : kPart);
    g.sk = 0; g.ns = 1; g.slot = cluster;
    return true;
  }
  __device__ __forceinline__ void next(const Seg& g) {
    if (mode == 0) x += C;
    else x += g.k1 - g.k0;
  }
};
// cluster whose stream-K range contains flattened position xx: max{c : floor(c*W/C) <= xx}
__device__ __forceinline__ int sk_cluster_of(long long xx, long long W, int C) {
  return (int)(((xx + 1) * C - 1) / W);
}

// Halo-mode tile geometry.  Tiles are enumerated class-major: full 8x8 blocks (2 per CTA,
// 10 halo rows each), then bottom-edge blocks (rb valid rows: rb+2 halo rows, up to 8 per
// CTA), then right-edge blocks (cr valid columns, loaded as rb+2... columns: the tile is
// "transposed", its 8-row UMMA groups run down a pixel column).
struct HaloTile {
  int bpt;       // blocks per CTA tile
  int lines;     // halo lines (rows, or columns if tr) loaded per block
  int tr;        // 1: column-oriented (right-edge class)
  int j0;        // index of this CTA's first block in the class list
  int nblk;      // blocks in the class
  const int32_t* list;
};

template <int CG>
__device__ __forceinline__ HaloTile halo_tile(int mt, int rank, int nF, int nB, const int32_t* list,
                                              int nR, const ConvParams& p) {
  HaloTile g;
  const int mF = (nF + 2 * CG - 1) / (2 * CG);
  const int mB = (nB + p.bpt_b * CG - 1) / (p.bpt_b * CG);
  int local;
  if (mt < mF) {
    g.bpt = 2; g.lines = 10; g.tr = 0; g.nblk = nF; g.list = list; local = mt;
  } else if (mt < mF + mB) {
    g.bpt = p.bpt_b; g.lines = p.rb + 2; g.tr = 0; g.nblk = nB; g.list = list + nF; local = mt - mF;
  } else {
    g.bpt = p.bpt_r; g.lines = p.cr + 2; g.tr = 1; g.nblk = nR; g.list = list + nF + nB;
    local = mt - mF - mB;
  }
  g.j0 = local * g.bpt * CG + rank * g.bpt;
  return g;
}

// Per-tap mode, bf16 y: one 32-column chunk of this WARP's 32 tile rows -> (bias already added,
// + residual) -> bf16 -> the warp's own staging buffer (32 rows of 64 B, SW64 swizzle), then one
// TMA tensor store per block quarter the warp covers (box {32 ch, BLK, 4, 1}: b = 8 -> rows
// [4(q&1), 4(q&1)+4) of block q/2; b = 4 -> two whole 4x4 blocks).  Out-of-image pixels of edge
// blocks and channels beyond C_out are clipped by the TMA unit; a short tile's padding blocks are
// skipped.  Warp-local: no barrier with the other epilogue warps.  Two buffers per warp: lane 0
// waits until the store that last read a buffer has read it.  Row r of the warp sits at byte
// r * 64 = (y, x) of the box layout (tile rows are block-major).
template <int BLK>
__device__ __forceinline__ void stage_chunk_tma_warp(const ConvParams& p, const CUtensorMap& tmY, uint8_t* buf,
                                                     int lane, int q, size_t pix, bool valid, int co,
                                                     float (&v)[32], int bn, int by, int bx, bool listed) {
  if (p.res && valid) add_residual<32>(p, pix, co, v);
  if (lane == 0) bulk_wait_group_read<1>();
  __syncwarp();
  const uint32_t base = smem_u32(buf) + (uint32_t)lane * 64u;
  const uint32_t sw = ((uint32_t)lane >> 1) & 3u;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint4 pk;
    __nv_bfloat162 t0 = __floats2bfloat162_rn(v[8 * g + 0], v[8 * g + 1]);
    __nv_bfloat162 t1 = __floats2bfloat162_rn(v[8 * g + 2], v[8 * g + 3]);
    __nv_bfloat162 t2 = __floats2bfloat162_rn(v[8 * g + 4], v[8 * g + 5]);
    __nv_bfloat162 t3 = __floats2bfloat162_rn(v[8 * g + 6], v[8 * g + 7]);
    pk.x = *reinterpret_cast<uint32_t*>(&t0);
    pk.y = *reinterpret_cast<uint32_t*>(&t1);
    pk.z = *reinterpret_cast<uint32_t*>(&t2);
    pk.w = *reinterpret_cast<uint32_t*>(&t3);
    sts128(base + (((uint32_t)g ^ sw) << 4), pk);
  }
  fence_proxy_async_shared();
  __syncwarp();
  // block coordinates of the (up to two) blocks of this warp's rows: lane 0's and lane 16's
  const int n1 = __shfl_sync(0xffffffffu, bn, 16), by1 = __shfl_sync(0xffffffffu, by, 16),
            bx1 = __shfl_sync(0xffffffffu, bx, 16);
  const bool l1 = __shfl_sync(0xffffffffu, listed ? 1 : 0, 16) != 0;
#ifdef SPHINX_TRACE
  if (p.dbg & 1) return;  // timing probe: stage, but issue no store
#endif
  if (lane == 0) {
    if constexpr (BLK == 8) {
      if (listed) tma_store_4d(&tmY, buf, co, bx * BLK, by * BLK + (q & 1) * 4, bn);
    } else {
      if (listed) tma_store_4d(&tmY, buf, co, bx * BLK, by * BLK, bn);
      if (l1) tma_store_4d(&tmY, buf + 1024, co, bx1 * BLK, by1 * BLK, n1);
    }
    bulk_commit_group();
  }
}

// CG = 1: one CTA per 128 x BN tile, tcgen05.mma.cta_group::1 (M = 128).
// CG = 2: a CTA pair (cluster of 2) per 256 x BN tile, tcgen05.mma.cta_group::2 (M = 256):
//   each CTA TMA-loads its own 128 rows of A and its half (BN/2 rows) of B; the leader
//   (rank 0) waits for both halves on its full barrier and issues the MMAs; commits are
//   multicast to both CTAs' barriers; each CTA's epilogue drains its own TMEM lanes and
//   arrives on the leader's accumulator-empty barrier.  B traffic per SM halves.
template <int BN, int CG, int BLK, bool HALO, bool EDGE, bool NORM>
__global__ void __launch_bounds__(NORM ? kThreadsNorm : kThreadsEpi8, 1)
    sparse_conv3x3_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                             const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmC,
                             const __grid_constant__ CUtensorMap tmY, const ConvParams p) {
  using Cfg = ConvCfg<BN, CG, HALO, EDGE, NORM>;
  static_assert(!NORM || HALO, "the fused GN+SiLU transform works on halo slots");
  static_assert(!EDGE || HALO, "edge packing is a halo-mode feature");
  static_assert(!HALO || BLK == 8, "halo staging needs 8x8 blocks");
  constexpr int S = Cfg::kStages;
  constexpr int NB = Cfg::kNumBars;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + (HALO ? Cfg::kARing : S * kStageA);
  uint8_t* s_store = smem + Cfg::kRingBytes;  // per-tap mode: [warp][buf][32 rows x 64 B], SW64
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kRingBytes + Cfg::kStoreBytes);
  uint64_t* empty = full + NB;
  uint64_t* tfull = empty + NB;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);
  uint64_t* red_bar = tempty + 2;  // [2] split-K / stream-K partial staging barriers
  // bias of the tile held in accumulator a: s_bias[a * 256 + column] (0 beyond cout / no bias)
  float* s_bias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 512 + kBM * 8);
  // NORM: per-chunk (scale, shift) of the tile's blocks [8 blocks][64 channels], then the
  // per-slot "halo landed" barriers (the A slots' full barriers become "transformed")
  // table row (block i, 8-channel group j) at s_tab + (i * 8 + j) * 20 floats: the 80-byte stride
  // puts the 8 groups a warp reads on disjoint bank quads (a 64-byte stride was 4-way conflicted)
  float* s_tab = s_bias + 2 * 256;
  uint8_t* s_rowinfo = reinterpret_cast<uint8_t*>(s_tab + 8 * 8 * 20);  // [<= 320 halo rows]: block or 255
  uint64_t* landed = tempty + 5;  // after tmem_slot (tempty + 4)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef SPHINX_TRACE
  if (threadIdx.x == 0) CONV_TRACE(0, gtimer());
#endif
  const int rank = CG == 2 ? (int)cluster_ctarank() : 0;
  const int cluster_id = blockIdx.x / CG, n_clusters = gridDim.x / CG;
  // early_list: the count and the plan's class counts are valid at launch, so their loads are
  // issued here and their latency hides under the setup below (asm with memory clobbers keeps the
  // compiler from sinking them)
  int e_count = 0, e_nF = 0, e_nB = 0, e_nR = 0;
  if (p.early_list) {
    e_count = __ldg(p.count);
    if (EDGE && p.plan_ids) {
      e_nF = __ldg(p.plan_meta + 0);
      e_nB = __ldg(p.plan_meta + 1);
      e_nR = __ldg(p.plan_meta + 2);
    }
  }
  // ---- setup that needs no upstream data (overlaps the previous kernel's tail under PDL)
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if constexpr (EDGE) tma_prefetch(&tmC);
    for (int s = 0; s < NB; ++s) {
      // NORM: an A slot is ready when BOTH CTAs' transform warps have arrived
      mbar_init(&full[s], (NORM && s < Cfg::kANum) ? CG : 1);
      mbar_init(&empty[s], 1);
    }
    if constexpr (NORM)
      for (int s = 0; s < Cfg::kANum; ++s) mbar_init(&landed[s], 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], (NORM ? 4 : 8) * CG);
    }
    mbar_init(&red_bar[0], 1);
    mbar_init(&red_bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc_cg2<Cfg::kTmemCols>(tmem_slot);
    else tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (!p.early_list) {
    pdl_wait();  // ids, count, plan and x are produced upstream
    pdl_trigger();
  }
  // early_list: the trigger follows the epilogue warps' griddepcontrol.wait (below), so a
  // dependent launched early has every kernel before this one complete -- its own early reads
  // of a list written two or more kernels back are then ordered transitively.
#ifdef SPHINX_TRACE
  if (threadIdx.x == 0) CONV_TRACE(1, gtimer());
#endif
  const int count = p.early_list ? e_count : *p.count;
  constexpr int BPT = kBM / (BLK * BLK);  // blocks per CTA tile (2 at b=8, 8 at b=4)
  constexpr int bb = BLK * BLK;
  const int bpt_pair = BPT * CG;  // blocks per (pair) tile
  // class counts (edge packing) -- without a plan every listed block is a "full" block
  const int32_t* list = (EDGE && p.plan_ids) ? p.plan_ids : p.ids;
  const bool planned = EDGE && p.plan_ids;
  const int nF = planned ? (p.early_list ? e_nF : __ldg(p.plan_meta + 0)) : count;
  const int nB = planned ? (p.early_list ? e_nB : __ldg(p.plan_meta + 1)) : 0;
  const int nR = planned ? (p.early_list ? e_nR : __ldg(p.plan_meta + 2)) : 0;
  const int m_tiles = HALO ? (nF + 2 * CG - 1) / (2 * CG) +
                                 (nB + p.bpt_b * CG - 1) / (p.bpt_b * CG) +
                                 (nR + p.bpt_r * CG - 1) / (p.bpt_r * CG)
                           : (count + bpt_pair - 1) / bpt_pair;
  const int tiles = m_tiles * p.n_tiles_n;
  const int ksteps = p.taps * p.kc;
  // halo mode splits K at 64-channel chunk boundaries (all 9 taps of a chunk stay together)
  // Full waves of tiles run unsplit; the last partial wave (rem tiles) is split nsplit ways
  // along K so that it fills one co-resident round (tail split-K).  Halo mode splits at
  // 64-channel chunk boundaries (the 9 taps of a chunk stay together).
  const int rem = tiles - (tiles / n_clusters) * n_clusters;
  const int nsplit = rem > 0 ? choose_split(rem, n_clusters, ksteps, HALO ? p.kc : 16, p) : 1;
  const int n_full = nsplit > 1 ? tiles - rem : tiles;
  const int total = n_full + (nsplit > 1 ? rem * nsplit : 0);  // work units
  // stream-K (halo mode) when it shortens the makespan (in chunk units, ~1 chunk of fixup)
  int sk_mode = 0;
  const long long Wk = (long long)tiles * p.kc;
  if (HALO && p.ws_part != nullptr && p.allow_streamk && Wk >= n_clusters &&
      n_clusters <= p.ws_slots && n_clusters * CG * 2 <= 1024) {
    const long long q = Wk / n_clusters;  // chunks per cluster (floor)
    // measured: the tail split's rendezvous + reduction costs ~2 chunks, stream-K's fixup ~1;
    // stream-K is taken only on a clear modelled win (it measured worse at model ties)
    const long long cost0 = nsplit > 1 ? (long long)(tiles / n_clusters) * p.kc + p.kc / nsplit + 2
                                       : (long long)((tiles + n_clusters - 1) / n_clusters) * p.kc;
    const long long cost1 = (Wk + n_clusters - 1) / n_clusters + 2;
    if ((cost1 < cost0 || p.allow_streamk == 2) && (p.kc + q - 1) / q <= Cfg::kMaxParts) sk_mode = 1;
  }
  SegIter it0;
  it0.mode = sk_mode; it0.cluster = cluster_id; it0.C = n_clusters; it0.total = total;
  it0.n_full = n_full; it0.nsplit = nsplit; it0.kc = p.kc; it0.W = Wk;
  it0.x = sk_mode ? (long long)cluster_id * Wk / n_clusters : cluster_id;
  it0.hi = sk_mode ? (long long)(cluster_id + 1) * Wk / n_clusters : 0;


#ifdef SPHINX_TRACE
  if (threadIdx.x == 0) CONV_TRACE(15, gtimer());
#endif
  if (warp == 0 || (HALO && warp == kAWarp)) {
    // early_list: the halo (A) producer -- also warp 0 when it issues A (per-tap path, or halo
    // mode without split producers) -- waits for the predecessor; the weight-only producer not
    if (p.early_list && !p.early_input && (warp == kAWarp || !HALO)) pdl_wait();
    // ===================== TMA producers (both CTAs) =====================
    // halo mode: warp 0 issues the weight (B) tiles and warp kAWarp the halos (A), so the two
    // streams of TMA issues overlap (a single issuing thread caps the per-SM TMA op rate)
    if (elect_one()) {
      const uint64_t pol_a = policy_evict_normal();
      const uint64_t pol_b = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      if constexpr (HALO) {
        // Two cursors over this CTA's flattened (unit, chunk) sequence: the A cursor (halo
        // loads) runs up to kAhead chunks ahead of the B cursor (weight tiles), so a chunk's
        // halo is requested long before its 9 taps' MMAs need it.  Before issuing B(c) the
        // producer may wait only on A slots the MMA frees while consuming B(c-1) or earlier
        // (otherwise the MMA would stall on B(c)): kAhead <= kANum - 1.
        struct Cur {
          SegIter it;
          Seg g;
          int ok, kc;
        };
        auto cur_init = [&](Cur& c) {
          c.it = it0;
          c.ok = c.it.get(c.g);
          c.kc = c.ok ? c.g.k0 : 0;
        };
        auto cur_next = [&](Cur& c) {
          if (++c.kc >= c.g.k1) {
            c.it.next(c.g);
            c.ok = c.it.get(c.g);
            c.kc = c.ok ? c.g.k0 : 0;
          }
        };
        Cur ca, cb;
        cur_init(ca);
        cur_init(cb);
        constexpr int kAhead = 2 < Cfg::kANum - 1 ? 2 : Cfg::kANum - 1;
        long long a_seg = -1;  // segment whose blocks are decoded in cx/cy/cn
        long long b_seg = -1;
        int b_n0 = 0;
        uint32_t b_bytes = Cfg::kStageB;  // this CTA's bytes per (tap, chunk) weight tile
        const CUtensorMap* b_tm = &tmB;
        HaloTile g{};
        int cx[8], cy[8], cn[8];
        int ahead = 0;  // chunks the A cursor is ahead of the B cursor
        int bs = 0;     // B ring position
        uint32_t bph = 0;
#ifdef SPHINX_TRACE
        bool tr_a = false, tr_b = false;
#endif
        constexpr bool split = true;
        const bool doA = split ? warp == kAWarp : warp == 0;
        const bool doB = warp == 0;
        while (doB ? cb.ok : ca.ok) {
          // ---- A: issue halos up to kAhead chunks ahead of the current B chunk (split: the A
          // thread runs on its own, bounded only by the A ring)
          while (doA && ca.ok && (split || ahead < kAhead)) {
            if (ca.it.x != a_seg) {  // new segment: decode its blocks once (kept in registers)
              a_seg = ca.it.x;
              g = halo_tile<CG>(ca.g.t / p.n_tiles_n, rank, nF, nB, list, nR, p);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                // pad a short tile with a real block of the same class (computed, never stored)
                const int j = min(g.j0 + i, g.nblk - 1);
                int n = 0, by = 0, bx = 0;
                if (i < g.bpt) decode_block(__ldg(g.list + j), p.hb, p.wb, n, by, bx);
                cn[i] = n;
                cy[i] = by * BLK - 1;
                cx[i] = bx * BLK - 1;
              }
            }
            const uint32_t a_bytes = (uint32_t)(g.lines * g.bpt * 10 * 128);  // real halo bytes
            // line l of block i lands in the (l * bpt + i)-th 1280-B line of the slot
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* a_dst = sA + stage * Cfg::kASlot;
            uint32_t bar;
            if constexpr (NORM) {
              // raw halos land on this CTA's own barrier; the transform warps hand the slot on
              mbar_arrive_expect_tx(&landed[stage], a_bytes);
              bar = smem_u32(&landed[stage]);
            } else if constexpr (CG == 1) {
              mbar_arrive_expect_tx(&full[stage], a_bytes);
              bar = smem_u32(&full[stage]);
            } else {
              if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * a_bytes);
              bar = leader_addr(&full[stage]);
            }
            for (int l = 0; l < g.lines; ++l) {
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                if (i >= g.bpt) break;
                uint8_t* dst = a_dst + (l * g.bpt + i) * Cfg::kHaloRow;
                const CUtensorMap* tm = g.tr ? &tmC : &tmA;
                const int xx = g.tr ? cx[i] + l : cx[i], yy = g.tr ? cy[i] : cy[i] + l;
                if constexpr (CG == 1 || NORM) tma_load_4d_bar(tm, bar, dst, ca.kc * kBK, xx, yy, cn[i], pol_a);
                else tma_load_4d_cg2(tm, bar, dst, ca.kc * kBK, xx, yy, cn[i], pol_a);
              }
            }
#ifdef SPHINX_TRACE
            if (!tr_a) {
              CONV_TRACE(8, gtimer());
              tr_a = true;
            }
#endif
            if (++stage == Cfg::kANum) {
              stage = 0;
              phase ^= 1;
            }
            cur_next(ca);
            ++ahead;
          }
          if (!doB) break;
          // ---- B: one (tap, chunk) weight tile per tap of the B cursor's chunk
          {
            if (cb.it.x != b_seg) {
              b_seg = cb.it.x;
              const int ntb = cb.g.t - (cb.g.t / p.n_tiles_n) * p.n_tiles_n;
              b_n0 = ntb * BN + rank * Cfg::kBNc;
              b_bytes = (uint32_t)Cfg::kStageB;
              b_tm = &tmB;
            }
            const int n0 = b_n0;
            for (int tap = 0; tap < 9; ++tap) {
              uint64_t* bf = &full[Cfg::kANum + bs];
              mbar_wait(&empty[Cfg::kANum + bs], bph ^ 1);
              uint8_t* b_dst = sB + bs * Cfg::kStageB;
              if constexpr (CG == 1) {
                mbar_arrive_expect_tx(bf, b_bytes);
                tma_load_3d(b_tm, bf, b_dst, cb.kc * kBK, tap, n0, pol_b);
              } else {
                if (rank == 0) mbar_arrive_expect_tx(bf, 2 * b_bytes);
                tma_load_3d_cg2(b_tm, leader_addr(bf), b_dst, cb.kc * kBK, tap, n0, pol_b);
              }
#ifdef SPHINX_TRACE
              if (!tr_b) {
                CONV_TRACE(9, gtimer());
                tr_b = true;
              }
#endif
              if (++bs == Cfg::kBNum) {
                bs = 0;
                bph ^= 1;
              }
            }
          }
          cur_next(cb);
          --ahead;
        }
#ifdef SPHINX_TRACE
        if (doB) CONV_TRACE(7, gtimer());
#endif
      } else if (warp == 0)
      for (int u = cluster_id; u < total; u += n_clusters) {
        const Unit U = decode_unit(u, n_full, nsplit);
        const int t = U.t;
        const int mt = t / p.n_tiles_n, nt = t - mt * p.n_tiles_n;
        const int ks0 = U.sk * ksteps / U.ns, ks1 = (U.sk + 1) * ksteps / U.ns;
        // TMA origin of every block of this CTA's half of the tile (kept in registers)
        int cx[BPT], cy[BPT], cn[BPT];
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
          // pad a short last tile with a real block (its rows are computed, never stored)
          const int j = min(mt * bpt_pair + rank * BPT + i, count - 1);
          int n, by, bx;
          decode_block(__ldg(p.ids + j), p.hb, p.wb, n, by, bx);
          cn[i] = n;
          cy[i] = by * BLK - 1;
          cx[i] = bx * BLK - 1;
        }
        const int n0 = nt * BN + rank * Cfg::kBNc;
        const uint32_t stage_bytes = (uint32_t)kStageA + (uint32_t)Cfg::kStageB;
        const CUtensorMap* b_tm = &tmB;
        int tap = ks0 / p.kc, kc = ks0 - (ks0 / p.kc) * p.kc;
        for (int ks = ks0; ks < ks1; ++ks) {
          {
            // 3x3: tap (dy, dx); pointwise: the block itself (centre tap)
            const int dy = p.taps == 9 ? tap / 3 : 1, dx = p.taps == 9 ? tap - 3 * (tap / 3) : 1;
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* a_dst = sA + stage * kStageA;
            uint8_t* b_dst = sB + stage * Cfg::kStageB;
            if constexpr (CG == 1) {
              mbar_arrive_expect_tx(&full[stage], stage_bytes);
#pragma unroll
              for (int i = 0; i < BPT; ++i)
                tma_load_4d(&tmA, &full[stage], a_dst + i * bb * 128, kc * kBK, cx[i] + dx,
                            cy[i] + dy, cn[i], pol_a);
              tma_load_3d(b_tm, &full[stage], b_dst, kc * kBK, tap, n0, pol_b);
            } else {
              if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * stage_bytes);
              const uint32_t bar = leader_addr(&full[stage]);
#pragma unroll
              for (int i = 0; i < BPT; ++i)
                tma_load_4d_cg2(&tmA, bar, a_dst + i * bb * 128, kc * kBK, cx[i] + dx, cy[i] + dy,
                                cn[i], pol_a);
              tma_load_3d_cg2(b_tm, bar, b_dst, kc * kBK, tap, n0, pol_b);
            }
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
            if (++kc == p.kc) {
              kc = 0;
              ++tap;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only) =====================
    if (rank == 0 && elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(kBM * CG, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      if constexpr (HALO) {
        int bs = 0;
        uint32_t bph = 0;
        SegIter it = it0;
        Seg sg;
#ifdef SPHINX_TRACE
        int n_chunks = 0;
        bool first = true;
#endif
        for (; it.get(sg); it.next(sg)) {
          const int kc0 = sg.k0, kc1 = sg.k1;
#ifdef SPHINX_TRACE
          n_chunks += kc1 - kc0;
#endif
          const HaloTile g = halo_tile<CG>(sg.t / p.n_tiles_n, 0, nF, nB, list, nR, p);
          const uint32_t line_stride = (uint32_t)(g.bpt * Cfg::kHaloRow);
          const bool nar = sg.t % p.n_tiles_n == p.n_tiles_n - 1 && p.n_last < BN;
          const uint32_t idesc_t = nar ? idesc_bf16_f32(kBM * CG, p.n_last) : idesc;
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
          for (int kc = kc0; kc < kc1; ++kc) {
            if constexpr (NORM) mbar_wait_acq_cluster(&full[stage], phase);
            else mbar_wait(&full[stage], phase);
            tc_fence_after();
#ifdef SPHINX_TRACE
            if (first) CONV_TRACE(10, gtimer());
#endif
            const uint32_t a_base = smem_u32(sA + stage * Cfg::kASlot);
            for (int tap = 0; tap < 9; ++tap) {
              const int dy = tap / 3, dx = tap - 3 * (tap / 3);
              mbar_wait(&full[Cfg::kANum + bs], bph);
              tc_fence_after();
#ifdef SPHINX_TRACE
              if (first) {
                CONV_TRACE(2, gtimer());
                first = false;
              }
#endif
              // tap (dy,dx): 8-row group q*bpt + block at a_start + group*2048; rows run along
              // the halo line, so the along-line shift is 128 B per pixel and the cross-line
              // shift is one line (bpt slots); transposed tiles swap the roles of dy and dx
              const int major = g.tr ? dx : dy, minor = g.tr ? dy : dx;
              const uint32_t a_start = a_base + (uint32_t)major * line_stride + (uint32_t)(minor * 128);
              const uint32_t b_addr = smem_u32(sB + bs * Cfg::kStageB);
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k) {
                const uint64_t ad = umma_desc_sw128(a_start + k * 32, Cfg::kHaloRow, 0u);
                const uint64_t bd = umma_desc_sw128(b_addr + k * 32, 1024);
                const uint32_t accum = (kc != kc0 || tap != 0 || k != 0) ? 1u : 0u;
                if constexpr (CG == 1) tc_mma_bf16(d_tmem, ad, bd, idesc_t, accum);
                else tc_mma_bf16_cg2(d_tmem, ad, bd, idesc_t, accum);
              }
              if constexpr (CG == 1) tc_commit(&empty[Cfg::kANum + bs]);
              else tc_commit_cg2_mc(&empty[Cfg::kANum + bs]);
              if (++bs == Cfg::kBNum) {
                bs = 0;
                bph ^= 1;
              }
            }
            if constexpr (CG == 1) tc_commit(&empty[stage]); else tc_commit_cg2_mc(&empty[stage]);
            if (++stage == Cfg::kANum) {
              stage = 0;
              phase ^= 1;
            }
          }
          if constexpr (CG == 1) tc_commit(&tfull[acc]); else tc_commit_cg2_mc(&tfull[acc]);
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
#ifdef SPHINX_TRACE
        CONV_TRACE(3, gtimer());
        CONV_TRACE(6, (unsigned long long)n_chunks);
#endif
      } else
      for (int u = cluster_id; u < total; u += n_clusters) {
        const Unit U = decode_unit(u, n_full, nsplit);
        const int ks0 = U.sk * ksteps / U.ns, ks1 = (U.sk + 1) * ksteps / U.ns;
        const bool nar = U.t % p.n_tiles_n == p.n_tiles_n - 1 && p.n_last < BN;
        const uint32_t idesc_t = nar ? idesc_bf16_f32(kBM * CG, p.n_last) : idesc;
        TWAIT(21, mbar_wait(&tempty[acc], acc_phase ^ 1));
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int ks = ks0; ks < ks1; ++ks) {
          TWAIT(20, mbar_wait(&full[stage], phase));
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * kStageA);
          const uint32_t b_addr = smem_u32(sB + stage * Cfg::kStageB);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ad = umma_desc_sw128(a_addr + k * 32, 1024);
            const uint64_t bd = umma_desc_sw128(b_addr + k * 32, 1024);
            const uint32_t accum = (ks != ks0 || k != 0) ? 1u : 0u;
            if constexpr (CG == 1) tc_mma_bf16(d_tmem, ad, bd, idesc_t, accum);
            else tc_mma_bf16_cg2(d_tmem, ad, bd, idesc_t, accum);
          }
          if constexpr (CG == 1) tc_commit(&empty[stage]); else tc_commit_cg2_mc(&empty[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CG == 1) tc_commit(&tfull[acc]); else tc_commit_cg2_mc(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp < kAWarp || (!NORM && warp >= kXWarp)) {
    if (p.early_list) {
      pdl_wait();  // stores / residual reads after the predecessor completes
      pdl_trigger();
    }
    // ============ epilogue (warps 2..5, and 7..10 for non-NORM kernels; both CTAs) ============
    constexpr int kEpiW = NORM ? 4 : 8, kEpiT = kEpiW * 32, kHalves = kEpiW / 4;
    const int half = warp >= kXWarp ? 1 : 0;  // which half of the 32-column chunks this warp drains
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    const int erow = half * kBM + row;  // epilogue thread index
    int st_cnt = 0;                      // staged chunks (TMA-store path): buffer = st_cnt & 1
    int acc = 0;
    uint32_t acc_phase = 0;
    // tile row -> (block, pixel): per-tap mode rows are block-major (b^2 rows per block);
    // halo mode rows are [line q][block][8 px along the line] (group = q * bpt + block)
    auto tile_geom = [&](int mt, int& bi, int& ry, int& rx, int& j, int& nblk, const int32_t*& lst) {
      if constexpr (HALO) {
        const HaloTile g = halo_tile<CG>(mt, rank, nF, nB, list, nR, p);
        bi = (row >> 3) % g.bpt;
        const int q = (row >> 3) / g.bpt;
        ry = g.tr ? (row & 7) : q;
        rx = g.tr ? q : (row & 7);
        j = g.j0 + bi;
        nblk = g.nblk;
        lst = g.list;
      } else {
        bi = row / bb;
        ry = (row - bi * bb) / BLK;
        rx = (row - bi * bb) % BLK;
        j = mt * bpt_pair + rank * BPT + bi;
        nblk = count;
        lst = p.ids;
      }
    };
    // One tile ahead: the next tile's block id and (per-tap unsplit tiles) bias columns are loaded
    // while this tile drains, so their global-load latency is off the epilogue's critical path.
    int pf_id = 0;
    float pf_b[4] = {0.f, 0.f, 0.f, 0.f};
    auto prefetch = [&](const Seg& g) {
      const int mt = g.t / p.n_tiles_n, nt = g.t - mt * p.n_tiles_n;
      int bi, ry, rx, j, nblk;
      const int32_t* lst;
      tile_geom(mt, bi, ry, rx, j, nblk, lst);
      pf_id = (bi < (HALO ? 8 : BPT) && j < nblk) ? __ldg(lst + j) : 0;
      if (!HALO && g.ns == 1) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = half * 32 + k * 64 + lane, co = nt * BN + c;
          pf_b[k] = (p.bias && c < BN && co < p.cout) ? __ldg(p.bias + co) : 0.f;
        }
      }
    };
    SegIter it = it0;
    Seg sg;
    bool have = it.get(sg);
    if (have) prefetch(sg);
    while (have) {
      const int t = sg.t, sk = sg.sk, ns = sg.ns;
      const Unit U{sg.t, sg.sk, sg.ns, sg.slot};
      const int mt = t / p.n_tiles_n, nt = t - mt * p.n_tiles_n;
      const int my_id = pf_id;
      float b_reg[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) b_reg[k] = pf_b[k];
      SegIter nit = it;
      nit.next(sg);
      Seg nsg;
      const bool nhave = nit.get(nsg);
      if (nhave) prefetch(nsg);
      int bi, ry, rx, j, nblk;
      const int32_t* lst;
      tile_geom(mt, bi, ry, rx, j, nblk, lst);
      bool valid = (bi < (HALO ? 8 : BPT)) && (j < nblk);
      size_t pix = 0;
      int n = 0, by = 0, bx = 0;
      if (valid) {
        decode_block(my_id, p.hb, p.wb, n, by, bx);
        const int yy = by * BLK + ry, xx = bx * BLK + rx;
        valid = (yy < p.h) && (xx < p.w);
        pix = (((size_t)n * p.h + yy) * p.w + xx) * p.cout;
      }
      const bool listed = (bi < (HALO ? 8 : BPT)) && (j < nblk);
      // split-K part: column-major [BN][128] (lanes = consecutive rows: coalesced)
      float* part = nullptr;
      if (ns > 1) part = p.ws_part + ((size_t)(U.slot * ns + sk) * CG + rank) * kBM * BN + row;
      // stream-K part: column-major [BN][128] slot of this cluster (coalesced per column)
      float* skpart = (sg.role == kPart)
                          ? p.ws_part + ((size_t)cluster_id * CG + rank) * kBM * BN + row : nullptr;
      // per-tap unsplit tiles: each warp holds its chunks' bias in registers (lane l: column
      // c0 + l of chunk k, c0 = half*32 + k*64) -- no barrier across the epilogue warps
      const bool regbias = !HALO && ns == 1;
      if (!regbias) {
        // this tile's bias slice -> s_bias[acc] (the slot was last read by a tile that used it
        // two or more tiles ago, before a barrier 1 every thread has passed since)
        float* sb = s_bias + acc * 256;
        const int nb = p.bias ? min(BN, p.cout - nt * BN) : 0;
        for (int c = erow; c < BN; c += kEpiT) sb[c] = c < nb ? __ldg(p.bias + nt * BN + c) : 0.f;
        named_bar_sync(1, kEpiT);
      }
      const float* sbt = s_bias + acc * 256;
      if (warp == 2 && lane == 0) TWAIT(23, mbar_wait(&tfull[acc], acc_phase));
      else mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#ifdef SPHINX_TRACE
      if (warp == 2 && lane == 0) {
        CONV_TRACE(11, gtimer());
        if (p.trace) ++g_conv_trace[blockIdx.x * 24 + 12];
      }
#endif
      if (sg.role == kOwner) {
       if (half == 0) {  // the owner reduction runs on warps 2..5 (barrier 3, 128 threads)
        // ---- stream-K owner: wait for the parts of tile t, then add them chunk by chunk
        const int c_last = sk_cluster_of((long long)(t + 1) * p.kc - 1, Wk, n_clusters);
        const int n_parts = c_last - cluster_id;
        int* cnt = p.ws_cnt + (cluster_id * CG + rank) * 2;
        if (row == 0) {
          int seen;
          do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
            if (seen < n_parts) __nanosleep(64);
          } while (seen < n_parts);
          fence_proxy_async_global();
        }
        named_bar_sync(3, 128);
        float* stage_buf = reinterpret_cast<float*>(sA);  // the operand ring is idle now
        const uint32_t chunk_bytes = 32u * kBM * 4u;          // 32 columns x 128 rows, fp32
        auto stage_chunk = [&](int c0, int buf) {             // issued by row 0 only
          mbar_arrive_expect_tx(&red_bar[buf], chunk_bytes * (uint32_t)n_parts);
          for (int j = 0; j < n_parts; ++j)
            bulk_g2s(stage_buf + ((size_t)buf * Cfg::kMaxParts + j) * 32 * kBM,
                     p.ws_part + ((size_t)(cluster_id + 1 + j) * CG + rank) * kBM * BN + (size_t)c0 * kBM,
                     chunk_bytes, &red_bar[buf]);
        };
        if (row == 0) stage_chunk(0, 0);
        uint32_t rph0 = 0, rph1 = 0;
#pragma unroll 1
        for (int c0 = 0, ci = 0; c0 < BN; c0 += 32, ++ci) {
          const int buf = ci & 1;
          if (row == 0 && c0 + 32 < BN) stage_chunk(c0 + 32, buf ^ 1);  // prefetch next chunk
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0), r);
          tc_wait_ld();
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          mbar_wait(&red_bar[buf], buf ? rph1 : rph0);
          if (buf) rph1 ^= 1; else rph0 ^= 1;
          for (int j = 0; j < n_parts; ++j) {
            const float* src = stage_buf + ((size_t)buf * Cfg::kMaxParts + j) * 32 * kBM + row;
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += src[i * kBM];  // lanes = consecutive rows
          }
          if (valid) store_row_chunk(p, pix, nt * BN + c0, v, sbt + c0);
          named_bar_sync(3, 128);  // every thread done with buf before it is refilled
        }
        if (row == 0) cnt[0] = 0;  // leave the counter zeroed for the next launch
       }
      } else if (regbias) {
        if constexpr (!HALO) {
          // per-tap unsplit tile: double-buffered TMEM drain (chunk k+1's tcgen05.ld is in flight
          // while chunk k is converted and stored), bias from registers, and with bf16 y a
          // warp-local staged TMA store per chunk
          int width = (nt == p.n_tiles_n - 1 && p.n_last < BN) ? p.n_last : BN;
#ifdef SPHINX_TRACE
          if (p.dbg & 4) width = 0;  // timing probe: release the accumulator without draining it
#endif
          uint8_t* wbuf = s_store + (size_t)((half * 4 + q) * 2) * 2048;
          uint32_t ra[32], rb[32];
          const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
          if (half * 32 < width) {
            tmem_ld_32x32b_x32(tbase + (uint32_t)(half * 32), ra);
            tc_wait_ld_dep(ra);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int c0 = half * 32 + k * 64;
            if (c0 >= width) break;
            uint32_t(&cur)[32] = (k & 1) ? rb : ra;
            uint32_t(&nxt)[32] = (k & 1) ? ra : rb;
            const bool more = c0 + 64 < width;
            if (more) tmem_ld_32x32b_x32(tbase + (uint32_t)(c0 + 64), nxt);
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(cur[i]) + __shfl_sync(0xffffffffu, b_reg[k], i);
            if (p.tma_y) {
              stage_chunk_tma_warp<BLK>(p, tmY, wbuf + (st_cnt & 1) * 2048, lane, q, pix, valid, nt * BN + c0, v,
                                        n, by, bx, listed);
              ++st_cnt;
            } else if (valid) {
              store_row_chunk(p, pix, nt * BN + c0, v, nullptr);
            }
            if (more) tc_wait_ld_dep(nxt);
          }
        }
      } else {
        // a ragged last C_out tile only has p.n_last valid accumulator columns (the rest are
        // beyond C_out: never stored, so they need not be drained or parked either)
        const int width = (nt == p.n_tiles_n - 1 && p.n_last < BN) ? p.n_last : BN;
        for (int c0 = half * 32; c0 < width; c0 += 32 * kHalves) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0), r);
          tc_wait_ld();
          if (sg.role == kPart) {
#pragma unroll
            for (int i = 0; i < 32; ++i) __stcg(skpart + (size_t)(c0 + i) * kBM, __uint_as_float(r[i]));
          } else if (ns > 1) {
            // split-K: park this split's fp32 partial (column-major, coalesced)
#pragma unroll
            for (int i = 0; i < 32; ++i) __stcg(part + (size_t)(c0 + i) * kBM, __uint_as_float(r[i]));
          } else if (valid) {
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
            store_row_chunk(p, pix, nt * BN + c0, v, sbt + c0);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
#ifdef SPHINX_TRACE
      if (warp == 2 && lane == 0 && p.trace) {
        const unsigned long long d = gtimer() - g_conv_trace[blockIdx.x * 24 + 11];
        g_conv_trace[blockIdx.x * 24 + 13] += d;
        g_conv_trace[blockIdx.x * 24 + 14] = d;
      }
#endif
      if (lane == 0) {
        if constexpr (CG == 1) mbar_arrive(&tempty[acc]);
        else mbar_arrive_cluster(leader_addr(&tempty[acc]));
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      if (sg.role == kPart) {
        // publish this part to the tile's owner (never waits)
        __threadfence();
        named_bar_sync(1, kEpiT);
        if (erow == 0) {
          const int owner = sk_cluster_of((long long)t * p.kc, Wk, n_clusters);
          atomicAdd(p.ws_cnt + (owner * CG + rank) * 2, 1);
        }
      }
      if (ns > 1) {
        // Rendezvous of the ns units of tile t (all co-resident in this single round),
        // then each reduces a 1/nsplit slice of the rows, summing partials in split order
        // (deterministic), with coalesced float4 loads across the epilogue threads.
        __threadfence();
        named_bar_sync(1, kEpiT);
#ifdef SPHINX_TRACE
        if (erow == 0) {
          CONV_TRACE(16, gtimer());
          CONV_TRACE(19, (unsigned long long)ns);
        }
#endif
        int* arrive = p.ws_cnt + (U.slot * CG + rank) * 2;
        if (erow == 0) {
          atomicAdd(arrive, 1);
          int seen;
          do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(seen) : "l"(arrive) : "memory");
            if (seen < ns) __nanosleep(64);
          } while (seen < ns);
        }
        named_bar_sync(1, kEpiT);
#ifdef SPHINX_TRACE
        if (erow == 0) CONV_TRACE(17, gtimer());
#endif
        // this unit reduces output columns [c0s, c1s) (multiples of 8) of all 128 rows: from every
        // part that column range is one contiguous column-major block -> one bulk copy each
        const int c0s = (sk * (BN / 8) / ns) * 8, c1s = ((sk + 1) * (BN / 8) / ns) * 8;
        const int ncol = c1s - c0s;
        const uint32_t slice_bytes = (uint32_t)(ncol * kBM * 4);
        const float* base = p.ws_part + ((size_t)(U.slot * ns) * CG + rank) * kBM * BN + (size_t)c0s * kBM;
        const size_t split_stride = (size_t)CG * kBM * BN;
        float* stage_buf = reinterpret_cast<float*>(sA);  // the operand ring is idle now
        if ((size_t)ns * slice_bytes > (size_t)Cfg::kRingBytes) __trap();  // never at BN <= 256
        if (erow == 0 && ncol > 0) {
          fence_proxy_async_global();
          mbar_arrive_expect_tx(red_bar, slice_bytes * (uint32_t)ns);
          for (int s2 = 0; s2 < ns; ++s2)
            bulk_g2s(stage_buf + (size_t)s2 * ncol * kBM, base + s2 * split_stride, slice_bytes, red_bar);
        }
        if (ncol > 0) {
          mbar_wait(red_bar, 0);
          if (valid) {
            // thread = row (its own pixel); partials summed in split order (deterministic)
            for (int c = half * 8; c < ncol; c += 8 * kHalves) {
              const int co = nt * BN + c0s + c;
              if (co >= p.cout) break;
              float v8[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) v8[i] = stage_buf[(size_t)(c + i) * kBM + row];
              for (int s2 = 1; s2 < ns; ++s2) {
                const float* sp = stage_buf + (size_t)s2 * ncol * kBM;
#pragma unroll
                for (int i = 0; i < 8; ++i) v8[i] += sp[(size_t)(c + i) * kBM + row];
              }
#pragma unroll
              for (int i = 0; i < 8; ++i) v8[i] += sbt[c0s + c + i];
              if (p.res) add_residual<8>(p, pix, co, v8);
              if (p.y_f32) {
                float* yp = static_cast<float*>(p.y) + pix + co;
                *reinterpret_cast<float4*>(yp) = make_float4(v8[0], v8[1], v8[2], v8[3]);
                *reinterpret_cast<float4*>(yp + 4) = make_float4(v8[4], v8[5], v8[6], v8[7]);
              } else {
                uint4 pk;
                __nv_bfloat162 t0 = __floats2bfloat162_rn(v8[0], v8[1]);
                __nv_bfloat162 t1 = __floats2bfloat162_rn(v8[2], v8[3]);
                __nv_bfloat162 t2 = __floats2bfloat162_rn(v8[4], v8[5]);
                __nv_bfloat162 t3 = __floats2bfloat162_rn(v8[6], v8[7]);
                pk.x = *reinterpret_cast<uint32_t*>(&t0);
                pk.y = *reinterpret_cast<uint32_t*>(&t1);
                pk.z = *reinterpret_cast<uint32_t*>(&t2);
                pk.w = *reinterpret_cast<uint32_t*>(&t3);
                *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + pix + co) = pk;
              }
            }
          }
        }
        // departure: the last unit to leave re-zeroes both counters for the next launch
        named_bar_sync(1, kEpiT);
#ifdef SPHINX_TRACE
        if (erow == 0) CONV_TRACE(18, gtimer());
#endif
        if (erow == 0) {
          const int old = atomicAdd(arrive + 1, 1);
          if (old == ns - 1) {
            arrive[0] = 0;
            arrive[1] = 0;
            __threadfence();
          }
        }
      }
      it = nit;
      sg = nsg;
      have = nhave;
    }
    // staged TMA stores: complete before the CTA exits (shared memory must outlive their reads)
    if constexpr (!HALO)
      if (p.tma_y && lane == 0) bulk_wait_group_all();
  } else if constexpr (NORM) {
    if (warp >= kXWarp) {
      // ============ fused GroupNorm + SiLU (NEXT-3): transform warps 7..14, both CTAs ============
      // Each raw halo slot lands on this CTA's `landed` barrier; the kXThreads transform threads apply
      // a = SiLU(x * scale + shift) in place (scale/shift per (frame, channel) from p.norm_tab),
      // leaving out-of-image halo pixels at zero (the conv's zero padding is in the activation
      // domain), fence the generic-proxy writes for the tensor core, and arrive on the leader's
      // A-slot barrier (count = CTAs per pair).  Thread xt always touches the physical 16-byte
      // unit xt & 7 of rows kXThreads/8 apart, so its SW128 phase -- and hence its logical 8-channel group
      // -- is fixed (rows kXThreads/8 apart, a multiple of 8).
      const int xt = threadIdx.x - kXWarp * 32;
      const int u16 = xt & 7;
      const int jl = u16 ^ ((xt >> 3) & 7);
      int stage = 0;
      uint32_t phase = 0;
      SegIter it = it0;
      Seg sg;
      long long a_seg = -1;
      HaloTile g{};
      int rows = 0;
      for (; it.get(sg); it.next(sg)) {
        if (it.x != a_seg) {
          // new tile: per halo row (= one pixel of one block's halo line) the block index, or 255
          // if the pixel lies outside the image (its zero fill must stay zero); chunk-invariant
          a_seg = it.x;
          g = halo_tile<CG>(sg.t / p.n_tiles_n, rank, nF, nB, list, nR, p);
          rows = g.lines * g.bpt * 10;
          for (int row = xt; row < rows; row += kXThreads) {
            const int lb = row / 10, px = row - lb * 10;
            const int l = lb / g.bpt, i = lb - l * g.bpt;
            int n = 0, by = 0, bx = 0;
            decode_block(__ldg(g.list + min(g.j0 + i, g.nblk - 1)), p.hb, p.wb, n, by, bx);
            const int y0 = by * BLK - 1, x0 = bx * BLK - 1;
            const int yy = g.tr ? y0 + px : y0 + l, xx = g.tr ? x0 + l : x0 + px;
            sts_u8(smem_u32(s_rowinfo) + row, (yy < 0 || yy >= p.h || xx < 0 || xx >= p.w) ? 255u : (uint32_t)i);
          }
        }
        for (int kc = sg.k0; kc < sg.k1; ++kc) {
          // this chunk's (scale, shift) for the tile's blocks x 64 channels
          for (int idx = xt; idx < g.bpt * 64; idx += kXThreads) {
            const int i = idx >> 6, ch = kc * kBK + (idx & 63);
            int n = 0, by = 0, bx = 0;
            decode_block(__ldg(g.list + min(g.j0 + i, g.nblk - 1)), p.hb, p.wb, n, by, bx);
            const float2 v2 = ch < p.cin ? __ldg(p.norm_tab + (size_t)n * p.cin + ch) : make_float2(0.f, 0.f);
            sts64f(smem_u32(s_tab + (i * 8 + ((idx & 63) >> 3)) * 20 + (idx & 7) * 2), v2.x, v2.y);
          }
          mbar_wait(&landed[stage], phase);
          named_bar_sync(2, kXThreads);
          const uint32_t slot = smem_u32(sA + stage * Cfg::kASlot + u16 * 16);
          const uint32_t rinfo = smem_u32(s_rowinfo), tab0 = smem_u32(s_tab);
          // 4 rows per iteration (rows kXThreads/8 apart keep this thread's SW128 phase):
          // independent LDS / SFU chains in flight
          constexpr int kRS = kXThreads / 8;
          for (int r0 = xt >> 3; r0 < rows; r0 += 4 * kRS) {
            uint4 v[4];
            int bi[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int row = r0 + kRS * q;
              bi[q] = row < rows ? (int)lds_u8(rinfo + row) : 255;
              if (bi[q] != 255) v[q] = lds128(slot + row * 128);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (bi[q] == 255) continue;
              const uint32_t w4[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
              const uint32_t tb = tab0 + (uint32_t)((bi[q] * 8 + jl) * 20) * 4;
              uint32_t o4[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint4 tu = lds128(tb + k * 16);  // (scale, shift) of channels 2k, 2k+1
                const float4 t = make_float4(__uint_as_float(tu.x), __uint_as_float(tu.y),
                                             __uint_as_float(tu.z), __uint_as_float(tu.w));
                const float a0 = fmaf(__uint_as_float(w4[k] << 16), t.x, t.y);
                const float a1 = fmaf(__uint_as_float(w4[k] & 0xffff0000u), t.z, t.w);
                const __nv_bfloat162 pk = __floats2bfloat162_rn(__fdividef(a0, 1.f + __expf(-a0)),
                                                                __fdividef(a1, 1.f + __expf(-a1)));
                o4[k] = *reinterpret_cast<const uint32_t*>(&pk);
              }
              sts128(slot + (r0 + kRS * q) * 128, make_uint4(o4[0], o4[1], o4[2], o4[3]));
            }
          }
          fence_proxy_async_smem();
          named_bar_sync(2, kXThreads);
          if (xt == 0) {
            if constexpr (CG == 1) mbar_arrive(&full[stage]);
            else mbar_arrive_release_cluster(leader_addr(&full[stage]));
          }
          if (++stage == Cfg::kANum) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  }
#ifdef SPHINX_TRACE
  if (warp == 2 && lane == 0) CONV_TRACE(4, gtimer());
#endif
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
#ifdef SPHINX_TRACE
  if (threadIdx.x == 0) CONV_TRACE(5, gtimer());
#endif
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_cg2<Cfg::kTmemCols>(tmem_base);
    else tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

// Edge-class plan (halo mode on maps with H % 8 or W % 8 != 0): partitions the ascending list
// into full, bottom-edge (incl. corner) and right-edge blocks, each kept ascending, with
// warp-ballot / popc prefix sums in one CTA (latency-bound: <= a few thousand ids).
__global__ void __launch_bounds__(1024) conv_plan_kernel(const int32_t* __restrict__ ids,
                                                         const int32_t* __restrict__ count, int hb,
                                                         int wb, int has_b, int has_r,
                                                         int32_t* __restrict__ plan_ids,
                                                         int32_t* __restrict__ meta) {
  pdl_wait();
  pdl_trigger();
  // pass 1: class totals (so the class sub-lists' offsets are known); pass 2: scatter, with
  // one ballot per class per round giving each id its in-class rank (order = list order)
  __shared__ int tot[3];
  __shared__ int warp_off[3][32];
  __shared__ int round_tot[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int cnt = *count;
  if (threadIdx.x < 3) tot[threadIdx.x] = 0;
  __syncthreads();
  auto cls_of = [&](int id) {
    const int r = id % (hb * wb), by = r / wb, bx = r - (r / wb) * wb;
    return (has_b && by == hb - 1) ? 1 : ((has_r && bx == wb - 1) ? 2 : 0);
  };
  int local[3] = {0, 0, 0};
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) ++local[cls_of(__ldg(ids + j))];
  for (int c = 0; c < 3; ++c) {
    int v = local[c];
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0 && v) atomicAdd(&tot[c], v);
  }
  __syncthreads();
  int base[3] = {0, tot[0], tot[0] + tot[1]};
  for (int start = 0; start < cnt; start += blockDim.x) {
    const int j = start + threadIdx.x;
    int id = 0, c = -1;
    if (j < cnt) {
      id = __ldg(ids + j);
      c = cls_of(id);
    }
    int pre = 0;
    for (int k = 0; k < 3; ++k) {
      const unsigned bal = __ballot_sync(0xffffffffu, c == k);
      if (c == k) pre = __popc(bal & ((1u << lane) - 1u));
      if (lane == 0) warp_off[k][warp] = __popc(bal);
    }
    __syncthreads();
    if (warp < 3) {  // warp k scans class k's per-warp counts
      const int v = lane < nwarps ? warp_off[warp][lane] : 0;
      int incl = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += o;
      }
      if (lane < nwarps) warp_off[warp][lane] = incl - v;
      if (lane == 31) round_tot[warp] = incl;
    }
    __syncthreads();
    if (c >= 0) plan_ids[base[c] + warp_off[c][warp] + pre] = id;
    for (int k = 0; k < 3; ++k) base[k] += round_tot[k];
    __syncthreads();
  }
  if (threadIdx.x < 3) meta[threadIdx.x] = tot[threadIdx.x];
}

// ------------------------------------------------------------------ host side

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t get_encode_tiled() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(ptr);
  }
  return fn;
}

template <int BN, int CG, int BLK, bool HALO, bool EDGE = false, bool NORM = false>
static sphinx_status launch_bn(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                               const CUtensorMap& tb2, const ConvParams& p, int grid, cudaStream_t s) {
  using Cfg = ConvCfg<BN, CG, HALO, EDGE, NORM>;
  auto kern = sparse_conv3x3_tc_kernel<BN, CG, BLK, HALO, EDGE, NORM>;
  static bool attr_set = false;  // per process; the attribute is per function
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (e != cudaSuccess) return cuda_fail(e);
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NORM ? kThreadsNorm : kThreadsEpi8);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  ConvParams pk = p;
  pk.ring_bytes = Cfg::kRingBytes;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, tb2, pk);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

template <int BN>
static sphinx_status launch_cg(int cg, const CUtensorMap& ta, const CUtensorMap& tb,
                               const CUtensorMap& tc, const CUtensorMap& tb2, const ConvParams& p, int grid,
                               cudaStream_t s) {
  if (p.norm_tab) {  // fused GN+SiLU (halo mode, CTA pair; checked by the caller)
    return p.plan_ids ? launch_bn<BN, 2, 8, true, true, true>(ta, tb, tc, tb2, p, grid, s)
                      : launch_bn<BN, 2, 8, true, false, true>(ta, tb, tc, tb2, p, grid, s);
  }
  if (p.b == 8 && p.halo && p.plan_ids)
    return cg == 2 ? launch_bn<BN, 2, 8, true, true>(ta, tb, tc, tb2, p, grid, s)
                   : launch_bn<BN, 1, 8, true, true>(ta, tb, tc, tb2, p, grid, s);
  if (p.b == 8 && p.halo)
    return cg == 2 ? launch_bn<BN, 2, 8, true>(ta, tb, tc, tb2, p, grid, s)
                   : launch_bn<BN, 1, 8, true>(ta, tb, tc, tb2, p, grid, s);
  if (p.b == 8)
    return cg == 2 ? launch_bn<BN, 2, 8, false>(ta, tb, tc, tb2, p, grid, s)
                   : launch_bn<BN, 1, 8, false>(ta, tb, tc, tb2, p, grid, s);
  return cg == 2 ? launch_bn<BN, 2, 4, false>(ta, tb, tc, tb2, p, grid, s)
                 : launch_bn<BN, 1, 4, false>(ta, tb, tc, tb2, p, grid, s);
}

// Widest tile that minimises padded output columns (ties -> wider).  (Ragged 256-wide tiles
// with a narrow last tile, e.g. 320 = 256 + 64, measured slower: DESIGN.md §6.4.)
static int pick_bn(int cout) {
  const int cands[] = {256, 160, 128, 64, 32};
  int best = 32, best_pad = 1 << 30;
  for (int bn : cands) {
    const int pad = cdiv(cout, bn) * bn;
    if (pad < best_pad) {
      best_pad = pad;
      best = bn;
    }
  }
  return best;
}

}  // namespace sphinx

using namespace sphinx;

// Workspace: [kCntBytes of int32 split-K arrival counters][plan meta (256 B)]
//            [plan ids: capacity int32, padded to 256 B][split-K partial-tile slots].
constexpr size_t kCntBytes = 4096;
static size_t plan_bytes(long long capacity) { return 256 + (((size_t)capacity * 4 + 255) & ~(size_t)255); }

static size_t slot_bytes(int cg, int bn) { return (size_t)cg * kBM * bn * sizeof(float); }

extern "C" size_t sphinx_conv_workspace_size(int32_t n, int32_t h, int32_t w_, int32_t c_in,
                                             int32_t c_out, int32_t block) {
  (void)c_in;
  if (c_out <= 0 || n <= 0 || h <= 0 || w_ <= 0 || block <= 0) return 0;
  const long long capacity = (long long)n * cdiv(h, block) * cdiv(w_, block);
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) sms = v;
  }
  // one slot per SM (two rounds of CTA pairs), sized for the CTA-pair kernel
  return kCntBytes + plan_bytes(capacity) + (size_t)sms * slot_bytes(2, pick_bn(c_out));
}

static sphinx_status conv_impl(const void* x, const void* w, const float* bias, const void* residual,
                               void* y, sphinx_dtype y_dtype, int32_t n, int32_t h, int32_t w_,
                               int32_t c_in, int32_t c_out, int32_t block, const int32_t* block_ids,
                               const int32_t* count, int32_t capacity, void* workspace,
                               size_t workspace_bytes, sphinx_stream_t stream, int taps = 9,
                               const float2* norm_tab = nullptr, int flags = 0) {
  if (!x || !w || !y || !block_ids || !count) return SPHINX_ERR_INVALID_ARGUMENT;
  if (residual && (residual == x || !aligned16(residual))) return SPHINX_ERR_INVALID_ARGUMENT;
  if (workspace && (reinterpret_cast<uintptr_t>(workspace) & 255u)) return SPHINX_ERR_INVALID_ARGUMENT;
  if (n <= 0 || h <= 0 || w_ <= 0 || c_in <= 0 || c_out <= 0 || block <= 0 || capacity < 0)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (y_dtype != SPHINX_BF16 && y_dtype != SPHINX_F32) return SPHINX_ERR_INVALID_ARGUMENT;
  const int hb = cdiv(h, block), wb = cdiv(w_, block);
  if ((int64_t)capacity > (int64_t)n * hb * wb) return SPHINX_ERR_INVALID_ARGUMENT;
  if (c_in % 8 || c_out % 8 || (block != 4 && block != 8)) return SPHINX_ERR_UNSUPPORTED;
  if (!aligned16(x) || !aligned16(w) || !aligned16(y)) return SPHINX_ERR_UNSUPPORTED;
  int sms = 0;
  sphinx_status st = check_device(&sms);
  if (st != SPHINX_OK) return st;
  if (capacity == 0) return SPHINX_OK;
  PFN_encodeTiled_t enc = get_encode_tiled();
  if (!enc) return cuda_fail(cudaErrorNotSupported);

  int bn = pick_bn(c_out);
  // pointwise projections (K = C_in only: 5 K-steps per tile at C_in = 320) issue many short
  // tiles; the 256-wide tile needs 1/3 fewer MMA instructions and tiles per output column than
  // the 160-wide one, worth up to 1/15 padded columns (q|k|v 960 -> 1024: 23.3 vs 25.5 us, §6.9)
  if (taps == 1 && bn != 256 && cdiv(c_out, 256) * 256 * 15 <= c_out * 16) bn = 256;
#ifdef SPHINX_DEV_KNOBS
  if (const char* env = getenv("SPHINX_BN")) {  // dev build A/B: force the C_out tile width
    const int v = atoi(env);
    if (v == 32 || v == 64 || v == 128 || v == 160 || v == 256) bn = v;
  }
#endif
  // CTA-pair (cta_group::2) unless the caller forces the 1-SM kernel: halves the weight traffic
  // per SM
  int cg = (flags & SPHINX_CONV_FORCE_CG1) ? 1 : 2;
  // halo-staged A for 8x8 blocks unless the caller forces a path: each activation read once per
  // chunk
  int halo = (block == 8 && taps == 9) ? 1 : 0;
  if (flags & (SPHINX_CONV_FORCE_HALO | SPHINX_CONV_FORCE_PERTAP)) {
    halo = halo && !(flags & SPHINX_CONV_FORCE_PERTAP);
  } else if (halo && !norm_tab) {
    // At most one wave of tiles even if every capacity block is listed (e.g. a single frame):
    // the problem is latency-bound, and the per-tap path's split-K over (tap, chunk) K-steps
    // (halo mode splits only at 64-channel chunks) fills more of the GPU.  Measured on one
    // 72x72x320 frame: 9.5 vs 12.6 us at 5% density, 15.5 vs 17.8 us dense.  With C_in <= 320
    // (per-tap A traffic = 9 shifted windows of 64 channels per chunk) the per-tap path also wins
    // up to ~16 waves at capacity: its (tap, chunk) tails are finer and, since the round-2 per-tap
    // epilogue, its tiles drain as fast (21 x 72x72x320, same box: 22.5 vs 25.8 us at 10%, 37.2 vs
    // 40.6 at 25%, 73.2 vs 73.9 at 50%, 148.0 vs 148.4 dense; the configs[2] step -1%; the
    // configs[3] level 0 (92 waves at capacity) stays in halo mode)
    const long long max_tiles = (long long)cdiv(capacity, (kBM / (block * block)) * 2) * cdiv(c_out, pick_bn(c_out));
    if (max_tiles <= sms / 2 || (c_in <= 320 && max_tiles <= 16LL * (sms / 2))) halo = 0;
  }
  if (norm_tab) {
    if (!halo) return SPHINX_ERR_UNSUPPORTED;  // the transform works on halo slots (b = 8, 3x3)
    cg = 2;
  }
  CUtensorMap ta, tb, tc, tb2;
  {
    const cuuint64_t dims[4] = {(cuuint64_t)c_in, (cuuint64_t)w_, (cuuint64_t)h, (cuuint64_t)n};
    const cuuint64_t strides[3] = {(cuuint64_t)c_in * 2, (cuuint64_t)w_ * c_in * 2,
                                   (cuuint64_t)h * w_ * c_in * 2};
    // per-tap: the b x b block window; halo: one halo row of b+2 pixels
    const cuuint32_t box[4] = {(cuuint32_t)kBK, (cuuint32_t)(halo ? block + 2 : block),
                               (cuuint32_t)(halo ? 1 : block), 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return SPHINX_ERR_UNSUPPORTED;
    // halo columns (transposed right-edge tiles): one pixel wide, b+2 tall
    const cuuint32_t boxc[4] = {(cuuint32_t)kBK, 1, (cuuint32_t)(block + 2), 1};
    r = enc(&tc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, boxc, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return SPHINX_ERR_UNSUPPORTED;
  }
  {
    const cuuint64_t dims[3] = {(cuuint64_t)c_in, (cuuint64_t)taps, (cuuint64_t)c_out};
    const cuuint64_t strides[2] = {(cuuint64_t)c_in * 2, (cuuint64_t)taps * c_in * 2};
    const cuuint32_t box[3] = {(cuuint32_t)kBK, 1, (cuuint32_t)(bn / cg)};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w), dims, strides,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return SPHINX_ERR_UNSUPPORTED;
  }
  // per-tap mode with bf16 y: the epilogue writes each 32-column chunk of a block with one TMA
  // tensor store (box {32 ch, b, b, 1} of the NHWC map; SW64 staging layout)
  int tma_y = (!halo && y_dtype == SPHINX_BF16 && !norm_tab && c_out >= 32) ? 1 : 0;
#ifdef SPHINX_DEV_KNOBS
  if (getenv("SPHINX_NO_TMA_Y")) tma_y = 0;  // dev build A/B: direct 16-byte stores instead
#endif
  if (tma_y) {
    const cuuint64_t dims[4] = {(cuuint64_t)c_out, (cuuint64_t)w_, (cuuint64_t)h, (cuuint64_t)n};
    const cuuint64_t strides[3] = {(cuuint64_t)c_out * 2, (cuuint64_t)w_ * c_out * 2,
                                   (cuuint64_t)h * w_ * c_out * 2};
    const cuuint32_t box[4] = {32, (cuuint32_t)block, 4, 1};  // one warp's 32 rows (stage_chunk_tma_warp)
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tb2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, y, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return SPHINX_ERR_UNSUPPORTED;
  } else {
    tb2 = tb;  // unused
  }
  ConvParams p;
  p.ids = block_ids;
  p.count = count;
  p.bias = bias;
  p.y = y;
  p.res = static_cast<const __nv_bfloat16*>(residual);
  p.norm_tab = norm_tab;
  p.cin = c_in;
  p.y_f32 = y_dtype == SPHINX_F32;
  p.h = h;
  p.w = w_;
  p.cout = c_out;
  p.b = block;
  p.hb = hb;
  p.wb = wb;
  p.kc = cdiv(c_in, kBK);
  p.taps = taps;
  p.n_tiles_n = cdiv(c_out, bn);
  p.n_last = bn;
  p.tma_y = tma_y;
  p.bpt = kBM / (block * block);
  p.halo = halo;
  p.trace = 0;
  p.early_list = 0;
  p.early_input = 0;
  p.dbg = 0;
#ifdef SPHINX_TRACE
  if (const char* env = getenv("SPHINX_DBG")) p.dbg = atoi(env);
  {
    static int launch_no = 0;
    const char* env = getenv("SPHINX_TRACE_LAUNCH");
    p.trace = env && atoi(env) == launch_no;
    ++launch_no;
  }
#endif
  p.allow_streamk = (flags & SPHINX_CONV_FORCE_STREAMK) ? 2 : (flags & SPHINX_CONV_NO_STREAMK) ? 0 : 1;
  p.ws_part = nullptr;
  p.ws_cnt = nullptr;
  p.ws_slots = 0;
  p.ws_tiles = 0;
  p.plan_ids = nullptr;
  p.plan_meta = nullptr;
  p.rb = h % 8;
  p.cr = w_ % 8;
  p.bpt_b = p.rb ? (16 / p.rb < 8 ? 16 / p.rb : 8) : 8;
  p.bpt_r = p.cr ? (16 / p.cr < 8 ? 16 / p.cr : 8) : 8;
  const size_t pl_bytes = plan_bytes(capacity);
  const bool allow_split = !(flags & SPHINX_CONV_NO_SPLIT), allow_edge = !(flags & SPHINX_CONV_NO_EDGE);
  const bool ws_ok = workspace && workspace_bytes >= kCntBytes + pl_bytes;
  uint8_t* ws8 = static_cast<uint8_t*>(workspace);
  if (ws_ok && allow_edge && halo && (p.rb || p.cr)) {
    p.plan_meta = reinterpret_cast<int32_t*>(ws8 + kCntBytes);
    p.plan_ids = reinterpret_cast<int32_t*>(ws8 + kCntBytes + 256);
  }
  if (allow_split && ws_ok && workspace_bytes >= kCntBytes + pl_bytes + slot_bytes(cg, bn)) {
    p.ws_cnt = reinterpret_cast<int32_t*>(ws8);
    p.ws_part = reinterpret_cast<float*>(ws8 + kCntBytes + pl_bytes);
    p.ws_slots = (int)((workspace_bytes - kCntBytes - pl_bytes) / slot_bytes(cg, bn));
    p.ws_tiles = (int)(kCntBytes / (2 * sizeof(int32_t))) / cg;
  }
  const long long max_tiles = (long long)cdiv(capacity, p.bpt * cg) * p.n_tiles_n;
  int max_clusters = sms / cg;
#ifdef SPHINX_DEV_KNOBS
  if (const char* env = getenv("SPHINX_GRID_CAP")) {  // dev build: fewer SMs (ingress-limit probe)
    const int v = atoi(env) / cg;
    if (v >= 1 && v < max_clusters) max_clusters = v;
  }
#endif
  const long long want = p.ws_part ? max_tiles * 16 : max_tiles;  // split-K may multiply units
  const int grid = cg * (int)(want < max_clusters ? want : max_clusters);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // SPHINX_CONV_LIST_READY: ids/count (and a reused plan) predate the preceding kernel; not when
  // this call launches the plan kernel (its output becomes the immediate predecessor's) or for
  // the fused-GN variant (its table comes from the preceding kernel)
  p.early_list = (flags & SPHINX_CONV_LIST_READY) && !norm_tab &&
                 !(p.plan_ids && !(flags & SPHINX_CONV_REUSE_PLAN)) ? 1 : 0;
  p.early_input = (p.early_list && (flags & SPHINX_CONV_INPUT_READY)) ? 1 : 0;
  // SPHINX_CONV_REUSE_PLAN: the workspace already holds the edge plan of this very list (the
  // caller's previous conv on this stream used the same list and workspace): skip the plan launch
  if (p.plan_ids && !(flags & SPHINX_CONV_REUSE_PLAN)) {
    cudaError_t e = launch_k(conv_plan_kernel, dim3(1), dim3(1024), 0, s, block_ids, count, hb, wb,
                             (int)(p.rb != 0), (int)(p.cr != 0), const_cast<int32_t*>(p.plan_ids),
                             const_cast<int32_t*>(p.plan_meta));
    if (e != cudaSuccess) return cuda_fail(e);
  }
  switch (bn) {
    case 256: return launch_cg<256>(cg, ta, tb, tc, tb2, p, grid, s);
    case 160: return launch_cg<160>(cg, ta, tb, tc, tb2, p, grid, s);
    case 128: return launch_cg<128>(cg, ta, tb, tc, tb2, p, grid, s);
    case 64: return launch_cg<64>(cg, ta, tb, tc, tb2, p, grid, s);
    default: return launch_cg<32>(cg, ta, tb, tc, tb2, p, grid, s);
  }
}

extern "C" sphinx_status sphinx_sparse_conv3x3(const void* x, const void* w, const float* bias,
                                               void* y, sphinx_dtype y_dtype, int32_t n, int32_t h,
                                               int32_t w_, int32_t c_in, int32_t c_out,
                                               int32_t block, const int32_t* block_ids,
                                               const int32_t* count, int32_t capacity,
                                               void* workspace, size_t workspace_bytes,
                                               sphinx_stream_t stream) {
  return conv_impl(x, w, bias, nullptr, y, y_dtype, n, h, w_, c_in, c_out, block, block_ids, count,
                   capacity, workspace, workspace_bytes, stream);
}

extern "C" sphinx_status sphinx_sparse_conv3x3_residual(
    const void* x, const void* w, const float* bias, const void* residual, void* y,
    sphinx_dtype y_dtype, int32_t n, int32_t h, int32_t w_, int32_t c_in, int32_t c_out,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity,
    void* workspace, size_t workspace_bytes, sphinx_stream_t stream) {
  if (!residual) return SPHINX_ERR_INVALID_ARGUMENT;
  return conv_impl(x, w, bias, residual, y, y_dtype, n, h, w_, c_in, c_out, block, block_ids, count,
                   capacity, workspace, workspace_bytes, stream);
}

extern "C" sphinx_status sphinx_sparse_pointwise(
    const void* x, const void* w, const float* bias, const void* residual, void* y,
    sphinx_dtype y_dtype, int32_t n, int32_t h, int32_t w_, int32_t c_in, int32_t c_out,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity,
    void* workspace, size_t workspace_bytes, sphinx_stream_t stream) {
  return conv_impl(x, w, bias, residual, y, y_dtype, n, h, w_, c_in, c_out, block, block_ids, count,
                   capacity, workspace, workspace_bytes, stream, 1);
}

extern "C" sphinx_status sphinx_conv_edge_plan(const int32_t* block_ids, const int32_t* count, int32_t n,
                                               int32_t h, int32_t w_, int32_t block, int32_t capacity,
                                               void* workspace, size_t workspace_bytes,
                                               sphinx_stream_t stream) {
  if (!block_ids || !count || !workspace || n <= 0 || h <= 0 || w_ <= 0 || capacity < 0)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (reinterpret_cast<uintptr_t>(workspace) & 255u) return SPHINX_ERR_INVALID_ARGUMENT;
  const int hb = cdiv(h, block), wb = cdiv(w_, block);
  if ((int64_t)capacity > (int64_t)n * hb * wb) return SPHINX_ERR_INVALID_ARGUMENT;
  // only the halo path (8x8 blocks) on maps with partial edge blocks uses a plan
  if (block != 8 || (h % 8 == 0 && w_ % 8 == 0)) return SPHINX_OK;
  if (workspace_bytes < kCntBytes + plan_bytes(capacity)) return SPHINX_ERR_INVALID_ARGUMENT;
  sphinx_status st = check_device();
  if (st != SPHINX_OK) return st;
  uint8_t* ws8 = static_cast<uint8_t*>(workspace);
  cudaError_t e = launch_k(conv_plan_kernel, dim3(1), dim3(1024), 0, reinterpret_cast<cudaStream_t>(stream),
                           block_ids, count, hb, wb, (int)(h % 8 != 0), (int)(w_ % 8 != 0),
                           reinterpret_cast<int32_t*>(ws8 + kCntBytes + 256),
                           reinterpret_cast<int32_t*>(ws8 + kCntBytes));
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}

extern "C" sphinx_status sphinx_sparse_conv3x3_ex(
    const void* x, const void* w, const float* bias, const void* residual, void* y,
    sphinx_dtype y_dtype, int32_t n, int32_t h, int32_t w_, int32_t c_in, int32_t c_out,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity,
    void* workspace, size_t workspace_bytes, int32_t flags, sphinx_stream_t stream) {
  if (flags & ~(SPHINX_CONV_REUSE_PLAN | SPHINX_CONV_LIST_READY | SPHINX_CONV_INPUT_READY |
                SPHINX_CONV_VARIANT_MASK))
    return SPHINX_ERR_INVALID_ARGUMENT;
  return conv_impl(x, w, bias, residual, y, y_dtype, n, h, w_, c_in, c_out, block, block_ids, count,
                   capacity, workspace, workspace_bytes, stream, 9, nullptr, (int)flags);
}

extern "C" sphinx_status sphinx_sparse_conv3x3_gn_silu(
    const void* x, const float* scale_shift, const void* w, const float* bias, const void* residual,
    void* y, sphinx_dtype y_dtype, int32_t n, int32_t h, int32_t w_, int32_t c_in, int32_t c_out,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity, void* workspace,
    size_t workspace_bytes, sphinx_stream_t stream) {
  if (!scale_shift || (reinterpret_cast<uintptr_t>(scale_shift) & 7u)) return SPHINX_ERR_INVALID_ARGUMENT;
  return conv_impl(x, w, bias, residual, y, y_dtype, n, h, w_, c_in, c_out, block, block_ids, count,
                   capacity, workspace, workspace_bytes, stream, 9,
                   reinterpret_cast<const float2*>(scale_shift));
}

#ifdef SPHINX_TRACE
extern "C" SPHINX_API int sphinx_debug_conv_trace_reset() {
  static unsigned long long zero[1024 * 24] = {};
  return cudaMemcpyToSymbol(sphinx::g_conv_trace, zero, sizeof(zero)) == cudaSuccess ? 0 : -1;
}
extern "C" SPHINX_API int sphinx_debug_conv_trace(unsigned long long* host, int n_ctas) {
  return cudaMemcpyFromSymbol(host, sphinx::g_conv_trace, sizeof(unsigned long long) * 24 * n_ctas) ==
                 cudaSuccess ? 0 : -1;
}
#endif
