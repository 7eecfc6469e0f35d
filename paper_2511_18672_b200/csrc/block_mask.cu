// block_mask.cu — step (1): per-pixel maps -> per-level block masks, counts, start steps.
//
// P:346-352 (opacity + blur masks, OR, block tiling), P:447 (tau_o = 0.5, "below"),
// P:489 (max-pool by the VAE factor and per UNet level), Alg1 lines 4-10, Eq. 2.
//
// Design: the pass over the two fp32 pixel maps is the only HBM-heavy
// part (8 B / pixel).  Kernel A streams the maps with 128-bit coalesced loads; each
// CTA covers a strip of rows inside one level-0 block row, every thread owns a fixed
// column vector so its level-0 block column is fixed, and the "any flagged pixel"
// reduction is a per-thread OR followed by a racy-but-idempotent byte store of 1.
// Level l >= 1 blocks nest exactly over 2^l x 2^l level-0 blocks (b*f*2^l pixel
// footprints), so kernel B derives them from the level-0 mask, counts per frame with
// __syncthreads_count, and its thread 0 evaluates the start step in fp64.
#include "common.cuh"

namespace sphinx {

struct KLogicSet {
  sphinx_klogic lg[SPHINX_MAX_LOGICS];
  int32_t n_logics;
  double gamma;
  int32_t enabled;
};

template <int V>
__global__ void __launch_bounds__(512) block_mask_l0_kernel(
    const float* __restrict__ O, const float* __restrict__ U, const float* __restrict__ tau_u,
    float tau_o, int hp, int wp, int cell_px, int hb0, int wb0, int rows_per_cta, int splits,
    uint8_t* __restrict__ mask0) {
  pdl_wait();
  pdl_trigger();
  const int cta = blockIdx.x;
  const int s = cta % splits;
  const int rest = cta / splits;
  const int by = rest % hb0;
  const int n = rest / hb0;
  const int y0 = by * cell_px + s * rows_per_cta;
  const int y1 = min(min(y0 + rows_per_cta, (by + 1) * cell_px), hp);
  if (y0 >= y1) return;
  const float tu = U ? __ldg(tau_u + n) : 0.0f;
  const int nvec = wp / V;
  const size_t frame_off = (size_t)n * hp * wp;
  for (int cv = threadIdx.x; cv < nvec; cv += blockDim.x) {
    const int bx = (cv * V) / cell_px;  // V divides cell_px: the V pixels share a block
    bool flag = false;
    int y = y0 + threadIdx.y;
#pragma unroll 4
    for (; y < y1; y += blockDim.y) {
      const size_t off = frame_off + (size_t)y * wp + (size_t)cv * V;
      if constexpr (V == 4) {
        const float4 o = __ldg(reinterpret_cast<const float4*>(O + off));
        // !(o >= tau): NaN refines (R-9), equality does not (R-8)
        flag |= !(o.x >= tau_o) | !(o.y >= tau_o) | !(o.z >= tau_o) | !(o.w >= tau_o);
        if (U) {
          const float4 u = __ldg(reinterpret_cast<const float4*>(U + off));
          flag |= !(u.x <= tu) | !(u.y <= tu) | !(u.z <= tu) | !(u.w <= tu);
        }
      } else {
        const float o = __ldg(O + off);
        flag |= !(o >= tau_o);
        if (U) flag |= !(__ldg(U + off) <= tu);
      }
    }
    if (flag) mask0[((size_t)n * hb0 + by) * wb0 + bx] = 1;
  }
}

// Eq. 2 + ratio + k-logic lookup, fp64, correctly rounded
// operations only (no FMA contraction) so that k is bit-identical to the oracle (R-16).
__device__ int32_t start_step_one(float qf, float c0f, float c1f, float tf, int lid,
                                  const KLogicSet& ks) {
  const double t = (double)tf, c0 = (double)c0f, c1 = (double)c1f, q = (double)qf;
  if (lid < 0 || lid >= ks.n_logics || !(t >= 0.0 && t <= 1.0)) return -1;
  const double g = ks.gamma;
  double f;
  if (c1 >= c0) {
    f = (g == 1.0) ? t : (g == 0.5) ? __dsqrt_rn(t) : pow(t, g);
  } else {
    const double omt = __dsub_rn(1.0, t);
    const double p = (g == 1.0) ? omt : (g == 0.5) ? __dsqrt_rn(omt) : pow(omt, g);
    f = __dsub_rn(1.0, p);
  }
  const double qs = __dadd_rn(c0, __dmul_rn(__dsub_rn(c1, c0), f));
  if (!(qs > 0.0)) return -1;
  const double r = __ddiv_rn(q, qs);
  if (r != r) return -1;
  const sphinx_klogic& lg = ks.lg[lid];
  int32_t k = lg.fallback_k;
  for (int i = 0; i < lg.m; ++i)
    if (lg.thr[i] <= r) k = lg.step[i];
  return k > lg.k_max ? lg.k_max : k;
}

struct LevelPtrs {
  uint8_t* mask[4];
  int hb[4];
  int wb[4];
};

__global__ void __launch_bounds__(256) block_mask_tail_kernel(
    LevelPtrs lv, int n_levels, int32_t* __restrict__ counts, const __grid_constant__ KLogicSet ks,
    const float* __restrict__ q, const float* __restrict__ c0, const float* __restrict__ c1,
    const float* __restrict__ t, const int32_t* __restrict__ logic_id,
    int32_t* __restrict__ start_step) {
  pdl_wait();
  pdl_trigger();
  const int n = blockIdx.x;
  const int hb0 = lv.hb[0], wb0 = lv.wb[0];
  const uint8_t* m0 = lv.mask[0] + (size_t)n * hb0 * wb0;
  for (int l = 0; l < n_levels; ++l) {
    const int hb = lv.hb[l], wb = lv.wb[l], span = 1 << l;
    uint8_t* ml = lv.mask[l] + (size_t)n * hb * wb;
    int local = 0;
    for (int j = threadIdx.x; j < hb * wb; j += blockDim.x) {
      uint8_t v;
      if (l == 0) {
        v = m0[j];
      } else {
        const int by = j / wb, bx = j % wb;
        v = 0;
        for (int yy = by * span; yy < min((by + 1) * span, hb0); ++yy)
          for (int xx = bx * span; xx < min((bx + 1) * span, wb0); ++xx) v |= m0[yy * wb0 + xx];
        ml[j] = v;
      }
      local += v;
    }
    __shared__ int acc;
    if (threadIdx.x == 0) acc = 0;
    __syncthreads();
    if (local) atomicAdd(&acc, local);
    __syncthreads();
    if (threadIdx.x == 0 && counts) counts[n * n_levels + l] = acc;
    __syncthreads();
  }
  if (ks.enabled && threadIdx.x == 0)
    start_step[n] = start_step_one(q[n], c0[n], c1[n], t[n], logic_id ? logic_id[n] : 0, ks);
}

}  // namespace sphinx

using namespace sphinx;

extern "C" sphinx_status sphinx_block_mask(const float* opacity, const float* uncertainty,
                                           const float* tau_u, float tau_o, int32_t n, int32_t hp,
                                           int32_t wp, int32_t f, int32_t b, int32_t n_levels,
                                           uint8_t* const* block_mask, int32_t* active_count,
                                           const sphinx_start_args* ss, int32_t* start_step,
                                           sphinx_stream_t stream) {
  if (!opacity || !block_mask || n <= 0 || hp <= 0 || wp <= 0 || f <= 0 || b <= 0 || b > 64)
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (n_levels < 1 || n_levels > 4 || !(tau_o >= 0.0f && tau_o <= 1.0f))
    return SPHINX_ERR_INVALID_ARGUMENT;
  if (uncertainty && !tau_u) return SPHINX_ERR_INVALID_ARGUMENT;
  if (hp % f || wp % f) return SPHINX_ERR_INVALID_ARGUMENT;
  const int h0 = hp / f, w0 = wp / f, div = 1 << (n_levels - 1);
  if (h0 % div || w0 % div) return SPHINX_ERR_INVALID_ARGUMENT;
  for (int l = 0; l < n_levels; ++l)
    if (!block_mask[l]) return SPHINX_ERR_INVALID_ARGUMENT;
  KLogicSet ks{};
  if (ss) {
    if (!start_step || !ss->q_reg || !ss->c0 || !ss->c1 || !ss->t || !ss->logics)
      return SPHINX_ERR_INVALID_ARGUMENT;
    if (!(ss->gamma > 0.0f && ss->gamma <= 1.0f)) return SPHINX_ERR_INVALID_ARGUMENT;
    if (ss->n_logics < 1 || ss->n_logics > SPHINX_MAX_LOGICS) return SPHINX_ERR_INVALID_ARGUMENT;
    for (int j = 0; j < ss->n_logics; ++j) {
      const sphinx_klogic& lg = ss->logics[j];
      if (lg.m < 1 || lg.m > 16) return SPHINX_ERR_INVALID_ARGUMENT;
      for (int i = 1; i < lg.m; ++i)
        if (!(lg.thr[i - 1] < lg.thr[i]) || lg.step[i - 1] > lg.step[i])
          return SPHINX_ERR_INVALID_ARGUMENT;
      ks.lg[j] = lg;
    }
    ks.n_logics = ss->n_logics;
    ks.gamma = (double)ss->gamma;
    ks.enabled = 1;
  }
  int sms = 0;
  sphinx_status st = check_device(&sms);
  if (st != SPHINX_OK) return st;

  const int cell_px = b * f;  // pixel footprint of one level-0 block
  const int hb0 = cdiv(h0, b), wb0 = cdiv(w0, b);
  LevelPtrs lv{};
  for (int l = 0; l < n_levels; ++l) {
    lv.mask[l] = block_mask[l];
    lv.hb[l] = cdiv(h0 >> l, b);
    lv.wb[l] = cdiv(w0 >> l, b);
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(block_mask[0], 0, (size_t)n * hb0 * wb0, s);
  if (e != cudaSuccess) return cuda_fail(e);

  const bool vec = (wp % 4 == 0) && (cell_px % 4 == 0) && aligned16(opacity) &&
                   (!uncertainty || aligned16(uncertainty));
  const int V = vec ? 4 : 1;
  const int nvec = wp / V;
  int bdx = nvec < 256 ? nvec : 256;
  int bdy = 512 / bdx;
  if (bdy < 1) bdy = 1;
  const int rows_per_cta = 4 * bdy;
  int splits = cdiv(cell_px, rows_per_cta);
  const dim3 block(bdx, bdy);
  const int grid = n * hb0 * splits;
  uint8_t* m0 = block_mask[0];
  e = launch_k(vec ? block_mask_l0_kernel<4> : block_mask_l0_kernel<1>, dim3(grid), block, 0, s,
               opacity, uncertainty, tau_u, tau_o, (int)hp, (int)wp, cell_px, hb0, wb0, rows_per_cta,
               splits, m0);
  if (e != cudaSuccess) return cuda_fail(e);
  const float* q = ss ? ss->q_reg : nullptr;
  const float* c0 = ss ? ss->c0 : nullptr;
  const float* c1 = ss ? ss->c1 : nullptr;
  const float* tt = ss ? ss->t : nullptr;
  const int32_t* lid = ss ? ss->logic_id : nullptr;
  e = launch_k(block_mask_tail_kernel, dim3(n), dim3(256), 0, s, lv, (int)n_levels, active_count, ks,
               q, c0, c1, tt, lid, start_step);
  if (e != cudaSuccess) return cuda_fail(e);
  return SPHINX_OK;
}
