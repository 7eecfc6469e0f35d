/*
 * sphinx_oracle.h — CPU ORACLE for the Sphinx selective-refinement hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load liboracle.so.
 * The product path (paper_2511_18672_b200/, libsphinx.so) never links,
 * imports or executes anything in this directory, and this directory shares
 * no code, header, table or constant with it.
 *
 * Plain, slow, obviously-correct C99, fp64 for every floating-point step,
 * compiled with -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 * Citation keys: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * "Alg1 line k" = the k-th statement of Algorithm 1, readings R-n =
 * DESIGN.md §3.
 *
 * Every function returns 0 on success and a negative value on invalid
 * arguments ("invalid-argument").
 */
#ifndef SPHINX_ORACLE_H
#define SPHINX_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* k-decision logic K_c (Fig. k_logic). */
typedef struct {
  int32_t m;            /* number of cut points, 1..16 */
  double thr[16];       /* strictly ascending ratio cut points, left-closed */
  int32_t step[16];     /* start steps, non-decreasing */
  int32_t fallback_k;   /* k when r < thr[0] */
  int32_t k_max;        /* clamp (40) */
} oracle_klogic;

/* O1a. Pixel refinement mask M = M_op OR M_blur (Alg1 lines 9-10).
 * M_op = 1[O < tau_o] ("below 0.5"); M_blur = 1[U > tau_u[n]] (P:348,
 * "1 indicates blurry").  NaN flags the pixel (reading R-9).  U may be NULL. */
int oracle_pixel_mask(const float* O, const float* U, const float* tau_u, float tau_o,
                      int n, int hp, int wp, uint8_t* m);

/* O1b. Non-overlapping f x f max-pool of a binary grid ("downsampled using
 * max-pooling at each layer").  Requires h % f == 0 and w % f == 0. */
int oracle_maxpool(const uint8_t* in, int n, int h, int w, int f, uint8_t* out);

/* O1c. SBNet-style block tiling ("marked for refinement if it contains at
 * least one pixel"): block (by,bx) of b x b cells is 1 iff any cell
 * of it is 1.  Edge blocks are truncated (reading R-2).  out: [n][ceil(h/b)][ceil(w/b)]. */
int oracle_tile_blocks(const uint8_t* grid, int n, int h, int w, int b, uint8_t* out);

/* O1. The composite step a1, in the paper's order: pixel mask -> max-pool by
 * the VAE factor f ("downsampled by a factor of 8") -> max-pool by 2 per
 * UNet level -> block tiling per level.  masks: concatenation of the
 * n_levels block masks [n][Hb_l][Wb_l]; counts: [n][n_levels] or NULL. */
int oracle_block_mask(const float* O, const float* U, const float* tau_u, float tau_o,
                      int n, int hp, int wp, int f, int b, int n_levels,
                      uint8_t* masks, int32_t* counts);

/* O2. Start step (Alg1 lines 4-6; Eq. 2 at P:270-281; ratio P:268; k-logic P:288).
 * All arithmetic in fp64.  k[i] = -1 for invalid per-frame input
 * (t outside [0,1], Q* <= 0 or NaN; reading R-15).  logic_id may be NULL. */
int oracle_start_step(const float* q, const float* c0, const float* c1, const float* t,
                      const int32_t* logic_id, double gamma,
                      const oracle_klogic* logics, int n_logics, int n, int32_t* k);

/* Eq. 2 alone, for pins. */
double oracle_eq2(double c0, double c1, double t, double gamma);
/* oracle_eq2 over n frames (marshalling only: out[i] = oracle_eq2(c0[i], c1[i], t[i], gamma)). */
void oracle_eq2_batch(const double* c0, const double* c1, const double* t, double gamma, int n,
                      double* out);
/* k-logic lookup alone. */
int32_t oracle_select_k(const oracle_klogic* lg, double r);

/* O3. Compaction (P:352 batched blocks; Alg1 lines 17, 19).
 * select: 0 = ACTIVE (mask && (k==NULL || 0<=k[n]<=u)),
 *         1 = INACTIVE_FRAMES (k!=NULL && k[n] > u), 2 = ALL (k==NULL || k[n] >= 0).
 * ids ascending flat (n*hb+by)*wb+bx; *count = list length. */
int oracle_compact(const uint8_t* mask, int n, int hb, int wb, const int32_t* k, int u,
                   int select, int32_t* ids, int32_t* count);

/* O4. Forward noise on listed blocks (Alg1 lines 12, 19):
 * x_t = sqrt(abar[u_n]) x0 + sqrt(1 - abar[u_n]) eps, fp64, abar widened from fp32.
 * NHWC [n][h][w][c]; out (double) receives xt_in for elements not listed. */
int oracle_noise(const float* x0, const float* eps, const float* xt_in, double* out,
                 int n, int h, int w, int c, int b, const int32_t* ids, int count,
                 const int32_t* step, const float* abar, int total_steps);

/* O5. 3x3 / stride 1 / zero-pad 1 convolution on the exact bf16 values
 * (inputs are bf16 bit patterns), fp64 accumulation, for every real pixel of
 * every listed block ("batched convolution over selected blocks").
 * x: [n][h][w][cin], wt: [cout][3][3][cin], bias: [cout] fp32 or NULL.
 * y, absacc: double [n][h][w][cout]; only listed pixels are written;
 * absacc = sum |w*x| (the tolerance scale, north_star). */
int oracle_conv3x3_blocks(const uint16_t* x, const uint16_t* wt, const float* bias,
                          int n, int h, int w, int cin, int cout, int b,
                          const int32_t* ids, int count, double* y, double* absacc,
                          int n_threads);

/* O5'. The textbook dense convolution over all pixels (same definition). */
int oracle_conv3x3_dense(const uint16_t* x, const uint16_t* wt, const float* bias,
                         int n, int h, int w, int cin, int cout,
                         double* y, double* absacc, int n_threads);

/* O6. Cached scatter ("reuses cached latents ... for unrefined regions"):
 * out = active(block) ? src : cache, bit copy of elem_bytes per element.
 * src_layout 0 = FULL NHWC, active from mask/k/u exactly as oracle_compact ACTIVE;
 * src_layout 1 = COMPACT [count][b][b][c] in ids order, active = listed. */
int oracle_scatter(const void* src, int src_layout, const void* cache, void* out, int elem_bytes,
                   int n, int h, int w, int c, int b,
                   const uint8_t* mask, const int32_t* k, int u,
                   const int32_t* ids, int count);

/* NEXT-1. Deterministic DDIM update (eta = 0) on listed blocks (Alg1 line 18 D.partial_step's
 * latent update): eps_hat = (z - sqrt(abar[u]) x0_hat) / sqrt(1 - abar[u]);
 * z' = sqrt(abar[u+1]) x0_hat + sqrt(1 - abar[u+1]) eps_hat, fp64 (abar widened from fp32).
 * 0 <= u < S.  out (double) receives z for elements not listed. */
int oracle_ddim_step(const float* z, const float* x0_hat, double* out, int n, int h, int w, int c,
                     int b, const int32_t* ids, int count, int u, const float* abar,
                     int total_steps);

/* NEXT-2a. Laplacian blur map (Alg1 line 7 laplacian_var):
 * luminance Y = 0.299 R + 0.587 G + 0.114 B (reading R-23) of NHWC rgb [n][h][w][3] ->
 * 3x3 Laplacian [[0,1,0],[1,-4,1],[0,1,0]] with edge replication -> population variance of the
 * Laplacian over the window x window neighbourhood (edge replication).  fp64 out [n][h][w].
 * window odd >= 3. */
int oracle_laplacian_var(const float* rgb, int n, int h, int w, int window, double* B);

/* NEXT-2b. k x k box mean with edge replication ("smoothed"; S:217 5x5). */
int oracle_box_smooth(const double* in, int n, int h, int w, int k, double* out);

/* NEXT-2c. Otsu threshold of `count` values in [0,1] (Alg1 line 8; S:205-214;
 * reading R-24): 256 bins, bin i = (i/256, (i+1)/256] (bin 0 also holds 0); split after bin
 * k (class 0 = bins <= k, i.e. v <= (k+1)/256), between-class variance maximised EXACTLY
 * (integer histogram, 128-bit rational comparison), ties to the smaller k; tau = (k+1)/256.
 * Degenerate (one non-empty bin): tau = max value, so no value is above it. */
int oracle_otsu(const float* values, long count, float* tau);
int oracle_otsu_f64(const double* values, long count, float* tau);

/* NEXT-2. The uncertainty producer (Alg1 lines 7-8; "smoothed, normalized, and
 * inverted, followed by Otsu"): B = laplacian_var(rgb), S = box(B, smooth), per frame
 * N = (S - min S)/(max S - min S) (constant -> 0), U = 1 - N, tau[n] = otsu(U[n]).
 * U fp64 [n][h][w]; tau fp32 [n].  The blur mask is U > tau (1 = blurry). */
int oracle_uncertainty(const float* rgb, int n, int h, int w, int window, int smooth, double* U,
                       float* tau);

/* NEXT-3 helpers.  Round a double to bfloat16 bits, nearest-even, directly from fp64. */
uint16_t oracle_bf16_rne(double v);

/* NEXT-3a. GroupNorm statistics over the full current map (reading R-26): per (frame i,
 * group g) mean and population variance of the h*w*c/G values of channels
 * [g*c/G, (g+1)*c/G), two passes in fp64.  mean, var: [n][groups]. */
int oracle_gn_stats(const double* x, int n, int h, int w, int c, int groups, double* mean,
                    double* var);

/* NEXT-3b. t = gamma[ch] (x - mean)/sqrt(var + eps) + beta[ch]; a = SiLU(t) = t/(1+exp(-t)),
 * every pixel (P:333 ResNet block normalisation/activation; R-26).  t may be NULL. */
int oracle_gn_silu(const double* x, int n, int h, int w, int c, int groups, const double* mean,
                   const double* var, const float* gamma, const float* beta, double eps,
                   double* t, double* a);

/* NEXT-3. Block-sparse ResNet block with latent reuse (R-26, R-27):
 *   a1 = bf16(SiLU(GN1(x)));  h = listed ? bf16(conv(a1;w1)+b1) : h_cache;
 *   a2 = bf16(SiLU(GN2(h)));  y = listed ? x + conv(a2;w2)+b2 : y_cache.
 * GN statistics over the full current maps.  See sphinx_oracle.c for the outputs. */
int oracle_resblock(const uint16_t* x, const uint16_t* h_cache, const double* y_cache,
                    const uint16_t* w1, const float* b1, const uint16_t* w2, const float* b2,
                    const float* g1, const float* be1, const float* g2, const float* be2,
                    int groups, double eps, int n, int h, int w, int c, int b,
                    const int32_t* ids, int count, double* a1_pre, uint16_t* a1_out,
                    double* h_pre, double* h_abs, uint16_t* h_out, double* a2_pre,
                    uint16_t* a2_out, double* y, double* y_abs, int n_threads);

/* NEXT-4. Frame-sparse temporal attention with the latent (K/V) cache (R-28):
 *   qkv = listed ? bf16(Wqkv x + bqkv) : qkv_cache;  per pixel and head, o[n] = softmax over
 *   the T frames m of n's sequence of q_n.k_m/sqrt(d), times v_m;  y = listed ? x + Wo bf16(o)
 *   + bo : y_cache.  See sphinx_oracle.c for the outputs. */
int oracle_temporal_attn(const uint16_t* x, const uint16_t* qkv_cache, const double* y_cache,
                         const uint16_t* wqkv, const float* bqkv, const uint16_t* wo,
                         const float* bo, int n, int h, int w, int c, int heads, int T, int b,
                         const int32_t* ids, int count, double* qkv_pre, uint16_t* qkv_out,
                         double* qkv_abs, double* o_pre, uint16_t* o_out, double* y, double* y_abs);

#ifdef __cplusplus
}
#endif
#endif
