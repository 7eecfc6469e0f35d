/*
 * sphinx.h — C ABI of the B200-native (sm_100a) Sphinx selective-refinement hot path.
 *
 * Paper: "Sphinx: Efficiently Serving Novel View Synthesis using Regression-Guided
 * Selective Refinement" (arXiv 2511.18672).  Citation keys: P:n = PAPER.md line n,
 * S:n = SPEC.md line n, "Alg1 line k" = k-th statement of Algorithm 1,
 * R-n = reading n in DESIGN.md §3.
 *
 * The five entry points are the five steps of the hot path (BASELINE north_star):
 *   (1) sphinx_block_mask      per-pixel maps -> per-level block masks + per-frame start step
 *   (2) sphinx_compact_blocks  block mask (+ frame eligibility) -> ascending block-id list
 *   (3) sphinx_noise_inject    x_t = sqrt(abar) x0 + sqrt(1-abar) eps on listed blocks
 *   (4) sphinx_sparse_conv3x3  halo gather + 3x3 implicit GEMM (tcgen05/TMEM) on listed blocks
 *   (5) sphinx_scatter_cached  out = active ? computed : latent cache
 * and the SURVEY §8(f) "next" rows built on them: sphinx_ddim_step (NEXT-1),
 * sphinx_uncertainty_map (NEXT-2), and the block-sparse ResNet block (NEXT-3:
 * sphinx_gn_block_stats, sphinx_gn_silu, sphinx_sparse_conv3x3_residual,
 * sphinx_sparse_resblock), and the temporal-attention latent cache (NEXT-4:
 * sphinx_sparse_pointwise, sphinx_temporal_attention, sphinx_temporal_block).
 *
 * CONVENTIONS (all entry points)
 *  - Ownership: every array pointer is caller-owned memory.  "device" pointers must be
 *    CUDA device (or managed) memory of the current device; "host" pointers are read
 *    synchronously before return.  The library never allocates, frees or retains
 *    caller pointers after it returns.
 *  - Asynchrony: arguments visible on the host are validated synchronously; the work is
 *    then enqueued on `stream` (NULL = legacy default stream) with no implicit
 *    synchronisation.  No call reads device memory on the host (device counts stay on
 *    the device), so every call is CUDA-graph capturable.
 *  - Errors: a non-zero sphinx_status is returned before anything is enqueued, except
 *    SPHINX_ERR_CUDA which may follow a failed launch.  Per-frame data errors that live
 *    in device memory cannot be reported synchronously; they are encoded in outputs as
 *    documented per call (start_step = -1).
 *  - Layouts: feature maps and latents are NHWC, C innermost (channels-last), densely
 *    packed.  Block (n, by, bx) of a level with Hb x Wb blocks has flat id
 *    (n*Hb + by)*Wb + bx (S:192 frame-major, row-major; R-20).  Edge blocks are
 *    truncated at the image border (R-2).
 *  - Determinism: outputs are bit-reproducible run to run: no floating-point
 *    atomics, list order defined by the flat id.
 *  - Thread safety: no global mutable state besides the thread-local last CUDA error.
 */
#ifndef SPHINX_H
#define SPHINX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SPHINX_API __attribute__((visibility("default")))
#else
#define SPHINX_API
#endif

typedef struct CUstream_st* sphinx_stream_t; /* == cudaStream_t */

typedef enum {
  SPHINX_OK = 0,
  SPHINX_ERR_INVALID_ARGUMENT = 1, /* null pointer, non-positive size, inconsistent dims,
                                      tau_o outside [0,1], gamma outside (0,1], bad k-logic,
                                      S < 2 ... */
  SPHINX_ERR_UNSUPPORTED = 2,      /* valid but not implemented on sm_100a (e.g. C % 8 != 0,
                                      block > 16); there is no fallback */
  SPHINX_ERR_CUDA = 3,             /* launch / driver failure: see sphinx_last_cuda_error() */
  SPHINX_ERR_DEVICE = 4            /* current device is not sm_100 */
} sphinx_status;

typedef enum { SPHINX_BF16 = 0, SPHINX_F32 = 1 } sphinx_dtype;

/* Which blocks compaction selects (Alg1 lines 17-19). */
typedef enum {
  SPHINX_SELECT_ACTIVE = 0,          /* mask == 1 and 0 <= k[n] <= u: A_u = 1[k <= u] (Alg1 line 17) */
  SPHINX_SELECT_INACTIVE_FRAMES = 1, /* every block of frames with k[n] > u: resampled (Alg1 line 19) */
  SPHINX_SELECT_ALL = 2,             /* every block of frames with k[n] >= 0 (or all if k == NULL) */
  SPHINX_SELECT_NOISE = 3            /* ACTIVE | INACTIVE_FRAMES: every block the step's noise pass
                                        touches (Alg1 lines 12 and 19 in one list); needs mask and k */
} sphinx_select;

typedef enum { SPHINX_SRC_FULL = 0, SPHINX_SRC_COMPACT = 1 } sphinx_src_layout;

/* k-decision logic K_c (Fig. k_logic).
 * k = step[i] for the largest i with thr[i] <= r (left-closed); fallback_k when
 * r < thr[0]; then min(k, k_max) ("We set the largest k=40"). */
typedef struct {
  int32_t m;         /* number of cut points, 1..16 */
  double thr[16];    /* strictly ascending ratio cut points */
  int32_t step[16];  /* non-decreasing start steps */
  int32_t fallback_k;
  int32_t k_max;
} sphinx_klogic;

#define SPHINX_MAX_LOGICS 8

/* Per-frame inputs of the start-step map (Alg1 lines 3-6; Eq. 2). */
typedef struct {
  const float* q_reg;        /* [N] device: no-reference score Q_reg of the regression frame */
  const float* c0;           /* [N] device: score of input view I0 of the frame's request */
  const float* c1;           /* [N] device: score of input view I1 */
  const float* t;            /* [N] device: normalised target position t in [0,1] (Eq. 2; R-12) */
  const int32_t* logic_id;   /* [N] device: cluster index c selecting the k-logic, or NULL = 0;
                                a negative id marks a conditioning (input) frame: k = -1 (R-14) */
  float gamma;               /* Eq. 2 exponent, in (0,1] */
  const sphinx_klogic* logics; /* host array of n_logics tables, copied by value into the launch */
  int32_t n_logics;          /* 1..SPHINX_MAX_LOGICS */
} sphinx_start_args;

SPHINX_API int32_t sphinx_abi_version(void);      /* returns SPHINX_ABI_VERSION */
SPHINX_API int32_t sphinx_last_cuda_error(void);  /* cudaError_t of the last SPHINX_ERR_CUDA on this thread */
#define SPHINX_ABI_VERSION 10

/* ---------------------------------------------------------------------------------
 * (1) Block mask + start step.
 * P:346 opacity mask M_op = 1[O < tau_o] ("opacity values below 0.5");
 * P:348 blur mask (1 = blurry) from the uncertainty map U and per-frame Otsu
 * threshold tau_u[n] (R-10: tau_u is an input); P:350 M = M_op OR M_blur;
 * P:489 M is max-pooled by the VAE factor f and by 2 at every UNet level;
 * P:352 block (n,by,bx) of level l is active iff it contains >= 1 masked cell.
 * Equivalently: active iff some pixel (i,j) with by*b*f*2^l <= i < (by+1)*b*f*2^l
 * (clipped to Hp), same for j, has !(O >= tau_o) || (U && !(U <= tau_u[n]))
 * (NaN refines, R-9; strict inequalities, R-8).
 *
 * opacity       [N][Hp][Wp] fp32 device.
 * uncertainty   [N][Hp][Wp] fp32 device, or NULL (then tau_u is ignored).
 * tau_u         [N] fp32 device.
 * tau_o         opacity threshold in [0,1] (0.5).
 * px_per_cell   f: image pixels per level-0 latent cell (8 = VAE factor; 1 allowed).
 * block         b in cells, same at every level, 1..64.
 * n_levels      1..4; level l has H_l = (Hp/f) >> l; requires Hp % f == 0 and
 *               (Hp/f) % 2^(n_levels-1) == 0 (and the same for W).
 * block_mask    HOST array of n_levels DEVICE pointers; level l is u8 [N][ceil(H_l/b)][ceil(W_l/b)]
 *               and receives 0/1.
 * active_count  [N][n_levels] int32 device, or NULL.
 * ss            host struct or NULL (skip the start-step map).
 * start_step    [N] int32 device out (required if ss != NULL): k_n = K_c(q/Q*) per Alg1 lines 4-6
 *               in fp64; -1 if t outside [0,1], Q* <= 0 / NaN, or logic_id out of range (R-15).
 *               gamma == 1 and gamma == 0.5 use t and sqrt(t) (exact); other gamma use pow (R-16).
 * ------------------------------------------------------------------------------- */
SPHINX_API sphinx_status sphinx_block_mask(const float* opacity, const float* uncertainty, const float* tau_u,
                                float tau_o, int32_t n, int32_t hp, int32_t wp,
                                int32_t px_per_cell, int32_t block, int32_t n_levels,
                                uint8_t* const* block_mask, int32_t* active_count,
                                const sphinx_start_args* ss, int32_t* start_step,
                                sphinx_stream_t stream);

/* ---------------------------------------------------------------------------------
 * (2) Compaction ("batched convolution over selected blocks").
 * Emits, in ascending flat-id order, the ids of the blocks selected by `select`
 * (see sphinx_select; k[n] < 0 excludes frame n from every selection, R-14), and
 * writes their number to *count.  The count stays on the device.
 *
 * block_mask   u8 [N][hb][wb] device (may be NULL only for SELECT_INACTIVE_FRAMES / SELECT_ALL).
 * start_step   int32 [N] device or NULL (all frames eligible; required for INACTIVE_FRAMES).
 * step_u       the denoising step u of Alg1's loop.
 * block_ids    int32 [N*hb*wb] device out (capacity = N*hb*wb).
 * count        int32 device scalar out.
 * ------------------------------------------------------------------------------- */
SPHINX_API sphinx_status sphinx_compact_blocks(const uint8_t* block_mask, int32_t n, int32_t hb, int32_t wb,
                                    const int32_t* start_step, int32_t step_u, sphinx_select select,
                                    int32_t* block_ids, int32_t* count, sphinx_stream_t stream);

/* Several compactions in ONE launch (one CTA per job; each job exactly as
 * sphinx_compact_blocks with the same arguments): e.g. the ACTIVE lists of every UNet level and
 * the INACTIVE_FRAMES list of one step.  jobs: host array, copied into the launch. */
#define SPHINX_MAX_COMPACT_JOBS 8
typedef struct {
  const uint8_t* block_mask;  /* device u8 [n][hb][wb] (may be NULL for INACTIVE_FRAMES / ALL) */
  int32_t n, hb, wb;
  const int32_t* start_step;  /* device [n] or NULL */
  int32_t step_u;
  sphinx_select select;
  int32_t* block_ids;         /* device out, capacity n*hb*wb */
  int32_t* count;             /* device out */
} sphinx_compact_job;
SPHINX_API sphinx_status sphinx_compact_blocks_batch(const sphinx_compact_job* jobs, int32_t n_jobs,
                                                     sphinx_stream_t stream);

/* ---------------------------------------------------------------------------------
 * Multi-GPU data plane (P:333 frames are the independent units; north_star "balanced
 * by active-block count"): the frame -> rank plan, computed on the device by every rank from the
 * all-gathered masks and start steps, identical on every rank (deterministic):
 *   cost[f] = sum_l count_l[f] * C_l^2, count_l[f] = blocks with mask 1 in frame f at level l if
 *             0 <= k[f] <= u, else 0 (the executed MMA work of frame f at this step);
 *   frames by cost descending (frame id ascending on ties) each go to the least-loaded rank
 *   (lowest rank on ties): longest processing time first.
 * block_mask        HOST array of n_levels DEVICE pointers, u8 [n][blocks_per_frame[l]].
 * blocks_per_frame  HOST [n_levels]: hb_l * wb_l.      channels  HOST [n_levels]: C_l.
 * start_step        int32 [n] device (all ranks' frames).   step_u  u of Alg1's loop.
 * owner             int32 [n] device: the rank that owns frame f's request (receives its blocks).
 * world, rank       ranks and this rank (1 <= world <= 32; n <= 4096).
 * Outputs (device): k_mine int32 [n] = start_step of this rank's frames, -1 elsewhere (the input of
 * this rank's compaction); rank_of int32 [n]; load int64 [world] (sum of the ranks' costs);
 * pair int32 [n_levels][world][world] = level-l blocks rank s computes for frames rank o owns;
 * recv int32 [n_levels] = blocks this rank receives per level (sum over s != rank of pair[l][s][rank]).
 * One 1024-thread CTA; no host synchronisation (the host reads pair back only to size the NCCL
 * send / recv of the owner gather).
 * ------------------------------------------------------------------------------- */
/* Halo windows of listed blocks, copied map to map (same NHWC geometry [n][h][w][c], bf16 or fp32):
 * for every listed block the pixels a 3x3 conv over it reads -- rows [by*b-1, by*b+b+1) x columns
 * [bx*b-1, bx*b+b+1), clipped to the image, all channels -- go from src to dst; nothing else of dst
 * is written.  src may be PINNED HOST memory (read by the GPU over PCIe through unified addressing):
 * a serving loop whose level features arrive from the host then moves only what its convs read
 * (refinement touches the selected blocks; their 1-pixel ring is the conv's halo).
 * block_ids/count/capacity: a list of this geometry (device).  c * elem % 16 == 0; src, dst 16-B
 * aligned.  Bit copy. */
SPHINX_API sphinx_status sphinx_gather_halo_windows(const void* src, void* dst, sphinx_dtype dtype, int32_t n,
                                                    int32_t h, int32_t w, int32_t c, int32_t block,
                                                    const int32_t* block_ids, const int32_t* count,
                                                    int32_t capacity, sphinx_stream_t stream);

SPHINX_API sphinx_status sphinx_shard_plan(uint8_t* const* block_mask, const int32_t* blocks_per_frame,
                                           const int32_t* channels, int32_t n_levels, int32_t n,
                                           const int32_t* start_step, int32_t step_u, const int32_t* owner,
                                           int32_t world, int32_t rank, int32_t* k_mine, int32_t* rank_of,
                                           int64_t* load, int32_t* pair, int32_t* recv,
                                           sphinx_stream_t stream);

/* ---------------------------------------------------------------------------------
 * (3) Forward noise on listed blocks (Alg1 line 12 add_noise(Z0, k_min); line 19
 * resampling of inactive frames to u+1; formula S:303 / north_star):
 *   x_t = sqrt(abar[u_n]) * x0 + sqrt(1 - abar[u_n]) * eps     (fp32)
 * for every element of every real pixel of every listed block; every other element of
 * x_t is left untouched.  u = 0 is the noisiest step, u = S clean (R-5).
 *
 * x0, eps, x_t  NHWC fp32 [N][h][w][c] device; x_t may alias x0 (in place).
 * block_ids/count/capacity  a list produced by sphinx_compact_blocks for this geometry.
 * step          int32 [N] device: u_n per frame; a frame with u_n outside [0,S] is left untouched.
 * abar          fp32 [S+1] device; total_steps = S >= 2.  eps is caller-generated (R-6).
 * ------------------------------------------------------------------------------- */
SPHINX_API sphinx_status sphinx_noise_inject(const float* x0, const float* eps, float* x_t,
                                  int32_t n, int32_t h, int32_t w, int32_t c, int32_t block,
                                  const int32_t* block_ids, const int32_t* count, int32_t capacity,
                                  const int32_t* step, const float* abar, int32_t total_steps,
                                  sphinx_stream_t stream);
/* The step's whole noise pass in one launch (Alg1 line 12 for active frames, line 19 for inactive
 * ones): for every listed block of frame n, u_n = start_step[n] if 0 <= start_step[n] <= step_u
 * (active: noised to its start step k) and u_n = step_u + 1 if start_step[n] > step_u (inactive:
 * resampled); frames with start_step < 0 are untouched.  Use with a SPHINX_SELECT_NOISE list.
 * Same arguments and results as two sphinx_noise_inject calls over the ACTIVE and
 * INACTIVE_FRAMES lists with those steps; step_u + 1 <= total_steps. */
SPHINX_API sphinx_status sphinx_noise_inject_step(const float* x0, const float* eps, float* x_t,
                                       int32_t n, int32_t h, int32_t w, int32_t c, int32_t block,
                                       const int32_t* block_ids, const int32_t* count, int32_t capacity,
                                       const int32_t* start_step, int32_t step_u, const float* abar,
                                       int32_t total_steps, sphinx_stream_t stream);

/* ---------------------------------------------------------------------------------
 * (4) Block-sparse 3x3 convolution ("tiles the feature maps into blocks ...
 * enables batched convolution over selected blocks"):
 *   y[n,p,co] = bias[co] + sum_{dy,dx in {-1,0,1}} sum_ci W[co][dy+1][dx+1][ci] * x[n,p+(dy,dx),ci]
 * with x = 0 outside the image (R-17), computed (bf16 x bf16, fp32 accumulation on the
 * tcgen05 tensor cores) for every real pixel of every listed block and written into the
 * full-resolution y at its own position (the scatter of computed blocks is fused).
 * Halo pixels are read from the full map as-is: inactive blocks there hold cached values
 * (P:352 latent reuse).  Pixels of unlisted blocks are NOT written (persistent-buffer
 * mode: pre-fill y with the cache, R-17).
 *
 * x      bf16 NHWC [N][h][w][c_in] device, 16-byte aligned.
 * w      bf16 [c_out][3][3][c_in] device (OHWI, R-19; torch OIHW -> permute(0,2,3,1)).
 * bias   fp32 [c_out] device or NULL.
 * y      NHWC [N][h][w][c_out] device, y_dtype bf16 or fp32; must not alias x.
 * c_in % 8 == 0, c_out % 8 == 0, block in {4, 8}  (else SPHINX_ERR_UNSUPPORTED).
 * block_ids/count/capacity  list from sphinx_compact_blocks (capacity = N*Hb*Wb upper bound).
 * workspace  device scratch of sphinx_conv_workspace_size(...) bytes, 256-byte aligned, ZERO-
 *            INITIALISED ONCE by the caller (the kernel leaves it zeroed); one per stream.  It
 *            holds the split-K arrival counters and fp32 partial tiles (used when the device-side
 *            block count leaves the last wave of tiles partial: the tail is split along K and
 *            reduced in a fixed order, so results stay bit-reproducible) and, for maps with
 *            H % 8 or W % 8 != 0, the edge-class plan (full / bottom-edge / right-edge blocks).
 *            NULL disables both (the conv is still complete and exact, only slower).
 * ------------------------------------------------------------------------------- */
SPHINX_API sphinx_status sphinx_sparse_conv3x3(const void* x, const void* w, const float* bias,
                                    void* y, sphinx_dtype y_dtype,
                                    int32_t n, int32_t h, int32_t w_, int32_t c_in, int32_t c_out,
                                    int32_t block, const int32_t* block_ids, const int32_t* count,
                                    int32_t capacity, void* workspace, size_t workspace_bytes,
                                    sphinx_stream_t stream);
SPHINX_API size_t sphinx_conv_workspace_size(int32_t n, int32_t h, int32_t w_, int32_t c_in, int32_t c_out,
                                  int32_t block);

/* sphinx_sparse_conv3x3 with an optional residual (as in _residual, NULL = none) and flags:
 * SPHINX_CONV_REUSE_PLAN  the workspace already holds the edge-class plan of THIS list (the
 *                         caller's previous conv on this stream used the same block_ids, count and
 *                         workspace, e.g. the second conv of a ResNet block): skip recomputing it.
 *                         Undefined results if the list changed in between.
 * SPHINX_CONV_LIST_READY  block_ids / count (and a reused plan) were written by a kernel that ran
 *                         BEFORE the immediately preceding kernel on this stream (e.g. compaction
 *                         earlier in the step): the conv reads them and starts its weight loads
 *                         before waiting for the preceding kernel (programmatic dependent launch);
 *                         its activation loads and stores still wait.  Ignored when the call
 *                         launches its own edge plan. */
#define SPHINX_CONV_REUSE_PLAN 1
#define SPHINX_CONV_LIST_READY 2
/* SPHINX_CONV_INPUT_READY (with LIST_READY): x was also written before the preceding kernel (e.g.
 * a level's input features): the activation loads and MMAs may run while the preceding kernel
 * drains; the epilogue (stores) still waits for it, so the kernel completes after it. */
#define SPHINX_CONV_INPUT_READY 4
/* PDL ordering: a LIST_READY conv signals its dependents only after its own epilogue has waited
 * for its predecessor, so any chain of LIST_READY convs (e.g. edge_plan(L1) -> conv(L0) ->
 * conv(L1, REUSE_PLAN | LIST_READY)) keeps "every kernel before the preceding one is complete"
 * transitively. */

/* Kernel-variant overrides (tests and tuning only; the default choice is the measured-fastest
 * one).  Every variant computes the same result within the conv bar and is
 * bit-reproducible on its own. */
#define SPHINX_CONV_FORCE_CG1 (1 << 8)      /* 1-SM tcgen05 kernel (cta_group::1) */
#define SPHINX_CONV_FORCE_HALO (1 << 9)     /* halo-staged A even when one wave fits (b = 8) */
#define SPHINX_CONV_FORCE_PERTAP (1 << 10)  /* per-tap A windows instead of halo staging */
#define SPHINX_CONV_NO_SPLIT (1 << 11)      /* never split K (one pass per tile) */
#define SPHINX_CONV_NO_EDGE (1 << 12)       /* no edge-class packing of partial edge blocks */
#define SPHINX_CONV_NO_STREAMK (1 << 13)    /* tail split-K only, never stream-K */
#define SPHINX_CONV_FORCE_STREAMK (1 << 14) /* stream-K whenever the workspace allows it */
#define SPHINX_CONV_VARIANT_MASK (0x7f << 8)

/* Computes the edge-class plan of a list into a conv workspace (what a conv call without
 * SPHINX_CONV_REUSE_PLAN does first), so that it can run early in a step and every conv over the
 * list passes SPHINX_CONV_REUSE_PLAN (| SPHINX_CONV_LIST_READY).  A no-op for maps without partial
 * edge blocks or block != 8. */
SPHINX_API sphinx_status sphinx_conv_edge_plan(const int32_t* block_ids, const int32_t* count, int32_t n,
                                               int32_t h, int32_t w_, int32_t block, int32_t capacity,
                                               void* workspace, size_t workspace_bytes,
                                               sphinx_stream_t stream);
SPHINX_API sphinx_status sphinx_sparse_conv3x3_ex(
    const void* x, const void* w, const float* bias, const void* residual, void* y,
    sphinx_dtype y_dtype, int32_t n, int32_t h, int32_t w_, int32_t c_in, int32_t c_out,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity,
    void* workspace, size_t workspace_bytes, int32_t flags, sphinx_stream_t stream);

/* ---------------------------------------------------------------------------------
 * (5) Cached scatter ("reuses cached latents from the last full denoising step for
 * unrefined regions"):  out[n,y,x,:] = active(n, y/b, x/b) ? src[...] : cache[n,y,x,:]
 * as a bit copy (NaN payloads and -0 preserved).
 *
 * src_layout FULL:    src NHWC [N][h][w][c]; active(n,by,bx) = block_mask[n][by][bx] &&
 *                     (start_step == NULL || 0 <= start_step[n] <= step_u)  (same predicate as
 *                     SELECT_ACTIVE).  out may alias src: then only inactive blocks are written.
 * src_layout COMPACT: src [count][b][b][c] holds the listed blocks in list order
 *                     (block_ids/count required, ascending); active = listed.
 * cache, out  NHWC device; dtype selects the element width (bf16 = 2 B, fp32 = 4 B);
 *             c * elem_size must be a multiple of 16 bytes; out must not alias cache.
 * ------------------------------------------------------------------------------- */
SPHINX_API sphinx_status sphinx_scatter_cached(const void* src, sphinx_src_layout src_layout,
                                    const void* cache, void* out, sphinx_dtype dtype,
                                    int32_t n, int32_t h, int32_t w, int32_t c, int32_t block,
                                    const uint8_t* block_mask, const int32_t* start_step,
                                    int32_t step_u, const int32_t* block_ids, const int32_t* count,
                                    sphinx_stream_t stream);

/* ---------------------------------------------------------------------------------
 * Multi-GPU data plane: pack / unpack of listed blocks.  P:352 "batched
 * convolution over selected blocks", "latent scatter-gather operations": refined blocks
 * computed on one GPU travel to the GPU owning the frame's request as a COMPACT array in list
 * order, then land at their NHWC positions.  Bit copies (NaN payloads, -0 preserved).
 *
 * sphinx_gather_blocks:  dst[j][py][px][:] = src[n, by*b+py, bx*b+px, :] for list entry j
 *                        (id = (n*Hb+by)*Wb+bx), real pixels only; dst's padding pixels of
 *                        truncated edge blocks are left untouched.
 * sphinx_scatter_blocks: out[n, by*b+py, bx*b+px, :] = src[j][py][px][:] for list entry j, real
 *                        pixels only; every other pixel of out is untouched.  The list may be in
 *                        any order (e.g. several senders' segments concatenated); duplicate ids
 *                        give an unspecified winner.
 * src/dst/out  device, 16-byte aligned; NHWC [N][h][w][c] on the map side, [capacity][b][b][c]
 *              on the compact side; dtype gives the element width; c * elem_size % 16 == 0
 *              (else SPHINX_ERR_UNSUPPORTED); src must not alias dst/out.
 * block_ids/count/capacity  device list (count <= capacity <= N*Hb*Wb; count read on device).
 * ------------------------------------------------------------------------------- */
SPHINX_API sphinx_status sphinx_gather_blocks(const void* src, void* dst, sphinx_dtype dtype, int32_t n,
                                              int32_t h, int32_t w, int32_t c, int32_t block,
                                              const int32_t* block_ids, const int32_t* count,
                                              int32_t capacity, sphinx_stream_t stream);
SPHINX_API sphinx_status sphinx_scatter_blocks(const void* src, void* out, sphinx_dtype dtype, int32_t n,
                                               int32_t h, int32_t w, int32_t c, int32_t block,
                                               const int32_t* block_ids, const int32_t* count,
                                               int32_t capacity, sphinx_stream_t stream);

/* ---------------------------------------------------------------------------------
 * NEXT-1. Partial-step latent update (Alg1 line 18; deterministic DDIM, eta = 0):
 *   eps_hat = (z - sqrt(abar[u]) x0_hat) / sqrt(1 - abar[u])
 *   z_out   = sqrt(abar[u+1]) x0_hat + sqrt(1 - abar[u+1]) eps_hat          (fp32)
 * for every element of every real pixel of every listed block (the refined blocks of the
 * active frames); other elements of z_out are untouched.  Inactive frames are resampled
 * with sphinx_noise_inject at step u+1 (Alg1 line 19).
 * z, x0_hat, z_out  NHWC fp32 [N][h][w][c] device; z_out may alias z.
 * step_u            0 <= u < total_steps (u = 0 noisiest).
 * abar              HOST fp32 [S+1] (read synchronously: the step is a scalar of the loop).
 * ------------------------------------------------------------------------------- */
SPHINX_API sphinx_status sphinx_ddim_step(const float* z, const float* x0_hat, float* z_out,
                                          int32_t n, int32_t h, int32_t w, int32_t c, int32_t block,
                                          const int32_t* block_ids, const int32_t* count,
                                          int32_t capacity, int32_t step_u, const float* abar,
                                          int32_t total_steps, sphinx_stream_t stream);

/* ---------------------------------------------------------------------------------
 * NEXT-2. Uncertainty (blur) producer feeding step (1) (Alg1 lines 7-8; "smoothed,
 * normalized, and inverted, followed by Otsu thresholding"; constants S:196-222, R-23/R-24):
 *   Y = 0.299 R + 0.587 G + 0.114 B; L = 3x3 Laplacian [[0,1,0],[1,-4,1],[0,1,0]] (edge
 *   replication); V = population variance of L over window x window (edge replication);
 *   S = smooth x smooth box mean of V; U = 1 - (S - min S)/(max S - min S) per frame
 *   (constant S -> U = 1); tau_u[n] = Otsu over 256 bins, bin i = (i/256, (i+1)/256],
 *   exact between-class-variance argmax, ties to the lower split, tau = (k+1)/256; a frame
 *   whose U occupies one bin gets tau = 1 (= max U: no pixel is blurry).
 * The outputs are exactly sphinx_block_mask's (uncertainty, tau_u): blurry iff U > tau_u.
 * rgb          NHWC fp32 [N][h][w][3] device (the regression frames X, values in [0,1]).
 * window       odd, 3..15 (SPEC default 7); smooth: odd, 1..15 (SPEC default 5).
 * uncertainty  fp32 [N][h][w] device out; tau_u: fp32 [N] device out.
 * workspace    device scratch of sphinx_uncertainty_workspace_size(N) bytes (re-initialised
 *              by every call on `stream`).
 * ------------------------------------------------------------------------------- */
SPHINX_API sphinx_status sphinx_uncertainty_map(const float* rgb, int32_t n, int32_t h, int32_t w,
                                                int32_t window, int32_t smooth, float* uncertainty,
                                                float* tau_u, void* workspace, size_t workspace_bytes,
                                                sphinx_stream_t stream);
SPHINX_API size_t sphinx_uncertainty_workspace_size(int32_t n);

/* ---------------------------------------------------------------------------------
 * NEXT-3. Block-sparse UNet ResNet block with latent reuse ("ResNet layers ...
 * operate independently on each frame ... can be safely applied only to frames selected for
 * refinement"; "reuses cached latents from the last full denoising step for unrefined
 * regions"; readings R-26, R-27 in DESIGN.md):
 *   a1 = bf16(SiLU(GN1(x)));   h = listed ? bf16(conv3x3(a1; w1) + b1) : h (cached)
 *   a2 = bf16(SiLU(GN2(h)));   y = listed ? x + conv3x3(a2; w2) + b2 : y (cached)
 * GroupNorm (torch.nn.GroupNorm semantics: `groups` consecutive-channel groups, population
 * variance, per-channel affine) takes its statistics over the FULL current map (fresh values
 * in listed blocks, cached values elsewhere).  They are maintained incrementally in a
 * persistent per-block statistics buffer so a partial step reads active bytes only.
 *
 * Statistics buffer (sphinx_gn_stats_size(...) bytes, 8-byte aligned, caller-owned):
 *   block entries fp32 [N][Hb][Wb][groups][2] = (mean, M2) of the block's real pixels x the
 *   group's c/groups channels, then frame entries fp32 [N][groups][2] = (mean, 1/sqrt(var+eps))
 *   written by sphinx_gn_silu.  Persistent: at a full step (every block listed, e.g.
 *   SELECT_ALL) every block entry is written; a partial step rewrites only listed blocks, the
 *   others keep describing the cached content (which is what the full-map statistics need).
 * ------------------------------------------------------------------------------- */
SPHINX_API size_t sphinx_gn_stats_size(int32_t n, int32_t h, int32_t w, int32_t groups, int32_t block);

/* Rewrites the statistics entries of the listed blocks of the bf16 NHWC map x [N][h][w][c]
 * (fp32 shifted sums per channel, Chan combination per group).  c % groups == 0 (else
 * INVALID_ARGUMENT); c % 8 == 0 and lcm(c/groups, 8) <= 2048 (else UNSUPPORTED). */
SPHINX_API sphinx_status sphinx_gn_block_stats(const void* x, int32_t n, int32_t h, int32_t w, int32_t c,
                                               int32_t groups, int32_t block, const int32_t* block_ids,
                                               const int32_t* count, int32_t capacity, float* stats,
                                               sphinx_stream_t stream);

/* a = bf16(SiLU(gamma[ch] (x - mean_g) / sqrt(var_g + eps) + beta[ch])), var = M2 / count,
 * with (mean_g, var_g) of every frame combined from ALL Hb*Wb block entries of `stats` (fp32;
 * written to the buffer's frame entries), applied to every pixel of every listed block AND its
 * 1-pixel ring clipped to the image (exactly the pixels a 3x3 conv over the listed blocks
 * reads); other pixels of `a` are untouched.
 * x, a: bf16 NHWC [N][h][w][c] device, a != x.  gamma, beta: fp32 [c] device, 16-byte aligned.
 * eps >= 0. */
SPHINX_API sphinx_status sphinx_gn_silu(const void* x, float* stats, const float* gamma,
                                        const float* beta, float eps, int32_t n, int32_t h, int32_t w,
                                        int32_t c, int32_t groups, int32_t block,
                                        const int32_t* block_ids, const int32_t* count,
                                        int32_t capacity, void* a, sphinx_stream_t stream);

/* sphinx_sparse_conv3x3 with a bf16 NHWC residual [N][h][w][c_out] (16-byte aligned, != x)
 * added in the epilogue: y = residual + bias + conv (the ResNet block's identity skip). */
SPHINX_API sphinx_status sphinx_sparse_conv3x3_residual(
    const void* x, const void* w, const float* bias, const void* residual, void* y,
    sphinx_dtype y_dtype, int32_t n, int32_t h, int32_t w_, int32_t c_in, int32_t c_out,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity,
    void* workspace, size_t workspace_bytes, sphinx_stream_t stream);

/* Fused-conv table: combines the frame statistics from ALL block entries of `stats` (also written to
 * its frame entries) into table fp32 [N][c][2] = (gamma[ch] rstd_g, beta[ch] - mean_g gamma[ch]
 * rstd_g), so that SiLU(GN(x)) = SiLU(x * scale + shift).  table: device, 8-byte aligned. */
SPHINX_API sphinx_status sphinx_gn_scale_shift(float* stats, const float* gamma, const float* beta,
                                               float eps, int32_t n, int32_t h, int32_t w, int32_t c,
                                               int32_t groups, int32_t block, float* table,
                                               sphinx_stream_t stream);

/* sphinx_sparse_conv3x3 of the activation a = SiLU(x * scale[n][ci] + shift[n][ci]) computed ON
 * THE FLY from the raw map x: the halo tiles are normalised in shared memory between their TMA
 * load and the MMA (out-of-image halo pixels stay zero: zero padding of a), so a never exists
 * in HBM.  scale_shift: sphinx_gn_scale_shift's table.  Residual optional (as in _residual).
 * Needs the halo-staged path: block == 8 (else UNSUPPORTED). */
SPHINX_API sphinx_status sphinx_sparse_conv3x3_gn_silu(
    const void* x, const float* scale_shift, const void* w, const float* bias, const void* residual,
    void* y, sphinx_dtype y_dtype, int32_t n, int32_t h, int32_t w_, int32_t c_in, int32_t c_out,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity, void* workspace,
    size_t workspace_bytes, sphinx_stream_t stream);

/* The whole block (6 launches, stream-ordered, graph capturable).  With env SPHINX_RB_FUSED=1
 * and block == 8:
 *   gn_block_stats(x) -> gn_scale_shift(x) -> conv_gn_silu(x; w1,b1) into h -> gn_block_stats(h)
 *   -> gn_scale_shift(h) -> conv_gn_silu(h; w2,b2, residual x) into y   (GN+SiLU fused into the
 *   convs; a_scratch holds the scale/shift table).  Default (measured faster, DESIGN 6.8):
 *   gn_block_stats(x) -> gn_silu(x) -> conv(w1,b1) into h -> gn_block_stats(h) -> gn_silu(h)
 *   -> conv_residual(w2,b2, residual x) into y.
 * x        bf16 NHWC [N][h][w][c]: the current full map (cached values in unlisted blocks).
 * w1, w2   bf16 OHWI [c][3][3][c]; b1, b2 fp32 [c] or NULL; gn*_gamma/beta fp32 [c].
 * h_buf    bf16 NHWC, persistent: holds the cached conv1 output; listed pixels are rewritten.
 * x_stats, h_stats  persistent per-block statistics of x and h (see above); listed entries
 *          are rewritten.  Initialise them (and h_buf, y) with a full step.
 * y        NHWC bf16 or fp32, persistent: the block output; listed pixels rewritten.
 * a_scratch bf16 NHWC [N][h][w][c] scratch (the normalised activations).
 * workspace as for sphinx_sparse_conv3x3 (c_in = c_out = c).
 * Buffers must be distinct (no aliasing among x, h_buf, y, a_scratch; x_stats != h_stats). */
SPHINX_API sphinx_status sphinx_sparse_resblock(
    const void* x, const void* w1, const float* b1, const void* w2, const float* b2,
    const float* gn1_gamma, const float* gn1_beta, const float* gn2_gamma, const float* gn2_beta,
    int32_t groups, float eps, void* h_buf, float* x_stats, float* h_stats, void* y,
    sphinx_dtype y_dtype, void* a_scratch, int32_t n, int32_t h, int32_t w, int32_t c,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity,
    void* workspace, size_t workspace_bytes, sphinx_stream_t stream);
/* sphinx_sparse_resblock with flags.  SPHINX_RB_FUSED_GN: GN+SiLU applied inside each conv's halo
 * path (sphinx_gn_scale_shift + sphinx_sparse_conv3x3_gn_silu; block must be 8, else
 * SPHINX_ERR_UNSUPPORTED) instead of the separate activation pass -- same result within the
 * NEXT-3 bar, measured slower; a_scratch then holds the [N][c] float2 table. */
#define SPHINX_RB_FUSED_GN 1
SPHINX_API sphinx_status sphinx_sparse_resblock_ex(
    const void* x, const void* w1, const float* b1, const void* w2, const float* b2,
    const float* gn1_gamma, const float* gn1_beta, const float* gn2_gamma, const float* gn2_beta,
    int32_t groups, float eps, void* h_buf, float* x_stats, float* h_stats, void* y,
    sphinx_dtype y_dtype, void* a_scratch, int32_t n, int32_t h, int32_t w, int32_t c,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity,
    void* workspace, size_t workspace_bytes, int32_t flags, sphinx_stream_t stream);

/* ---------------------------------------------------------------------------------
 * NEXT-4. Temporal-attention latent cache ("Every T steps, the model performs a full
 * denoising pass over all input and target frames, during which the intermediate latent
 * representations from each temporal attention layer are cached.  In the subsequent (T-1)
 * partial denoising steps, frames that are not actively refined simply retrieve and reuse these
 * cached latents"; reading R-28).  Tokens of temporal attention are the frames of one sequence
 * (frames_per_seq consecutive frames of the batch) at the same pixel.  The cache is the
 * persistent q|k|v buffer: listed (frame, block) tokens are re-projected, every other token keeps
 * the K/V of the last full step.
 * ------------------------------------------------------------------------------- */

/* Pointwise (1x1) projection on listed blocks, the tcgen05 kernel of sphinx_sparse_conv3x3 with
 * one tap:  y[n,p,co] = (residual[n,p,co]) + bias[co] + sum_ci W[co][ci] x[n,p,ci]  for every
 * real pixel of every listed block; other pixels untouched.  w: bf16 [c_out][c_in] (row-major =
 * OHWI with 1x1 taps); residual: bf16 NHWC [N][h][w][c_out] or NULL (16-byte aligned, != x);
 * other arguments, constraints and the workspace as for sphinx_sparse_conv3x3. */
SPHINX_API sphinx_status sphinx_sparse_pointwise(
    const void* x, const void* w, const float* bias, const void* residual, void* y,
    sphinx_dtype y_dtype, int32_t n, int32_t h, int32_t w_, int32_t c_in, int32_t c_out,
    int32_t block, const int32_t* block_ids, const int32_t* count, int32_t capacity,
    void* workspace, size_t workspace_bytes, sphinx_stream_t stream);

/* Attention of the listed tokens over the frames of their sequence:
 *   o[n,p, head hd] = sum_m softmax_m(q[n,p,hd] . k[m,p,hd] / sqrt(64)) v[m,p,hd]
 * m over the frames_per_seq frames of n's sequence, q|k|v read from qkv (listed tokens fresh,
 * unlisted tokens cached), fp32 arithmetic, bf16 output written for listed pixels only.
 * qkv  bf16 NHWC [N][h][w][3c] = q | k | v, each head-major (head hd = channels [64 hd, 64 hd+64)).
 * o    bf16 NHWC [N][h][w][c].  qkv and o 16-byte aligned; c / heads must be 64;
 *      frames_per_seq <= 32 and divides N; 128 + frames_per_seq * (6c + 16) bytes <= 227 KB
 *      (else UNSUPPORTED).  A pixel's frames_per_seq tokens are staged in shared memory by one
 *      TMA tensor copy when two staging buffers fit (else per (pixel, group of heads) when
 *      a group's buffers fit twice per SM, else by frames_per_seq bulk copies); identical
 *      results; SPHINX_ERR_UNSUPPORTED if the driver rejects the tensor map.
 * workspace  sphinx_temporal_attention_workspace_size(...) bytes (4-byte aligned): the per
 *      (sequence, block position) listed-frame bitmasks, rebuilt by every call. */
SPHINX_API size_t sphinx_temporal_attention_workspace_size(int32_t n, int32_t h, int32_t w,
                                                           int32_t frames_per_seq, int32_t block);
SPHINX_API sphinx_status sphinx_temporal_attention(const void* qkv, void* o, int32_t n, int32_t h,
                                                   int32_t w, int32_t c, int32_t heads,
                                                   int32_t frames_per_seq, int32_t block,
                                                   const int32_t* block_ids, const int32_t* count,
                                                   int32_t capacity, void* workspace,
                                                   size_t workspace_bytes, sphinx_stream_t stream);
/* sphinx_temporal_attention with an explicit head grouping (tests and tuning): head_group = k > 0
 * stages units of (pixel, k heads) with one 5-D tensor copy (k divides heads; k = heads: no
 * grouping); 0 = the default choice (groups only when the all-heads ring does not fit twice per
 * SM).  Same result for every k. */
SPHINX_API sphinx_status sphinx_temporal_attention_ex(const void* qkv, void* o, int32_t n, int32_t h,
                                                      int32_t w, int32_t c, int32_t heads,
                                                      int32_t frames_per_seq, int32_t block,
                                                      const int32_t* block_ids, const int32_t* count,
                                                      int32_t capacity, void* workspace,
                                                      size_t workspace_bytes, int32_t head_group,
                                                      sphinx_stream_t stream);

/* The temporal block (3 launches + 1 plan kernel, graph capturable):
 *   qkv_buf[listed] = bf16(Wqkv x + bqkv)       (sphinx_sparse_pointwise, c -> 3c)
 *   o = attention(qkv_buf)                      (sphinx_temporal_attention)
 *   y[listed] = x + Wo o + bo                   (sphinx_sparse_pointwise with residual x)
 * x bf16 NHWC [N][h][w][c]; wqkv bf16 [3c][c]; wo bf16 [c][c]; bqkv [3c], bo [c] fp32 or NULL.
 * qkv_buf bf16 [N][h][w][3c] and y (bf16/fp32 [N][h][w][c]) are persistent (initialise with a
 * full step: every block listed); o_scratch bf16 [N][h][w][c].  workspace: a conv workspace for
 * c_out = 3c (sphinx_conv_workspace_size); attn_workspace as above.  Buffers must not alias. */
SPHINX_API sphinx_status sphinx_temporal_block(
    const void* x, const void* wqkv, const float* bqkv, const void* wo, const float* bo,
    int32_t heads, int32_t frames_per_seq, void* qkv_buf, void* o_scratch, void* y,
    sphinx_dtype y_dtype, int32_t n, int32_t h, int32_t w, int32_t c, int32_t block,
    const int32_t* block_ids, const int32_t* count, int32_t capacity, void* workspace,
    size_t workspace_bytes, void* attn_workspace, size_t attn_workspace_bytes,
    sphinx_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SPHINX_H */
