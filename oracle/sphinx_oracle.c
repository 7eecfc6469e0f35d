/*
 * sphinx_oracle.c — CPU ORACLE (test infrastructure only; see sphinx_oracle.h).
 *
 * Plain C99, fp64, scalar loops in the paper's order.  No blocking, fusion or
 * reordering beyond what the definitions state.  OpenMP is used only to run
 * independent output pixels of the convolution concurrently; every output
 * element is still the same strictly ordered sum.
 */
#include "sphinx_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define BAD (-1)

/* ---------------------------------------------------------------- a1 ---- */

/* Alg1 line 9: M_op = 1[O < tau_o]; line 10: M = M_op v M_blur.
 * P:447 "Pixels with opacity values below 0.5 or identified as blurry are selected".
 * Reading R-9: a NaN is never "confident", so !(o >= tau_o) and !(u <= tau). */
int oracle_pixel_mask(const float* O, const float* U, const float* tau_u, float tau_o,
                      int n, int hp, int wp, uint8_t* m) {
  if (!O || !m || n <= 0 || hp <= 0 || wp <= 0) return BAD;
  if (!(tau_o >= 0.0f && tau_o <= 1.0f)) return BAD;
  if (U && !tau_u) return BAD;
  for (int i = 0; i < n; ++i) {
    for (int y = 0; y < hp; ++y) {
      for (int x = 0; x < wp; ++x) {
        size_t p = ((size_t)i * hp + y) * wp + x;
        int m_op = !(O[p] >= tau_o);
        int m_blur = 0;
        if (U) m_blur = !(U[p] <= tau_u[i]);
        m[p] = (uint8_t)(m_op || m_blur);
      }
    }
  }
  return 0;
}

/* P:489 "the confidence mask is downsampled using max-pooling at each layer";
 * S:246 non-overlapping window, 1 iff any input pixel is 1. */
int oracle_maxpool(const uint8_t* in, int n, int h, int w, int f, uint8_t* out) {
  if (!in || !out || n <= 0 || h <= 0 || w <= 0 || f <= 0) return BAD;
  if (h % f != 0 || w % f != 0) return BAD;
  int ho = h / f, wo = w / f;
  for (int i = 0; i < n; ++i)
    for (int y = 0; y < ho; ++y)
      for (int x = 0; x < wo; ++x) {
        uint8_t v = 0;
        for (int dy = 0; dy < f; ++dy)
          for (int dx = 0; dx < f; ++dx)
            if (in[((size_t)i * h + y * f + dy) * w + x * f + dx]) v = 1;
        out[((size_t)i * ho + y) * wo + x] = v;
      }
  return 0;
}

/* P:352 "tiles the feature maps into blocks ... Each block is marked for
 * refinement if it contains at least one pixel within the refinement mask";
 * S:253 last row/col blocks may be smaller (reading R-2). */
int oracle_tile_blocks(const uint8_t* grid, int n, int h, int w, int b, uint8_t* out) {
  if (!grid || !out || n <= 0 || h <= 0 || w <= 0 || b <= 0) return BAD;
  int hb = (h + b - 1) / b, wb = (w + b - 1) / b;
  for (int i = 0; i < n; ++i)
    for (int by = 0; by < hb; ++by)
      for (int bx = 0; bx < wb; ++bx) {
        uint8_t v = 0;
        for (int y = by * b; y < by * b + b && y < h; ++y)
          for (int x = bx * b; x < bx * b + b && x < w; ++x)
            if (grid[((size_t)i * h + y) * w + x]) v = 1;
        out[((size_t)i * hb + by) * wb + bx] = v;
      }
  return 0;
}

int oracle_block_mask(const float* O, const float* U, const float* tau_u, float tau_o,
                      int n, int hp, int wp, int f, int b, int n_levels,
                      uint8_t* masks, int32_t* counts) {
  if (!O || !masks || n <= 0 || hp <= 0 || wp <= 0 || f <= 0 || b <= 0) return BAD;
  if (n_levels < 1 || n_levels > 4) return BAD;
  if (hp % f != 0 || wp % f != 0) return BAD;
  int h0 = hp / f, w0 = wp / f;
  int div = 1 << (n_levels - 1);
  if (h0 % div != 0 || w0 % div != 0) return BAD;

  size_t npx = (size_t)n * hp * wp;
  uint8_t* pix = (uint8_t*)malloc(npx);
  uint8_t* cur = (uint8_t*)malloc((size_t)n * h0 * w0);
  uint8_t* nxt = (uint8_t*)malloc((size_t)n * h0 * w0);
  if (!pix || !cur || !nxt) { free(pix); free(cur); free(nxt); return -2; }
  int rc = oracle_pixel_mask(O, U, tau_u, tau_o, n, hp, wp, pix); /* Alg1 lines 9-10 */
  if (rc == 0) rc = oracle_maxpool(pix, n, hp, wp, f, cur);      /* VAE /8 */
  size_t off = 0;
  int hl = h0, wl = w0;
  for (int l = 0; rc == 0 && l < n_levels; ++l) {
    if (l > 0) { /* UNet level l: max-pool by 2 */
      rc = oracle_maxpool(cur, n, hl, wl, 2, nxt);
      hl /= 2; wl /= 2;
      uint8_t* t = cur; cur = nxt; nxt = t;
      if (rc) break;
    }
    int hb = (hl + b - 1) / b, wb = (wl + b - 1) / b;
    rc = oracle_tile_blocks(cur, n, hl, wl, b, masks + off);
    if (rc) break;
    if (counts) {
      for (int i = 0; i < n; ++i) {
        int32_t c = 0;
        for (int j = 0; j < hb * wb; ++j) c += masks[off + (size_t)i * hb * wb + j];
        counts[i * n_levels + l] = c;
      }
    }
    off += (size_t)n * hb * wb;
  }
  free(pix); free(cur); free(nxt);
  return rc;
}

/* ---------------------------------------------------------------- a2 ---- */

/* x^gamma with the exact definitions where they exist (reading R-16): x^1 = x and
 * x^(1/2) = sqrt(x), which C99 / IEEE 754 round correctly.  glibc pow(x, 0.5) is NOT
 * correctly rounded (it differs from sqrt for ~1.4e5 fp32 inputs in [2^-20, 1]), so it
 * is used only for the remaining gamma, where no exact reference exists. */
static double eq2_pow(double x, double gamma) {
  if (gamma == 1.0) return x;
  if (gamma == 0.5) return sqrt(x);
  return pow(x, gamma);
}

/* Eq. 2: Q* = c0 + (c1 - c0) f(t); f = t^gamma if c1 >= c0,
 * else 1 - (1 - t)^gamma.  Literal transcription (reading R-11). */
double oracle_eq2(double c0, double c1, double t, double gamma) {
  double f;
  if (c1 >= c0) f = eq2_pow(t, gamma);
  else f = 1.0 - eq2_pow(1.0 - t, gamma);
  return c0 + (c1 - c0) * f;
}

void oracle_eq2_batch(const double* c0, const double* c1, const double* t, double gamma, int n,
                      double* out) {
  for (int i = 0; i < n; ++i) out[i] = oracle_eq2(c0[i], c1[i], t[i], gamma);
}

/* S:143 k = steps[i] for the largest i with thresholds[i] <= r (left-closed,
 * S:166); fallback_k if r is below all; clamp to k_max ("largest k=40"). */
int32_t oracle_select_k(const oracle_klogic* lg, double r) {
  int32_t k = lg->fallback_k;
  for (int i = 0; i < lg->m; ++i)
    if (lg->thr[i] <= r) k = lg->step[i];
  if (k > lg->k_max) k = lg->k_max;
  return k;
}

int oracle_start_step(const float* q, const float* c0, const float* c1, const float* t,
                      const int32_t* logic_id, double gamma,
                      const oracle_klogic* logics, int n_logics, int n, int32_t* k) {
  if (!q || !c0 || !c1 || !t || !logics || !k || n <= 0 || n_logics < 1) return BAD;
  if (!(gamma > 0.0 && gamma <= 1.0)) return BAD;
  for (int j = 0; j < n_logics; ++j) {
    const oracle_klogic* lg = &logics[j];
    if (lg->m < 1 || lg->m > 16) return BAD;
    for (int i = 1; i < lg->m; ++i)
      if (!(lg->thr[i - 1] < lg->thr[i]) || lg->step[i - 1] > lg->step[i]) return BAD;
  }
  for (int i = 0; i < n; ++i) {
    int lid = logic_id ? logic_id[i] : 0;
    double ti = (double)t[i];
    if (lid < 0 || lid >= n_logics || !(ti >= 0.0 && ti <= 1.0)) { k[i] = -1; continue; }
    double qs = oracle_eq2((double)c0[i], (double)c1[i], ti, gamma); /* Alg1 line 4 */
    if (!(qs > 0.0)) { k[i] = -1; continue; }
    double r = (double)q[i] / qs;                                    /* Alg1 line 5 */
    if (r != r) { k[i] = -1; continue; }
    k[i] = oracle_select_k(&logics[lid], r);                         /* Alg1 line 6 */
  }
  return 0;
}

/* ---------------------------------------------------------------- a3 ---- */

int oracle_compact(const uint8_t* mask, int n, int hb, int wb, const int32_t* k, int u,
                   int select, int32_t* ids, int32_t* count) {
  if (!ids || !count || n <= 0 || hb <= 0 || wb <= 0) return BAD;
  if (select < 0 || select > 3) return BAD;
  if ((select == 0 || select == 3) && !mask) return BAD;
  if ((select == 1 || select == 3) && !k) return BAD;
  int32_t c = 0;
  for (int i = 0; i < n; ++i)
    for (int by = 0; by < hb; ++by)
      for (int bx = 0; bx < wb; ++bx) {
        int32_t id = (i * hb + by) * wb + bx;
        int take;
        if (select == 0)      /* A_u = 1[k <= u] (Alg1 line 17) and M (Alg1 line 18) */
          take = mask[id] && (!k || (k[i] >= 0 && k[i] <= u));
        else if (select == 1) /* frames not in A_u are resampled (Alg1 line 19) */
          take = k[i] > u;
        else if (select == 3) /* the step's noise pass: line 12's blocks or line 19's frames */
          take = (mask[id] && k[i] >= 0 && k[i] <= u) || k[i] > u;
        else
          take = !k || k[i] >= 0;
        if (take) ids[c++] = id;
      }
  *count = c;
  return 0;
}

/* ---------------------------------------------------------------- a4 ---- */

/* add_noise (Alg1 lines 12, 19): z_u = sqrt(abar[u]) z0 + sqrt(1 - abar[u]) eps
 * (BASELINE north_star).  u = 0 noisiest, u = S clean. */
int oracle_noise(const float* x0, const float* eps, const float* xt_in, double* out,
                 int n, int h, int w, int c, int b, const int32_t* ids, int count,
                 const int32_t* step, const float* abar, int total_steps) {
  if (!x0 || !eps || !xt_in || !out || !step || !abar) return BAD;
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || b <= 0 || count < 0 || total_steps < 2) return BAD;
  if (count > 0 && !ids) return BAD;
  size_t total = (size_t)n * h * w * c;
  for (size_t e = 0; e < total; ++e) out[e] = (double)xt_in[e];
  int hb = (h + b - 1) / b, wb = (w + b - 1) / b;
  for (int j = 0; j < count; ++j) {
    int id = ids[j];
    int i = id / (hb * wb), by = (id / wb) % hb, bx = id % wb;
    int u = step[i];
    if (u < 0 || u > total_steps) continue; /* left untouched */
    double ab = (double)abar[u];
    double a = sqrt(ab), s = sqrt(1.0 - ab);
    for (int y = by * b; y < by * b + b && y < h; ++y)
      for (int x = bx * b; x < bx * b + b && x < w; ++x)
        for (int ch = 0; ch < c; ++ch) {
          size_t e = (((size_t)i * h + y) * w + x) * c + ch;
          out[e] = a * (double)x0[e] + s * (double)eps[e];
        }
  }
  return 0;
}

/* ---------------------------------------------------------------- a5 ---- */

static double bf16_to_double(uint16_t v) {
  uint32_t bits = (uint32_t)v << 16; /* bf16 is the top half of an IEEE binary32 */
  float f;
  memcpy(&f, &bits, sizeof f);
  return (double)f;
}

/* y[n,p,co] = bias[co] + sum_{dy,dx} sum_ci W[co,dy+1,dx+1,ci] x[n,p+(dy,dx),ci],
 * x = 0 outside the image (reading R-17).  Order: taps row-major, then ci. */
static void conv_pixel(const double* xd, const double* wd, const float* bias,
                       int i, int y, int x, int h, int w, int cin, int cout,
                       double* yo, double* ao) {
  for (int co = 0; co < cout; ++co) {
    double acc = bias ? (double)bias[co] : 0.0;
    double aab = bias ? fabs((double)bias[co]) : 0.0;
    for (int ky = 0; ky < 3; ++ky) {
      int yy = y + ky - 1;
      if (yy < 0 || yy >= h) continue;
      for (int kx = 0; kx < 3; ++kx) {
        int xx = x + kx - 1;
        if (xx < 0 || xx >= w) continue;
        const double* xp = xd + (((size_t)i * h + yy) * w + xx) * cin;
        const double* wp = wd + (((size_t)co * 3 + ky) * 3 + kx) * cin;
        for (int ci = 0; ci < cin; ++ci) {
          double p = wp[ci] * xp[ci];
          acc += p;
          aab += fabs(p);
        }
      }
    }
    yo[co] = acc;
    if (ao) ao[co] = aab;
  }
}

static double* widen(const uint16_t* v, size_t cnt) {
  double* d = (double*)malloc(cnt * sizeof(double));
  if (!d) return NULL;
  for (size_t j = 0; j < cnt; ++j) d[j] = bf16_to_double(v[j]);
  return d;
}

int oracle_conv3x3_blocks(const uint16_t* x, const uint16_t* wt, const float* bias,
                          int n, int h, int w, int cin, int cout, int b,
                          const int32_t* ids, int count, double* y, double* absacc,
                          int n_threads) {
  if (!x || !wt || !y || n <= 0 || h <= 0 || w <= 0 || cin <= 0 || cout <= 0 || b <= 0) return BAD;
  if (count < 0 || (count > 0 && !ids)) return BAD;
  int hb = (h + b - 1) / b, wb = (w + b - 1) / b;
  for (int j = 0; j < count; ++j)
    if (ids[j] < 0 || ids[j] >= n * hb * wb) return BAD;
  double* xd = widen(x, (size_t)n * h * w * cin);
  double* wd = widen(wt, (size_t)cout * 9 * cin);
  if (!xd || !wd) { free(xd); free(wd); return -2; }
  long total = (long)count * b * b;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (long q = 0; q < total; ++q) {
    int j = (int)(q / (b * b));
    int p = (int)(q % (b * b));
    int id = ids[j];
    int i = id / (hb * wb), by = (id / wb) % hb, bx = id % wb;
    int yy = by * b + p / b, xx = bx * b + p % b;
    if (yy >= h || xx >= w) continue; /* truncated edge block (reading R-2) */
    size_t o = (((size_t)i * h + yy) * w + xx) * cout;
    conv_pixel(xd, wd, bias, i, yy, xx, h, w, cin, cout, y + o, absacc ? absacc + o : NULL);
  }
  free(xd); free(wd);
  return 0;
}

int oracle_conv3x3_dense(const uint16_t* x, const uint16_t* wt, const float* bias,
                         int n, int h, int w, int cin, int cout,
                         double* y, double* absacc, int n_threads) {
  if (!x || !wt || !y || n <= 0 || h <= 0 || w <= 0 || cin <= 0 || cout <= 0) return BAD;
  double* xd = widen(x, (size_t)n * h * w * cin);
  double* wd = widen(wt, (size_t)cout * 9 * cin);
  if (!xd || !wd) { free(xd); free(wd); return -2; }
  long total = (long)n * h * w;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (long q = 0; q < total; ++q) {
    int i = (int)(q / ((long)h * w));
    int yy = (int)((q / w) % h), xx = (int)(q % w);
    size_t o = (size_t)q * cout;
    conv_pixel(xd, wd, bias, i, yy, xx, h, w, cin, cout, y + o, absacc ? absacc + o : NULL);
  }
  free(xd); free(wd);
  return 0;
}

/* ---------------------------------------------------------------- a6 ---- */

/* P:352 "reuses cached latents from the last full denoising step for unrefined
 * regions".  A pixel takes src iff its block is refined. */
int oracle_scatter(const void* src, int src_layout, const void* cache, void* out, int elem_bytes,
                   int n, int h, int w, int c, int b,
                   const uint8_t* mask, const int32_t* k, int u,
                   const int32_t* ids, int count) {
  if (!src || !cache || !out || n <= 0 || h <= 0 || w <= 0 || c <= 0 || b <= 0) return BAD;
  if (elem_bytes != 2 && elem_bytes != 4) return BAD;
  if (src_layout != 0 && src_layout != 1) return BAD;
  if (src_layout == 0 && !mask) return BAD;
  if (src_layout == 1 && (count < 0 || (count > 0 && !ids))) return BAD;
  int hb = (h + b - 1) / b, wb = (w + b - 1) / b;
  size_t px_bytes = (size_t)c * elem_bytes;
  const uint8_t* s = (const uint8_t*)src;
  const uint8_t* ca = (const uint8_t*)cache;
  uint8_t* o = (uint8_t*)out;
  /* start from the cache everywhere ... */
  memcpy(o, ca, (size_t)n * h * w * px_bytes);
  if (src_layout == 0) {
    /* ... and take src on every pixel of an active block */
    for (int i = 0; i < n; ++i)
      for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
          int id = (i * hb + y / b) * wb + x / b;
          int act = mask[id] && (!k || (k[i] >= 0 && k[i] <= u));
          if (act) {
            size_t e = (((size_t)i * h + y) * w + x) * px_bytes;
            memcpy(o + e, s + e, px_bytes);
          }
        }
  } else {
    for (int j = 0; j < count; ++j) {
      int id = ids[j];
      if (id < 0 || id >= n * hb * wb) return BAD;
      int i = id / (hb * wb), by = (id / wb) % hb, bx = id % wb;
      for (int py = 0; py < b; ++py)
        for (int px = 0; px < b; ++px) {
          int y = by * b + py, x = bx * b + px;
          if (y >= h || x >= w) continue;
          size_t e = (((size_t)i * h + y) * w + x) * px_bytes;
          size_t se = (((size_t)j * b + py) * b + px) * px_bytes;
          memcpy(o + e, s + se, px_bytes);
        }
    }
  }
  return 0;
}

/* -------------------------------------------------------------- NEXT-1 ---- */

/* S:312 ddim_full_step / partial_step update: eps_hat = (z - sqrt(abar[u]) x0_hat) /
 * sqrt(1 - abar[u]); z' = sqrt(abar[u+1]) x0_hat + sqrt(1 - abar[u+1]) eps_hat (eta = 0).
 * Written in that order, in fp64. */
int oracle_ddim_step(const float* z, const float* x0_hat, double* out, int n, int h, int w, int c,
                     int b, const int32_t* ids, int count, int u, const float* abar,
                     int total_steps) {
  if (!z || !x0_hat || !out || !abar || n <= 0 || h <= 0 || w <= 0 || c <= 0 || b <= 0) return BAD;
  if (count < 0 || (count > 0 && !ids) || total_steps < 2) return BAD;
  if (u < 0 || u >= total_steps) return BAD;
  size_t total = (size_t)n * h * w * c;
  for (size_t e = 0; e < total; ++e) out[e] = (double)z[e];
  int hb = (h + b - 1) / b, wb = (w + b - 1) / b;
  double a0 = sqrt((double)abar[u]), s0 = sqrt(1.0 - (double)abar[u]);
  double a1 = sqrt((double)abar[u + 1]), s1 = sqrt(1.0 - (double)abar[u + 1]);
  for (int j = 0; j < count; ++j) {
    int id = ids[j];
    if (id < 0 || id >= n * hb * wb) return BAD;
    int i = id / (hb * wb), by = (id / wb) % hb, bx = id % wb;
    for (int y = by * b; y < by * b + b && y < h; ++y)
      for (int x = bx * b; x < bx * b + b && x < w; ++x)
        for (int ch = 0; ch < c; ++ch) {
          size_t e = (((size_t)i * h + y) * w + x) * c + ch;
          double eps_hat = ((double)z[e] - a0 * (double)x0_hat[e]) / s0;
          out[e] = a1 * (double)x0_hat[e] + s1 * eps_hat;
        }
  }
  return 0;
}

/* -------------------------------------------------------------- NEXT-2 ---- */

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

int oracle_laplacian_var(const float* rgb, int n, int h, int w, int window, double* B) {
  if (!rgb || !B || n <= 0 || h <= 0 || w <= 0) return BAD;
  if (window < 3 || window % 2 == 0) return BAD; /* S:199 even window -> invalid */
  size_t plane = (size_t)h * w;
  double* Y = (double*)malloc(plane * sizeof(double));
  double* L = (double*)malloc(plane * sizeof(double));
  if (!Y || !L) { free(Y); free(L); return -2; }
  int r = window / 2;
  for (int i = 0; i < n; ++i) {
    /* luminance (R-23) */
    for (size_t p = 0; p < plane; ++p) {
      const float* px = rgb + ((size_t)i * plane + p) * 3;
      Y[p] = 0.299 * (double)px[0] + 0.587 * (double)px[1] + 0.114 * (double)px[2];
    }
    /* 3x3 Laplacian with edge replication */
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        double up = Y[(size_t)clampi(y - 1, 0, h - 1) * w + x];
        double dn = Y[(size_t)clampi(y + 1, 0, h - 1) * w + x];
        double lf = Y[(size_t)y * w + clampi(x - 1, 0, w - 1)];
        double rt = Y[(size_t)y * w + clampi(x + 1, 0, w - 1)];
        L[(size_t)y * w + x] = up + dn + lf + rt - 4.0 * Y[(size_t)y * w + x];
      }
    /* population variance over the window (two-pass: mean, then mean squared deviation) */
    double cnt = (double)window * window;
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        double mean = 0.0;
        for (int dy = -r; dy <= r; ++dy)
          for (int dx = -r; dx <= r; ++dx)
            mean += L[(size_t)clampi(y + dy, 0, h - 1) * w + clampi(x + dx, 0, w - 1)];
        mean /= cnt;
        double var = 0.0;
        for (int dy = -r; dy <= r; ++dy)
          for (int dx = -r; dx <= r; ++dx) {
            double d = L[(size_t)clampi(y + dy, 0, h - 1) * w + clampi(x + dx, 0, w - 1)] - mean;
            var += d * d;
          }
        B[(size_t)i * plane + (size_t)y * w + x] = var / cnt;
      }
  }
  free(Y); free(L);
  return 0;
}

int oracle_box_smooth(const double* in, int n, int h, int w, int k, double* out) {
  if (!in || !out || n <= 0 || h <= 0 || w <= 0 || k < 1 || k % 2 == 0) return BAD;
  int r = k / 2;
  size_t plane = (size_t)h * w;
  for (int i = 0; i < n; ++i)
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        double s = 0.0;
        for (int dy = -r; dy <= r; ++dy)
          for (int dx = -r; dx <= r; ++dx)
            s += in[(size_t)i * plane + (size_t)clampi(y + dy, 0, h - 1) * w + clampi(x + dx, 0, w - 1)];
        out[(size_t)i * plane + (size_t)y * w + x] = s / ((double)k * k);
      }
  return 0;
}

typedef unsigned __int128 u128;

/* Between-class variance of the split after bin k, exactly:  with n0, n1 the class counts,
 * N = n0 + n1, S0 the sum of class-0 bin indices and S the total, sigma_b^2 * N^2 =
 * (n0 S - N S0)^2 / (n0 n1).  Returned as quotient + remainder over den = n0 n1. */
static void otsu_score(const long long* hist, int k, long long N, long long S, u128* q, u128* rem,
                       u128* den) {
  long long n0 = 0, s0 = 0;
  for (int i = 0; i <= k; ++i) { n0 += hist[i]; s0 += (long long)i * hist[i]; }
  long long n1 = N - n0;
  if (n0 == 0 || n1 == 0) { *q = 0; *rem = 0; *den = 1; return; }
  __int128 d = (__int128)n0 * S - (__int128)N * s0;
  u128 num = (u128)(d < 0 ? -d : d);
  num = num * num;
  *den = (u128)n0 * (u128)n1;
  *q = num / *den;
  *rem = num % *den;
}

static int otsu_from_hist(const long long* hist, float vmax, float* tau) {
  long long N = 0, S = 0;
  int nonempty = 0;
  for (int i = 0; i < 256; ++i) { N += hist[i]; S += (long long)i * hist[i]; nonempty += hist[i] > 0; }
  if (N <= 0) return BAD;
  if (nonempty <= 1) { *tau = vmax; return 0; } /* constant grid: nothing above */
  int best = 0;
  u128 bq, br, bd;
  otsu_score(hist, 0, N, S, &bq, &br, &bd);
  for (int k = 1; k < 255; ++k) {
    u128 q, r, d;
    otsu_score(hist, k, N, S, &q, &r, &d);
    /* strictly greater only: ties go to the smaller k */
    if (q > bq || (q == bq && r * bd > br * d)) { best = k; bq = q; br = r; bd = d; }
  }
  *tau = (float)(best + 1) / 256.0f;
  return 0;
}

static int bin_of(double v) {
  /* bin i = (i/256, (i+1)/256]; v * 256 is exact in binary floating point */
  double t = ceil(v * 256.0) - 1.0;
  if (t < 0.0) t = 0.0;
  if (t > 255.0) t = 255.0;
  return (int)t;
}

int oracle_otsu(const float* values, long count, float* tau) {
  if (!values || !tau || count <= 0) return BAD;
  long long hist[256] = {0};
  float vmax = values[0];
  for (long j = 0; j < count; ++j) {
    hist[bin_of((double)values[j])]++;
    if (values[j] > vmax) vmax = values[j];
  }
  return otsu_from_hist(hist, vmax, tau);
}

int oracle_otsu_f64(const double* values, long count, float* tau) {
  if (!values || !tau || count <= 0) return BAD;
  long long hist[256] = {0};
  double vmax = values[0];
  for (long j = 0; j < count; ++j) {
    hist[bin_of(values[j])]++;
    if (values[j] > vmax) vmax = values[j];
  }
  return otsu_from_hist(hist, (float)vmax, tau);
}

int oracle_uncertainty(const float* rgb, int n, int h, int w, int window, int smooth, double* U,
                       float* tau) {
  if (!rgb || !U || !tau || n <= 0 || h <= 0 || w <= 0) return BAD;
  size_t plane = (size_t)h * w;
  double* B = (double*)malloc((size_t)n * plane * sizeof(double));
  if (!B) return -2;
  int rc = oracle_laplacian_var(rgb, n, h, w, window, B);         /* Alg1 line 7 */
  if (rc == 0) rc = oracle_box_smooth(B, n, h, w, smooth, U);     /* "smoothed" */
  for (int i = 0; rc == 0 && i < n; ++i) {
    double* u = U + (size_t)i * plane;
    double lo = u[0], hi = u[0];
    for (size_t p = 0; p < plane; ++p) { if (u[p] < lo) lo = u[p]; if (u[p] > hi) hi = u[p]; }
    for (size_t p = 0; p < plane; ++p) {
      double nrm = hi > lo ? (u[p] - lo) / (hi - lo) : 0.0;       /* "normalized" */
      u[p] = 1.0 - nrm;                                           /* "inverted" */
    }
    rc = oracle_otsu_f64(u, (long)plane, &tau[i]);                /* Alg1 line 8 "otsu" */
  }
  free(B);
  return rc;
}

/* ------------------------------------------------------------- NEXT-3 ---- */

/* Round a double to the nearest bfloat16 (8 significant bits), ties to even, directly
 * from the fp64 value (no intermediate fp32 rounding).  Overflow -> +-inf; NaN -> qNaN. */
uint16_t oracle_bf16_rne(double v) {
  if (isnan(v)) return 0x7fc0;
  double a = fabs(v);
  double r;
  if (a == 0.0) {
    r = 0.0;
  } else {
    int e = ilogb(a);            /* a in [2^e, 2^(e+1)) */
    if (e < -126) e = -126;      /* bf16 subnormals share the binary32 minimum exponent */
    double ulp = ldexp(1.0, e - 7);
    double q = a / ulp;          /* exact: power-of-two scaling */
    double fl = floor(q);
    double rem = q - fl;
    if (rem > 0.5 || (rem == 0.5 && fmod(fl, 2.0) != 0.0)) fl += 1.0;
    r = fl * ulp;
    if (r > 3.3895313892515355e38) r = INFINITY;  /* above the largest bf16 */
  }
  float f = (float)(signbit(v) ? -r : r);  /* exact: r has <= 8 significant bits; keeps -0 */
  uint32_t bits;
  memcpy(&bits, &f, sizeof bits);
  return (uint16_t)(bits >> 16);
}

/* GroupNorm statistics over the full current map (reading R-26): for frame i and group g
 * (channels [g*c/G, (g+1)*c/G), consecutive as in torch.nn.GroupNorm), mean and population
 * variance of the h*w*c/G values, two passes in fp64. */
int oracle_gn_stats(const double* x, int n, int h, int w, int c, int groups, double* mean,
                    double* var) {
  if (!x || !mean || !var || n <= 0 || h <= 0 || w <= 0 || c <= 0 || groups <= 0 ||
      c % groups != 0)
    return BAD;
  int cg = c / groups;
  size_t plane = (size_t)h * w;
  for (int i = 0; i < n; ++i)
    for (int g = 0; g < groups; ++g) {
      double s = 0.0;
      for (size_t p = 0; p < plane; ++p)
        for (int k = 0; k < cg; ++k) s += x[((size_t)i * plane + p) * c + g * cg + k];
      double cnt = (double)plane * cg;
      double m = s / cnt;
      double ss = 0.0;
      for (size_t p = 0; p < plane; ++p)
        for (int k = 0; k < cg; ++k) {
          double d = x[((size_t)i * plane + p) * c + g * cg + k] - m;
          ss += d * d;
        }
      mean[i * groups + g] = m;
      var[i * groups + g] = ss / cnt;
    }
  return 0;
}

/* GroupNorm + SiLU (the normalisation/activation in front of each conv of a UNet ResNet
 * block; reading R-26): t = gamma[ch] (x - mean) / sqrt(var + eps) + beta[ch],
 * a = SiLU(t) = t / (1 + exp(-t)).  Every pixel of the map.  t may be NULL. */
int oracle_gn_silu(const double* x, int n, int h, int w, int c, int groups, const double* mean,
                   const double* var, const float* gamma, const float* beta, double eps,
                   double* t, double* a) {
  if (!x || !mean || !var || !gamma || !beta || !a || n <= 0 || h <= 0 || w <= 0 || c <= 0 ||
      groups <= 0 || c % groups != 0 || !(eps >= 0.0))
    return BAD;
  int cg = c / groups;
  size_t plane = (size_t)h * w;
  for (int i = 0; i < n; ++i)
    for (size_t p = 0; p < plane; ++p)
      for (int ch = 0; ch < c; ++ch) {
        size_t o = ((size_t)i * plane + p) * c + ch;
        int g = ch / cg;
        double sd = sqrt(var[i * groups + g] + eps);
        double tt = (double)gamma[ch] * (x[o] - mean[i * groups + g]) / sd + (double)beta[ch];
        if (t) t[o] = tt;
        a[o] = tt / (1.0 + exp(-tt));
      }
  return 0;
}

/* NEXT-3. Block-sparse UNet ResNet block with latent reuse ("ResNet layers ... can be
 * safely applied only to frames selected for refinement"; "reuses cached latents from
 * the last full denoising step for unrefined regions"; readings R-26, R-27):
 *   a1 = bf16(SiLU(GN1(x)))                       GN statistics over the full current map x
 *   h  = listed ? bf16(conv3x3(a1; w1) + b1) : h_cache
 *   a2 = bf16(SiLU(GN2(h)))                       GN statistics over the full map h
 *   y  = listed ? x + conv3x3(a2; w2) + b2 : y_cache       (identity skip, C_in = C_out)
 * x, h_cache: bf16 bits NHWC [n][h][w][c]; y_cache: double.  w1, w2: bf16 bits [c][3][3][c];
 * b1, b2, g1, be1, g2, be2: fp32 [c].  Outputs (every pixel, double unless noted):
 * a1_pre / a2_pre = the SiLU values before bf16 rounding; a1, a2 = their bf16 bits;
 * h_pre = listed ? conv1 value (before rounding) : decoded h_cache; h_out = bf16 bits of h;
 * h_abs / y_abs = sum |w*a| (+|b|) at listed pixels (0 elsewhere); y.  Any output may be
 * NULL except y. */
int oracle_resblock(const uint16_t* x, const uint16_t* h_cache, const double* y_cache,
                    const uint16_t* w1, const float* b1, const uint16_t* w2, const float* b2,
                    const float* g1, const float* be1, const float* g2, const float* be2,
                    int groups, double eps, int n, int h, int w, int c, int b,
                    const int32_t* ids, int count, double* a1_pre, uint16_t* a1_out,
                    double* h_pre, double* h_abs, uint16_t* h_out, double* a2_pre,
                    uint16_t* a2_out, double* y, double* y_abs, int n_threads) {
  if (!x || !h_cache || !y_cache || !w1 || !w2 || !g1 || !be1 || !g2 || !be2 || !y) return BAD;
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || b <= 0 || groups <= 0 || c % groups != 0) return BAD;
  if (count < 0 || (count > 0 && !ids)) return BAD;
  int hb = (h + b - 1) / b, wb = (w + b - 1) / b;
  for (int j = 0; j < count; ++j)
    if (ids[j] < 0 || ids[j] >= n * hb * wb) return BAD;
  size_t npx = (size_t)n * h * w, tot = npx * c;
  /* listed[pixel]: the pixel's block is in the list (P:352 block granularity) */
  uint8_t* listed = (uint8_t*)calloc(npx, 1);
  double* xd = widen(x, tot);
  double* m = (double*)malloc((size_t)n * groups * sizeof(double));
  double* v = (double*)malloc((size_t)n * groups * sizeof(double));
  double* act = (double*)malloc(tot * sizeof(double));
  uint16_t* abits = (uint16_t*)malloc(tot * sizeof(uint16_t));
  double* cv = (double*)malloc(tot * sizeof(double));
  double* ca = (double*)malloc(tot * sizeof(double));
  uint16_t* hb16 = (uint16_t*)malloc(tot * sizeof(uint16_t));
  double* hd = (double*)malloc(tot * sizeof(double));
  int rc = 0;
  if (!listed || !xd || !m || !v || !act || !abits || !cv || !ca || !hb16 || !hd) { rc = -2; goto done; }
  for (int j = 0; j < count; ++j) {
    int id = ids[j];
    int i = id / (hb * wb), by = (id / wb) % hb, bx = id % wb;
    for (int yy = by * b; yy < by * b + b && yy < h; ++yy)
      for (int xx = bx * b; xx < bx * b + b && xx < w; ++xx) listed[((size_t)i * h + yy) * w + xx] = 1;
  }
  /* 1. a1 = bf16(SiLU(GN1(x))) over the full map */
  if ((rc = oracle_gn_stats(xd, n, h, w, c, groups, m, v)) != 0) goto done;
  if ((rc = oracle_gn_silu(xd, n, h, w, c, groups, m, v, g1, be1, eps, NULL, act)) != 0) goto done;
  for (size_t e = 0; e < tot; ++e) abits[e] = oracle_bf16_rne(act[e]);
  if (a1_pre) memcpy(a1_pre, act, tot * sizeof(double));
  if (a1_out) memcpy(a1_out, abits, tot * sizeof(uint16_t));
  /* 2. h = listed ? bf16(conv1) : h_cache */
  for (size_t e = 0; e < tot; ++e) { cv[e] = 0.0; ca[e] = 0.0; }
  if ((rc = oracle_conv3x3_blocks(abits, w1, b1, n, h, w, c, c, b, ids, count, cv, ca, n_threads)) != 0)
    goto done;
  for (size_t p = 0; p < npx; ++p)
    for (int ch = 0; ch < c; ++ch) {
      size_t e = p * c + ch;
      hb16[e] = listed[p] ? oracle_bf16_rne(cv[e]) : h_cache[e];
      hd[e] = bf16_to_double(hb16[e]);
      if (h_pre) h_pre[e] = listed[p] ? cv[e] : hd[e];
      if (h_abs) h_abs[e] = listed[p] ? ca[e] : 0.0;
    }
  if (h_out) memcpy(h_out, hb16, tot * sizeof(uint16_t));
  /* 3. a2 = bf16(SiLU(GN2(h))) over the full map */
  if ((rc = oracle_gn_stats(hd, n, h, w, c, groups, m, v)) != 0) goto done;
  if ((rc = oracle_gn_silu(hd, n, h, w, c, groups, m, v, g2, be2, eps, NULL, act)) != 0) goto done;
  for (size_t e = 0; e < tot; ++e) abits[e] = oracle_bf16_rne(act[e]);
  if (a2_pre) memcpy(a2_pre, act, tot * sizeof(double));
  if (a2_out) memcpy(a2_out, abits, tot * sizeof(uint16_t));
  /* 4. y = listed ? x + conv2 : y_cache  (identity skip) */
  for (size_t e = 0; e < tot; ++e) { cv[e] = 0.0; ca[e] = 0.0; }
  if ((rc = oracle_conv3x3_blocks(abits, w2, b2, n, h, w, c, c, b, ids, count, cv, ca, n_threads)) != 0)
    goto done;
  for (size_t p = 0; p < npx; ++p)
    for (int ch = 0; ch < c; ++ch) {
      size_t e = p * c + ch;
      y[e] = listed[p] ? xd[e] + cv[e] : y_cache[e];
      if (y_abs) y_abs[e] = listed[p] ? ca[e] + fabs(xd[e]) : 0.0;
    }
done:
  free(listed); free(xd); free(m); free(v); free(act); free(abits); free(cv); free(ca);
  free(hb16); free(hd);
  return rc;
}

/* ------------------------------------------------------------- NEXT-4 ---- */

/* NEXT-4. Frame-sparse temporal attention with the latent cache ("every T steps, the
 * model performs a full denoising pass ... the intermediate latent representations from each
 * temporal attention layer are cached.  In the subsequent (T-1) partial denoising steps,
 * frames that are not actively refined simply retrieve and reuse these cached latents";
 * reading R-28).  Per pixel p, the frames of a sequence (T consecutive frames) are the tokens:
 *   qkv = listed ? bf16(Wqkv x + bqkv) : qkv_cache                   (K/V cache of every frame)
 *   o[n,p] = softmax_m(q_n . k_m / sqrt(d)) v_m, m over n's sequence, per head of d = c/heads
 *   y = listed ? x + Wo bf16(o) + bo : y_cache                       (identity residual)
 * x: bf16 bits [n][h][w][c]; qkv_cache: bf16 bits [n][h][w][3c] (q | k | v, head-major);
 * wqkv: bf16 bits [3c][c]; wo: bf16 bits [c][c]; bqkv [3c], bo [c] fp32 or NULL.
 * Outputs (every pixel): qkv_pre (listed: fp64 projection, else decoded cache), qkv_out
 * (bits), qkv_abs (sum |w x| + |b| at listed, else 0), o_pre / o_out (listed only, else 0),
 * y, y_abs (|x| + |bo| + sum |wo o| at listed, else 0).  Outputs other than y may be NULL. */
int oracle_temporal_attn(const uint16_t* x, const uint16_t* qkv_cache, const double* y_cache,
                         const uint16_t* wqkv, const float* bqkv, const uint16_t* wo,
                         const float* bo, int n, int h, int w, int c, int heads, int T, int b,
                         const int32_t* ids, int count, double* qkv_pre, uint16_t* qkv_out,
                         double* qkv_abs, double* o_pre, uint16_t* o_out, double* y, double* y_abs) {
  if (!x || !qkv_cache || !y_cache || !wqkv || !wo || !y) return BAD;
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || b <= 0 || heads <= 0 || c % heads != 0 || T <= 0 ||
      n % T != 0)
    return BAD;
  if (count < 0 || (count > 0 && !ids)) return BAD;
  int hb = (h + b - 1) / b, wb = (w + b - 1) / b;
  for (int j = 0; j < count; ++j)
    if (ids[j] < 0 || ids[j] >= n * hb * wb) return BAD;
  int c3 = 3 * c, d = c / heads;
  size_t npx = (size_t)n * h * w, plane = (size_t)h * w;
  uint8_t* listed = (uint8_t*)calloc(npx, 1);
  double* xd = widen(x, npx * c);
  double* wq = widen(wqkv, (size_t)c3 * c);
  double* wd = widen(wo, (size_t)c * c);
  uint16_t* qb = (uint16_t*)malloc(npx * c3 * sizeof(uint16_t));
  double* qv = (double*)malloc(npx * c3 * sizeof(double));
  uint16_t* ob = (uint16_t*)calloc(npx * c, sizeof(uint16_t));
  double* sc = (double*)malloc((size_t)T * sizeof(double));
  int rc = 0;
  if (!listed || !xd || !wq || !wd || !qb || !qv || !ob || !sc) { rc = -2; goto done4; }
  for (int j = 0; j < count; ++j) {
    int id = ids[j];
    int i = id / (hb * wb), by = (id / wb) % hb, bx = id % wb;
    for (int yy = by * b; yy < by * b + b && yy < h; ++yy)
      for (int xx = bx * b; xx < bx * b + b && xx < w; ++xx) listed[((size_t)i * h + yy) * w + xx] = 1;
  }
  /* 1. projections of the listed (frame, pixel) tokens; cached K/V (and Q) elsewhere */
  for (size_t p = 0; p < npx; ++p)
    for (int j = 0; j < c3; ++j) {
      size_t e = p * c3 + j;
      if (listed[p]) {
        double acc = bqkv ? (double)bqkv[j] : 0.0, aab = bqkv ? fabs((double)bqkv[j]) : 0.0;
        for (int ci = 0; ci < c; ++ci) {
          double pr = wq[(size_t)j * c + ci] * xd[p * c + ci];
          acc += pr;
          aab += fabs(pr);
        }
        if (qkv_pre) qkv_pre[e] = acc;
        if (qkv_abs) qkv_abs[e] = aab;
        qb[e] = oracle_bf16_rne(acc);
      } else {
        qb[e] = qkv_cache[e];
        if (qkv_pre) qkv_pre[e] = bf16_to_double(qkv_cache[e]);
        if (qkv_abs) qkv_abs[e] = 0.0;
      }
      qv[e] = bf16_to_double(qb[e]);
    }
  if (qkv_out) memcpy(qkv_out, qb, npx * c3 * sizeof(uint16_t));
  /* 2. attention over the frames of the sequence at the same pixel, listed queries only */
  double inv = 1.0 / sqrt((double)d);
  for (int i = 0; i < n; ++i)
    for (size_t p = 0; p < plane; ++p) {
      size_t pi = (size_t)i * plane + p;
      for (int hd = 0; hd < heads; ++hd)
        for (int k = 0; k < d; ++k) {
          size_t eo = pi * c + hd * d + k;
          if (o_pre) o_pre[eo] = 0.0;
        }
      if (!listed[pi]) continue;
      int s0 = (i / T) * T;
      for (int hd = 0; hd < heads; ++hd) {
        const double* q = qv + pi * c3 + hd * d;
        double mx = -INFINITY;
        for (int m = 0; m < T; ++m) {
          const double* kk = qv + ((size_t)(s0 + m) * plane + p) * c3 + c + hd * d;
          double s = 0.0;
          for (int k = 0; k < d; ++k) s += q[k] * kk[k];
          sc[m] = s * inv;
          if (sc[m] > mx) mx = sc[m];
        }
        double den = 0.0;
        for (int m = 0; m < T; ++m) { sc[m] = exp(sc[m] - mx); den += sc[m]; }
        for (int k = 0; k < d; ++k) {
          double o = 0.0;
          for (int m = 0; m < T; ++m)
            o += sc[m] / den * qv[((size_t)(s0 + m) * plane + p) * c3 + 2 * c + hd * d + k];
          size_t eo = pi * c + hd * d + k;
          if (o_pre) o_pre[eo] = o;
          ob[eo] = oracle_bf16_rne(o);
        }
      }
    }
  if (o_out) memcpy(o_out, ob, npx * c * sizeof(uint16_t));
  /* 3. output projection + identity residual on listed pixels, cache elsewhere */
  for (size_t p = 0; p < npx; ++p)
    for (int co = 0; co < c; ++co) {
      size_t e = p * c + co;
      if (!listed[p]) {
        y[e] = y_cache[e];
        if (y_abs) y_abs[e] = 0.0;
        continue;
      }
      double acc = (bo ? (double)bo[co] : 0.0), aab = (bo ? fabs((double)bo[co]) : 0.0);
      for (int ci = 0; ci < c; ++ci) {
        double pr = wd[(size_t)co * c + ci] * bf16_to_double(ob[p * c + ci]);
        acc += pr;
        aab += fabs(pr);
      }
      y[e] = xd[e] + acc;
      if (y_abs) y_abs[e] = aab + fabs(xd[e]);
    }
done4:
  free(listed); free(xd); free(wq); free(wd); free(qb); free(qv); free(ob); free(sc);
  return rc;
}
