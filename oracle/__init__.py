"""CPU ORACLE for the Sphinx selective-refinement hot path — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The product
path (``paper_2511_18672_b200``) never imports it and shares no code with it.

The arithmetic lives in ``sphinx_oracle.c`` (plain C99, fp64, cited per
function against PAPER.md / SPEC.md).  This module only marshals numpy arrays
through ctypes.

Parity status per function:
  pixel_mask / maxpool / tile_blocks / block_mask   pinned (TV-1..5, brute force)
  eq2 / select_k / start_step                       pinned (TV-6..8; gamma=0.5
                                                    is the correctly rounded sqrt, checked exactly
                                                    with rationals; realized-ratio cut points);
                                                    the k-logic TABLE values are parity unpinned
                                                    (Fig. k_logic is an image)
  compact                                           pinned (popcount, brute-force order, identity)
  noise                                             pinned (TV-9..11, Monte Carlo)
  conv3x3_blocks / conv3x3_dense                    pinned (shift kernels, torch fp64 conv2d, linearity)
  scatter                                           pinned (density 0/1, composition O7)
  ddim_step (NEXT-1)                                pinned (S:315 collapse to the clean latent,
                                                    S:316 flat segment, eps-direction invariant)
  laplacian_var / box_smooth / otsu / uncertainty   pinned (S:201-213 examples, brute-force Otsu
    (NEXT-2)                                        argmax, variance identities)
  bf16_rne / gn_stats / gn_silu / resblock          pinned (torch RNE float->bfloat16 incl. ties,
    (NEXT-3)                                        torch fp64 group_norm/silu/conv2d dense
                                                    formulation, density 0, cache consistency)
  temporal_attn (NEXT-4)                            pinned (T=1 closed form o = v, torch fp64
                                                    linear + scaled_dot_product_attention,
                                                    frame-permutation equivariance, uniform keys,
                                                    cache consistency, stale-cache locality)
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

SELECT_ACTIVE, SELECT_INACTIVE_FRAMES, SELECT_ALL, SELECT_NOISE = 0, 1, 2, 3
SRC_FULL, SRC_COMPACT = 0, 1


class KLogic(ctypes.Structure):
    """Mirror of ``oracle_klogic``."""
    _fields_ = [("m", ctypes.c_int32), ("thr", ctypes.c_double * 16),
                ("step", ctypes.c_int32 * 16), ("fallback_k", ctypes.c_int32),
                ("k_max", ctypes.c_int32)]


def make_klogic(thr, steps, fallback_k=0, k_max=40):
    lg = KLogic()
    lg.m = len(thr)
    for i, (t, s) in enumerate(zip(thr, steps)):
        lg.thr[i] = float(t)
        lg.step[i] = int(s)
    lg.fallback_k = fallback_k
    lg.k_max = k_max
    return lg


def build(force=False):
    """Compile liboracle.so with gcc (no CUDA headers, no fast-math, no FMA contraction)."""
    src = os.path.join(_HERE, "sphinx_oracle.c")
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= os.path.getmtime(src):
        return _SO
    cmd = ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-fno-fast-math", "-o", _SO, src, "-lm"]
    subprocess.check_call(cmd)
    return _SO


def load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        I = ctypes.c_int
        F = ctypes.c_float
        D = ctypes.c_double
        sig = {
            "oracle_pixel_mask": [P, P, P, F, I, I, I, P],
            "oracle_maxpool": [P, I, I, I, I, P],
            "oracle_tile_blocks": [P, I, I, I, I, P],
            "oracle_block_mask": [P, P, P, F, I, I, I, I, I, I, P, P],
            "oracle_start_step": [P, P, P, P, P, D, P, I, I, P],
            "oracle_compact": [P, I, I, I, P, I, I, P, P],
            "oracle_noise": [P, P, P, P, I, I, I, I, I, P, I, P, P, I],
            "oracle_conv3x3_blocks": [P, P, P, I, I, I, I, I, I, P, I, P, P, I],
            "oracle_conv3x3_dense": [P, P, P, I, I, I, I, I, P, P, I],
            "oracle_scatter": [P, I, P, P, I, I, I, I, I, I, P, P, I, P, I],
            "oracle_ddim_step": [P, P, P, I, I, I, I, I, P, I, I, P, I],
            "oracle_laplacian_var": [P, I, I, I, I, P],
            "oracle_box_smooth": [P, I, I, I, I, P],
            "oracle_otsu": [P, ctypes.c_long, P],
            "oracle_otsu_f64": [P, ctypes.c_long, P],
            "oracle_uncertainty": [P, I, I, I, I, I, P, P],
            "oracle_gn_stats": [P, I, I, I, I, I, P, P],
            "oracle_gn_silu": [P, I, I, I, I, I, P, P, P, P, D, P, P],
            "oracle_resblock": [P, P, P, P, P, P, P, P, P, P, P, I, D, I, I, I, I, I, P, I,
                                P, P, P, P, P, P, P, P, P, I],
            "oracle_temporal_attn": [P, P, P, P, P, P, P, I, I, I, I, I, I, I, P, I,
                                     P, P, P, P, P, P, P],
        }
        for name, args in sig.items():
            fn = getattr(_lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        _lib.oracle_eq2.argtypes = [D, D, D, D]
        _lib.oracle_eq2.restype = D
        _lib.oracle_eq2_batch.argtypes = [P, P, P, D, I, P]
        _lib.oracle_eq2_batch.restype = None
        _lib.oracle_select_k.argtypes = [P, D]
        _lib.oracle_select_k.restype = ctypes.c_int32
        _lib.oracle_bf16_rne.argtypes = [D]
        _lib.oracle_bf16_rne.restype = ctypes.c_uint16
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def _check(rc, name):
    if rc != 0:
        raise ValueError(f"{name}: invalid argument (rc={rc})")


def level_dims(hp, wp, f, b, n_levels):
    """Geometry only: (H_l, W_l, Hb_l, Wb_l) per level (/f then /2 per level)."""
    out = []
    h, w = hp // f, wp // f
    for l in range(n_levels):
        out.append((h, w, -(-h // b), -(-w // b)))
        h, w = h // 2, w // 2
    return out


def pixel_mask(O, U, tau_u, tau_o):
    lib = load()
    O = _c(O, np.float32); U = _c(U, np.float32); tau_u = _c(tau_u, np.float32)
    n, hp, wp = O.shape
    m = np.zeros((n, hp, wp), np.uint8)
    _check(lib.oracle_pixel_mask(_p(O), _p(U), _p(tau_u), tau_o, n, hp, wp, _p(m)), "pixel_mask")
    return m


def maxpool(grid, f):
    lib = load()
    g = _c(grid, np.uint8)
    n, h, w = g.shape
    out = np.zeros((n, h // f, w // f), np.uint8)
    _check(lib.oracle_maxpool(_p(g), n, h, w, f, _p(out)), "maxpool")
    return out


def tile_blocks(grid, b):
    lib = load()
    g = _c(grid, np.uint8)
    n, h, w = g.shape
    out = np.zeros((n, -(-h // b), -(-w // b)), np.uint8)
    _check(lib.oracle_tile_blocks(_p(g), n, h, w, b, _p(out)), "tile_blocks")
    return out


def block_mask(O, U, tau_u, tau_o, f, b, n_levels):
    """Returns (list of per-level u8 masks [n,Hb,Wb], counts int32 [n, n_levels])."""
    lib = load()
    O = _c(O, np.float32); U = _c(U, np.float32); tau_u = _c(tau_u, np.float32)
    n, hp, wp = O.shape
    dims = level_dims(hp, wp, f, b, n_levels)
    sizes = [n * hb * wb for (_, _, hb, wb) in dims]
    flat = np.zeros(sum(sizes), np.uint8)
    counts = np.zeros((n, n_levels), np.int32)
    _check(lib.oracle_block_mask(_p(O), _p(U), _p(tau_u), tau_o, n, hp, wp, f, b, n_levels,
                                 _p(flat), _p(counts)), "block_mask")
    masks, off = [], 0
    for (sz, (_, _, hb, wb)) in zip(sizes, dims):
        masks.append(flat[off:off + sz].reshape(n, hb, wb).copy())
        off += sz
    return masks, counts


def eq2(c0, c1, t, gamma):
    return load().oracle_eq2(c0, c1, t, gamma)


def eq2_batch(c0, c1, t, gamma):
    c0 = _c(c0, np.float64); c1 = _c(c1, np.float64); t = _c(t, np.float64)
    out = np.empty(len(t), np.float64)
    load().oracle_eq2_batch(_p(c0), _p(c1), _p(t), float(gamma), len(t), _p(out))
    return out


def select_k(logic, r):
    return load().oracle_select_k(ctypes.byref(logic), r)


def start_step(q, c0, c1, t, gamma, logics, logic_id=None):
    lib = load()
    q = _c(q, np.float32); c0 = _c(c0, np.float32); c1 = _c(c1, np.float32); t = _c(t, np.float32)
    lid = _c(logic_id, np.int32)
    n = q.shape[0]
    arr = (KLogic * len(logics))(*logics)
    k = np.zeros(n, np.int32)
    _check(lib.oracle_start_step(_p(q), _p(c0), _p(c1), _p(t), _p(lid), gamma,
                                 ctypes.cast(arr, ctypes.c_void_p), len(logics), n, _p(k)),
           "start_step")
    return k


def compact(mask, k=None, u=0, select=SELECT_ACTIVE, shape=None):
    lib = load()
    m = _c(mask, np.uint8) if mask is not None else None
    n, hb, wb = m.shape if m is not None else shape
    kk = _c(k, np.int32)
    ids = np.zeros(max(n * hb * wb, 1), np.int32)
    cnt = np.zeros(1, np.int32)
    _check(lib.oracle_compact(_p(m), n, hb, wb, _p(kk), int(u), select, _p(ids), _p(cnt)), "compact")
    return ids[:cnt[0]].copy()


def noise(x0, eps, xt_in, b, ids, step, abar):
    lib = load()
    x0 = _c(x0, np.float32); eps = _c(eps, np.float32); xt_in = _c(xt_in, np.float32)
    ids = _c(ids, np.int32); step = _c(step, np.int32); abar = _c(abar, np.float32)
    n, h, w, c = x0.shape
    out = np.zeros(x0.shape, np.float64)
    _check(lib.oracle_noise(_p(x0), _p(eps), _p(xt_in), _p(out), n, h, w, c, b,
                            _p(ids), len(ids), _p(step), _p(abar), len(abar) - 1), "noise")
    return out


def conv3x3_blocks(x_bf16bits, w_bf16bits, bias, b, ids, n_threads=0, y_init=None):
    """x: uint16 [n,h,w,cin] bf16 bits; w: uint16 [cout,3,3,cin]; returns (y, absacc) fp64.
    Pixels outside listed blocks hold y_init (default NaN) / NaN."""
    lib = load()
    x = _c(x_bf16bits, np.uint16); w = _c(w_bf16bits, np.uint16)
    bias = _c(bias, np.float32); ids = _c(ids, np.int32)
    n, h, wd, cin = x.shape
    cout = w.shape[0]
    y = np.full((n, h, wd, cout), np.nan) if y_init is None else np.array(y_init, np.float64)
    a = np.full((n, h, wd, cout), np.nan)
    _check(lib.oracle_conv3x3_blocks(_p(x), _p(w), _p(bias), n, h, wd, cin, cout, b,
                                     _p(ids), len(ids), _p(y), _p(a), n_threads), "conv3x3_blocks")
    return y, a


def conv3x3_dense(x_bf16bits, w_bf16bits, bias, n_threads=0):
    lib = load()
    x = _c(x_bf16bits, np.uint16); w = _c(w_bf16bits, np.uint16); bias = _c(bias, np.float32)
    n, h, wd, cin = x.shape
    cout = w.shape[0]
    y = np.zeros((n, h, wd, cout)); a = np.zeros((n, h, wd, cout))
    _check(lib.oracle_conv3x3_dense(_p(x), _p(w), _p(bias), n, h, wd, cin, cout,
                                    _p(y), _p(a), n_threads), "conv3x3_dense")
    return y, a


def scatter(src, cache, b, mask=None, k=None, u=0, ids=None, src_layout=SRC_FULL):
    """Bit copy; src/cache any 2- or 4-byte dtype, NHWC (or COMPACT [count,b,b,c])."""
    lib = load()
    cache = np.ascontiguousarray(cache)
    src = np.ascontiguousarray(src, dtype=cache.dtype)
    n, h, w, c = cache.shape
    out = np.empty_like(cache)
    m = _c(mask, np.uint8); kk = _c(k, np.int32); ids = _c(ids, np.int32)
    cnt = 0 if ids is None else len(ids)
    _check(lib.oracle_scatter(_p(src), src_layout, _p(cache), _p(out), cache.dtype.itemsize,
                              n, h, w, c, b, _p(m), _p(kk), int(u), _p(ids), cnt), "scatter")
    return out


def ddim_step(z, x0_hat, b, ids, u, abar):
    """NEXT-1 DDIM update on listed blocks, fp64; unlisted elements = z."""
    lib = load()
    z = _c(z, np.float32); x0_hat = _c(x0_hat, np.float32); ids = _c(ids, np.int32)
    abar = _c(abar, np.float32)
    n, h, w, c = z.shape
    out = np.zeros(z.shape, np.float64)
    _check(lib.oracle_ddim_step(_p(z), _p(x0_hat), _p(out), n, h, w, c, b, _p(ids), len(ids), int(u),
                                _p(abar), len(abar) - 1), "ddim_step")
    return out


def laplacian_var(rgb, window=7):
    lib = load()
    rgb = _c(rgb, np.float32)
    n, h, w, _ = rgb.shape
    B = np.zeros((n, h, w))
    _check(lib.oracle_laplacian_var(_p(rgb), n, h, w, window, _p(B)), "laplacian_var")
    return B


def box_smooth(x, k=5):
    lib = load()
    x = _c(x, np.float64)
    n, h, w = x.shape
    out = np.zeros_like(x)
    _check(lib.oracle_box_smooth(_p(x), n, h, w, k, _p(out)), "box_smooth")
    return out


def otsu(values):
    """tau for one grid (float32 values, the kernel's precision) -- NEXT-2c."""
    lib = load()
    v = _c(values, np.float32).ravel()
    tau = np.zeros(1, np.float32)
    _check(lib.oracle_otsu(_p(v), v.size, _p(tau)), "otsu")
    return float(tau[0])


def otsu_f64(values):
    lib = load()
    v = _c(values, np.float64).ravel()
    tau = np.zeros(1, np.float32)
    _check(lib.oracle_otsu_f64(_p(v), v.size, _p(tau)), "otsu_f64")
    return float(tau[0])


def uncertainty(rgb, window=7, smooth=5):
    """(U fp64 [n,h,w], tau fp32 [n]) -- NEXT-2."""
    lib = load()
    rgb = _c(rgb, np.float32)
    n, h, w, _ = rgb.shape
    U = np.zeros((n, h, w))
    tau = np.zeros(n, np.float32)
    _check(lib.oracle_uncertainty(_p(rgb), n, h, w, window, smooth, _p(U), _p(tau)), "uncertainty")
    return U, tau


def bf16_rne(v):
    """NEXT-3: bfloat16 bits of each double, round to nearest even (from fp64 directly)."""
    lib = load()
    v = np.asarray(v, np.float64)
    return np.array([lib.oracle_bf16_rne(float(t)) for t in v.ravel()], np.uint16).reshape(v.shape)


def gn_stats(x, groups):
    """NEXT-3a: per (frame, group) mean and population variance over the full NHWC map."""
    lib = load()
    x = _c(x, np.float64)
    n, h, w, c = x.shape
    mean = np.zeros((n, groups)); var = np.zeros((n, groups))
    _check(lib.oracle_gn_stats(_p(x), n, h, w, c, groups, _p(mean), _p(var)), "gn_stats")
    return mean, var


def gn_silu(x, groups, gamma, beta, eps, mean=None, var=None):
    """NEXT-3b: (t, SiLU(t)) with t = GroupNorm(x) (statistics of x unless given)."""
    lib = load()
    x = _c(x, np.float64)
    if mean is None:
        mean, var = gn_stats(x, groups)
    mean = _c(mean, np.float64); var = _c(var, np.float64)
    gamma = _c(gamma, np.float32); beta = _c(beta, np.float32)
    n, h, w, c = x.shape
    t = np.zeros(x.shape); a = np.zeros(x.shape)
    _check(lib.oracle_gn_silu(_p(x), n, h, w, c, groups, _p(mean), _p(var), _p(gamma), _p(beta),
                              float(eps), _p(t), _p(a)), "gn_silu")
    return t, a


def resblock(x_bits, h_cache_bits, y_cache, w1_bits, b1, w2_bits, b2, g1, be1, g2, be2,
             groups, eps, b, ids, n_threads=0):
    """NEXT-3 sparse ResNet block (R-26, R-27).  Returns a dict of fp64 / bf16-bit arrays:
    a1_pre, a1, h_pre, h_abs, h, a2_pre, a2, y, y_abs (see sphinx_oracle.c)."""
    lib = load()
    x = _c(x_bits, np.uint16); hc = _c(h_cache_bits, np.uint16); yc = _c(y_cache, np.float64)
    w1 = _c(w1_bits, np.uint16); w2 = _c(w2_bits, np.uint16)
    b1 = _c(b1, np.float32); b2 = _c(b2, np.float32)
    g1 = _c(g1, np.float32); be1 = _c(be1, np.float32)
    g2 = _c(g2, np.float32); be2 = _c(be2, np.float32)
    ids = _c(ids, np.int32)
    n, h, w, c = x.shape
    o = {k: np.zeros(x.shape) for k in ("a1_pre", "h_pre", "h_abs", "a2_pre", "y", "y_abs")}
    o.update({k: np.zeros(x.shape, np.uint16) for k in ("a1", "h", "a2")})
    _check(lib.oracle_resblock(_p(x), _p(hc), _p(yc), _p(w1), _p(b1), _p(w2), _p(b2),
                               _p(g1), _p(be1), _p(g2), _p(be2), int(groups), float(eps),
                               n, h, w, c, b, _p(ids), len(ids),
                               _p(o["a1_pre"]), _p(o["a1"]), _p(o["h_pre"]), _p(o["h_abs"]),
                               _p(o["h"]), _p(o["a2_pre"]), _p(o["a2"]), _p(o["y"]),
                               _p(o["y_abs"]), n_threads), "resblock")
    return o


def temporal_attn(x_bits, qkv_cache_bits, y_cache, wqkv_bits, bqkv, wo_bits, bo, heads, T, b, ids):
    """NEXT-4 frame-sparse temporal attention with the K/V cache (R-28).  Returns a dict:
    qkv_pre, qkv (bits), qkv_abs, o_pre, o (bits), y, y_abs (see sphinx_oracle.c)."""
    lib = load()
    x = _c(x_bits, np.uint16); qc = _c(qkv_cache_bits, np.uint16); yc = _c(y_cache, np.float64)
    wq = _c(wqkv_bits, np.uint16); wo = _c(wo_bits, np.uint16)
    bq = _c(bqkv, np.float32); bo = _c(bo, np.float32); ids = _c(ids, np.int32)
    n, h, w, c = x.shape
    o = {"qkv_pre": np.zeros((n, h, w, 3 * c)), "qkv": np.zeros((n, h, w, 3 * c), np.uint16),
         "qkv_abs": np.zeros((n, h, w, 3 * c)), "o_pre": np.zeros(x.shape),
         "o": np.zeros(x.shape, np.uint16), "y": np.zeros(x.shape), "y_abs": np.zeros(x.shape)}
    _check(lib.oracle_temporal_attn(_p(x), _p(qc), _p(yc), _p(wq), _p(bq), _p(wo), _p(bo), n, h, w, c,
                                    int(heads), int(T), int(b), _p(ids), len(ids), _p(o["qkv_pre"]),
                                    _p(o["qkv"]), _p(o["qkv_abs"]), _p(o["o_pre"]), _p(o["o"]),
                                    _p(o["y"]), _p(o["y_abs"])), "temporal_attn")
    return o
