"""GPU parity of NEXT-3, the block-sparse ResNet block (readings R-26, R-27),
through the C ABI against the CPU oracle on the same seeded inputs.

Bars (derived from the arithmetic):
* GroupNorm+SiLU: the GPU computes the activation in fp32 from fp32 statistics and rounds it
  once to bf16; the oracle computes it in fp64.  Given a bound d on the fp32 pre-rounding error,
  the GPU value must lie within half a bf16 ulp + d of the oracle's unrounded value, i.e. it is
  the oracle's own bf16 rounding except where the fp64 value is within d of a rounding midpoint.
  d = 1.1 (|gamma| 1e-5 (1 + (|mean| + |x - mean|)/sd) + 1e-6 |t|) + 1e-6 |a| + 1e-7
  (fp32 statistics: relative 1e-5 of the scale; |SiLU'| <= 1.1).
* Shift weights (one tap, no bias): each conv is an exact copy, so the block output differs from
  the oracle only by these roundings and their propagation through GN2 (first-order bound, h
  allowed one bf16 ulp): tight, any wiring bug (wrong stats, frame, group, halo, cache, skip)
  is O(1).
* Random weights: the same chain with the conv bound 1e-3 sum|w a| (+ one ulp of every a1)
  feeding GN2, and 1e-3 sum|w a2| + sum|w2| E_a2 at the output.
* Unlisted pixels of h and y, and statistics entries of unlisted blocks: untouched, bitwise.
"""
import numpy as np
import pytest

import oracle
import synthetic as syn

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
dev = "cuda"
G, EPS = syn.GN_GROUPS, syn.GN_EPS


def T(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(dev)


def bf16(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(dev)


def bits_of(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def dec(bits):
    return syn.bf16_bits_to_f32(bits).astype(np.float64)


def half_ulp(v):
    """Half a bf16 ulp at |v| (8 significant bits): v = m 2^e, m in [0.5, 1) -> 2^(e-9)."""
    _, e = np.frexp(np.abs(np.asarray(v, np.float64)))
    return np.ldexp(1.0, e - 9)


def gpu_ids(sp, mask):
    n, hb, wb = mask.shape
    ids = torch.full((n * hb * wb,), -7, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    sp.sphinx_compact_blocks(T(mask.astype(np.uint8)), None, 0, 0, ids, cnt, shape=(n, hb, wb))
    return ids, cnt


def block_mask(n, h, w, b, density, pattern, tag):
    hb, wb = -(-h // b), -(-w // b)
    rg = syn.rng("rb-mask", tag)
    return np.stack([syn.choose_cells(rg, hb, wb, round(density * hb * wb), pattern)
                     for _ in range(n)]).astype(np.uint8)


def dilated_px(mask, h, w, b):
    """Pixels of listed blocks and their 1-pixel ring (what a 3x3 conv over the list reads)."""
    n, hb, wb = mask.shape
    m = np.zeros((n, h, w), bool)
    for i, by, bx in zip(*np.nonzero(mask)):
        m[i, max(by * b - 1, 0):min(by * b + b + 1, h), max(bx * b - 1, 0):min(bx * b + b + 1, w)] = True
    return m


def listed_px(mask, h, w, b):
    n, hb, wb = mask.shape
    m = np.zeros((n, h, w), bool)
    for i, by, bx in zip(*np.nonzero(mask)):
        m[i, by * b:by * b + b, bx * b:bx * b + b] = True
    return m


def act_err_bound(x, t, a, gamma, groups):
    """d of the module docstring, per element (oracle values only)."""
    n, h, w, c = x.shape
    mean, var = oracle.gn_stats(x, groups)
    cg = c // groups
    mu = np.repeat(mean, cg, axis=1)[:, None, None, :]
    sd = np.sqrt(np.repeat(var, cg, axis=1) + EPS)[:, None, None, :]
    g = np.abs(gamma.astype(np.float64))
    dt = g * 1e-5 * (1.0 + (np.abs(mu) + np.abs(x - mu)) / sd) + 1e-6 * np.abs(t)
    return 1.1 * dt + 1e-6 * np.abs(a) + 1e-7, mu, sd


def _inputs(n, h, w, c, tag):
    x = syn.resblock_features_bf16((n, h, w, c), tag)
    g1, be1 = syn.gn_affine_f32(c, tag + "-1")
    return x, g1, be1


# ------------------------------------------------------------ GroupNorm + SiLU

@pytest.mark.parametrize("n,h,w,c,b,groups,dens,pattern", [
    (2, 16, 16, 32, 4, 8, 0.25, "scattered"),
    (2, 72, 72, 320, 8, 32, 0.25, "clustered"),
    (2, 36, 36, 640, 8, 32, 0.4, "scattered"),
    (3, 18, 18, 1280, 8, 32, 0.5, "checker"),
    (2, 20, 13, 64, 8, 16, 0.6, "scattered"),
    (1, 24, 24, 2048, 8, 32, 0.3, "clustered"),
])
def test_gn_silu_vs_oracle_incremental_stats(sphinx, n, h, w, c, b, groups, dens, pattern):
    """Full step: statistics of x_old for EVERY block.  Partial step: listed blocks of x_new
    (= x_old with fresh listed blocks) rewrite their entries only; the activation of x_new on
    listed blocks + ring equals the oracle's full-map GroupNorm of x_new (R-26)."""
    tag = f"gn{n}{h}{w}{c}"
    x_old, g1, be1 = _inputs(n, h, w, c, tag)
    mask = block_mask(n, h, w, b, dens, pattern, tag)
    L = listed_px(mask, h, w, b)
    x_new = x_old.copy()
    x_new[L] = syn.resblock_features_bf16((n, h, w, c), tag + "-fresh")[L]
    hb, wb = mask.shape[1:]
    stats = sphinx.gn_stats_buffer(n, h, w, groups, b, dev)
    all_ids, all_cnt = gpu_ids(sphinx, np.ones_like(mask))
    sphinx.sphinx_gn_block_stats(bf16(x_old), groups, b, all_ids, all_cnt, stats)
    before = sphinx.gn_block_entries(stats, n, h, w, groups, b).cpu().numpy().copy()
    ids, cnt = gpu_ids(sphinx, mask)
    xg = bf16(x_new)
    sphinx.sphinx_gn_block_stats(xg, groups, b, ids, cnt, stats)
    a = torch.full((n, h, w, c), 77.0, dtype=torch.bfloat16, device=dev)
    sphinx.sphinx_gn_silu(xg, stats, T(g1), T(be1), EPS, groups, b, ids, cnt, a)
    torch.cuda.synchronize()
    after = sphinx.gn_block_entries(stats, n, h, w, groups, b).cpu().numpy()
    assert np.array_equal(after[mask == 0], before[mask == 0])   # unlisted entries untouched
    xd = dec(x_new)
    t, a_ref = oracle.gn_silu(xd, groups, g1, be1, EPS)
    d, _, _ = act_err_bound(xd, t, a_ref, g1, groups)
    got = dec(bits_of(a))
    D = dilated_px(mask, h, w, b)
    err = np.abs(got[D] - a_ref[D])
    tol = half_ulp(a_ref[D]) + d[D]
    assert np.all(err <= tol), f"max err/tol {np.max(err / tol)}"
    assert np.all(got[~D] == 77.0)                                  # outside the ring untouched


def test_gn_silu_exact_rounding_fraction(sphinx):
    """Sanity of the bound: >= 97% of activations are bit-identical to the oracle's own
    round-to-nearest-even of its fp64 value."""
    n, h, w, c, b, groups = 1, 16, 16, 64, 8, 8
    x, g1, be1 = _inputs(n, h, w, c, "gnexact")
    mask = np.ones((n, 2, 2), np.uint8)
    ids, cnt = gpu_ids(sphinx, mask)
    stats = sphinx.gn_stats_buffer(n, h, w, groups, b, dev)
    a = torch.zeros((n, h, w, c), dtype=torch.bfloat16, device=dev)
    sphinx.sphinx_gn_block_stats(bf16(x), groups, b, ids, cnt, stats)
    sphinx.sphinx_gn_silu(bf16(x), stats, T(g1), T(be1), EPS, groups, b, ids, cnt, a)
    _, a_ref = oracle.gn_silu(dec(x), groups, g1, be1, EPS)
    same = bits_of(a) == oracle.bf16_rne(a_ref)
    assert same.mean() >= 0.97, same.mean()


# ------------------------------------------------------------ conv + residual

@pytest.mark.parametrize("n,h,c,b,dens", [(2, 16, 32, 4, 0.3), (2, 72, 320, 8, 0.25), (2, 36, 640, 8, 0.4),
                                          (2, 18, 1280, 8, 0.5), (3, 20, 96, 8, 0.6)])
@pytest.mark.parametrize("out", ["f32", "bf16"])
def test_conv_residual_vs_oracle(sphinx, n, h, c, b, dens, out):
    """y = residual + bias + conv (the identity skip fused in the epilogue), all kernel paths
    (split-K reduction included: the last wave of a small list is split on the device)."""
    tag = f"res{n}{h}{c}"
    x = syn.features_bf16((n, h, h, c), tag)
    r = syn.features_bf16((n, h, h, c), tag + "-r")
    wt = syn.weights_bf16(c, c, tag)
    bs = syn.bias_f32(c, tag)
    mask = block_mask(n, h, h, b, dens, "scattered", tag)
    ids, cnt = gpu_ids(sphinx, mask)
    dt = torch.float32 if out == "f32" else torch.bfloat16
    y = torch.full((n, h, h, c), -5.0, dtype=dt, device=dev)
    sphinx.sphinx_sparse_conv3x3(bf16(x), bf16(wt), T(bs), y, b, ids, cnt, residual=bf16(r))
    torch.cuda.synchronize()
    want, acc = oracle.conv3x3_blocks(x, wt, bs, b, oracle.compact(mask))
    L = ~np.isnan(want[..., 0])
    ref = want[L] + dec(r)[L]
    got = y.float().cpu().numpy().astype(np.float64)
    tol = 1e-3 * acc[L] + 1e-6 + 2.0 ** -23 * (np.abs(ref) + np.abs(dec(r)[L]))
    if out == "bf16":
        tol = tol + 2.0 ** -8 * np.abs(ref)
    err = np.abs(got[L] - ref)
    assert np.all(err <= tol), f"max err/tol {np.max(err / tol)}"
    assert np.all(got[~L] == -5.0)


# ------------------------------------------------------------ the whole block

def _shift_w(c, ky, kx):
    wt = np.zeros((c, 3, 3, c), np.float32)
    for i in range(c):
        wt[i, ky, kx, i] = 1.0
    return syn.to_bf16_bits(wt)


class RB:
    """GPU state of one ResNet block: persistent h/y buffers and per-block statistics."""

    def __init__(self, sp, n, h, w, c, b, groups, h_cache, y_cache, y_dtype=torch.float32):
        self.sp, self.b, self.groups = sp, b, groups
        self.h = bf16(h_cache)
        self.y = T(y_cache.astype(np.float32)).to(y_dtype)
        self.xs = sp.gn_stats_buffer(n, h, w, groups, b, dev)
        self.hs = sp.gn_stats_buffer(n, h, w, groups, b, dev)
        self.a = torch.zeros((n, h, w, c), dtype=torch.bfloat16, device=dev)

    def run(self, x_bits, params, ids, cnt):
        w1, b1, w2, b2, g1, be1, g2, be2 = params
        self.sp.sphinx_sparse_resblock(bf16(x_bits), bf16(w1), None if b1 is None else T(b1), bf16(w2),
                                       None if b2 is None else T(b2), (T(g1), T(be1)), (T(g2), T(be2)),
                                       self.groups, EPS, self.h, self.xs, self.hs, self.y, self.a,
                                       self.b, ids, cnt)


def _params(c, tag, shift=None):
    g1, be1 = syn.gn_affine_f32(c, tag + "-1")
    g2, be2 = syn.gn_affine_f32(c, tag + "-2")
    if shift is not None:
        w = _shift_w(c, *shift)
        return (w, None, w, None, g1, be1, g2, be2)
    return (syn.weights_bf16(c, c, tag + "-1"), syn.bias_f32(c, tag + "-1"),
            syn.weights_bf16(c, c, tag + "-2"), syn.bias_f32(c, tag + "-2"), g1, be1, g2, be2)


def _stats_init(sp, rb, x_bits, h_bits, mask):
    all_ids, all_cnt = gpu_ids(sp, np.ones_like(mask))
    sp.sphinx_gn_block_stats(bf16(x_bits), rb.groups, rb.b, all_ids, all_cnt, rb.xs)
    sp.sphinx_gn_block_stats(rb.h, rb.groups, rb.b, all_ids, all_cnt, rb.hs)


def shift_map(arr, shift):
    """out[p] = arr[p + (ky-1, kx-1)] (0 outside the image): where a shift conv reads."""
    ky, kx = shift
    dy, dx = ky - 1, kx - 1
    hh, ww = arr.shape[1:3]
    out = np.zeros_like(arr)
    out[:, max(0, -dy):hh - max(0, dy), max(0, -dx):ww - max(0, dx)] = \
        arr[:, max(0, dy):hh - max(0, -dy), max(0, dx):ww - max(0, -dx)]
    return out


def _h_tol(o, x_bits, params, groups, shift):
    """Bound on |h_gpu - h_pre| (h_pre = the oracle's unrounded conv1 value) at listed pixels:
    GPU a1 within half-ulp + d1 of a1_pre, oracle a1 within half-ulp of a1_pre, then conv1
    (exact copy for shift weights; else 1e-3 sum|w a1| + sum|w1| (ulp(a1) + d1)) and the
    GPU's bf16 rounding of h (half an ulp; one ulp allowed)."""
    w1, b1, w2, b2, g1, be1, g2, be2 = params
    xd = dec(x_bits)
    t1, _ = oracle.gn_silu(xd, groups, g1, be1, EPS)
    d1, _, _ = act_err_bound(xd, t1, o["a1_pre"], g1, groups)
    E_a1 = 2.0 * half_ulp(o["a1_pre"]) + d1
    if shift is not None:
        return shift_map(E_a1, shift) + 2.0 * half_ulp(o["h_pre"])
    w_abs_sum = np.abs(dec(w1)).reshape(w1.shape[0], -1).sum(axis=1)
    return ((1e-3 + 2.0 ** -8) * o["h_abs"] + d1.max() * w_abs_sum + 2.0 * half_ulp(o["h_pre"])
            + 1e-6)


def _chain_tol(o, x_bits, params, groups, shift):
    """Per-element bound on |y_gpu - y_ref| at listed pixels (module docstring)."""
    w1, b1, w2, b2, g1, be1, g2, be2 = params
    h_ref = dec(o["h"])
    # |h_gpu - h_ref| <= |h_gpu - h_pre| + |h_pre - h_ref| (the oracle's own rounding)
    E_h = _h_tol(o, x_bits, params, groups, shift) + half_ulp(o["h_pre"])
    n, hh, ww, c = h_ref.shape
    cg = c // groups
    Eg = E_h.reshape(n, hh * ww, groups, cg).max(axis=(1, 3))          # [n, groups]
    Eg = np.repeat(Eg, cg, axis=1)[:, None, None, :]
    t2, _ = oracle.gn_silu(h_ref, groups, g2, be2, EPS)
    d2, mu, sd = act_err_bound(h_ref, t2, o["a2_pre"], g2, groups)
    gam = np.abs(g2.astype(np.float64))
    E_t2 = gam / sd * (E_h + Eg + np.abs(h_ref - mu) * Eg / sd)
    # |a2_gpu - a2_bits_ref| <= half-ulp (GPU rounding) + half-ulp (oracle rounding) + drift
    E_a2 = 1.1 * E_t2 + d2 + 2.0 * half_ulp(o["a2_pre"])
    if shift is not None:
        return shift_map(E_a2, shift) + 2.0 ** -23 * np.abs(o["y"]) + 1e-7
    # conv of |w2| with E_a2 (oracle conv, inputs rounded UP to bf16 so the bound stays a bound)
    up = syn.to_bf16_bits((E_a2 * (1 + 2.0 ** -7)).astype(np.float32))
    w_abs = syn.to_bf16_bits(np.abs(dec(w2)).astype(np.float32))
    prop, _ = oracle.conv3x3_dense(up, w_abs, None)
    return 1e-3 * o["y_abs"] + prop + 2.0 ** -23 * np.abs(o["y"]) + 1e-6


@pytest.fixture(params=["fused", "unfused"])
def rb_path(request, monkeypatch, sphinx):
    """The block with GN+SiLU fused into the conv's halo path (SPHINX_RB_FUSED_GN, 8x8 blocks) and
    with the separate gn_silu activation pass (the default)."""
    if request.param == "fused":
        plain = sphinx.sphinx_sparse_resblock

        def fused(*a, **k):
            bl = a[14] if len(a) > 14 else k["block"]
            return plain(*a, fused=bl == 8, **k)
        monkeypatch.setattr(sphinx, "sphinx_sparse_resblock", fused)
    return request.param


@pytest.mark.parametrize("n,h,w,c,b,groups,dens,pattern,shift", [
    (2, 16, 16, 32, 4, 8, 0.3, "scattered", (2, 2)),
    (2, 20, 13, 64, 8, 16, 0.5, "scattered", (0, 1)),
    (2, 72, 72, 320, 8, 32, 0.25, "clustered", (2, 0)),
    (2, 36, 36, 640, 8, 32, 0.4, "checker", (1, 2)),
    (2, 18, 18, 1280, 8, 32, 0.5, "scattered", (0, 0)),
    (2, 20, 13, 64, 8, 16, 0.5, "scattered", None),
    (2, 72, 72, 320, 8, 32, 0.25, "clustered", None),
    (2, 18, 18, 1280, 8, 32, 0.5, "scattered", None),
])
def test_resblock_vs_oracle(sphinx, rb_path, n, h, w, c, b, groups, dens, pattern, shift):
    tag = f"rb{n}{h}{w}{c}{shift}"
    x = syn.resblock_features_bf16((n, h, w, c), tag)
    h_cache = syn.resblock_features_bf16((n, h, w, c), tag + "-hc")
    y_cache = dec(syn.features_bf16((n, h, w, c), tag + "-yc"))
    mask = block_mask(n, h, w, b, dens, pattern, tag)
    params = _params(c, tag, shift)
    rb = RB(sphinx, n, h, w, c, b, groups, h_cache, y_cache)
    _stats_init(sphinx, rb, x, h_cache, mask)
    hs_before = sphinx.gn_block_entries(rb.hs, n, h, w, groups, b).cpu().numpy().copy()
    ids, cnt = gpu_ids(sphinx, mask)
    rb.run(x, params, ids, cnt)
    torch.cuda.synchronize()
    o = oracle.resblock(x, h_cache, y_cache, *params, groups, EPS, b, oracle.compact(mask))
    L = listed_px(mask, h, w, b)
    h_got = bits_of(rb.h)
    y_got = rb.y.cpu().numpy().astype(np.float64)
    # unlisted pixels and statistics entries: untouched, bitwise
    assert np.array_equal(h_got[~L], h_cache[~L])
    assert np.array_equal(y_got[~L], y_cache[~L].astype(np.float32).astype(np.float64))
    hs_after = sphinx.gn_block_entries(rb.hs, n, h, w, groups, b).cpu().numpy()
    assert np.array_equal(hs_after[mask == 0], hs_before[mask == 0])
    # h on listed pixels: conv1 bound (shift: exact copy of a1 up to its rounding)
    h_tol = _h_tol(o, x, params, groups, shift)
    herr = np.abs(dec(h_got) - o["h_pre"])
    assert np.all(herr[L] <= h_tol[L]), f"h max err/tol {np.max(herr[L] / h_tol[L])}"
    tol = _chain_tol(o, x, params, groups, shift)
    err = np.abs(y_got - o["y"])
    assert np.all(err[L] <= tol[L]), f"y max err/tol {np.max(err[L] / tol[L])}"


def test_resblock_density_zero(sphinx, rb_path):
    n, h, w, c, b = 1, 16, 16, 64, 8
    x = syn.resblock_features_bf16((n, h, w, c), "rb0")
    hc = syn.resblock_features_bf16((n, h, w, c), "rb0-h")
    yc = dec(syn.features_bf16((n, h, w, c), "rb0-y"))
    mask = np.zeros((n, 2, 2), np.uint8)
    rb = RB(sphinx, n, h, w, c, b, 8, hc, yc)
    ids, cnt = gpu_ids(sphinx, mask)
    rb.run(x, _params(c, "rb0"), ids, cnt)
    torch.cuda.synchronize()
    assert np.array_equal(bits_of(rb.h), hc)
    assert np.array_equal(rb.y.cpu().numpy(), yc.astype(np.float32))


def test_resblock_full_step_then_partial_steps(sphinx, rb_path):
    """The serving loop (R-17): a full step (every block) fills h, y and both
    statistics buffers; partial steps with a growing active set (A_u monotone) and
    fresh x on listed blocks rewrite listed data only.  Each partial step equals the oracle
    whose caches are the oracle's own previous results (shift weights: tight chain bound)."""
    n, h, w, c, b, groups = 2, 24, 24, 64, 8, 16
    shift = (2, 1)
    params = _params(c, "rbloop", shift)
    x = syn.resblock_features_bf16((n, h, w, c), "rbloop-x0")
    hc0 = syn.resblock_features_bf16((n, h, w, c), "rbloop-h")
    yc0 = dec(syn.features_bf16((n, h, w, c), "rbloop-y"))
    full = np.ones((n, 3, 3), np.uint8)
    rb = RB(sphinx, n, h, w, c, b, groups, hc0, yc0)
    _stats_init(sphinx, rb, x, hc0, full)
    ids, cnt = gpu_ids(sphinx, full)
    rb.run(x, params, ids, cnt)
    o = oracle.resblock(x, hc0, yc0, *params, groups, EPS, b, oracle.compact(full))
    rg = syn.rng("rbloop-masks")
    mask = np.zeros((n, 3, 3), np.uint8)
    for step in range(3):
        mask |= (rg.random((n, 3, 3)) < 0.3).astype(np.uint8)   # A_u grows
        L = listed_px(mask, h, w, b)
        x = x.copy()
        x[L] = syn.resblock_features_bf16((n, h, w, c), f"rbloop-x{step + 1}")[L]
        ids, cnt = gpu_ids(sphinx, mask)
        rb.run(x, params, ids, cnt)
        torch.cuda.synchronize()
        o = oracle.resblock(x, o["h"], o["y"], *params, groups, EPS, b, oracle.compact(mask))
        y_got = rb.y.cpu().numpy().astype(np.float64)
        tol = _chain_tol(o, x, params, groups, shift)
        # caches carry the earlier steps' (bounded) differences: allow the full-step bound there
        err = np.abs(y_got - o["y"])
        assert np.all(err[L] <= 2 * tol[L]), f"step {step}: y max err/tol {np.max(err[L] / tol[L])}"


def test_resblock_full_size_bench_config(sphinx):
    """BASELINE configs[2] level-0 size in the bench's launch configuration: 21 frames x 72x72x320,
    clustered ~25% of blocks, persistent buffers after a full step; shift weights (tight bound)."""
    n, h, w, c, b, groups = 21, 72, 72, 320, 8, 32
    shift = (2, 1)
    x = syn.resblock_features_bf16((n, h, w, c), "rbfull")
    h_cache = syn.resblock_features_bf16((n, h, w, c), "rbfull-hc")
    y_cache = dec(syn.features_bf16((n, h, w, c), "rbfull-yc"))
    mask = block_mask(n, h, w, b, 0.25, "clustered", "rbfull")
    params = _params(c, "rbfull", shift)
    rb = RB(sphinx, n, h, w, c, b, groups, h_cache, y_cache)
    _stats_init(sphinx, rb, x, h_cache, mask)
    ids, cnt = gpu_ids(sphinx, mask)
    rb.run(x, params, ids, cnt)
    torch.cuda.synchronize()
    o = oracle.resblock(x, h_cache, y_cache, *params, groups, EPS, b, oracle.compact(mask))
    L = listed_px(mask, h, w, b)
    assert np.array_equal(bits_of(rb.h)[~L], h_cache[~L])
    y_got = rb.y.cpu().numpy().astype(np.float64)
    tol = _chain_tol(o, x, params, groups, shift)
    err = np.abs(y_got - o["y"])
    assert np.all(err[L] <= tol[L]), f"y max err/tol {np.max(err[L] / tol[L])}"
