"""Pins the CPU oracle to what the paper, SPEC and mathematics fix (no GPU).

Each test names the passage or property it checks.  None of them re-types the
oracle's formula: they use worked values (tests/golden/worked_examples.json),
closed forms, brute force on tiny inputs, library routines (torch fp64
conv2d), exact invariants, or Monte-Carlo statistics.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synthetic as syn

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


# ------------------------------------------------------------------ a1 masks

@pytest.mark.parametrize("case", GOLD["block_mask"], ids=lambda c: c["name"])
def test_block_mask_worked_examples(case):
    O = np.ones((case["n"], case["hp"], case["wp"]), np.float32)
    for (y, x, v) in case["pixels"]:
        O[0, y, x] = np.nan if v == "nan" else v
    masks, counts = oracle.block_mask(O, None, None, 0.5, case["f"], case["b"], case["levels"])
    for l, want in enumerate(case["ids"]):
        assert np.flatnonzero(masks[l]).tolist() == want, (case["cite"], l)
        assert counts[0, l] == len(want)


def test_opacity_mask_spec_row():
    g = GOLD["opacity_mask_spec"]
    O = np.array([[g["row"]]], np.float32)
    assert oracle.pixel_mask(O, None, None, g["tau_o"])[0, 0].tolist() == g["mask"]


def test_opacity_mask_trivial_and_union():
    ones = np.ones((2, 4, 4), np.float32)
    assert oracle.pixel_mask(ones, None, None, 0.5).sum() == 0
    assert oracle.pixel_mask(0 * ones, None, None, 0.5).all()
    # M = M_op OR M_blur (Alg1 line 10): blur full, opacity empty -> full
    U = np.ones((2, 4, 4), np.float32)
    tau = np.full(2, 0.5, np.float32)
    assert oracle.pixel_mask(ones, U, tau, 0.5).all()
    # strict '>' for the blur map (reading R-8): U == tau is not blurry
    assert oracle.pixel_mask(ones, 0.5 * U, tau, 0.5).sum() == 0
    # disjoint single pixels -> exactly two set pixels
    O = ones.copy(); O[0, 1, 1] = 0.0
    U2 = np.zeros_like(ones); U2[0, 2, 3] = 1.0
    assert oracle.pixel_mask(O, U2, tau, 0.5).sum() == 2
    with pytest.raises(ValueError):
        oracle.pixel_mask(ones, None, None, 1.5)


def test_maxpool_spec_examples():
    m = np.zeros((1, 8, 8), np.uint8); m[0, 3, 5] = 1
    assert oracle.maxpool(m, 8).tolist() == [[[1]]]
    assert oracle.maxpool(np.zeros((1, 16, 16), np.uint8), 4).sum() == 0
    rg = syn.rng("pin-maxpool")
    for _ in range(200):
        g = (rg.random((1, 16, 16)) < 0.05).astype(np.uint8)
        assert np.array_equal(oracle.maxpool(oracle.maxpool(g, 2), 2), oracle.maxpool(g, 4))
    with pytest.raises(ValueError):
        oracle.maxpool(np.zeros((1, 6, 6), np.uint8), 4)


def test_tile_blocks_spec_and_brute_force():
    assert oracle.tile_blocks(np.ones((1, 8, 8), np.uint8), 4).sum() == 4
    g = np.zeros((1, 9, 9), np.uint8); g[0, 8, 2] = 1
    t = oracle.tile_blocks(g, 4)
    assert t.shape == (1, 3, 3) and t.sum() == 1 and t[0, 2, 0] == 1        # S:257, edge block
    rg = syn.rng("pin-tile")
    for _ in range(50):
        h, w, b = rg.integers(1, 30), rg.integers(1, 30), int(rg.integers(1, 9))
        g = (rg.random((2, h, w)) < 0.03).astype(np.uint8)
        want = np.zeros((2, -(-h // b), -(-w // b)), np.uint8)
        for i in range(2):
            for by in range(want.shape[1]):
                for bx in range(want.shape[2]):
                    want[i, by, bx] = g[i, by * b:(by + 1) * b, bx * b:(bx + 1) * b].any()
        assert np.array_equal(oracle.tile_blocks(g, b), want)


def test_block_mask_exhaustive_config1_patterns():
    """All 2^16 block patterns of config-1 geometry (16x16, f=1, b=4): paint one
    flagged pixel at a random spot of every chosen block; the oracle must return
    exactly the pattern (coverage + no false positives)."""
    n = 1 << 16
    pat = ((np.arange(n)[:, None] >> np.arange(16)[None, :]) & 1).astype(bool)  # [n,16]
    rg = syn.rng("pin-exhaustive")
    O = rg.uniform(0.5, 1.0, size=(n, 16, 16)).astype(np.float32)  # 0.5 itself is not flagged
    oy = rg.integers(0, 4, size=(n, 16)); ox = rg.integers(0, 4, size=(n, 16))
    fi, bi = np.nonzero(pat)
    by, bx = bi // 4, bi % 4
    O[fi, by * 4 + oy[fi, bi], bx * 4 + ox[fi, bi]] = rg.uniform(0, 0.4999, size=len(fi))
    masks, counts = oracle.block_mask(O, None, None, 0.5, 1, 4, 1)
    assert np.array_equal(masks[0].reshape(n, 16).astype(bool), pat)
    assert np.array_equal(counts[:, 0], pat.sum(1))


def test_block_mask_sparse_pixels_brute_force():
    """Isolated random pixels on footprint boundaries, equality and NaN pixels (R-8, R-9) at
    576x576, f=8, b=8, L=3: every level equals a brute-force any() over the block's truncated
    b*f*2^l footprint of the raw pixel flags."""
    O, U, tau = syn.sparse_pixel_maps(6, 576, 576, 64, 9, tag="pin-sparse")
    masks, counts = oracle.block_mask(O, U, tau, 0.5, 8, 8, 3)
    flag = ~(O >= 0.5) | ~(U <= tau[:, None, None])
    for l in range(3):
        fp = 64 << l
        nb = -(-576 // fp)
        want = np.zeros((6, nb, nb), np.uint8)
        for by in range(nb):
            for bx in range(nb):
                want[:, by, bx] = flag[:, by * fp:(by + 1) * fp, bx * fp:(bx + 1) * fp].any(axis=(1, 2))
        assert np.array_equal(masks[l], want), l
        assert np.array_equal(counts[:, l], want.reshape(6, -1).sum(1))


def test_block_mask_pyramid_nesting_and_counts():
    """Coarser levels never drop a refined region (S:232 'every coarser level >=
    max-pool of the finer'): with b=8 and /2 per level, a level-l block covers the
    2x2 level-(l-1) blocks below it (edge blocks truncated), so it is their OR."""
    n = 3
    O, cells = syn.opacity_maps(n, 576, 576, 64, [0.05, 0.25, 0.6], "scattered", tag="pin-pyr")
    U, tau = syn.uncertainty_maps(n, 576, 576, 64, cells, tag="pin-pyr")
    masks, counts = oracle.block_mask(O, U, tau, 0.5, 8, 8, 3)
    assert [m.shape for m in masks] == [(n, 9, 9), (n, 5, 5), (n, 3, 3)]
    # level 0 equals the cells the generator painted (each painted cell has >= 1 flagged px,
    # unpainted cells have opacity >= 0.8 and uncertainty blobs only inside painted cells)
    assert np.array_equal(masks[0].astype(bool), cells)
    for l in (1, 2):
        fine, coarse = masks[l - 1], masks[l]
        for i in range(n):
            for by in range(coarse.shape[1]):
                for bx in range(coarse.shape[2]):
                    assert coarse[i, by, bx] == fine[i, 2 * by:2 * by + 2, 2 * bx:2 * bx + 2].any()
    for l in range(3):
        assert np.array_equal(counts[:, l], masks[l].reshape(n, -1).sum(1))


# --------------------------------------------------------------- a2 start step

@pytest.mark.parametrize("case", GOLD["eq2"], ids=lambda c: c["cite"][:12])
def test_eq2_worked(case):
    got = oracle.eq2(case["c0"], case["c1"], case["t"], case["gamma"])
    assert abs(got - case["expect"]) <= case["tol"], case["cite"]


def test_eq2_gamma1_is_linear_and_endpoints():
    for t in np.linspace(0, 1, 100):
        for (c0, c1) in ((60.0, 70.0), (70.0, 60.0), (55.5, 55.5)):
            assert abs(oracle.eq2(c0, c1, t, 1.0) - (c0 + (c1 - c0) * t)) <= 1e-12
    for g in (0.1, 0.5, 0.9, 1.0):                                         # f(0)=0, f(1)=1
        for (c0, c1) in ((60.0, 70.0), (70.0, 60.0)):
            assert oracle.eq2(c0, c1, 0.0, g) == c0
            assert oracle.eq2(c0, c1, 1.0, g) == c1


def _is_correctly_rounded_sqrt(f, x):
    """Exact check from the definition: f is the double nearest to sqrt(x) iff x lies between
    the squares of the midpoints to f's neighbours (rational arithmetic, no rounding)."""
    from fractions import Fraction as Fr
    if x == 0.0:
        return f == 0.0
    lo, hi = Fr(math.nextafter(f, -math.inf)), Fr(math.nextafter(f, math.inf))
    F = Fr(f)
    return ((lo + F) / 2) ** 2 <= Fr(x) <= ((F + hi) / 2) ** 2


def test_eq2_gamma_half_is_correctly_rounded_sqrt():
    """Eq. 2 at gamma = 0.5 is c0 + (c1-c0) sqrt(t).  Reading R-16: both sides use
    the correctly rounded sqrt, so k is bit-exact.  (c0, c1) = (0, 1) exposes f(t) itself; it
    must be the correctly rounded sqrt -- checked exactly with rationals on a sample, and bit
    for bit against IEEE sqrt (numpy) over > 10^6 fp32 t in [0, 1] incl. 0x3d00e96f, where
    glibc pow(t, 0.5) is one ulp off."""
    bits = np.arange(0, 0x3F800001, 1009, dtype=np.uint32)
    bits = np.concatenate([bits, np.uint32([0x3D00E96F, 0x3F800000, 0x00000001, 0x3E800000])])
    t = bits.view(np.float32).astype(np.float64)
    assert len(t) > 10 ** 6
    f = oracle.eq2_batch(np.zeros_like(t), np.ones_like(t), t, 0.5)
    assert np.array_equal(f.view(np.uint64), np.sqrt(t).view(np.uint64))
    # c1 < c0 branch: f = 1 - (1-t)^0.5 with (c0, c1) = (1, 0): Q* = 1 - f
    g = oracle.eq2_batch(np.ones_like(t), np.zeros_like(t), t, 0.5)
    assert np.array_equal(g.view(np.uint64), (1.0 - (1.0 - np.sqrt(1.0 - t))).view(np.uint64))
    rg = syn.rng("pin-sqrt")
    for i in list(rg.integers(0, len(t), 3000)) + [len(t) - 4]:
        assert _is_correctly_rounded_sqrt(float(f[i]), float(t[i])), float(t[i])
    # gamma = 1 is t itself (not pow): bitwise
    f1 = oracle.eq2_batch(np.zeros_like(t), np.ones_like(t), t, 1.0)
    assert np.array_equal(f1, t)


GOLD_EQ2R = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "eq2_realized_ratio.json")))


@pytest.mark.parametrize("case", GOLD_EQ2R["cases"], ids=lambda c: f"{c['t_bits']}-{c['c0']}-{c['c1']}")
def test_start_step_cut_point_at_realized_ratio(case):
    """A k-logic cut point exactly at the realized ratio r (what a decile calibration emits,
    S:149): thresholds are left-closed, so thr = r selects the step and
    thr = next double above r does not.  One ulp of Q* flips k here."""
    import struct
    t = struct.unpack("<f", struct.pack("<I", int(case["t_bits"], 16)))[0]
    qs = float.fromhex(case["qstar_hex"])
    assert oracle.eq2(case["c0"], case["c1"], t, 0.5) == qs
    r = float.fromhex(case["r_hex"])
    for thr, want in (([r], 25), ([math.nextafter(r, math.inf)], 0), ([math.nextafter(r, -math.inf)], 25),
                      ([r - 0.1, r, r + 0.1], 30)):
        steps = [25] if len(thr) == 1 else [10, 30, 40]
        lg = oracle.make_klogic(thr, steps, 0, 40)
        k = oracle.start_step([np.float32(case["q"])], [case["c0"]], [case["c1"]], [np.float32(t)], 0.5, [lg])
        assert k[0] == want, (thr, want)


def test_select_k_spec_and_monotone():
    g = GOLD["select_k"]
    lg = oracle.make_klogic(g["logic"]["thr"], g["logic"]["steps"], g["logic"]["fallback_k"],
                            g["logic"]["k_max"])
    for c in g["cases"]:
        assert oracle.select_k(lg, c["r"]) == c["k"], c["cite"]
    ks = [oracle.select_k(lg, r) for r in np.linspace(0, 2, 2001)]       # S:157 monotone
    assert all(a <= b for a, b in zip(ks, ks[1:]))
    big = oracle.make_klogic([0.5, 0.9], [30, 48], 0, 40)                  # S:160 never above k_max
    assert max(oracle.select_k(big, r) for r in np.linspace(0, 2, 101)) == 40


def test_start_step_fp32_tie_cases():
    lg = oracle.make_klogic(**{k: v for k, v in syn.SPEC_KLOGIC.items() if k in ("thr",)},
                            steps=syn.SPEC_KLOGIC["steps"])
    for c in GOLD["start_step_fp32"]:
        q = np.float32(0.97 * 65) if c["q"] == "fp32(0.97*65)" else np.float32(c["q"])
        k = oracle.start_step([q], [c["c0"]], [c["c1"]], [c["t"]], c["gamma"], [lg])
        assert k[0] == c["k"], c["cite"]


def test_start_step_invalid_and_logic_id():
    lg0 = oracle.make_klogic([0.85, 0.92, 0.97], [10, 25, 40])
    lg1 = oracle.make_klogic([0.5], [5], 1, 40)
    k = oracle.start_step([60, 60, 60, 60], [60, 0, 60, 60], [70, 0, 70, 70],
                          [1.5, 0.5, 0.5, 0.5], 0.5, [lg0, lg1], logic_id=[0, 0, 1, 2])
    # t outside [0,1] -> -1; Q* = 0 -> -1; logic 1 -> 5; bad logic id -> -1
    assert k.tolist() == [-1, -1, 5, -1]


# ---------------------------------------------------------------- a3 compaction

def test_compact_brute_force_and_selections():
    rg = syn.rng("pin-compact")
    for trial in range(30):
        n, hb, wb = int(rg.integers(1, 6)), int(rg.integers(1, 10)), int(rg.integers(1, 10))
        m = (rg.random((n, hb, wb)) < rg.random()).astype(np.uint8)
        k = rg.integers(-1, 45, size=n).astype(np.int32)
        u = int(rg.integers(0, 50))
        ids = oracle.compact(m, k, u)
        elig = (k >= 0) & (k <= u)                                          # Alg1 line 17
        want = np.flatnonzero((m.astype(bool) & elig[:, None, None]).ravel())
        assert np.array_equal(ids, want)
        assert len(ids) == int((m * elig[:, None, None]).sum())
        inact = oracle.compact(m, k, u, oracle.SELECT_INACTIVE_FRAMES)      # Alg1 line 19
        assert np.array_equal(inact, np.flatnonzero(np.repeat(k > u, hb * wb)))
        allb = oracle.compact(None, k, u, oracle.SELECT_ALL, shape=(n, hb, wb))
        assert np.array_equal(allb, np.flatnonzero(np.repeat(k >= 0, hb * wb)))
        noise = oracle.compact(m, k, u, oracle.SELECT_NOISE)               # lines 12 + 19 together
        assert np.array_equal(noise, np.union1d(want, np.flatnonzero(np.repeat(k > u, hb * wb))))
    m = np.ones((3, 5, 5), np.uint8)
    assert np.array_equal(oracle.compact(m), np.arange(75))                 # density 1 -> identity
    assert len(oracle.compact(0 * m)) == 0                                  # density 0 -> empty


# --------------------------------------------------------------------- a4 noise

@pytest.mark.parametrize("case", GOLD["noise"], ids=lambda c: c["name"])
def test_noise_worked(case):
    abar = syn.abar_linear(case["S"]) if case["schedule"] == "linear" else syn.abar_cosine(case["S"])
    x0 = np.full((1, 4, 4, 2), case["x0"], np.float32)
    eps = np.full_like(x0, case["eps"])
    out = oracle.noise(x0, eps, np.zeros_like(x0), 4, [0], [case["u"]], abar)
    assert np.all(np.abs(out - case["expect"]) <= case["tol"]), case["cite"]


def test_noise_clean_endpoint_and_untouched():
    abar = syn.abar_cosine(50)
    x0 = syn.latents_f32((2, 9, 9, 4), "pin-n-x0")
    eps = syn.latents_f32((2, 9, 9, 4), "pin-n-eps")
    xt = syn.latents_f32((2, 9, 9, 4), "pin-n-xt")
    out = oracle.noise(x0, eps, xt, 4, [0, 1, 2, 3, 4, 5, 6, 7, 8, 9], [50, 10], abar)
    assert np.array_equal(out[0].astype(np.float32), x0[0])                 # S:306, frame 0 all listed
    # frame 1: only block ids 9 (=frame1 block (0,0)) listed -> rest untouched, bitwise
    touched = np.zeros((9, 9), bool); touched[0:4, 0:4] = True
    assert np.array_equal(out[1][~touched].astype(np.float32), xt[1][~touched])
    assert not np.array_equal(out[1][touched].astype(np.float32), xt[1][touched])


def test_noise_monte_carlo_marginals():
    """S:308 / S:577: over 10 000 draws, mean within 3 sigma of sqrt(abar)z0 and
    variance within 5% of 1-abar, at u in {0,10,25,40}."""
    abar = syn.abar_cosine(50)
    z0 = np.float32(0.7)
    draws = 10000
    x0 = np.full((1, 1, draws, 1), z0, np.float32)
    eps = syn.rng("pin-mc").standard_normal((1, 1, draws, 1)).astype(np.float32)
    for u in (0, 10, 25, 40):
        out = oracle.noise(x0, eps, np.zeros_like(x0), draws, [0], [u], abar).ravel()
        a = float(abar[u])
        sigma = math.sqrt((1 - a) / draws)
        assert abs(out.mean() - math.sqrt(a) * z0) <= 3 * sigma
        assert abs(out.var() / (1 - a) - 1) <= 0.05


# ---------------------------------------------------------------------- a5 conv

def _shift_weights(c, ky, kx):
    w = np.zeros((c, 3, 3, c), np.float32)
    for i in range(c):
        w[i, ky, kx, i] = 1.0
    return syn.to_bf16_bits(w)


@pytest.mark.parametrize("ky,kx", [(a, c) for a in range(3) for c in range(3)])
def test_conv_shift_kernels_exact(ky, kx):
    """W = delta(co=ci) delta(tap) gives y(p) = x(p + (ky-1, kx-1)) exactly, zero
    outside the image (TV-12/13), across block boundaries and ragged edges."""
    n, h, w, c, b = 2, 10, 11, 8, 4
    x = syn.features_bf16((n, h, w, c), "pin-shift")
    xf = syn.bf16_bits_to_f32(x).astype(np.float64)
    want = np.zeros((n, h, w, c))
    dy, dx = ky - 1, kx - 1
    for yy in range(h):
        for xx in range(w):
            if 0 <= yy + dy < h and 0 <= xx + dx < w:
                want[:, yy, xx] = xf[:, yy + dy, xx + dx]
    y, a = oracle.conv3x3_dense(x, _shift_weights(c, ky, kx), None)
    assert np.array_equal(y, want)
    hb, wb = -(-h // b), -(-w // b)
    ids = np.arange(0, n * hb * wb, 2)
    ys, _ = oracle.conv3x3_blocks(x, _shift_weights(c, ky, kx), None, b, ids)
    listed = np.zeros((n, h, w), bool)
    for id_ in ids:
        i, r = divmod(int(id_), hb * wb)
        by, bx = divmod(r, wb)
        listed[i, by * b:(by + 1) * b, bx * b:(bx + 1) * b] = True
    assert np.array_equal(ys[listed], want[listed])
    assert np.isnan(ys[~listed]).all()


def test_conv_dense_matches_torch_fp64():
    """Library sanity check: torch.nn.functional.conv2d in fp64 on CPU."""
    torch = pytest.importorskip("torch")
    n, h, w, cin, cout = 2, 9, 7, 24, 16
    x = syn.features_bf16((n, h, w, cin), "pin-torch")
    wt = syn.weights_bf16(cout, cin, "pin-torch")
    bias = syn.bias_f32(cout, "pin-torch")
    y, a = oracle.conv3x3_dense(x, wt, bias)
    xt = torch.from_numpy(syn.bf16_bits_to_f32(x).astype(np.float64)).permute(0, 3, 1, 2)
    wtt = torch.from_numpy(syn.bf16_bits_to_f32(wt).astype(np.float64)).permute(0, 3, 1, 2)
    ref = torch.nn.functional.conv2d(xt, wtt, torch.from_numpy(bias.astype(np.float64)), padding=1)
    ref = ref.permute(0, 2, 3, 1).numpy()
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(a)
    assert np.all(a >= np.abs(y - bias) - 1e-12)


def test_conv_zero_input_bias_and_abs_sum():
    n, h, w, c = 1, 5, 6, 8
    zero = np.zeros((n, h, w, c), np.uint16)
    bias = syn.bias_f32(c, "pin-zero")
    y, _ = oracle.conv3x3_dense(zero, syn.weights_bf16(c, c, "pin-zero"), bias)
    assert np.array_equal(y, np.broadcast_to(bias.astype(np.float64), y.shape))
    # non-negative operands: sum |w x| == sum w x exactly (same order, no cancellation)
    xp = syn.to_bf16_bits(np.abs(syn.bf16_bits_to_f32(syn.features_bf16((n, h, w, c), "pz"))))
    wp = syn.to_bf16_bits(np.abs(syn.bf16_bits_to_f32(syn.weights_bf16(c, c, "pz"))))
    y, a = oracle.conv3x3_dense(xp, wp, None)
    assert np.array_equal(y, a)


def test_conv_blocks_equal_dense_on_listed_pixels():
    """P:352 / S:326: block-sparse output equals the dense conv on active blocks."""
    n, h, w, c, b = 2, 18, 18, 16, 8
    x = syn.features_bf16((n, h, w, c), "pin-bd")
    wt = syn.weights_bf16(c, c, "pin-bd")
    bias = syn.bias_f32(c, "pin-bd")
    yd, ad = oracle.conv3x3_dense(x, wt, bias)
    ids = np.array([0, 4, 8, 9, 13, 17])  # includes truncated edge blocks (3x3 grid)
    ys, as_ = oracle.conv3x3_blocks(x, wt, bias, b, ids)
    got = ~np.isnan(ys[..., 0])
    assert got.sum() == sum(min(b, h - (r // 3) * b) * min(b, w - (r % 3) * b)
                            for r in (i % 9 for i in ids))
    assert np.array_equal(ys[got], yd[got]) and np.array_equal(as_[got], ad[got])


# ------------------------------------------------------------------- a6 scatter

def test_scatter_density_0_1_and_composition():
    n, h, w, c, b = 2, 18, 18, 8, 8
    src = syn.features_bf16((n, h, w, c), "pin-sc-src")
    cache = syn.features_bf16((n, h, w, c), "pin-sc-cache")
    m0 = np.zeros((n, 3, 3), np.uint8)
    assert np.array_equal(oracle.scatter(src, cache, b, mask=m0), cache)        # density 0
    m1 = np.ones((n, 3, 3), np.uint8)
    assert np.array_equal(oracle.scatter(src, cache, b, mask=m1), src)          # density 1
    k = np.array([5, 30], np.int32)
    out = oracle.scatter(src, cache, b, mask=m1, k=k, u=10)                     # frame 1 inactive
    assert np.array_equal(out[0], src[0]) and np.array_equal(out[1], cache[1])
    # O7: scatter(conv_sparse(x), cache) == where(active, dense(x), cache)
    rg = syn.rng("pin-o7")
    m = (rg.random((n, 3, 3)) < 0.5).astype(np.uint8)
    ids = oracle.compact(m)
    x = syn.features_bf16((n, h, w, c), "pin-o7x")
    wt = syn.weights_bf16(c, c, "pin-o7")
    cache32 = syn.latents_f32((n, h, w, c), "pin-o7c")
    ys, _ = oracle.conv3x3_blocks(x, wt, None, b, ids, y_init=cache32.astype(np.float64))
    yd, _ = oracle.conv3x3_dense(x, wt, None)
    act = np.kron(m, np.ones((1, b, b), np.uint8))[:, :h, :w].astype(bool)
    want = np.where(act[..., None], yd.astype(np.float32), cache32)
    got = oracle.scatter(ys.astype(np.float32), cache32, b, mask=m)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    # COMPACT source layout gives the same result
    comp = np.zeros((len(ids), b, b, c), np.float32)
    for j, id_ in enumerate(ids):
        i, r = divmod(int(id_), 9)
        by, bx = divmod(r, 3)
        blk = ys[i, by * b:(by + 1) * b, bx * b:(bx + 1) * b].astype(np.float32)
        comp[j, :blk.shape[0], :blk.shape[1]] = blk
    got2 = oracle.scatter(comp, cache32, b, ids=ids, src_layout=oracle.SRC_COMPACT)
    assert np.array_equal(got2.view(np.uint32), want.view(np.uint32))


# ------------------------------------------------------------- NEXT-1 DDIM update

def test_ddim_collapses_to_clean_latent():
    """with x0_hat = the true clean latent, running u from k to S collapses z to x0
    (within 1e-5), for the cosine and linear schedules and several start steps."""
    x0 = syn.latents_f32((2, 16, 16, 4), "ddim-x0")
    eps = syn.latents_f32((2, 16, 16, 4), "ddim-eps")
    ids = np.arange(2 * 16)  # every 4x4 block
    for abar in (syn.abar_cosine(50), syn.abar_linear(50)):
        for k in (0, 10, 25, 40, 49):
            z = oracle.noise(x0, eps, x0, 4, ids, [k, k], abar).astype(np.float32)
            for u in range(k, 50):
                z = oracle.ddim_step(z, x0, 4, ids, u, abar).astype(np.float32)
            assert np.max(np.abs(z - x0)) <= 1e-5


def test_ddim_flat_segment_identity_and_last_step():
    z = syn.latents_f32((1, 8, 8, 4), "ddim-z")
    xh = syn.latents_f32((1, 8, 8, 4), "ddim-xh")
    ids = np.arange(4)
    abar = syn.abar_cosine(50).copy()
    abar[11] = abar[10]                          # S:316 hypothetical flat segment
    out = oracle.ddim_step(z, xh, 4, ids, 10, abar)
    assert np.max(np.abs(out - z)) <= 1e-12
    out = oracle.ddim_step(z, xh, 4, ids, 49, syn.abar_cosine(50))  # abar[S] = 1 -> x0_hat
    assert np.array_equal(out, xh.astype(np.float64))


def test_ddim_preserves_noise_direction_and_untouched():
    """eta = 0: if z = sqrt(abar_u) x0_hat + sqrt(1-abar_u) e then z' = sqrt(abar_u+1) x0_hat +
    sqrt(1-abar_u+1) e (up to the fp32 rounding of z); unlisted blocks keep z bitwise."""
    abar = syn.abar_cosine(50)
    xh = syn.latents_f32((2, 12, 12, 4), "ddim-dir-x")
    e = syn.latents_f32((2, 12, 12, 4), "ddim-dir-e")
    for u in (0, 13, 37, 48):
        a0, s0 = np.sqrt(np.float64(abar[u])), np.sqrt(1 - np.float64(abar[u]))
        a1, s1 = np.sqrt(np.float64(abar[u + 1])), np.sqrt(1 - np.float64(abar[u + 1]))
        z = (a0 * xh + s0 * e).astype(np.float32)
        ids = np.array([0, 4, 8, 9, 17])          # 3x3 blocks of 4 per frame, ragged
        out = oracle.ddim_step(z, xh, 4, ids, u, abar)
        want = a1 * xh + s1 * e
        listed = np.zeros((2, 12, 12), bool)
        for id_ in ids:
            i, r = divmod(int(id_), 9)
            by, bx = divmod(r, 3)
            listed[i, by * 4:(by + 1) * 4, bx * 4:(bx + 1) * 4] = True
        tol = 1e-6 * (s1 / s0) * np.abs(z) + 1e-12
        assert np.all(np.abs(out - want)[listed] <= tol[listed])
        assert np.array_equal(out[~listed].astype(np.float32), z[~listed])
    with pytest.raises(ValueError):
        oracle.ddim_step(z, xh, 4, [0], 50, abar)  # u must be < S


# ------------------------------------------------------- NEXT-2 uncertainty producer

def _rgb(shape, tag):
    return syn.rng("rgb", tag, shape).uniform(0, 1, size=shape + (3,)).astype(np.float32)


def test_laplacian_var_constant_and_point():
    """S:201 constant image -> all-zero map; S:202 a single bright pixel -> the map is largest
    around it and exactly zero where the window cannot see the Laplacian's support."""
    const = np.full((1, 12, 9, 3), 0.37, np.float32)
    assert np.all(oracle.laplacian_var(const, 7) == 0.0)
    img = np.zeros((1, 21, 21, 3), np.float32)
    img[0, 10, 10, :] = 1.0
    B = oracle.laplacian_var(img, 7)[0]
    yy, xx = np.mgrid[0:21, 0:21]
    cheb = np.maximum(np.abs(yy - 10), np.abs(xx - 10))
    assert np.all(B[cheb > 4] == 0.0) and np.all(B[cheb <= 3] > 0)
    assert B.argmax() // 21 in range(6, 15)
    # mirror symmetry of the configuration (to summation-order rounding)
    assert np.allclose(B, B[::-1, ::-1], rtol=1e-12, atol=0) and np.allclose(B, B.T, rtol=1e-12, atol=0)
    for k in range(20):  # S:203 non-negative
        assert oracle.laplacian_var(_rgb((2, 17, 13), f"nn{k}"), 3 + 2 * (k % 3)).min() >= 0.0
    with pytest.raises(ValueError):
        oracle.laplacian_var(img, 6)  # S:199 even window


def test_laplacian_var_and_box_match_scipy_ndimage():
    """Library cross-check: scipy.ndimage.laplace / uniform_filter with mode='nearest'
    (= edge replication) give the same Laplacian variance and box mean in fp64."""
    nd = pytest.importorskip("scipy.ndimage")
    rgb = _rgb((2, 23, 31), "scipy")
    Y = rgb.astype(np.float64) @ np.array([0.299, 0.587, 0.114])
    for win in (3, 7):
        B = oracle.laplacian_var(rgb, win)
        for i in range(2):
            L = nd.laplace(Y[i], mode="nearest")
            m1 = nd.uniform_filter(L, win, mode="nearest")
            m2 = nd.uniform_filter(L * L, win, mode="nearest")
            assert np.max(np.abs(B[i] - (m2 - m1 * m1))) <= 1e-9 * max(1.0, m2.max())
    S = oracle.box_smooth(B, 5)
    for i in range(2):
        assert np.max(np.abs(S[i] - nd.uniform_filter(B[i], 5, mode="nearest"))) <= 1e-12 * B.max()


def _brute_otsu(v):
    """Exhaustive search over the 255 splits of the 256-bin histogram (bin i = (i/256,(i+1)/256],
    R-24), between-class variance in fp64, first maximum."""
    b = np.clip(np.ceil(v.astype(np.float64) * 256) - 1, 0, 255).astype(int)
    if len(np.unique(b)) == 1:
        return float(v.max())
    best, bk = -1.0, 0
    for k in range(255):
        c0, c1 = b[b <= k], b[b > k]
        if len(c0) == 0 or len(c1) == 0:
            s = 0.0
        else:
            w0, w1 = len(c0) / len(b), len(c1) / len(b)
            s = w0 * w1 * (c0.mean() - c1.mean()) ** 2
        if s > best:
            best, bk = s, k
    return (bk + 1) / 256.0


def test_otsu_spec_examples_and_brute_force():
    v = np.concatenate([np.full(500, 0.1), np.full(500, 0.9)]).astype(np.float32)
    tau = oracle.otsu(v)
    assert 0.1 < tau <= 0.9 and np.array_equal(v > tau, np.arange(1000) >= 500)
    assert oracle.otsu(np.full(64, 0.5, np.float32)) == 0.5
    assert not np.any(np.full(64, 0.5, np.float32) > 0.5)
    rg = syn.rng("pin-otsu")
    for t in range(50):
        kind = t % 3
        if kind == 0:
            v = rg.random(400)
        elif kind == 1:
            v = np.concatenate([rg.normal(0.3, 0.05, 300), rg.normal(0.7, 0.1, 200)])
        else:
            v = rg.beta(0.5, 2.0, 700)
        v = np.clip(v, 0, 1).astype(np.float32)
        assert oracle.otsu(v) == np.float32(_brute_otsu(v)), t
    with pytest.raises(ValueError):
        oracle.otsu(np.zeros(0, np.float32))


def test_uncertainty_blur_mask_properties():
    """S:219 constant map -> empty mask; S:220 half sharp checkerboard / half flat gray ->
    the mask (U > tau: 1 = blurry) covers the flat half and not the sharp half (>= 95%)."""
    U, tau = oracle.uncertainty(np.full((1, 32, 32, 3), 0.4, np.float32))
    assert np.all(U == 1.0) and tau[0] == 1.0 and not np.any(U > tau[0])
    img = np.full((1, 64, 64, 3), 0.5, np.float32)
    yy, xx = np.mgrid[0:64, 0:32]
    img[0, :, :32, :] = ((yy + xx) % 2)[..., None].astype(np.float32)
    U, tau = oracle.uncertainty(img)
    m = U[0] > tau[0]
    assert m[:, 40:].mean() >= 0.95 and m[:, :24].mean() <= 0.05
    assert set(np.unique(m)) <= {False, True}


# ------------------------------------------------------- NEXT-3 sparse ResNet block

def _listed_px(ids, n, h, w, b):
    hb, wb = -(-h // b), -(-w // b)
    m = np.zeros((n, h, w), bool)
    for id_ in ids:
        i, r = divmod(int(id_), hb * wb)
        by, bx = divmod(r, wb)
        m[i, by * b:(by + 1) * b, bx * b:(bx + 1) * b] = True
    return m


def test_bf16_rne_matches_torch_including_ties():
    """oracle_bf16_rne == torch's float32 -> bfloat16 conversion (round to nearest even) on
    fp32-representable doubles, including exact ties (low 16 bits 0x8000) and signed zero."""
    torch = pytest.importorskip("torch")
    rg = np.random.default_rng(11)
    f = rg.standard_normal(20000).astype(np.float32) * np.float32(3.0)
    bits = f.view(np.uint32)
    ties = ((bits[:4000] & 0xFFFF0000) | 0x8000).view(np.float32)   # exact halfway cases
    vals = np.concatenate([f, ties, np.float32([0.0, -0.0, 1e-30, -2.5e-39, 3.3e38])])
    want = torch.from_numpy(vals).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = oracle.bf16_rne(vals.astype(np.float64))
    assert np.array_equal(got, want)


def test_gn_silu_matches_torch_group_norm():
    """GroupNorm (consecutive channel groups, population variance, per-sample statistics)
    + SiLU equals torch.nn.functional.group_norm / silu in fp64 on the NCHW view."""
    torch = pytest.importorskip("torch")
    n, h, w, c, G = 2, 9, 7, 40, 4
    x = syn.bf16_bits_to_f32(syn.resblock_features_bf16((n, h, w, c), "pin-gn")).astype(np.float64)
    g, be = syn.gn_affine_f32(c, "pin-gn")
    t, a = oracle.gn_silu(x, G, g, be, 1e-6)
    xt = torch.from_numpy(x).permute(0, 3, 1, 2)
    ref = torch.nn.functional.group_norm(xt, G, torch.from_numpy(g.astype(np.float64)),
                                         torch.from_numpy(be.astype(np.float64)), eps=1e-6)
    assert np.max(np.abs(t - ref.permute(0, 2, 3, 1).numpy())) <= 1e-12
    assert np.max(np.abs(a - torch.nn.functional.silu(ref).permute(0, 2, 3, 1).numpy())) <= 1e-12
    m, v = oracle.gn_stats(x, G)
    assert np.allclose(m[1, 2], x[1, :, :, 20:30].mean(), rtol=0, atol=1e-13)


def _rb_inputs(n, h, w, c, tag):
    x = syn.resblock_features_bf16((n, h, w, c), tag)
    hc = syn.resblock_features_bf16((n, h, w, c), tag + "-hc")
    yc = syn.bf16_bits_to_f32(syn.features_bf16((n, h, w, c), tag + "-yc")).astype(np.float64)
    w1, w2 = syn.weights_bf16(c, c, tag + "-1"), syn.weights_bf16(c, c, tag + "-2")
    b1, b2 = syn.bias_f32(c, tag + "-1"), syn.bias_f32(c, tag + "-2")
    g1, be1 = syn.gn_affine_f32(c, tag + "-1")
    g2, be2 = syn.gn_affine_f32(c, tag + "-2")
    return x, hc, yc, w1, b1, w2, b2, g1, be1, g2, be2


def test_resblock_matches_torch_dense_formulation():
    """R-26/R-27 written as torch fp64 dense ops + where(): h = where(listed, conv2d(a1)+b1,
    h_cache), GroupNorm of the FULL map h (fresh + cached), y = where(listed, x + conv2d(a2)
    + b2, y_cache).  Each rounding point uses the oracle's a1/h/a2 bits (bf16_rne is pinned
    above), each arithmetic stage is re-derived with library ops."""
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    n, h, w, c, b, G = 2, 12, 10, 32, 4, 8
    x, hc, yc, w1, b1, w2, b2, g1, be1, g2, be2 = _rb_inputs(n, h, w, c, "pin-rb")
    hb, wb = 3, 3
    ids = np.array([0, 1, 4, 8, 9, 12, 17])
    o = oracle.resblock(x, hc, yc, w1, b1, w2, b2, g1, be1, g2, be2, G, 1e-6, b, ids)
    L = _listed_px(ids, n, h, w, b)[..., None]
    d = lambda bits: torch.from_numpy(syn.bf16_bits_to_f32(bits).astype(np.float64)).permute(0, 3, 1, 2)
    nhwc = lambda t: t.permute(0, 2, 3, 1).numpy()
    t64 = lambda a: torch.from_numpy(np.asarray(a, np.float64))
    a1 = nhwc(F.silu(F.group_norm(d(x), G, t64(g1), t64(be1), eps=1e-6)))
    assert np.max(np.abs(o["a1_pre"] - a1)) <= 1e-12
    assert np.array_equal(o["a1"], oracle.bf16_rne(o["a1_pre"]))
    c1 = nhwc(F.conv2d(d(o["a1"]), d(w1), t64(b1), padding=1))
    assert np.max(np.abs(np.where(L, o["h_pre"], 0) - np.where(L, c1, 0))) <= 1e-12
    assert np.array_equal(o["h"], np.where(L, oracle.bf16_rne(c1), hc))
    a2 = nhwc(F.silu(F.group_norm(d(o["h"]), G, t64(g2), t64(be2), eps=1e-6)))
    assert np.max(np.abs(o["a2_pre"] - a2)) <= 1e-12
    c2 = nhwc(F.conv2d(d(o["a2"]), d(w2), t64(b2), padding=1))
    xd = nhwc(d(x))
    assert np.max(np.abs(o["y"] - np.where(L, xd + c2, yc))) <= 1e-12


def test_resblock_density_0_and_full_cache_consistency():
    """Density 0: y == y_cache and h == h_cache exactly.  Latent reuse: with caches
    from the dense pass (every block listed) on the same x, ANY block list reproduces the
    dense output bit for bit (the sparse block is exact, not an approximation, when the
    cache is current)."""
    n, h, w, c, b, G = 2, 16, 16, 16, 8, 4
    x, hc, yc, w1, b1, w2, b2, g1, be1, g2, be2 = _rb_inputs(n, h, w, c, "pin-rb0")
    args = (w1, b1, w2, b2, g1, be1, g2, be2, G, 1e-6, b)
    o0 = oracle.resblock(x, hc, yc, *args, np.zeros(0, np.int32))
    assert np.array_equal(o0["y"], yc) and np.array_equal(o0["h"], hc)
    dense = oracle.resblock(x, hc, yc, *args, np.arange(n * 4))
    for ids in ([0], [1, 2, 7], [3, 4, 5, 6]):
        o = oracle.resblock(x, dense["h"], dense["y"], *args, np.array(ids))
        assert np.array_equal(o["y"], dense["y"]) and np.array_equal(o["h"], dense["h"])
    # and a stale cache is visible through the halo and the statistics: change the cached h
    # of an unlisted block -> listed outputs change (GN2 over the full map, halo reads cache)
    hc2 = dense["h"].copy()
    hc2[0, 0:8, 8:16] = syn.resblock_features_bf16((8, 8, c), "pin-rb0-stale")
    o = oracle.resblock(x, hc2, dense["y"], *args, np.array([0]))
    assert not np.array_equal(o["y"][0, 0:8, 0:8], dense["y"][0, 0:8, 0:8])
    assert np.array_equal(o["y"][1], dense["y"][1])   # frame 1: nothing listed


# --------------------------------------------- NEXT-4 temporal attention + K/V cache

def _ta_inputs(n, h, w, c, tag, gain=1.0):
    x = syn.resblock_features_bf16((n, h, w, c), tag)
    qc = syn.resblock_features_bf16((n, h, w, 3 * c), tag + "-qc")
    yc = syn.bf16_bits_to_f32(syn.features_bf16((n, h, w, c), tag + "-yc")).astype(np.float64)
    wq = syn.linear_weights_bf16(3 * c, c, tag + "-q", gain)
    wo = syn.linear_weights_bf16(c, c, tag + "-o")
    bq, bo = syn.bias_f32(3 * c, tag + "-q"), syn.bias_f32(c, tag + "-o")
    return x, qc, yc, wq, bq, wo, bo


def test_temporal_attn_single_frame_is_value():
    """T = 1: the softmax over one key is exactly 1, so o = v of the same token (closed form)."""
    n, h, w, c, b = 3, 8, 8, 128, 4
    x, qc, yc, wq, bq, wo, bo = _ta_inputs(n, h, w, c, "pin-ta1")
    o = oracle.temporal_attn(x, qc, yc, wq, bq, wo, bo, 2, 1, b, np.arange(n * 4))
    v = syn.bf16_bits_to_f32(o["qkv"][..., 2 * c:]).astype(np.float64)
    assert np.array_equal(o["o_pre"], v)


def test_temporal_attn_matches_torch_dense():
    """Every block listed: qkv = torch fp64 linear(x); o = torch fp64 scaled_dot_product_attention
    over the frames of each sequence at each pixel (on the oracle's bf16 qkv, whose rounding is
    pinned above); y = x + linear(o bits)."""
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    n, h, w, c, b, heads, T = 4, 8, 6, 128, 4, 2, 2
    x, qc, yc, wq, bq, wo, bo = _ta_inputs(n, h, w, c, "pin-ta2")
    ids = np.arange(n * 2 * 2)
    o = oracle.temporal_attn(x, qc, yc, wq, bq, wo, bo, heads, T, b, ids)
    dec = lambda bits: torch.from_numpy(syn.bf16_bits_to_f32(bits).astype(np.float64))
    t64 = lambda a: torch.from_numpy(np.asarray(a, np.float64))
    q_ref = F.linear(dec(x), dec(wq), t64(bq)).numpy()
    assert np.max(np.abs(o["qkv_pre"] - q_ref)) <= 1e-12
    qkv = dec(o["qkv"]).reshape(n // T, T, h * w, 3, heads, c // heads)    # [s, t, p, qkv, hd, d]
    qkv = qkv.permute(3, 0, 2, 4, 1, 5)                                      # [qkv, s, p, hd, t, d]
    att = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2])            # [s, p, hd, t, d]
    att = att.permute(0, 3, 1, 2, 4).reshape(n, h, w, c).numpy()
    assert np.max(np.abs(o["o_pre"] - att)) <= 1e-12
    y_ref = dec(x).numpy() + F.linear(dec(o["o"]), dec(wo), t64(bo)).numpy()
    assert np.max(np.abs(o["y"] - y_ref)) <= 1e-12


def test_temporal_attn_permutation_uniform_and_cache():
    """Permuting the frames of a sequence permutes the outputs (no positional term); identical
    keys give the mean of the values; caches from the dense pass make ANY list reproduce the
    dense output bit for bit; a stale cached K/V of an unlisted frame changes listed outputs at
    the same pixel only (the cache is read, per pixel)."""
    n, h, w, c, b, heads, T = 3, 8, 8, 64, 4, 1, 3
    x, qc, yc, wq, bq, wo, bo = _ta_inputs(n, h, w, c, "pin-ta3")
    all_ids = np.arange(n * 4)
    d0 = oracle.temporal_attn(x, qc, yc, wq, bq, wo, bo, heads, T, b, all_ids)
    perm = [2, 0, 1]
    dp = oracle.temporal_attn(x[perm], qc[perm], yc[perm], wq, bq, wo, bo, heads, T, b, all_ids)
    assert np.array_equal(dp["y"], d0["y"][perm])
    # uniform keys: Wk = 0 and bk = 0 -> every score 0 -> o = mean over frames of v
    wq0 = wq.copy(); wq0[c:2 * c] = 0
    bq0 = bq.copy(); bq0[c:2 * c] = 0
    du = oracle.temporal_attn(x, qc, yc, wq0, bq0, wo, bo, heads, T, b, all_ids)
    v = syn.bf16_bits_to_f32(du["qkv"][..., 2 * c:]).astype(np.float64)
    assert np.allclose(du["o_pre"], np.broadcast_to(v.mean(axis=0), v.shape), rtol=0, atol=1e-12)
    for ids in ([0], [1, 5, 6], [3, 4, 8, 11]):
        o = oracle.temporal_attn(x, d0["qkv"], d0["y"], wq, bq, wo, bo, heads, T, b, np.array(ids))
        assert np.array_equal(o["y"], d0["y"]) and np.array_equal(o["qkv"], d0["qkv"])
    stale = d0["qkv"].copy()
    stale[2, 0, 0, c:] = syn.resblock_features_bf16((2 * c,), "pin-ta3-stale")  # frame 2, pixel (0,0)
    o = oracle.temporal_attn(x, stale, d0["y"], wq, bq, wo, bo, heads, T, b, np.array([0]))  # frame 0 blk 0
    assert not np.array_equal(o["y"][0, 0, 0], d0["y"][0, 0, 0])
    assert np.array_equal(o["y"][0, 1:4], d0["y"][0, 1:4]) and np.array_equal(o["y"][0, 0, 1:4], d0["y"][0, 0, 1:4])
    o0 = oracle.temporal_attn(x, qc, yc, wq, bq, wo, bo, heads, T, b, np.zeros(0, np.int32))
    assert np.array_equal(o0["y"], yc) and np.array_equal(o0["qkv"], qc)
