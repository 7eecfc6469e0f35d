"""GPU parity: every C-ABI entry point against the CPU oracle on the same seeded inputs.

Bars (BASELINE north_star): masks, counts, id lists, start steps and scatter bit-exact;
conv |y - y_ref| <= 1e-3 * sum|w x| + 1e-6 per element (fp32 output); noise within
1e-6 relative to |a x0| + |s eps| (reading R-3).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synthetic as syn

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
dev = "cuda"


def T(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(dev)


def bf16(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(dev)


def gpu_block_mask(sp, O, U, tau_u, tau_o, f, b, L, start=None):
    n, hp, wp = O.shape
    dims = oracle.level_dims(hp, wp, f, b, L)
    masks = [torch.full((n, hb, wb), 7, dtype=torch.uint8, device=dev) for (_, _, hb, wb) in dims]
    counts = torch.full((n, L), -5, dtype=torch.int32, device=dev)
    k = torch.full((n,), -9, dtype=torch.int32, device=dev) if start else None
    sp.sphinx_block_mask(T(O), None if U is None else T(U), None if tau_u is None else T(tau_u),
                         tau_o, f, b, masks, counts, start, k)
    torch.cuda.synchronize()
    return [m.cpu().numpy() for m in masks], counts.cpu().numpy(), None if k is None else k.cpu().numpy()


def gpu_compact(sp, mask, k, u, select=0, shape=None):
    n, hb, wb = mask.shape if mask is not None else shape
    ids = torch.full((n * hb * wb,), -7, dtype=torch.int32, device=dev)
    cnt = torch.full((1,), -1, dtype=torch.int32, device=dev)
    sp.sphinx_compact_blocks(None if mask is None else T(mask), None if k is None else T(k, torch.int32),
                             u, select, ids, cnt, shape=(n, hb, wb))
    c = int(cnt.item())
    return ids, cnt, ids[:c].cpu().numpy()


# ----------------------------------------------------------------- step 1

@pytest.mark.parametrize("case", GOLD["block_mask"], ids=lambda c: c["name"])
def test_block_mask_worked_examples(sphinx, case):
    O = np.ones((case["n"], case["hp"], case["wp"]), np.float32)
    for (y, x, v) in case["pixels"]:
        O[0, y, x] = np.nan if v == "nan" else v
    masks, counts, _ = gpu_block_mask(sphinx, O, None, None, 0.5, case["f"], case["b"], case["levels"])
    for l, want in enumerate(case["ids"]):
        assert np.flatnonzero(masks[l]).tolist() == want


@pytest.mark.parametrize("geom", [
    dict(n=4, hp=16, wp=16, f=1, b=4, L=1, d=[0.25, 0.0, 1.0, 0.5]),     # configs[0] geometry
    dict(n=3, hp=18, wp=18, f=1, b=8, L=1, d=[0.3, 0.6, 1.0]),           # scalar path, ragged
    dict(n=21, hp=576, wp=576, f=8, b=8, L=3, d=list(syn.request_densities(21))),  # configs[2]
    dict(n=2, hp=64, wp=96, f=2, b=4, L=3, d=[0.1, 0.4]),
])
@pytest.mark.parametrize("pattern", ["clustered", "scattered"])
def test_block_mask_vs_oracle(sphinx, geom, pattern):
    n, hp, wp, f, b, L = geom["n"], geom["hp"], geom["wp"], geom["f"], geom["b"], geom["L"]
    O, cells = syn.opacity_maps(n, hp, wp, b * f, geom["d"], pattern, tag=f"gm{hp}{wp}")
    U, tau = syn.uncertainty_maps(n, hp, wp, b * f, cells, tag=f"gm{hp}{wp}")
    O[0, 0, 1] = np.nan
    U[-1, hp - 1, wp - 1] = tau[-1]  # equality: not blurry
    for uu, tt in ((U, tau), (None, None)):
        want_m, want_c = oracle.block_mask(O, uu, tt, 0.5, f, b, L)
        got_m, got_c, _ = gpu_block_mask(sphinx, O, uu, tt, 0.5, f, b, L)
        for l in range(L):
            assert np.array_equal(got_m[l], want_m[l]), l
        assert np.array_equal(got_c, want_c)


def test_start_steps_vs_oracle(sphinx):
    lg0 = oracle.make_klogic(**{"thr": syn.SPEC_KLOGIC["thr"], "steps": syn.SPEC_KLOGIC["steps"]})
    lg1 = oracle.make_klogic([0.6, 0.8, 0.9, 1.0], [5, 15, 30, 45], 2, 40)
    glg = [sphinx.make_klogic(syn.SPEC_KLOGIC["thr"], syn.SPEC_KLOGIC["steps"]),
           sphinx.make_klogic([0.6, 0.8, 0.9, 1.0], [5, 15, 30, 45], 2, 40)]
    reqs = [syn.request_scores(21, c0, c1, tag=f"r{i}") for i, (c0, c1) in
            enumerate([(62, 66), (70, 58), (50, 50), (64, 61)])]
    q, c0, c1, t = (np.concatenate([r[j] for r in reqs]) for j in range(4))
    n = len(q)
    # tie cases TV-6..8 and invalid inputs appended
    q = np.concatenate([q, np.float32([61.75, 59.8, np.float32(0.97 * 65), 60, 60])])
    c0 = np.concatenate([c0, np.float32([60, 60, 60, 0, 60])])
    c1 = np.concatenate([c1, np.float32([70, 70, 70, 0, 70])])
    t = np.concatenate([t, np.float32([0.25, 0.25, 0.25, 0.5, 1.5])])
    lid = (np.arange(len(q)) % 2).astype(np.int32)
    lid[n:] = 0
    O = np.ones((len(q), 16, 16), np.float32)
    thr_all = np.array(syn.SPEC_KLOGIC["thr"] + [0.6, 0.8, 0.9, 1.0])
    for gamma in (0.5, 1.0, 0.7):
        want = oracle.start_step(q, c0, c1, t, gamma, [lg0, lg1], logic_id=lid)
        start = dict(q_reg=T(q), c0=T(c0), c1=T(c1), t=T(t), gamma=gamma, logics=glg,
                     logic_id=T(lid))
        _, _, k = gpu_block_mask(sphinx, O, None, None, 0.5, 1, 4, 1, start=start)
        keep = np.ones(len(q), bool)
        if gamma not in (0.5, 1.0):
            # R-16 near-tie exclusion: CUDA pow and glibc pow may differ by an ulp, so frames whose
            # ratio lies within 1e-12 (relative) of a cut point are not compared for these gamma
            qs = np.array([oracle.eq2(float(a), float(b), float(ti), gamma) for a, b, ti in zip(c0, c1, t)])
            with np.errstate(divide="ignore", invalid="ignore"):
                r = q.astype(np.float64) / qs
            near = np.abs(r[:, None] - thr_all[None, :]) <= 1e-12 * thr_all[None, :]
            keep = ~near.any(1)
            assert keep.sum() >= len(q) - 5
        assert np.array_equal(k[keep], want[keep]), gamma
        assert k[n:].tolist() == [25, 10, 25, -1, -1] or gamma != 0.5


GOLD_EQ2R = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "eq2_realized_ratio.json")))


@pytest.mark.parametrize("gamma", [0.5, 1.0])
def test_start_steps_cut_points_at_realized_ratios(sphinx, gamma):
    """k-logic cut points placed EXACTLY at realized ratios r = q / Q* (a decile calibration
    emits such cut points; left-closed): 8 logics x 16 cut points, each the
    ratio of one of 128 frames (random fp32 t, c0, c1, q), plus the golden VERDICT-r01 vectors.
    Any 1-ulp difference in Eq. 2 or the division flips k, so this is the bit-exact bar of
    R-16 for gamma = 0.5 (correctly rounded sqrt) and 1 (t itself)."""
    import struct
    rg = syn.rng("gpu-realized", gamma)
    n = 125  # + 3 golden vectors: at most 16 frames (= cut points) per logic
    t = rg.random(n).astype(np.float32)
    c0 = rg.uniform(40, 80, n).astype(np.float32)
    c1 = rg.uniform(40, 80, n).astype(np.float32)
    q = (rg.uniform(0.8, 1.1, n) * 60).astype(np.float32)
    gold = GOLD_EQ2R["cases"] if gamma == 0.5 else []
    for c in gold:
        t = np.append(t, np.float32(struct.unpack("<f", struct.pack("<I", int(c["t_bits"], 16)))[0]))
        c0 = np.append(c0, np.float32(c["c0"])); c1 = np.append(c1, np.float32(c["c1"]))
        q = np.append(q, np.float32(c["q"]))
    r = np.array([float(qi) / oracle.eq2(float(a), float(b), float(ti), gamma)
                  for qi, a, b, ti in zip(q, c0, c1, t)])
    for i, c in enumerate(gold):
        assert r[n + i] == float.fromhex(c["r_hex"])
    m = len(q)
    lid = (np.arange(m) % 8).astype(np.int32)
    olg, glg, want_k = [], [], np.full(m, -9, np.int32)
    for j in range(8):
        idx = np.flatnonzero(lid == j)
        thr = np.unique(r[idx])[:16]
        steps = list(range(1, len(thr) + 1))
        olg.append(oracle.make_klogic(thr, steps, 0, 40))
        glg.append(sphinx.make_klogic(thr, steps, 0, 40))
        for i in idx:
            want_k[i] = int(np.searchsorted(thr, r[i], side="right"))  # left-closed: r == thr_i -> step i
    want = oracle.start_step(q, c0, c1, t, gamma, olg, logic_id=lid)
    assert np.array_equal(want, want_k)
    O = np.ones((m, 16, 16), np.float32)
    start = dict(q_reg=T(q), c0=T(c0), c1=T(c1), t=T(t), gamma=gamma, logics=glg, logic_id=T(lid))
    _, _, k = gpu_block_mask(sphinx, O, None, None, 0.5, 1, 4, 1, start=start)
    assert np.array_equal(k, want)
    # one ulp above every realized ratio: each frame drops one step (thresholds strictly above r)
    olg2, glg2 = [], []
    for j in range(8):
        idx = np.flatnonzero(lid == j)
        thr = np.nextafter(np.unique(r[idx])[:16], np.inf)
        steps = list(range(1, len(thr) + 1))
        olg2.append(oracle.make_klogic(thr, steps, 0, 40))
        glg2.append(sphinx.make_klogic(thr, steps, 0, 40))
    want2 = oracle.start_step(q, c0, c1, t, gamma, olg2, logic_id=lid)
    assert np.array_equal(want2, want - 1)
    start["logics"] = glg2
    _, _, k2 = gpu_block_mask(sphinx, O, None, None, 0.5, 1, 4, 1, start=start)
    assert np.array_equal(k2, want2)


def test_block_mask_exhaustive_config1_patterns(sphinx):
    """All 2^16 block patterns at configs[0] geometry (16x16, f=1, b=4) on the GPU: one painted
    pixel per chosen block must give exactly the pattern back (coverage + no false positives,
    S:261-264), bit-identical to the oracle."""
    O, pat = syn.exhaustive_block_patterns()
    n = len(O)
    got_m, got_c, _ = gpu_block_mask(sphinx, O, None, None, 0.5, 1, 4, 1)
    assert np.array_equal(got_m[0].reshape(n, 16).astype(bool), pat)
    assert np.array_equal(got_c[:, 0], pat.sum(1))
    want_m, want_c = oracle.block_mask(O, None, None, 0.5, 1, 4, 1)
    assert np.array_equal(got_m[0], want_m[0]) and np.array_equal(got_c, want_c)


@pytest.mark.parametrize("n_px", [1, 7, 60])
def test_block_mask_sparse_random_pixels(sphinx, n_px):
    """Uniformly random isolated flagged pixels (half on footprint-boundary rows/columns),
    equality pixels and NaNs at the bench geometry (576x576, f=8, b=8, L=3): masks and counts
    bit-exact vs the oracle at every level."""
    n = 12
    O, U, tau = syn.sparse_pixel_maps(n, 576, 576, 64, n_px)
    for uu, tt in ((U, tau), (None, None)):
        want_m, want_c = oracle.block_mask(O, uu, tt, 0.5, 8, 8, 3)
        got_m, got_c, _ = gpu_block_mask(sphinx, O, uu, tt, 0.5, 8, 8, 3)
        for l in range(3):
            assert np.array_equal(got_m[l], want_m[l]), l
        assert np.array_equal(got_c, want_c)


# ----------------------------------------------------------------- step 2

def test_compact_vs_oracle(sphinx):
    rg = syn.rng("gpu-compact")
    for (n, hb, wb) in [(1, 4, 4), (21, 9, 9), (168, 9, 9), (168, 5, 5), (3, 1, 1), (7, 33, 31)]:
        for dens in (0.0, 0.05, 0.25, 1.0):
            m = (rg.random((n, hb, wb)) < dens).astype(np.uint8)
            k = rg.integers(-1, 45, size=n).astype(np.int32)
            for u in (0, 25, 49):
                for sel in (0, 1, 2, 3):
                    if sel == 3:  # NOISE = ACTIVE | INACTIVE_FRAMES
                        _, _, got = gpu_compact(sphinx, m, k, u, sel)
                        assert np.array_equal(got, oracle.compact(m, k, u, sel))
                    elif sel == 0:
                        for kk in (k, None):
                            _, _, got = gpu_compact(sphinx, m, kk, u, sel)
                            assert np.array_equal(got, oracle.compact(m, kk, u, sel))
                    else:
                        _, _, got = gpu_compact(sphinx, None, k, u, sel, shape=(n, hb, wb))
                        assert np.array_equal(got, oracle.compact(None, k, u, sel, shape=(n, hb, wb)))


# ----------------------------------------------------------------- step 3

@pytest.mark.parametrize("shape,b", [((1, 16, 16, 4), 4), ((21, 72, 72, 4), 8), ((3, 36, 36, 4), 8),
                                     ((2, 18, 18, 3), 8)])
def test_noise_vs_oracle(sphinx, shape, b):
    n, h, w, c = shape
    hb, wb = -(-h // b), -(-w // b)
    rg = syn.rng("gpu-noise", shape)
    m = (rg.random((n, hb, wb)) < 0.4).astype(np.uint8)
    ids = oracle.compact(m)
    step = rg.integers(-1, 52, size=n).astype(np.int32)  # includes out-of-range u: untouched
    abar = syn.abar_cosine(50)
    x0, eps, xt = (syn.latents_f32(shape, f"gn{j}") for j in range(3))
    want = oracle.noise(x0, eps, xt, b, ids, step, abar)
    g_ids, g_cnt, _ = gpu_compact(sphinx, m, None, 0)
    out = T(xt)
    sphinx.sphinx_noise_inject(T(x0), T(eps), out, b, g_ids, g_cnt, T(step), T(abar))
    got = out.cpu().numpy()
    touched = want != xt.astype(np.float64)
    assert np.array_equal(got[~touched], xt[~touched])
    # tolerance relative to the term magnitudes |a x0| + |s eps| (reading R-3)
    u = np.clip(step, 0, 50)
    a = np.sqrt(abar[u].astype(np.float64))[:, None, None, None]
    s = np.sqrt(1.0 - abar[u].astype(np.float64))[:, None, None, None]
    scale = np.abs(a * x0) + np.abs(s * eps)
    assert np.all(np.abs(got - want) <= 1e-6 * scale + 1e-30)
    # in place (x_t aliases x0)
    inplace = T(x0)
    sphinx.sphinx_noise_inject(inplace, T(eps), inplace, b, g_ids, g_cnt, T(step), T(abar))
    want2 = oracle.noise(x0, eps, x0, b, ids, step, abar)
    assert np.all(np.abs(inplace.cpu().numpy() - want2) <= 1e-6 * scale + 1e-30)


@pytest.mark.parametrize("shape,b", [((21, 72, 72, 4), 8), ((5, 20, 13, 8), 4)])
def test_noise_step_fused_vs_oracle(sphinx, shape, b):
    """sphinx_noise_inject_step over a SELECT_NOISE list == Alg1 line 12 (active blocks at their
    start step k) and line 19 (inactive frames at u+1) in one pass; conditioning frames (k = -1)
    untouched; within 1e-6 of |a x0| + |s eps| (R-3)."""
    n, h, w, c = shape
    hb, wb = -(-h // b), -(-w // b)
    rg = syn.rng("gpu-noise-step", shape)
    m = (rg.random((n, hb, wb)) < 0.4).astype(np.uint8)
    k = rg.integers(-1, 45, size=n).astype(np.int32)
    u = 25
    abar = syn.abar_cosine(50)
    x0, eps, xt = (syn.latents_f32(shape, f"gns{j}") for j in range(3))
    step = np.where((k >= 0) & (k <= u), k, np.where(k > u, u + 1, -1)).astype(np.int32)
    want = oracle.noise(x0, eps, xt, b, oracle.compact(m, k, u, oracle.SELECT_NOISE), step, abar)
    g_ids, g_cnt, _ = gpu_compact(sphinx, m, k, u, 3)
    out = T(xt)
    sphinx.sphinx_noise_inject_step(T(x0), T(eps), out, b, g_ids, g_cnt, T(k), u, T(abar))
    got = out.cpu().numpy()
    touched = want != xt.astype(np.float64)
    assert touched.any() and np.array_equal(got[~touched], xt[~touched])
    uu = np.clip(step, 0, 50)
    a = np.sqrt(abar[uu].astype(np.float64))[:, None, None, None]
    s_ = np.sqrt(1.0 - abar[uu].astype(np.float64))[:, None, None, None]
    assert np.all(np.abs(got - want) <= 1e-6 * (np.abs(a * x0) + np.abs(s_ * eps)) + 1e-30)


# ----------------------------------------------------------------- step 4

@pytest.fixture(params=[(1, 0, 1, 1, 1), (2, 0, 1, 1, 1), (1, 1, 1, 1, 1), (2, 1, 1, 1, 1),
                        (2, 1, 1, 0, 1), (2, 0, 0, 0, 1), (2, 1, 0, 0, 1), (2, 1, 1, 1, 2),
                        (1, 1, 1, 1, 2)],
                ids=["cta1", "pair", "cta1-splitk", "pair-splitk", "pair-splitk-noedge", "pair-pertap",
                     "pair-pertap-splitk", "pair-streamk", "cta1-streamk"])
def conv_cg(request, monkeypatch, sphinx):
    """Runs a conv test with the 1-SM (cta_group::1) and the CTA-pair (cta_group::2) kernels,
    without and with device-chosen split-K, with halo-staged (b=8 default, with and without
    edge-class packing) and per-tap A, and with stream-K forced where feasible -- the variant
    flags of sphinx_sparse_conv3x3_ex (sphinx.h), passed explicitly on every conv call."""
    cg, split, halo, edge, streamk = request.param
    flags = ((sphinx.CONV_FORCE_CG1 if cg == 1 else 0) | (0 if split else sphinx.CONV_NO_SPLIT) |
             (sphinx.CONV_FORCE_HALO if halo else sphinx.CONV_FORCE_PERTAP) |
             (0 if edge else sphinx.CONV_NO_EDGE) |
             {0: sphinx.CONV_NO_STREAMK, 1: 0, 2: sphinx.CONV_FORCE_STREAMK}[streamk])
    plain = sphinx.sphinx_sparse_conv3x3

    def with_variant(*a, **k):
        return plain(*a, variant=flags | k.pop("variant", 0), **k)
    monkeypatch.setattr(sphinx, "sphinx_sparse_conv3x3", with_variant)
    return request.param


def _conv_check(sphinx, n, h, w, cin, cout, b, density, pattern, tag, out_dtype=torch.float32,
                bias=True, weights=None, x_bits=None, sample_ids=None):
    hb, wb = -(-h // b), -(-w // b)
    x = syn.features_bf16((n, h, w, cin), tag) if x_bits is None else x_bits
    wt = syn.weights_bf16(cout, cin, tag) if weights is None else weights
    bs = syn.bias_f32(cout, tag) if bias else None
    rg = syn.rng("conv-mask", tag)
    m = np.stack([syn.choose_cells(rg, hb, wb, round(density * hb * wb), pattern) for _ in range(n)])
    m = m.astype(np.uint8)
    ids_all = oracle.compact(m)
    g_ids, g_cnt, _ = gpu_compact(sphinx, m, None, 0)
    sentinel = -12345.0
    y = torch.full((n, h, w, cout), sentinel, dtype=out_dtype, device=dev)
    sphinx.sphinx_sparse_conv3x3(bf16(x), bf16(wt), None if bs is None else T(bs), y, b, g_ids, g_cnt)
    torch.cuda.synchronize()
    got = y.float().cpu().numpy().astype(np.float64)
    check_ids = ids_all if sample_ids is None else ids_all[sample_ids(len(ids_all))]
    want, acc = oracle.conv3x3_blocks(x, wt, bs, b, check_ids)
    listed = ~np.isnan(want[..., 0])
    tol = 1e-3 * acc[listed] + 1e-6
    if out_dtype == torch.bfloat16:
        tol = tol + 2.0 ** -8 * np.abs(want[listed])
    err = np.abs(got[listed] - want[listed])
    assert np.all(err <= tol), f"max err/tol {np.max(err / tol)}"
    if sample_ids is None:  # unlisted pixels untouched
        assert np.all(got[~listed] == np.float64(np.float32(sentinel)) if out_dtype == torch.float32
                      else got[~listed] == float(torch.tensor(sentinel, dtype=out_dtype).float()))
    return err, tol


def test_conv_config0(sphinx, conv_cg):
    """configs[0]: 1 frame, 16x16x32, 3x3 32->32, block 4, 25% active."""
    _conv_check(sphinx, 1, 16, 16, 32, 32, 4, 0.25, "scattered", "cfg0")


@pytest.mark.parametrize("h,c,pattern,dens", [(72, 320, "clustered", 0.25), (36, 640, "scattered", 0.4),
                                              (18, 1280, "checker", 0.5), (72, 320, "checker", 1.0)])
def test_conv_unet_levels(sphinx, conv_cg, h, c, pattern, dens):
    """configs[1]/[2] geometries: 72x72x320, 36x36x640 (ragged 5x5 blocks), 18x18x1280."""
    _conv_check(sphinx, 2, h, h, c, c, 8, dens, pattern, f"lvl{h}")


@pytest.mark.parametrize("cin,cout,b", [(64, 64, 8), (128, 32, 4), (320, 160, 8), (8, 16, 4),
                                        (96, 264, 8)])
def test_conv_shapes_bf16_out(sphinx, conv_cg, cin, cout, b):
    _conv_check(sphinx, 3, 20, 28, cin, cout, b, 0.5, "scattered", f"shape{cin}{cout}",
                out_dtype=torch.bfloat16)


@pytest.mark.parametrize("h,w", [(17, 9), (20, 28), (13, 11), (22, 15), (19, 23), (14, 30)])
@pytest.mark.parametrize("pattern", ["checker", "scattered"])
def test_conv_ragged_edges(sphinx, conv_cg, h, w, pattern):
    """Every remainder H % 8, W % 8 in 1..7: bottom-edge, right-edge and corner blocks (the
    edge-class packing of the halo kernel) against the oracle, bf16 and fp32 outputs."""
    for dt in (torch.float32, torch.bfloat16):
        _conv_check(sphinx, 3, h, w, 64, 96, 8, 0.6, pattern, f"rag{h}x{w}{pattern}", out_dtype=dt)


@pytest.mark.parametrize("ky,kx", [(0, 0), (1, 1), (2, 1), (0, 2)])
def test_conv_shift_kernels_exact(sphinx, conv_cg, ky, kx):
    """TV-12/13: a shift kernel reproduces the shifted input exactly, incl. halos across
    blocks (active and inactive neighbours) and zero padding at the border."""
    n, h, w, c, b = 2, 18, 18, 64, 8
    wt = np.zeros((c, 3, 3, c), np.float32)
    for i in range(c):
        wt[i, ky, kx, i] = 1.0
    err, _ = _conv_check(sphinx, n, h, w, c, c, b, 0.6, "scattered", "shift", bias=False,
                         weights=syn.to_bf16_bits(wt))
    assert np.all(err == 0)


def test_conv_density_zero_and_count_zero(sphinx, conv_cg):
    n, h, w, c, b = 1, 16, 16, 32, 4
    g_ids, g_cnt, got = gpu_compact(sphinx, np.zeros((n, 4, 4), np.uint8), None, 0)
    assert len(got) == 0
    y = torch.full((n, h, w, c), 3.0, device=dev)
    sphinx.sphinx_sparse_conv3x3(bf16(syn.features_bf16((n, h, w, c), "z")),
                                 bf16(syn.weights_bf16(c, c, "z")), None, y, b, g_ids, g_cnt)
    assert torch.all(y == 3.0)


def test_conv_deterministic_and_split_consistent(sphinx, monkeypatch):
    """S:350 bit-reproducible; split-K (fixed-order fp32 reduction) agrees with one pass
    within the conv tolerance on a latency-bound shape where the device picks S > 1."""
    n, h, c, b = 1, 18, 1280, 8
    x = bf16(syn.features_bf16((n, h, h, c), "det"))
    w = bf16(syn.weights_bf16(c, c, "det"))
    m = np.zeros((n, 3, 3), np.uint8); m[0, 0, :] = 1; m[0, 2, 2] = 1
    g_ids, g_cnt, _ = gpu_compact(sphinx, m, None, 0)
    outs = []
    for split in (True, True, False):
        y = torch.zeros((n, h, h, c), dtype=torch.float32, device=dev)
        sphinx.sphinx_sparse_conv3x3(x, w, None, y, b, g_ids, g_cnt,
                                     variant=0 if split else sphinx.CONV_NO_SPLIT)
        outs.append(y.cpu().numpy())
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
    xb = x.view(torch.int16).cpu().numpy().view(np.uint16)
    wb = w.view(torch.int16).cpu().numpy().view(np.uint16)
    want, acc = oracle.conv3x3_blocks(xb, wb, None, b, oracle.compact(m))
    listed = ~np.isnan(want[..., 0])
    for o in outs:
        assert np.all(np.abs(o[listed] - want[listed]) <= 1e-3 * acc[listed] + 1e-6)


def test_conv_full_size_sampled(sphinx, conv_cg):
    """BASELINE configs[3] size at level 1 (168 frames x 72x72x320, 25%): sampled blocks."""
    _conv_check(sphinx, 168, 72, 72, 320, 320, 8, 0.25, "clustered", "full168",
                sample_ids=lambda m: np.linspace(0, m - 1, 24).astype(int))


# ----------------------------------------------------------------- step 5

@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_scatter_vs_oracle(sphinx, dtype):
    n, h, w, c, b = 5, 36, 36, 64, 8
    hb, wb = 5, 5
    rg = syn.rng("gpu-scatter", dtype)
    m = (rg.random((n, hb, wb)) < 0.4).astype(np.uint8)
    k = np.array([0, 10, 30, -1, 45], np.int32)
    u = 25
    if dtype == "bf16":
        src, cache = syn.features_bf16((n, h, w, c), "s1"), syn.features_bf16((n, h, w, c), "s2")
        src[0, 0, 0, 0] = 0x7FC1  # NaN payload
        src[0, 0, 0, 1] = 0x8000  # -0
        tt = lambda a: bf16(a)
        back = lambda t: t.view(torch.int16).cpu().numpy().view(np.uint16)
    else:
        src, cache = syn.latents_f32((n, h, w, c), "s1"), syn.latents_f32((n, h, w, c), "s2")
        tt = lambda a: T(a)
        back = lambda t: t.cpu().numpy()
    want = oracle.scatter(src, cache, b, mask=m, k=k, u=u)
    out = tt(np.zeros_like(cache))
    sphinx.sphinx_scatter_cached(tt(src), tt(cache), out, b, block_mask=T(m), start_step=T(k), step_u=u)
    assert np.array_equal(back(out).view(np.uint8), want.view(np.uint8))
    # in place: out aliases src -> only inactive blocks written
    s2 = tt(src)
    sphinx.sphinx_scatter_cached(s2, tt(cache), s2, b, block_mask=T(m), start_step=T(k), step_u=u)
    assert np.array_equal(back(s2).view(np.uint8), want.view(np.uint8))
    # COMPACT layout
    ids = oracle.compact(m, k, u)
    comp = np.zeros((max(len(ids), 1), b, b, c), cache.dtype)
    for j, id_ in enumerate(ids):
        i, r = divmod(int(id_), hb * wb)
        by, bx = divmod(r, wb)
        blk = src[i, by * b:(by + 1) * b, bx * b:(bx + 1) * b]
        comp[j, :blk.shape[0], :blk.shape[1]] = blk
    want_c = oracle.scatter(comp, cache, b, ids=ids, src_layout=oracle.SRC_COMPACT)
    g_ids, g_cnt, _ = gpu_compact(sphinx, m, k, u)
    out2 = tt(np.zeros_like(cache))
    sphinx.sphinx_scatter_cached(tt(comp), tt(cache), out2, b, block_ids=g_ids, count=g_cnt,
                                 src_layout=sphinx.SRC_COMPACT)
    assert np.array_equal(back(out2).view(np.uint8), want_c.view(np.uint8))
    assert np.array_equal(want_c.view(np.uint8), want.view(np.uint8))


def test_invalid_arguments_raise(sphinx):
    with pytest.raises(sphinx.SphinxError):
        sphinx.sphinx_block_mask(T(np.ones((1, 16, 16), np.float32)), None, None, 2.0, 1, 4,
                                 [torch.zeros((1, 4, 4), dtype=torch.uint8, device=dev)])


# ----------------------------------------------------------------- NEXT-1 DDIM update

@pytest.mark.parametrize("shape,b", [((21, 72, 72, 4), 8), ((3, 18, 18, 4), 8), ((2, 16, 16, 3), 4)])
@pytest.mark.parametrize("u", [0, 17, 40, 49])
def test_ddim_step_vs_oracle(sphinx, shape, b, u):
    n, h, w, c = shape
    hb, wb = -(-h // b), -(-w // b)
    rg = syn.rng("gpu-ddim", shape, u)
    m = (rg.random((n, hb, wb)) < 0.4).astype(np.uint8)
    ids = oracle.compact(m)
    abar = syn.abar_cosine(50)
    z, xh = syn.latents_f32(shape, "gd-z"), syn.latents_f32(shape, "gd-x")
    want = oracle.ddim_step(z, xh, b, ids, u, abar)
    g_ids, g_cnt, _ = gpu_compact(sphinx, m, None, 0)
    out = T(z)  # in place: z_out aliases z
    sphinx.sphinx_ddim_step(out, T(xh), out, b, g_ids, g_cnt, u, abar)
    got = out.cpu().numpy()
    a0, s0 = np.sqrt(np.float64(abar[u])), np.sqrt(1 - np.float64(abar[u]))
    a1, s1 = np.sqrt(np.float64(abar[u + 1])), np.sqrt(1 - np.float64(abar[u + 1]))
    tol = 1e-6 * (np.abs(a1 * xh) + (s1 / s0) * (np.abs(z) + np.abs(a0 * xh))) + 1e-30
    assert np.all(np.abs(got - want) <= tol), np.max(np.abs(got - want) / tol)
    untouched = want == z.astype(np.float64)
    assert np.array_equal(got[untouched], z[untouched])


# ----------------------------------------------------------- NEXT-2 uncertainty producer

def _rgb_frames(n, h, w, tag):
    """Synthetic regression frames: smooth gradients + sharp texture + flat (blurry) patches."""
    return syn.rgb_frames(n, h, w, tag)


@pytest.mark.parametrize("n,h,w,win,sm", [(2, 64, 64, 7, 5), (3, 576, 576, 7, 5), (2, 37, 53, 3, 1),
                                          (1, 40, 30, 9, 3)])
def test_uncertainty_map_vs_oracle(sphinx, n, h, w, win, sm):
    rgb = _rgb_frames(n, h, w, f"{h}x{w}")
    U_ref, _ = oracle.uncertainty(rgb, win, sm)
    U = torch.empty((n, h, w), dtype=torch.float32, device=dev)
    tau = torch.empty((n,), dtype=torch.float32, device=dev)
    sphinx.sphinx_uncertainty_map(T(rgb), U, tau, win, sm)
    Ug, tg = U.cpu().numpy(), tau.cpu().numpy()
    # fp32 stencil (two-pass variance, box mean) and normalisation vs fp64: the map lives in
    # [0,1] and the fp32 rounding of S relative to the frame's range (max S - min S) stays
    # ~1e-6; 1e-4 absolute leaves two decades of margin (reading R-24)
    assert np.max(np.abs(Ug - U_ref)) <= 1e-4
    # the Otsu decision is taken in the kernel's precision: the oracle's exact Otsu on the
    # GPU's own U must give the GPU's tau bit for bit
    for i in range(n):
        assert tg[i] == np.float32(oracle.otsu(Ug[i])), i
    assert Ug.min() >= 0.0 and Ug.max() == 1.0


def test_uncertainty_map_degenerate_and_semantics(sphinx):
    # S:219 constant frame -> U == 1, tau == 1 -> empty blur mask
    rgb = np.full((2, 24, 24, 3), 0.3, np.float32)
    U = torch.empty((2, 24, 24), dtype=torch.float32, device=dev)
    tau = torch.empty((2,), dtype=torch.float32, device=dev)
    sphinx.sphinx_uncertainty_map(T(rgb), U, tau)
    assert torch.all(U == 1.0) and torch.all(tau == 1.0)
    # S:220 half sharp checkerboard / half flat gray: blurry = flat half
    img = np.full((1, 64, 64, 3), 0.5, np.float32)
    yy, xx = np.mgrid[0:64, 0:32]
    img[0, :, :32, :] = ((yy + xx) % 2)[..., None]
    U = torch.empty((1, 64, 64), dtype=torch.float32, device=dev)
    tau = torch.empty((1,), dtype=torch.float32, device=dev)
    sphinx.sphinx_uncertainty_map(T(img), U, tau)
    m = (U > tau[0]).cpu().numpy()[0]
    assert m[:, 40:].mean() >= 0.95 and m[:, :24].mean() <= 0.05
    # chained into step 1: the produced (U, tau) drive sphinx_block_mask exactly like the oracle
    O = np.ones((1, 64, 64), np.float32)
    masks, counts, _ = gpu_block_mask(sphinx, O, U.cpu().numpy(), tau.cpu().numpy(), 0.5, 1, 8, 1)
    want, _ = oracle.block_mask(O, U.cpu().numpy(), tau.cpu().numpy(), 0.5, 1, 8, 1)
    assert np.array_equal(masks[0], want[0])


def test_compact_batch_equals_single_calls(sphinx):
    """sphinx_compact_blocks_batch (one launch, one CTA per list) = the single calls, bit for bit."""
    rg = np.random.default_rng(5)
    jobs, want = [], []
    for (n, hb, wb, sel) in [(21, 9, 9, 0), (21, 5, 5, 0), (21, 3, 3, 0), (21, 9, 9, 1), (3, 4, 7, 2)]:
        m = (rg.random((n, hb, wb)) < 0.3).astype(np.uint8)
        k = rg.integers(-1, 45, n).astype(np.int32)
        ids = torch.full((n * hb * wb,), -3, dtype=torch.int32, device=dev)
        cnt = torch.zeros(1, dtype=torch.int32, device=dev)
        jobs.append(dict(block_mask=T(m), start_step=T(k, torch.int32), step_u=25, select=sel, block_ids=ids,
                         count=cnt))
        want.append(oracle.compact(m, k, 25, sel))
    sphinx.sphinx_compact_blocks_batch(jobs)
    torch.cuda.synchronize()
    for jb, w in zip(jobs, want):
        c = int(jb["count"].item())
        assert np.array_equal(jb["block_ids"][:c].cpu().numpy(), w)


def test_conv_reuse_plan(sphinx):
    """SPHINX_CONV_REUSE_PLAN: a second conv over the same list/workspace (edge-class maps) that
    skips the plan launch gives bit-identical output to a conv that recomputes it."""
    n, h, c, b = 3, 36, 64, 8
    x = bf16(syn.features_bf16((n, h, h, c), "reuse"))
    w = bf16(syn.weights_bf16(c, c, "reuse"))
    m = (np.random.default_rng(2).random((n, 5, 5)) < 0.5).astype(np.uint8)
    g_ids, g_cnt, _ = gpu_compact(sphinx, m, None, 0)
    ws = torch.zeros(sphinx.load().sphinx_conv_workspace_size(n, h, h, c, c, b), dtype=torch.uint8, device=dev)
    y0 = torch.zeros((n, h, h, c), device=dev)
    y1 = torch.zeros((n, h, h, c), device=dev)
    sphinx.sphinx_sparse_conv3x3(x, w, None, y0, b, g_ids, g_cnt, workspace=ws)
    sphinx.sphinx_sparse_conv3x3(x, w, None, y1, b, g_ids, g_cnt, workspace=ws, reuse_plan=True)
    torch.cuda.synchronize()
    assert np.array_equal(y0.cpu().numpy().view(np.uint32), y1.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("h,c", [(36, 64), (18, 640)])
def test_conv_early_start_flags(sphinx, h, c):
    """SPHINX_CONV_LIST_READY / SPHINX_CONV_INPUT_READY (loads before griddepcontrol.wait, stores
    after it): bit-identical to the plain launch, also when the preceding kernel is a long conv
    that writes a different output (the stores still follow it)."""
    n, b = 3, 8
    x = bf16(syn.features_bf16((n, h, h, c), "early"))
    w = bf16(syn.weights_bf16(c, c, "early"))
    m = (np.random.default_rng(5).random((n, h // b + (h % b > 0), h // b + (h % b > 0))) < 0.6).astype(np.uint8)
    g_ids, g_cnt, _ = gpu_compact(sphinx, m, None, 0)
    ws = torch.zeros(sphinx.load().sphinx_conv_workspace_size(n, h, h, c, c, b), dtype=torch.uint8, device=dev)
    ws2 = torch.zeros_like(ws)
    ys = [torch.zeros((n, h, h, c), device=dev) for _ in range(4)]
    sphinx.sphinx_sparse_conv3x3(x, w, None, ys[0], b, g_ids, g_cnt, workspace=ws)
    sphinx.sphinx_sparse_conv3x3(x, w, None, ys[1], b, g_ids, g_cnt, workspace=ws2)  # plan for ws2
    sphinx.sphinx_sparse_conv3x3(x, w, None, ys[2], b, g_ids, g_cnt, workspace=ws2, reuse_plan=True,
                                 list_ready=True)
    sphinx.sphinx_sparse_conv3x3(x, w, None, ys[3], b, g_ids, g_cnt, workspace=ws, reuse_plan=True,
                                 list_ready=True, input_ready=True)
    torch.cuda.synchronize()
    ref = ys[0].cpu().numpy().view(np.uint32)
    for y in ys[1:]:
        assert np.array_equal(ref, y.cpu().numpy().view(np.uint32))


def test_conv_back_to_back_list_ready(sphinx):
    """edge_plan(level 1) -> conv(level 0, LIST_READY) -> conv(level 1, LIST_READY |
    REUSE_PLAN), the call order the contract allows.  The level-1 conv reads its plan (written two
    kernels back) before its own griddepcontrol.wait; the level-0 conv only signals its dependents
    after its epilogue waited, so the plan is complete.  Repeated with fresh lists each round so a
    stale plan would show; results bit-identical to plain launches with their own (equally sized,
    zeroed) workspaces, so the device-side split decisions are the same."""
    rg = np.random.default_rng(11)
    n = 4
    x0 = bf16(syn.features_bf16((n, 72, 72, 320), "b2b0"))
    w0 = bf16(syn.weights_bf16(320, 320, "b2b0"))
    x1 = bf16(syn.features_bf16((n, 36, 36, 640), "b2b1"))
    w1 = bf16(syn.weights_bf16(640, 640, "b2b1"))
    sz0 = sphinx.load().sphinx_conv_workspace_size(n, 72, 72, 320, 320, 8)
    sz1 = sphinx.load().sphinx_conv_workspace_size(n, 36, 36, 640, 640, 8)
    ws0, ws0r = (torch.zeros(sz0, dtype=torch.uint8, device=dev) for _ in range(2))
    ws1, ws1r = (torch.zeros(sz1, dtype=torch.uint8, device=dev) for _ in range(2))
    for rnd in range(4):
        m0 = (rg.random((n, 9, 9)) < 0.3 + 0.1 * rnd).astype(np.uint8)
        m1 = (rg.random((n, 5, 5)) < 0.7 - 0.1 * rnd).astype(np.uint8)
        i0, c0, _ = gpu_compact(sphinx, m0, None, 0)
        i1, c1, _ = gpu_compact(sphinx, m1, None, 0)
        ya = [torch.zeros((n, 72, 72, 320), device=dev), torch.zeros((n, 36, 36, 640), device=dev)]
        yb = [torch.zeros_like(ya[0]), torch.zeros_like(ya[1])]
        sphinx.sphinx_sparse_conv3x3(x0, w0, None, ya[0], 8, i0, c0, workspace=ws0r)
        sphinx.sphinx_sparse_conv3x3(x1, w1, None, ya[1], 8, i1, c1, workspace=ws1r)
        sphinx.sphinx_conv_edge_plan(i1, c1, n, 36, 36, 8, 640, workspace=ws1)
        sphinx.sphinx_sparse_conv3x3(x0, w0, None, yb[0], 8, i0, c0, workspace=ws0, list_ready=True)
        sphinx.sphinx_sparse_conv3x3(x1, w1, None, yb[1], 8, i1, c1, workspace=ws1, reuse_plan=True,
                                     list_ready=True)
        torch.cuda.synchronize()
        for a, b in zip(ya, yb):
            assert np.array_equal(a.cpu().numpy().view(np.uint32), b.cpu().numpy().view(np.uint32)), rnd
