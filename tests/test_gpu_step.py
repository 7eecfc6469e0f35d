"""GPU parity of the WHOLE hot-path step at BASELINE configs[2] size, in the launch configuration
bench.py times: bench.GpuStep on one 21-frame request (576x576 maps, UNet levels 72x72x320,
36x36x640, 18x18x1280), captured as a CUDA graph and replayed, against the CPU oracle on the same
seeded inputs.

* a1/a2 block masks, per-frame counts and start steps, a3 id lists (3 levels + inactive frames):
  bit-exact.
* a4 noised latent: within 1e-6 of |a x0| + |s eps| (R-3), every element.
* a5 the first conv of every level on sampled listed blocks: the conv bar (bf16 output:
  1e-3 sum|w x| + 1e-6 + 2^-8 |y|); the second conv (which reads the first one's bf16 output,
  cached values elsewhere) on the same samples with the first conv's bound propagated through
  |W|: 1e-3 sum|w y| + conv(|W|, E_y) with E_y = 1e-3 sum|w x| + 2^-8 |y| + 1e-6.
* a6 latent scatter: cache values bitwise; refined blocks within the noise bar.
"""
import numpy as np
import pytest

import bench
import oracle
import synthetic as syn

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def dec(bits):
    return syn.bf16_bits_to_f32(bits).astype(np.float64)


def bits_of(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.fixture(scope="module")
def step_run(sphinx):
    dev = torch.device("cuda", 0)
    req = bench.make_request("r0")
    st = bench.GpuStep(req, dev)
    g, _ = bench.capture_step(torch, st, with_conv_events=False)
    # the persistent buffers are pre-filled with the cache once; replay the captured step
    for l in range(3):
        st.y[l].copy_(st.d[f"cache{l}"])
        st.z[l].copy_(st.d[f"cache{l}"])
    g.replay()
    torch.cuda.synchronize()
    return req, st


def _oracle_front(req):
    lg = oracle.make_klogic(syn.SPEC_KLOGIC["thr"], syn.SPEC_KLOGIC["steps"])
    masks, counts = oracle.block_mask(req["O"], req["U"], req["tau_u"], 0.5, bench.F, bench.B, 3)
    k = oracle.start_step(req["q"], req["c0"], req["c1"], req["t"], bench.GAMMA, [lg], req["lid"])
    return masks, counts, k


def test_step_masks_ids_start_steps_exact(step_run):
    req, st = step_run
    masks, counts, k = _oracle_front(req)
    for l in range(3):
        assert np.array_equal(st.masks[l].cpu().numpy(), masks[l])
        ids = oracle.compact(masks[l], k, bench.U_STEP, oracle.SELECT_ACTIVE)
        c = int(st.cnt[l].item())
        assert np.array_equal(st.ids[l][:c].cpu().numpy(), ids)
    assert np.array_equal(st.counts.cpu().numpy(), counts)
    assert np.array_equal(st.k.cpu().numpy(), k)
    inact = oracle.compact(None, k, bench.U_STEP, oracle.SELECT_INACTIVE_FRAMES, shape=masks[0].shape)
    assert np.array_equal(st.ids_in[:int(st.cnt_in.item())].cpu().numpy(), inact)


def test_step_noise_and_latent_scatter(step_run):
    req, st = step_run
    masks, _, k = _oracle_front(req)
    ids_a = oracle.compact(masks[0], k, bench.U_STEP, oracle.SELECT_ACTIVE)
    ids_i = oracle.compact(None, k, bench.U_STEP, oracle.SELECT_INACTIVE_FRAMES, shape=masks[0].shape)
    zt_gpu = st.zt.cpu().numpy().astype(np.float64)
    # Alg1 line 12 (active blocks at their start step k) then line 19 (inactive frames at u+1);
    # only the elements these lists write are compared
    zero = np.zeros(zt_gpu.shape, np.float32)
    z1 = oracle.noise(req["x0"], req["eps"], zero, bench.B, ids_a, k, req["abar"])
    step_u1 = np.full(bench.N_FRAMES, bench.U_STEP + 1, np.int32)
    z2 = oracle.noise(req["x0"], req["eps"], z1.astype(np.float32), bench.B, ids_i, step_u1, req["abar"])
    # tolerance on the written elements (others are the GPU's own untouched values by construction)
    hb = masks[0].shape[1]
    touched = np.zeros(zt_gpu.shape[:3], bool)
    for ids in (ids_a, ids_i):
        for id_ in ids:
            i, r = divmod(int(id_), hb * hb)
            by, bx = divmod(r, hb)
            touched[i, by * 8:by * 8 + 8, bx * 8:bx * 8 + 8] = True
    ab = req["abar"].astype(np.float64)
    u_frame = np.where(k <= bench.U_STEP, k, bench.U_STEP + 1)
    a = np.sqrt(ab[np.clip(u_frame, 0, bench.S)])[:, None, None, None]
    s = np.sqrt(1 - ab[np.clip(u_frame, 0, bench.S)])[:, None, None, None]
    tol = 1e-6 * (np.abs(a * req["x0"]) + np.abs(s * req["eps"])) + 1e-12
    assert touched.sum() > 0
    err = np.abs(zt_gpu - z2)
    assert np.all(err[touched] <= tol[touched])
    # a6: refined latent blocks from this step, the latent cache elsewhere (bitwise)
    out = st.lat_out.cpu().numpy()
    active_px = np.zeros(zt_gpu.shape[:3], bool)
    for id_ in ids_a:
        i, r = divmod(int(id_), hb * hb)
        by, bx = divmod(r, hb)
        active_px[i, by * 8:by * 8 + 8, bx * 8:bx * 8 + 8] = True
    assert np.array_equal(out[~active_px].view(np.uint32), req["lat_cache"][~active_px].view(np.uint32))
    assert np.all(np.abs(out[active_px] - z2[active_px]) <= tol[active_px])


def _sample(ids, hb, m=4):
    """First, middle, last listed block and one block on the last block row/column if any."""
    pick = [ids[0], ids[len(ids) // 2], ids[-1]]
    edge = [i for i in ids if (i % (hb * hb)) // hb == hb - 1 or (i % (hb * hb)) % hb == hb - 1]
    if edge:
        pick.append(edge[len(edge) // 2])
    return np.unique(np.array(pick[:m], np.int64)).astype(np.int32)


@pytest.mark.parametrize("level", [0, 1, 2])
def test_step_convs_sampled(step_run, level):
    req, st = step_run
    masks, _, k = _oracle_front(req)
    h, c = bench.LEVELS[level]
    hb = masks[level].shape[1]
    ids = oracle.compact(masks[level], k, bench.U_STEP, oracle.SELECT_ACTIVE)
    samp = _sample(ids, hb)
    x, cache = req[f"feat{level}"], req[f"cache{level}"]
    w0, b0, w1, b1 = req[f"w{level}0"], req[f"b{level}0"], req[f"w{level}1"], req[f"b{level}1"]
    # conv a on the samples and on every listed block in their 3x3 block neighbourhood (halo of b)
    listed = set(int(i) for i in ids)
    need = set()
    for id_ in samp:
        n, r = divmod(int(id_), hb * hb)
        by, bx = divmod(r, hb)
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                yy, xx = by + dy, bx + dx
                if 0 <= yy < hb and 0 <= xx < hb and (n * hb + yy) * hb + xx in listed:
                    need.add((n * hb + yy) * hb + xx)
    need = np.array(sorted(need), np.int32)
    ya, aa = oracle.conv3x3_blocks(x, w0, b0, bench.B, need)
    got_a = st.y[level].float().cpu().numpy().astype(np.float64)
    la = ~np.isnan(ya[..., 0])
    tol_a = 1e-3 * aa[la] + 1e-6 + 2.0 ** -8 * np.abs(ya[la])
    assert np.all(np.abs(got_a[la] - ya[la]) <= tol_a)
    # conv b reads y = listed ? bf16(conv a) : cache; the oracle uses its own conv a (rounded as the
    # GPU stores it) and the bound of conv a propagated through |W1|
    y_ref = np.where(la[..., None], ya, dec(cache))
    y_bits = cache.copy()
    y_bits[la] = oracle.bf16_rne(ya[la])
    E_y = np.where(la[..., None], 1e-3 * aa + 2.0 ** -8 * np.abs(y_ref) + 1e-6, 0.0)
    zb, ab_ = oracle.conv3x3_blocks(y_bits, w1, b1, bench.B, samp)
    up = syn.to_bf16_bits((E_y * (1 + 2.0 ** -7)).astype(np.float32))
    w_abs = syn.to_bf16_bits(np.abs(dec(w1)).astype(np.float32))
    prop, _ = oracle.conv3x3_blocks(up, w_abs, None, bench.B, samp)
    lb = ~np.isnan(zb[..., 0])
    got_b = st.z[level].float().cpu().numpy().astype(np.float64)
    tol_b = 1e-3 * ab_[lb] + prop[lb] + 1e-6 + 2.0 ** -8 * np.abs(zb[lb])
    assert np.all(np.abs(got_b[lb] - zb[lb]) <= tol_b), np.max(np.abs(got_b[lb] - zb[lb]) / tol_b)
