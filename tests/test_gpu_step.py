"""GPU parity of the WHOLE hot-path step in the launch configuration bench.py times:
paper_2511_18672_b200.step.RefinementStep, captured as a CUDA graph and replayed, against the
CPU oracle on the same seeded inputs, at two workloads:

* configs[2]: one 21-frame request (576x576 maps, UNet levels 72x72x320, 36x36x640,
  18x18x1280) -- every frame's masks, ids and latents; sampled conv blocks;
* configs[3]: 8 requests x 21 frames = 168 frames with request densities
  [5,10,25,50,75,25,10,5]% -- masks, counts, start steps, id lists and latents of the whole
  batch; convs on SURVEY 8(d)'s subsample: every listed block of request 0 plus every 8th
  listed block elsewhere (conv a), and every 64th (conv b, which needs conv a on its halo
  neighbourhood).

Bars: a1/a2 masks, counts, start steps and a3 id lists (L levels + inactive frames) bit-exact;
a4 noised latent within 1e-6 of |a x0| + |s eps| (R-3) on every written element; a5 first conv
of every level within 1e-3 sum|w x| + 1e-6 + 2^-8 |y| (bf16 output); the second conv (reading
the first one's bf16 output, cached values elsewhere) with the first conv's bound propagated
through |W|; a6 latent scatter: cache values bitwise, refined blocks within the noise bar.
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


@pytest.fixture(scope="module", params=["configs2", "configs3"])
def step_run(request, sphinx):
    from paper_2511_18672_b200.step import RefinementStep
    name = request.param
    dev = torch.device("cuda", 0)
    batch = bench.make_batch(name)
    cfg = bench.step_config(bench.WORKLOADS[name]["means"])
    st = RefinementStep(cfg, batch, dev, sphinx)
    g, _ = bench.capture_step(torch, st, with_conv_events=False)
    # the persistent buffers are pre-filled with the cache once; replay the captured step
    for l in range(cfg.L):
        st.y[l].copy_(st.d[f"cache{l}"])
        st.z[l].copy_(st.d[f"cache{l}"])
    st.lat_out.copy_(st.d["lat_cache"])
    g.replay()
    torch.cuda.synchronize()
    yield name, cfg, batch, st
    del g, st
    torch.cuda.empty_cache()


def _oracle_front(cfg, batch):
    kl = batch["klogic"]
    lg = oracle.make_klogic(kl["thr"], kl["steps"], kl["fallback_k"], kl["k_max"])
    masks, counts = oracle.block_mask(batch["O"], batch["U"], batch["tau_u"], cfg.tau_o, cfg.f, cfg.b, cfg.L)
    k = oracle.start_step(batch["q"], batch["c0"], batch["c1"], batch["t"], cfg.gamma, [lg], batch["lid"])
    return masks, counts, k


def test_step_masks_ids_start_steps_exact(step_run):
    name, cfg, batch, st = step_run
    masks, counts, k = _oracle_front(cfg, batch)
    for l in range(cfg.L):
        assert np.array_equal(st.masks[l].cpu().numpy(), masks[l])
        ids = oracle.compact(masks[l], k, cfg.u, oracle.SELECT_ACTIVE)
        c = int(st.cnt[l].item())
        assert np.array_equal(st.ids[l][:c].cpu().numpy(), ids)
    assert np.array_equal(st.counts.cpu().numpy(), counts)
    assert np.array_equal(st.k.cpu().numpy(), k)
    noise = oracle.compact(masks[0], k, cfg.u, oracle.SELECT_NOISE)
    assert np.array_equal(st.ids_noise[:int(st.cnt_noise.item())].cpu().numpy(), noise)
    if name == "configs3":  # the mixed densities reach the batch (8 requests, 5..75% means)
        d0 = masks[0].reshape(8, -1).mean(1)
        assert d0.min() < 0.12 and d0.max() > 0.6


def _block_px(ids, hb, b, shape):
    m = np.zeros(shape, bool)
    for id_ in ids:
        i, r = divmod(int(id_), hb * hb)
        by, bx = divmod(r, hb)
        m[i, by * b:by * b + b, bx * b:bx * b + b] = True
    return m


def test_step_noise_and_latent_scatter(step_run):
    name, cfg, batch, st = step_run
    masks, _, k = _oracle_front(cfg, batch)
    b, hb = cfg.b, cfg.hb[0]
    ids_a = oracle.compact(masks[0], k, cfg.u, oracle.SELECT_ACTIVE)
    ids_i = oracle.compact(None, k, cfg.u, oracle.SELECT_INACTIVE_FRAMES, shape=masks[0].shape)
    zt_gpu = st.zt.cpu().numpy().astype(np.float64)
    # Alg1 line 12 (active blocks at their start step k) then line 19 (inactive frames at u+1);
    # only the elements these lists write are compared
    zero = np.zeros(zt_gpu.shape, np.float32)
    z1 = oracle.noise(batch["x0"], batch["eps"], zero, b, ids_a, k, batch["abar"])
    step_u1 = np.full(cfg.n_frames, cfg.u + 1, np.int32)
    z2 = oracle.noise(batch["x0"], batch["eps"], z1.astype(np.float32), b, ids_i, step_u1, batch["abar"])
    touched = _block_px(ids_a, hb, b, zt_gpu.shape[:3]) | _block_px(ids_i, hb, b, zt_gpu.shape[:3])
    ab = batch["abar"].astype(np.float64)
    S = len(ab) - 1
    u_frame = np.where(k <= cfg.u, k, cfg.u + 1)
    a = np.sqrt(ab[np.clip(u_frame, 0, S)])[:, None, None, None]
    s = np.sqrt(1 - ab[np.clip(u_frame, 0, S)])[:, None, None, None]
    tol = 1e-6 * (np.abs(a * batch["x0"]) + np.abs(s * batch["eps"])) + 1e-12
    assert touched.sum() > 0
    err = np.abs(zt_gpu - z2)
    assert np.all(err[touched] <= tol[touched])
    # a6: refined latent blocks from this step, the latent cache elsewhere (bitwise)
    out = st.lat_out.cpu().numpy()
    active_px = _block_px(ids_a, hb, b, zt_gpu.shape[:3])
    assert np.array_equal(out[~active_px].view(np.uint32), batch["lat_cache"][~active_px].view(np.uint32))
    assert np.all(np.abs(out[active_px] - z2[active_px]) <= tol[active_px])


def _sample(name, cfg, l, ids, every):
    """configs[3]: every listed block of request 0 + every `every`-th listed block elsewhere
    (SURVEY 8(d)); configs[2]: first, middle, last listed block and one on the last block
    row/column."""
    hb = cfg.hb[l]
    if name == "configs3":
        fpb = hb * hb * cfg.frames_per_request
        r0 = ids[ids < fpb]
        rest = ids[ids >= fpb][::every]
        return np.unique(np.concatenate([r0 if every == 8 else r0[::8], rest])).astype(np.int32)
    pick = [ids[0], ids[len(ids) // 2], ids[-1]]
    edge = [i for i in ids if (i % (hb * hb)) // hb == hb - 1 or (i % (hb * hb)) % hb == hb - 1]
    if edge:
        pick.append(edge[len(edge) // 2])
    return np.unique(np.array(pick, np.int64)).astype(np.int32)


def _neighbourhood(samp, ids, hb):
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
    return np.array(sorted(need), np.int32)


@pytest.mark.parametrize("level", [0, 1, 2])
def test_step_convs_sampled(step_run, level):
    name, cfg, batch, st = step_run
    masks, _, k = _oracle_front(cfg, batch)
    b, hb = cfg.b, cfg.hb[level]
    ids = oracle.compact(masks[level], k, cfg.u, oracle.SELECT_ACTIVE)
    x, cache = batch[f"feat{level}"], batch[f"cache{level}"]
    w0, b0, w1, b1 = batch[f"w{level}0"], batch[f"b{level}0"], batch[f"w{level}1"], batch[f"b{level}1"]
    # conv a on its sample
    samp_a = _sample(name, cfg, level, ids, 8)
    ya, aa = oracle.conv3x3_blocks(x, w0, b0, b, samp_a)
    got_a = st.y[level].float().cpu().numpy().astype(np.float64)
    la = ~np.isnan(ya[..., 0])
    tol_a = 1e-3 * aa[la] + 1e-6 + 2.0 ** -8 * np.abs(ya[la])
    assert np.all(np.abs(got_a[la] - ya[la]) <= tol_a)
    # conv b on a smaller sample; it reads y = listed ? bf16(conv a) : cache, so the oracle runs
    # its own conv a on the halo neighbourhood (rounded as the GPU stores it) and propagates conv
    # a's bound through |W1|
    samp_b = _sample(name, cfg, level, ids, 64)
    need = _neighbourhood(samp_b, ids, hb)
    ya, aa = oracle.conv3x3_blocks(x, w0, b0, b, need)
    la = ~np.isnan(ya[..., 0])
    y_ref = np.where(la[..., None], ya, dec(cache))
    y_bits = cache.copy()
    y_bits[la] = oracle.bf16_rne(ya[la])
    E_y = np.where(la[..., None], 1e-3 * aa + 2.0 ** -8 * np.abs(y_ref) + 1e-6, 0.0)
    zb, ab_ = oracle.conv3x3_blocks(y_bits, w1, b1, b, samp_b)
    up = syn.to_bf16_bits((E_y * (1 + 2.0 ** -7)).astype(np.float32))
    w_abs = syn.to_bf16_bits(np.abs(dec(w1)).astype(np.float32))
    prop, _ = oracle.conv3x3_blocks(up, w_abs, None, b, samp_b)
    lb = ~np.isnan(zb[..., 0])
    got_b = st.z[level].float().cpu().numpy().astype(np.float64)
    tol_b = 1e-3 * ab_[lb] + prop[lb] + 1e-6 + 2.0 ** -8 * np.abs(zb[lb])
    assert np.all(np.abs(got_b[lb] - zb[lb]) <= tol_b), np.max(np.abs(got_b[lb] - zb[lb]) / tol_b)
    # unlisted pixels of both persistent buffers still hold the cache, bitwise
    listed = _block_px(ids, hb, b, got_a.shape[:3])
    for buf in (st.y[level], st.z[level]):
        v = buf.view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(v[~listed], cache[~listed])
