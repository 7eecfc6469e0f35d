"""Guard-band (canary) tests: every kernel of the step and of the NEXT rows writes only inside its
output arrays.  Each output is a view into a larger buffer whose head and tail guard bands are
filled with a canary bit pattern; after the call the guards must be bit-identical.  (Inside the
outputs, "unlisted elements untouched" is checked by the parity tests.)  compute-sanitizer cannot
see these overruns: the caching allocator hands out sub-ranges of larger allocations."""
import numpy as np
import pytest

import oracle
import synthetic as syn

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
dev = "cuda"
G = 256  # guard elements on each side (keeps 16-byte alignment for every dtype)


class Guarded:
    """A contiguous output of `shape` inside a buffer with canary guards on both sides."""

    def __init__(self, shape, dtype, canary=0x5A):
        n = int(np.prod(shape))
        self.raw = torch.empty(n + 2 * G, dtype=dtype, device=dev)
        self.raw.view(torch.uint8).fill_(canary)
        self.t = self.raw[G:G + n].view(shape)
        self.canary = canary

    def fill(self, v):
        self.t.fill_(v)
        return self

    def check(self, what):
        torch.cuda.synchronize()
        b = self.raw.view(torch.uint8)
        es = self.raw.element_size()
        head, tail = b[:G * es], b[b.numel() - G * es:]
        assert bool((head == self.canary).all()), f"{what}: write before the output"
        assert bool((tail == self.canary).all()), f"{what}: write past the output"


def T(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return (t.to(dtype) if dtype is not None else t).to(dev)


def bf16(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(dev)


def _lists(rg, n, hb, wb, frac):
    m = (rg.random((n, hb, wb)) < frac).astype(np.uint8)
    ids = np.flatnonzero(m.ravel()).astype(np.int32)
    return m, ids


def test_canary_step_kernels(sphinx):
    rg = np.random.default_rng(11)
    n, hp, f, b, L = 3, 64 * 3, 8, 8, 3   # 24x24 level-0 map, 3 levels (24, 12, 6)
    O = rg.random((n, hp, hp)).astype(np.float32)
    U = rg.random((n, hp, hp)).astype(np.float32)
    tau = np.full(n, 0.9, np.float32)
    dims = oracle.level_dims(hp, hp, f, b, L)
    masks = [Guarded((n, hb, wb), torch.uint8) for (_, _, hb, wb) in dims]
    counts = Guarded((n, L), torch.int32)
    k = Guarded((n,), torch.int32)
    lg = sphinx.make_klogic(syn.SPEC_KLOGIC["thr"], syn.SPEC_KLOGIC["steps"])
    start = dict(q_reg=T(np.full(n, 61.0, np.float32)), c0=T(np.full(n, 60.0, np.float32)),
                 c1=T(np.full(n, 70.0, np.float32)), t=T(np.linspace(0, 1, n).astype(np.float32)), gamma=0.5,
                 logics=[lg])
    sphinx.sphinx_block_mask(T(O), T(U), T(tau), 0.5, f, b, [m.t for m in masks], counts.t, start, k.t)
    for i, m in enumerate(masks):
        m.check(f"block_mask level {i}")
    counts.check("active counts")
    k.check("start steps")
    # compaction (single and batched): ids beyond the count keep their values, guards intact
    hb = dims[0][2]
    ids = Guarded((n * hb * hb,), torch.int32).fill(-7)
    cnt = Guarded((1,), torch.int32)
    sphinx.sphinx_compact_blocks(masks[0].t, k.t, 40, sphinx.SELECT_ACTIVE, ids.t, cnt.t)
    ids.check("compact ids")
    cnt.check("compact count")
    c = int(cnt.t.item())
    assert bool((ids.t[c:] == -7).all()), "compaction wrote past its count"
    jobs, gs = [], []
    for l, (_, _, hbl, wbl) in enumerate(dims):
        gi, gc = Guarded((n * hbl * wbl,), torch.int32), Guarded((1,), torch.int32)
        jobs.append(dict(block_mask=masks[l].t, start_step=k.t, step_u=40, select=sphinx.SELECT_ACTIVE,
                         block_ids=gi.t, count=gc.t))
        gs += [(gi, f"batch ids {l}"), (gc, f"batch count {l}")]
    sphinx.sphinx_compact_blocks_batch(jobs)
    for g_, what in gs:
        g_.check(what)
    # noise (and the fused per-step pass) on the latent
    h0 = hp // f
    x0 = rg.standard_normal((n, h0, h0, 4)).astype(np.float32)
    eps = rg.standard_normal((n, h0, h0, 4)).astype(np.float32)
    abar = T(syn.abar_cosine(50))
    xt = Guarded((n, h0, h0, 4), torch.float32).fill(0.0)
    sphinx.sphinx_noise_inject(T(x0), T(eps), xt.t, b, ids.t, cnt.t, k.t, abar)
    xt.check("noise")
    xt2 = Guarded((n, h0, h0, 4), torch.float32).fill(0.0)
    sphinx.sphinx_noise_inject_step(T(x0), T(eps), xt2.t, b, ids.t, cnt.t, k.t, 40, abar)
    xt2.check("noise step")
    # latent scatter (out of place) and DDIM update
    out = Guarded((n, h0, h0, 4), torch.float32)
    sphinx.sphinx_scatter_cached(xt.t, T(x0), out.t, b, block_mask=masks[0].t, start_step=k.t, step_u=40)
    out.check("scatter_cached")
    zo = Guarded((n, h0, h0, 4), torch.float32).fill(0.0)
    sphinx.sphinx_ddim_step(xt.t, T(x0), zo.t, b, ids.t, cnt.t, 25, syn.abar_cosine(50))
    zo.check("ddim")


@pytest.mark.parametrize("h,c,blk,y_f32", [(24, 64, 8, False), (20, 64, 8, True), (12, 32, 4, False),
                                           (18, 256, 8, False)])
def test_canary_conv(sphinx, h, c, blk, y_f32):
    rg = np.random.default_rng(h * c)
    n = 3
    hb = -(-h // blk)
    _, ids_np = _lists(rg, n, hb, hb, 0.5)
    # the list's last block is a bottom-right edge block when the map is ragged
    ids_np = np.unique(np.concatenate([ids_np, [n * hb * hb - 1]])).astype(np.int32)
    x = bf16(syn.features_bf16((n, h, h, c), f"canary-{h}"))
    w = bf16(syn.weights_bf16(c, c, f"canary-{h}"))
    bias = T(syn.bias_f32(c, f"canary-{h}"))
    y = Guarded((n, h, h, c), torch.float32 if y_f32 else torch.bfloat16)
    ids, cnt = T(ids_np), T(np.array([len(ids_np)], np.int32))
    for variant in (0, sphinx.CONV_FORCE_PERTAP, sphinx.CONV_FORCE_HALO, sphinx.CONV_NO_SPLIT):
        if variant == 0 or blk == 8:
            sphinx.sphinx_sparse_conv3x3(x, w, bias, y.t, blk, ids, cnt, variant=variant)
            y.check(f"conv variant {variant}")
    # pointwise projection (q|k|v width: a ragged last C_out tile)
    wq = bf16(syn.linear_weights_bf16(3 * c, c, "canary-q"))
    yq = Guarded((n, h, h, 3 * c), torch.bfloat16)
    sphinx.sphinx_sparse_pointwise(x, wq, T(np.zeros(3 * c, np.float32)), yq.t, blk, ids, cnt)
    yq.check("pointwise")


def test_canary_gather_scatter_and_uncertainty(sphinx):
    rg = np.random.default_rng(5)
    n, h, c, b = 2, 36, 64, 8
    hb = -(-h // b)
    _, ids_np = _lists(rg, n, hb, hb, 0.6)
    ids, cnt = T(ids_np), T(np.array([len(ids_np)], np.int32))
    src = bf16(syn.features_bf16((n, h, h, c), "canary-g"))
    pay = Guarded((len(ids_np), b, b, c), torch.bfloat16)
    sphinx.sphinx_gather_blocks(src, pay.t, b, ids, cnt)
    pay.check("gather_blocks")
    out = Guarded((n, h, h, c), torch.bfloat16).fill(0.0)
    sphinx.sphinx_scatter_blocks(pay.t, out.t, b, ids, cnt)
    out.check("scatter_blocks")
    rgb = T(syn.rgb_frames(2, 53, 37, "canary"))
    U = Guarded((2, 53, 37), torch.float32)
    tau = Guarded((2,), torch.float32)
    sphinx.sphinx_uncertainty_map(rgb, U.t, tau.t)
    U.check("uncertainty map")
    tau.check("tau_u")


def test_canary_shard_plan(sphinx):
    """sphinx_shard_plan writes exactly its five outputs (k_mine, rank_of, load, pair, recv)."""
    rg = np.random.default_rng(5)
    F, world, u = 50, 4, 25
    masks = [T((rg.random((F, hb, hb)) < 0.3).astype(np.uint8)) for hb in (9, 5, 3)]
    k = T(rg.integers(-1, 40, F).astype(np.int32))
    owner = T((np.arange(F) * world // F).astype(np.int32))
    outs = dict(k_mine=Guarded((F,), torch.int32), rank_of=Guarded((F,), torch.int32),
                rank_load=Guarded((world,), torch.int64), pair=Guarded((3, world, world), torch.int32),
                recv=Guarded((3,), torch.int32))
    sphinx.sphinx_shard_plan(masks, [320, 640, 1280], k, u, owner, world, 1, **{k_: g.t for k_, g in outs.items()})
    for k_, g in outs.items():
        g.check(f"shard_plan {k_}")
