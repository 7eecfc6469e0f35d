"""Test-only stand-in for the binding's calls used by RefinementStep, computed by the CPU ORACLE
on CPU torch tensors.  It lets the multi-rank data plane (paper_2511_18672_b200.step: mask
slices, all-gather, LPT plan, compaction over assigned frames, owner gather) run under gloo on
CPU, where no GPU exists; its results are compared across world sizes, never against the GPU.
"""
import numpy as np
import torch

import oracle
import synthetic as syn

SELECT_ACTIVE, SELECT_INACTIVE_FRAMES, SELECT_ALL, SELECT_NOISE = 0, 1, 2, 3


def _np(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def make_klogic(thr, steps, fallback_k=0, k_max=40):
    return oracle.make_klogic(thr, steps, fallback_k, k_max)


def load():
    return None


def sphinx_block_mask(O, U, tau_u, tau_o, f, b, masks, counts, start, k):
    m, c = oracle.block_mask(_np(O), None if U is None else _np(U), None if tau_u is None else _np(tau_u),
                             tau_o, f, b, len(masks))
    for l, t in enumerate(masks):
        t.copy_(torch.from_numpy(m[l]))
    if counts is not None:
        counts.copy_(torch.from_numpy(c))
    if start is not None:
        kk = oracle.start_step(_np(start["q_reg"]), _np(start["c0"]), _np(start["c1"]), _np(start["t"]),
                               start["gamma"], start["logics"],
                               None if start.get("logic_id") is None else _np(start["logic_id"]))
        k.copy_(torch.from_numpy(kk))


def sphinx_compact_blocks_batch(jobs):
    for j in jobs:
        m = None if j["block_mask"] is None else _np(j["block_mask"])
        kk = None if j["start_step"] is None else _np(j["start_step"])
        ids = oracle.compact(m, kk, j["step_u"], j["select"], shape=j.get("shape"))
        j["block_ids"][:len(ids)] = torch.from_numpy(ids.astype(np.int32))
        j["count"].fill_(len(ids))


def sphinx_shard_plan(masks, channels, k, u, owner, world, rank, k_mine, rank_of, rank_load, pair, recv):
    """Host twin of the device plan (the rule of sphinx.h / dist.lpt_assign) on CPU tensors."""
    from paper_2511_18672_b200 import dist as sdist
    kk = _np(k)
    act = (kk >= 0) & (kk <= u)
    F = len(kk)
    cnt = np.stack([_np(m).reshape(F, -1).astype(np.int64).sum(1) * act for m in masks], 1)
    assign, load = sdist.lpt_assign(sdist.frame_costs(cnt, channels), world)
    ro = np.zeros(F, np.int64)
    for r, fr in enumerate(assign):
        ro[fr] = r
    own = _np(owner).astype(np.int64)
    pr = np.zeros((len(masks), world, world), np.int64)
    for l in range(len(masks)):
        np.add.at(pr[l], (ro, own), cnt[:, l])
    rank_of.copy_(torch.from_numpy(ro.astype(np.int32)))
    rank_load.copy_(torch.from_numpy(load.astype(np.int64)))
    pair.copy_(torch.from_numpy(pr.astype(np.int32)))
    k_mine.copy_(torch.from_numpy(np.where(ro == rank, kk, -1).astype(np.int32)))
    recv.copy_(torch.from_numpy((pr[:, :, rank].sum(1) - pr[:, rank, rank]).astype(np.int32)))


def sphinx_conv_edge_plan(*a, **k):
    pass


def sphinx_noise_inject(x0, eps, x_t, b, ids, cnt, step, abar):
    n = int(cnt.item())
    z = oracle.noise(_np(x0), _np(eps), _np(x_t).copy(), b, _np(ids)[:n], _np(step), _np(abar))
    x_t.copy_(torch.from_numpy(z.astype(np.float32)))


def sphinx_noise_inject_step(x0, eps, x_t, b, ids, cnt, start_step, u, abar):
    k = _np(start_step)
    step = np.where((k >= 0) & (k <= u), k, np.where(k > u, u + 1, -1)).astype(np.int32)
    sphinx_noise_inject(x0, eps, x_t, b, ids, cnt, torch.from_numpy(step), abar)


def sphinx_sparse_conv3x3(x, w, bias, y, b, ids, cnt, **kw):
    n = int(cnt.item())
    lst = _np(ids)[:n]
    yv, _ = oracle.conv3x3_blocks(_np(x), _np(w), None if bias is None else _np(bias), b, lst)
    listed = ~np.isnan(yv[..., 0])
    out = _np(y)
    out[listed] = syn.to_bf16_bits(yv[listed].astype(np.float32))


def sphinx_scatter_cached(src, cache, out, b, block_mask=None, start_step=None, step_u=0):
    r = oracle.scatter(_np(src), _np(cache), b, mask=_np(block_mask), k=_np(start_step), u=step_u)
    out.copy_(torch.from_numpy(np.ascontiguousarray(r)))


def _blocks(ids, cnt, shape, b):
    n, h, w, _ = shape
    hb, wb = -(-h // b), -(-w // b)
    for j, id_ in enumerate(ids[:cnt]):
        f, r = divmod(int(id_), hb * wb)
        by, bx = divmod(r, wb)
        ry, rx = min(b, h - by * b), min(b, w - bx * b)
        yield j, f, by * b, bx * b, ry, rx


def sphinx_gather_blocks(src, dst, b, ids, cnt, capacity=None):
    s, d = _np(src), _np(dst)
    for j, f, y0, x0, ry, rx in _blocks(_np(ids), int(cnt.item()), src.shape, b):
        d[j, :ry, :rx] = s[f, y0:y0 + ry, x0:x0 + rx]


def sphinx_scatter_blocks(src, out, b, ids, cnt, capacity=None):
    s, o = _np(src), _np(out)
    for j, f, y0, x0, ry, rx in _blocks(_np(ids), int(cnt.item()), out.shape, b):
        o[f, y0:y0 + ry, x0:x0 + rx] = s[j, :ry, :rx]
