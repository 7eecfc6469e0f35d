"""Dev tool: time sphinx_temporal_attention per level under staging variants (SPHINX_TA_NBUF,
SPHINX_TA_THREADS), one process, CUDA graphs of 20 calls; outputs checked bit-identical to the
default.    python tools/ta_ab.py"""
import os
import sys

import numpy as np
import torch

sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_18672_b200 as sp  # noqa: E402
import synthetic as syn  # noqa: E402

LEVELS = [(72, 320), (36, 640), (18, 1280)]
VARIANTS = {0: [(None, None, None)], 1: [(None, None, None)], 2: [(None, None, None)]}
if os.environ.get("TA_AB_TMAP"):
    VARIANTS = {0: [(None, None, None), ("notmap", None, None)], 1: [(None, None, None), ("notmap", None, None)],
                2: [(None, None, None), ("tmap", None, None)]}
if os.environ.get("TA_AB_HG"):
    VARIANTS = {0: [(None, None, None)], 1: [(None, None, None), ("hg5", None, None)],
                2: [(None, None, None), ("hg0", None, None), ("hg10", None, None)]}
if os.environ.get("TA_AB_PPU"):
    VARIANTS = {0: [(None, None, None), ("ppu2", None, None), ("ppu2", 256, None), ("ppu2", None, 0)],
                1: [(None, None, None)], 2: [(None, None, None)]}
if os.environ.get("TA_AB_ALL"):
    VARIANTS = {0: [(None, None, None), (None, None, 0), (1, 256, 0)],
                1: [(None, None, None), (None, None, 0), (1, 256, 0)],
                2: [(None, None, None), (None, None, 1)]}
dev = torch.device("cuda", 0)
n, b, T = 21, 8, 21
bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
for l, (h, c) in enumerate(LEVELS):
    hb = -(-h // b)
    x = bf(syn.features_bf16((n, h, h, c), "t"))
    wq, wo = bf(syn.linear_weights_bf16(3 * c, c, "tq", 0.5)), bf(syn.linear_weights_bf16(c, c, "to"))
    qkv = torch.zeros((n, h, h, 3 * c), dtype=torch.bfloat16, device=dev)
    o, y = torch.zeros_like(x), torch.zeros_like(x)
    rg = syn.rng("taprof", l)
    m = np.stack([syn.choose_cells(rg, hb, hb, round(0.25 * hb * hb), "clustered") for _ in range(n)])
    ids = torch.from_numpy(np.flatnonzero(m.ravel()).astype(np.int32)).to(dev)
    cnt = torch.tensor([ids.numel()], dtype=torch.int32, device=dev)
    all_ids = torch.arange(n * hb * hb, dtype=torch.int32, device=dev)
    all_cnt = torch.tensor([n * hb * hb], dtype=torch.int32, device=dev)
    sp.sphinx_temporal_block(x, wq, None, wo, None, c // 64, T, qkv, o, y, b, all_ids, all_cnt)
    ws = sp.attn_workspace(n, h, h, T, b, dev) if hasattr(sp, "attn_workspace") else None
    ref = None
    for nb, th, pm in VARIANTS[l]:
        os.environ.pop("SPHINX_TA_PPU", None)
        os.environ.pop("SPHINX_TA_TMAP", None)
        os.environ.pop("SPHINX_TA_HGROUP", None)
        if isinstance(nb, str) and nb.startswith("hg"):
            os.environ["SPHINX_TA_HGROUP"] = nb[2:]
            nb = None
        if nb in ("tmap", "notmap"):
            os.environ["SPHINX_TA_TMAP"] = "1" if nb == "tmap" else "0"
            nb = None
        if nb == "ppu2":
            os.environ["SPHINX_TA_PPU"] = "2"
            nb = None
        for k, v in (("SPHINX_TA_NBUF", nb), ("SPHINX_TA_THREADS", th), ("SPHINX_TA_STREAM", pm)):
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = str(v)
        o.zero_()
        call = lambda: sp.sphinx_temporal_attention(qkv, o, c // 64, T, b, ids, cnt)
        call()
        torch.cuda.synchronize()
        got = o.clone()
        if ref is None:
            ref = got
        same = bool(torch.equal(got.view(torch.int16), ref.view(torch.int16)))
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            call()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    call()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 20 * 1e3)
        print(f"level {l} nbuf={nb} threads={th} stream={pm}: {min(ts):.1f} us (median {sorted(ts)[2]:.1f}) same={same}",
              flush=True)
