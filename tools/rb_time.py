"""Dev tool: graph-timed NEXT-3 block, its GN part and one plain conv per level (L2-warm, 20
replays), printing one JSON line.  Package chosen by sys.path (A/B of builds: PYTHONPATH)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_18672_b200 as sp  # noqa: E402
import synthetic as syn  # noqa: E402

LEVELS = [(72, 320), (36, 640), (18, 1280)]
n, b, G = 21, 8, syn.GN_GROUPS
dev = torch.device("cuda", 0)
bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)


def gtime(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    return sorted(ts)[2]


res = {"pkg": os.path.dirname(sp.__file__)}
for l, (h, c) in enumerate(LEVELS):
    hb = -(-h // b)
    x = bf(syn.features_bf16((n, h, h, c), "p"))
    w1, w2 = bf(syn.weights_bf16(c, c, "p1")), bf(syn.weights_bf16(c, c, "p2"))
    b1, b2 = (torch.from_numpy(syn.bias_f32(c, t)).to(dev) for t in ("p1", "p2"))
    gn1 = tuple(torch.from_numpy(a).to(dev) for a in syn.gn_affine_f32(c, "p1"))
    gn2 = tuple(torch.from_numpy(a).to(dev) for a in syn.gn_affine_f32(c, "p2"))
    hbuf, y, a = torch.zeros_like(x), torch.zeros_like(x), torch.zeros_like(x)
    xs, hs = sp.gn_stats_buffer(n, h, h, G, b, dev), sp.gn_stats_buffer(n, h, h, G, b, dev)
    rg = syn.rng("rbprof", l)
    m = np.stack([syn.choose_cells(rg, hb, hb, round(0.25 * hb * hb), "clustered") for _ in range(n)])
    ids = torch.from_numpy(np.flatnonzero(m.ravel()).astype(np.int32)).to(dev)
    cnt = torch.tensor([ids.numel()], dtype=torch.int32, device=dev)
    all_ids = torch.arange(n * hb * hb, dtype=torch.int32, device=dev)
    all_cnt = torch.tensor([n * hb * hb], dtype=torch.int32, device=dev)

    def block(i=ids, k=cnt):
        sp.sphinx_sparse_resblock(x, w1, b1, w2, b2, gn1, gn2, G, syn.GN_EPS, hbuf, xs, hs, y, a, b, i, k)
    block(all_ids, all_cnt)
    res[f"l{l}_block_us"] = round(gtime(block) * 1e3, 1)
    res[f"l{l}_gn_us"] = round(gtime(lambda: (sp.sphinx_gn_block_stats(x, G, b, ids, cnt, xs),
                                              sp.sphinx_gn_silu(x, xs, *gn1, syn.GN_EPS, G, b, ids, cnt, a))) * 1e3, 1)
    res[f"l{l}_conv_us"] = round(gtime(lambda: sp.sphinx_sparse_conv3x3(a, w1, b1, hbuf, b, ids, cnt)) * 1e3, 1)
print(json.dumps(res), flush=True)
