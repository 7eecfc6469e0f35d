"""Dev tool: one level's NEXT-3 ResNet block (full step, then 3 partial steps) for ncu.
    python tools/rb_profile.py [level]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_18672_b200 as sp  # noqa: E402
import synthetic as syn  # noqa: E402

LEVELS = [(72, 320), (36, 640), (18, 1280)]
l = int(sys.argv[1]) if len(sys.argv) > 1 else 0
h, c = LEVELS[l]
n, b, G = 21, 8, syn.GN_GROUPS
hb = -(-h // b)
dev = torch.device("cuda", 0)
bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
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
sp.sphinx_sparse_resblock(x, w1, b1, w2, b2, gn1, gn2, G, syn.GN_EPS, hbuf, xs, hs, y, a, b, all_ids, all_cnt)
for _ in range(3):
    sp.sphinx_sparse_resblock(x, w1, b1, w2, b2, gn1, gn2, G, syn.GN_EPS, hbuf, xs, hs, y, a, b, ids, cnt)
torch.cuda.synchronize()
print("done", ids.numel())
