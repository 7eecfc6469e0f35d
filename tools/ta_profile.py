"""Dev tool: one level's NEXT-4 temporal block (full step, then 2 partial steps) for ncu.
    python tools/ta_profile.py [level]"""
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
n, b, T = 21, 8, 21
hb = -(-h // b)
dev = torch.device("cuda", 0)
bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
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
for _ in range(2):
    sp.sphinx_temporal_block(x, wq, None, wo, None, c // 64, T, qkv, o, y, b, ids, cnt)
torch.cuda.synchronize()
print("done", ids.numel())
