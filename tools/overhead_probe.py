"""Fixed-overhead probe for sphinx_sparse_conv3x3: device time per launch (CUDA-graph
replay) for count = 0 and tiny counts, per CTA-group mode, vs an empty torch kernel."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_18672_b200 as sp  # noqa: E402
import synthetic as syn  # noqa: E402
from tools.conv_bench import timed  # noqa: E402

sp.load()
dev = torch.device("cuda")
bf = lambda bits: torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).to(dev)
z = torch.zeros(1, device=dev)
print(json.dumps({"empty_torch_fill_us": round(timed(lambda: z.fill_(1.0), 50) * 1e3, 2)}))
for (h, c) in [(72, 320), (18, 1280)]:
    x = bf(syn.features_bf16((1, h, h, c), "ov"))
    w = bf(syn.weights_bf16(c, c, "ov"))
    y = torch.zeros((1, h, h, c), dtype=torch.bfloat16, device=dev)
    hb = -(-h // 8)
    ids = torch.arange(hb * hb, dtype=torch.int32, device=dev)
    for cnt_v in (0, 1, 4):
        cnt = torch.tensor([cnt_v], dtype=torch.int32, device=dev)
        for cg in (1, 2):
            for split in (0, 1):
                os.environ["SPHINX_CONV_CG"] = str(cg)
                os.environ["SPHINX_CONV_SPLIT"] = str(split)
                t = timed(lambda: sp.sphinx_sparse_conv3x3(x, w, None, y, 8, ids, cnt), 50)
                print(json.dumps({"h": h, "c": c, "count": cnt_v, "cg": cg, "split": split, "us": round(t * 1e3, 2)}))
