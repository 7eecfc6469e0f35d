"""Dev A/B: the configs[1] single-frame density sweep under the current env (conv mode knobs)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2511_18672_b200 as sp  # noqa: E402

torch.cuda.set_device(0)
out = bench.density_sweep(torch, sp, torch.device("cuda", 0), frames_list=(1,))
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("SPHINX")},
                  "rows": [(r["density"], r["sparse_ms"], r["speedup_vs_cudnn"]) for r in out[0]["rows"]],
                  "cudnn_ms": out[0]["dense_cudnn_ms"]}))
