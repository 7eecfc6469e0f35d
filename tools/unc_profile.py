"""Dev tool: NEXT-2 uncertainty map on one 21-frame request (576x576) for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_18672_b200 as sp  # noqa: E402

dev = torch.device("cuda", 0)
n, hp = 21, 576
rgb = torch.rand((n, hp, hp, 3), device=dev, dtype=torch.float32)
U = torch.empty((n, hp, hp), device=dev, dtype=torch.float32)
tau = torch.empty((n,), device=dev, dtype=torch.float32)
for _ in range(3):
    sp.sphinx_uncertainty_map(rgb, U, tau)
torch.cuda.synchronize()
print("done")
