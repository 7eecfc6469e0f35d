"""ncu probe: one sphinx_uncertainty_map call on 21 x 576 x 576 RGB (after a warm-up)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_18672_b200 as sp  # noqa: E402

sp.load()
rgb = torch.rand((21, 576, 576, 3), device="cuda")
U = torch.empty((21, 576, 576), device="cuda")
tau = torch.empty((21,), device="cuda")
for _ in range(2):
    sp.sphinx_uncertainty_map(rgb, U, tau)
torch.cuda.synchronize()
