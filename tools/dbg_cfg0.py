import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2511_18672_b200 as sp
sp.load()
dev = torch.device("cuda:0")
n, h, c, b = 1, 16, 32, 4
x = torch.randn(n, h, h, c, device=dev).to(torch.bfloat16)
w = (torch.randn(c, 3, 3, c, device=dev) * 0.05).to(torch.bfloat16)
bias = torch.zeros(c, device=dev)
y = torch.zeros(n, h, h, c, device=dev)
ids = torch.arange(0, 16, 3, dtype=torch.int32, device=dev)
cnt = torch.tensor([ids.numel()], dtype=torch.int32, device=dev)
print("launch", flush=True)
sp.sphinx_sparse_conv3x3(x, w, bias, y, b, ids, cnt)
torch.cuda.synchronize()
print("ok", float(y.abs().sum()), flush=True)
