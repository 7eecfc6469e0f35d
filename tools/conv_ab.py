"""Per-level conv timing for same-box A/B of two library builds (run under gpurun):
    SPHINX_LIB=<path> python tools/conv_ab.py
168-frame maps at the three UNet levels, 25%/35%/45% clustered lists (the configs[3] step's
densities), default kernel choice; CUDA-graph replay of 20 launches, L2-warm."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18672_b200 as sp  # noqa: E402
import synthetic as syn  # noqa: E402


def main():
    lib = sp.load(os.environ["SPHINX_LIB"]) if os.environ.get("SPHINX_LIB") else sp.load()
    dev = torch.device("cuda", 0)
    out = {"lib": os.path.basename(os.environ.get("SPHINX_LIB", "libsphinx.so"))}
    for (h, c, d) in ((72, 320, 0.25), (36, 640, 0.35), (18, 1280, 0.45)):
        nf, b = 168, 8
        hb = -(-h // b)
        x = torch.from_numpy(syn.features_bf16((nf, h, h, c), "convab").view(np.int16)).view(torch.bfloat16).to(dev)
        w = torch.from_numpy(syn.weights_bf16(c, c, "convab").view(np.int16)).view(torch.bfloat16).to(dev)
        y = torch.zeros((nf, h, h, c), dtype=torch.bfloat16, device=dev)
        rg = syn.rng("convab-mask", h)
        m = np.stack([syn.choose_cells(rg, hb, hb, max(1, round(d * hb * hb)), "clustered") for _ in range(nf)])
        ids_np = np.flatnonzero(m.ravel()).astype(np.int32)
        ids = torch.from_numpy(ids_np).to(dev)
        cnt = torch.tensor([len(ids_np)], dtype=torch.int32, device=dev)
        ws = torch.zeros(int(lib.sphinx_conv_workspace_size(nf, h, h, c, c, b)), dtype=torch.uint8, device=dev)
        t = bench.graph_time(torch, lambda: sp.sphinx_sparse_conv3x3(x, w, None, y, b, ids, cnt, workspace=ws))
        out[f"L{h}x{c}"] = round(t, 5)
        del x, w, y, ws
        torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
