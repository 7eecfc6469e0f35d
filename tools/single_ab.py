"""Dev A/B: configs[1] (one 72x72x320 frame, block 8) conv time per kernel configuration.

    python -m paper_2511_18672_b200.build --trace
    SPHINX_LIB=paper_2511_18672_b200/libsphinx_trace.so python tools/single_ab.py

C_out tile width (dev knob SPHINX_BN of the trace build) x CTA group, over the bench's
clustered lists at 4..81 blocks; CUDA-graph replay of 20 launches, L2-warm (as bench.py's
density_sweep).  Prints one JSON line per configuration."""
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
    h, c, hb, nf = 72, 320, 9, 1
    x = torch.from_numpy(syn.features_bf16((nf, h, h, c), "sweep").view(np.int16)).view(torch.bfloat16).to(dev)
    w = torch.from_numpy(syn.weights_bf16(c, c, "sweep").view(np.int16)).view(torch.bfloat16).to(dev)
    y = torch.zeros((nf, h, h, c), dtype=torch.bfloat16, device=dev)
    ws = torch.zeros(int(lib.sphinx_conv_workspace_size(nf, h, h, c, c, 8)) * 4, dtype=torch.uint8, device=dev)
    lists = []
    for d in (0.05, 0.10, 0.25, 0.50, 1.0):
        rg = syn.rng("sweep-mask", nf, d)
        m = np.stack([syn.choose_cells(rg, hb, hb, round(d * 81), "clustered") for _ in range(nf)])
        ids_np = np.flatnonzero(m.ravel()).astype(np.int32)
        lists.append((torch.from_numpy(ids_np).to(dev), torch.tensor([len(ids_np)], dtype=torch.int32, device=dev)))
    for bn in (sys.argv[1:] or ["", "160", "128", "64", "32"]):
        for cg1 in (0, 1):
            if bn:
                os.environ["SPHINX_BN"] = bn
            else:
                os.environ.pop("SPHINX_BN", None)
            row = {"bn": bn or "default", "cg": 1 if cg1 else 2}
            for ids, cnt in lists:
                var = sp.CONV_FORCE_CG1 if cg1 else 0
                t = bench.graph_time(torch, lambda: sp.sphinx_sparse_conv3x3(x, w, None, y, 8, ids, cnt, workspace=ws,
                                                                             variant=var))
                row[str(int(cnt.item()))] = round(t * 1e3, 2)
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
