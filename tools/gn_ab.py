"""Dev A/B (dev build libsphinx_trace.so, SPHINX_GN_RG): NEXT-3 GroupNorm stage (block stats +
finalize + GN/SiLU) at the three UNet levels, 21 frames, 25% / 40% / 45% clustered lists; CUDA-graph
replay, L2-warm.   python -m paper_2511_18672_b200.build --trace && python tools/gn_ab.py"""
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
    sp.load(os.path.join(ROOT, "paper_2511_18672_b200", "libsphinx_trace.so"))
    dev = torch.device("cuda", 0)
    for (h, c, d) in ((72, 320, 0.25), (36, 640, 0.40), (18, 1280, 0.45)):
        n, b = 21, 8
        hb = -(-h // b)
        x = torch.from_numpy(syn.features_bf16((n, h, h, c), "gnab").view(np.int16)).view(torch.bfloat16).to(dev)
        g1, be1 = (torch.from_numpy(a).to(dev) for a in syn.gn_affine_f32(c, "gnab"))
        a = torch.empty_like(x)
        xs = sp.gn_stats_buffer(n, h, h, syn.GN_GROUPS, b, dev)
        rg = syn.rng("gnab-mask", h)
        m = np.stack([syn.choose_cells(rg, hb, hb, max(1, round(d * hb * hb)), "clustered") for _ in range(n)])
        ids_np = np.flatnonzero(m.ravel()).astype(np.int32)
        ids, cnt = torch.from_numpy(ids_np).to(dev), torch.tensor([len(ids_np)], dtype=torch.int32, device=dev)
        all_ids = torch.arange(n * hb * hb, dtype=torch.int32, device=dev)
        all_cnt = torch.tensor([n * hb * hb], dtype=torch.int32, device=dev)
        sp.sphinx_gn_block_stats(x, syn.GN_GROUPS, b, all_ids, all_cnt, xs)
        res = {}
        for r in ("default", "1", "2", "5", "10"):
            if r == "default":
                os.environ.pop("SPHINX_GN_RG", None)
            else:
                os.environ["SPHINX_GN_RG"] = r
            f = lambda: (sp.sphinx_gn_block_stats(x, syn.GN_GROUPS, b, ids, cnt, xs),
                         sp.sphinx_gn_silu(x, xs, g1, be1, syn.GN_EPS, syn.GN_GROUPS, b, ids, cnt, a))
            res[r] = round(bench.graph_time(torch, f), 5)
        os.environ.pop("SPHINX_GN_RG", None)
        print(json.dumps({"level": f"{h}x{c}", "blocks": len(ids_np), "gn_stage_ms": res}), flush=True)


if __name__ == "__main__":
    main()
