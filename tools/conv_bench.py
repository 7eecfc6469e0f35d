"""Microbenchmark of sphinx_sparse_conv3x3 (own kernel) vs cuDNN dense, per shape/density/CG.

    python tools/conv_bench.py [--cg 1 2] [--frames 21] [--reps 30]
Prints one JSON line per (level, density, cg).  L2-warm timing (back-to-back launches).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_18672_b200 as sp  # noqa: E402
import synthetic as syn  # noqa: E402


def timed(fn, reps):
    """Device time per launch: `reps` launches captured in one CUDA graph, replayed."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cg", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--frames", type=int, nargs="+", default=[21])
    ap.add_argument("--dens", type=float, nargs="+", default=[0.05, 0.1, 0.25, 0.5, 1.0])
    ap.add_argument("--levels", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--split", type=int, nargs="+", default=[0, 1])
    ap.add_argument("--halo", type=int, nargs="+", default=[1])
    a = ap.parse_args()
    sp.load()
    dev = torch.device("cuda")
    levels = [(72, 320), (36, 640), (18, 1280)]
    for nf in a.frames:
        for li in a.levels:
            h, c = levels[li]
            hb = -(-h // 8)
            bf = lambda bits: torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).to(dev)
            x = bf(syn.features_bf16((nf, h, h, c), f"mb{li}"))
            w = bf(syn.weights_bf16(c, c, f"mb{li}"))
            y = torch.zeros((nf, h, h, c), dtype=torch.bfloat16, device=dev)
            xn = x.permute(0, 3, 1, 2)
            wn = w.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
            t_cudnn = timed(lambda: torch.nn.functional.conv2d(xn, wn, padding=1), a.reps)
            sp.conv_workspace(c, dev, nf, h, h, 8)
            dense_flops = nf * h * h * 2 * 9 * c * c
            for d in a.dens:
                rg = syn.rng("mbmask", nf, li, d)
                m = np.stack([syn.choose_cells(rg, hb, hb, round(d * hb * hb), "clustered") for _ in range(nf)])
                ids_np = np.flatnonzero(m.ravel()).astype(np.int32)
                if len(ids_np) == 0:
                    continue
                r = ids_np % (hb * hb)
                px = int((np.minimum(8, h - (r // hb) * 8) * np.minimum(8, h - (r % hb) * 8)).sum())
                ids = torch.from_numpy(ids_np).to(dev)
                cnt = torch.tensor([len(ids_np)], dtype=torch.int32, device=dev)
                for cg in a.cg:
                  for split in a.split:
                   for halo in a.halo:
                    os.environ["SPHINX_CONV_HALO"] = str(halo)
                    os.environ["SPHINX_CONV_CG"] = str(cg)
                    os.environ["SPHINX_CONV_SPLIT"] = str(split)
                    t = timed(lambda: sp.sphinx_sparse_conv3x3(x, w, None, y, 8, ids, cnt), a.reps)
                    f = px * 2 * 9 * c * c
                    print(json.dumps({"frames": nf, "level": li, "shape": [h, c], "density": round(len(ids_np) / (nf * hb * hb), 3),
                                      "cg": cg, "split": split, "halo": halo, "ms": round(t, 5), "eff_tflops": round(f / t / 1e9, 1),
                                      "cudnn_ms": round(t_cudnn, 5), "cudnn_tflops": round(dense_flops / t_cudnn / 1e9, 1),
                                      "speedup_vs_cudnn": round(t_cudnn / t, 3)}), flush=True)


if __name__ == "__main__":
    main()
