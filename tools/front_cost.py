"""Dev: how much of the step the front chain (mask, compaction, edge plans, noise, latent scatter)
leaves exposed: the step graph vs a graph of the same six convs alone (same order and flags, over
the lists the step just produced).  Same box, alternating, L2 flushed between replays.

    python tools/front_cost.py [configs2 configs3]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18672_b200 as sp  # noqa: E402
from paper_2511_18672_b200.step import RefinementStep  # noqa: E402


def convs_only(st):
    cfg, d = st.cfg, st.d
    src = [d[f"feat{l}"] for l in range(cfg.L)]
    prev = None
    for (l, j) in st.conv_order():
        dst = st.y[l] if j % 2 == 0 else st.z[l]
        sp.sphinx_sparse_conv3x3(src[l], d[f"w{l}{j}"], d[f"b{l}{j}"], dst, cfg.b, st.ids[l], st.cnt[l],
                                 workspace=st.ws[l], reuse_plan=True, list_ready=True,
                                 input_ready=(j == 0 or prev != (l, j - 1)))
        src[l] = dst
        prev = (l, j)


def capture(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    return g


def main():
    sp.load()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for name in (sys.argv[1:] or ["configs2", "configs3"]):
        st = RefinementStep(bench.step_config(bench.WORKLOADS[name]["means"]), bench.make_batch(name), dev, sp)
        g_step = capture(st.run)
        g_conv = capture(lambda: convs_only(st))
        ms = {"step": [], "convs": []}
        for _ in range(6):
            for k, g in (("step", g_step), ("convs", g_conv)):
                for _ in range(10):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    g.replay()
                    e1.record()
                    flush.fill_(1.0)
                    torch.cuda.synchronize()
                    ms[k].append(e0.elapsed_time(e1))
        r = {k: round(float(np.median(v)), 4) for k, v in ms.items()}
        r["front_exposed_ms"] = round(r["step"] - r["convs"], 4)
        print(json.dumps({name: r}), flush=True)
        del st, g_step, g_conv
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
