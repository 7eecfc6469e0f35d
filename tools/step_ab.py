"""Same-box A/B of per-level conv kernel variants on the bench steps (run under gpurun):
default choice vs the per-tap path forced on some levels.  Outputs must agree within the conv bar
(different kernels sum in different orders); prints the median device step time of each.

    python tools/step_ab.py [configs2 configs3 ...]
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


def main():
    sp.load()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    P = sp.CONV_FORCE_PERTAP
    variants = {"default": None, "pertap_l0": [P, 0, 0], "pertap_l01": [P, P, 0], "pertap_all": [P, P, P]}
    for name in (sys.argv[1:] or ["configs2", "configs3"]):
        batch = bench.make_batch(name)
        steps, graphs = {}, {}
        for k, v in variants.items():
            cfg = bench.step_config(bench.WORKLOADS[name]["means"])
            cfg.conv_variant = v
            st = RefinementStep(cfg, batch, dev, sp)
            g, _ = bench.capture_step(torch, st, with_conv_events=False)
            steps[k], graphs[k] = st, g
        for k in variants:
            graphs[k].replay()
        torch.cuda.synchronize()
        for l in range(steps["default"].cfg.L):
            a = steps["default"].out(l).float()
            for k in variants:
                d = (steps[k].out(l).float() - a).abs().max().item()
                assert d <= 0.05 * a.abs().max().item(), (name, k, l, d)
        ms = {k: [] for k in variants}
        for _ in range(5):
            for k in variants:
                for _ in range(10):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    graphs[k].replay()
                    e1.record()
                    flush.fill_(1.0)
                    torch.cuda.synchronize()
                    ms[k].append(e0.elapsed_time(e1))
        print(json.dumps({name: {k: round(float(np.median(v)), 5) for k, v in ms.items()}}), flush=True)
        del steps, graphs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
