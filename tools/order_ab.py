"""Same-box A/B of the step's conv launch order (run under gpurun): level by level vs the
interleaved anti-diagonal order (RefinementStep.conv_order).  Outputs must be bitwise equal
(the order changes no arithmetic); prints the median device step time of each, alternating
A and B rounds so clock drift hits both.

    python tools/order_ab.py [configs2 configs3 ...]
    AB_KNOB=fused_compaction python tools/order_ab.py ...   # another boolean StepConfig knob
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
    # SPHINX_LIB: time another build of the library (same-box A/B of compile-time variants)
    sp.load(os.environ["SPHINX_LIB"]) if os.environ.get("SPHINX_LIB") else sp.load()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    res = {}
    knob = os.environ.get("AB_KNOB", "interleave_levels")
    for name in (sys.argv[1:] or ["configs2", "configs3"]):
        batch = bench.make_batch(name)
        steps, graphs = {}, {}
        for il in (False, True):
            cfg = bench.step_config(bench.WORKLOADS[name]["means"])
            setattr(cfg, knob, il)
            st = RefinementStep(cfg, batch, dev, sp)
            g, _ = bench.capture_step(torch, st, with_conv_events=False)
            steps[il], graphs[il] = st, g
        for il in (False, True):
            graphs[il].replay()
        torch.cuda.synchronize()
        for l in range(steps[True].cfg.L):
            a = steps[False].out(l).view(torch.int16)
            b = steps[True].out(l).view(torch.int16)
            assert torch.equal(a, b), (name, l)
        assert torch.equal(steps[False].lat_out, steps[True].lat_out)
        ms = {False: [], True: []}
        for _ in range(6):
            for il in (False, True):
                for _ in range(10):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    graphs[il].replay()
                    e1.record()
                    flush.fill_(1.0)
                    torch.cuda.synchronize()
                    ms[il].append(e0.elapsed_time(e1))
        if knob == "interleave_levels":
            res[name] = {"level_order_ms": float(np.median(ms[False])), "interleaved_ms": float(np.median(ms[True])),
                         "order": steps[True].conv_order()}
        else:
            res[name] = {f"{knob}=False_ms": float(np.median(ms[False])), f"{knob}=True_ms": float(np.median(ms[True]))}
        print(json.dumps({name: res[name]}), flush=True)
        del steps, graphs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
