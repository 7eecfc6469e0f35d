"""Dev tool: per-CTA timelines of conv launches from the trace build (libsphinx_trace.so).

    python -m paper_2511_18672_b200.build --trace
    python tools/conv_trace.py step [configs2|configs3]   # the bench step's six convs
    python tools/conv_trace.py pointwise                  # NEXT-4 q|k|v projections (3 levels)
    python tools/conv_trace.py single                     # configs[1]: one 72x72x320 frame

The trace build records per CTA (globaltimer, ns): entry, after pdl_wait, first MMA, last MMA
commit, epilogue done, exit, chunks issued, split-K park / rendezvous / reduce, TMEM drain
durations.  Printed relative to the earliest entry: launch skew, prologue, fill, main loop vs
the ideal, drain and tail.  Timings also come from the release build in a separate process
(`time` lines: CUDA-graph replay of 20 launches, L2-warm).
"""
import ctypes
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def show(lib, sms, title):
    buf = (ctypes.c_ulonglong * (sms * 24))()
    assert lib.sphinx_debug_conv_trace(buf, sms) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(sms, 24).astype(np.int64)
    live = a[:, 0] > 0
    a = a[live]
    if not len(a):
        print(f"{title}: no trace")
        return
    t0 = a[:, 0].min()
    rel = lambda c: (a[:, c] - t0) / 1e3  # us
    lead = a[:, 2] > 0
    chunks = a[lead, 6]
    print(f"{title}: {live.sum()} CTAs, kernel span {(a[:, 5].max() - t0) / 1e3:.1f} us")
    for name, c in (("entry", 0), ("after pdl_wait", 1), ("setup done", 15), ("first A issued", 8),
                    ("first B issued", 9), ("first A full", 10), ("first MMA", 2), ("last MMA", 3),
                    ("last acc ready", 11), ("epilogue done", 4), ("exit", 5), ("B producer done", 7),
                    ("split parked", 16), ("split rendezvous", 17), ("split reduced", 18)):
        v = rel(c)[a[:, c] > 0]
        if len(v):
            print(f"   {name:16s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f}")
    nt_ = np.maximum(a[:, 12], 1)
    print(f"   epilogue tiles med {np.median(a[:, 12]):.0f}; TMEM drain per tile med "
          f"{np.median(a[:, 13] / nt_) / 1e3:.2f} us, last tile med {np.median(a[:, 14]) / 1e3:.2f} us; "
          f"last acc -> epilogue done per CTA med {np.median((a[:, 4] - a[:, 11]) / 1e3):.2f} us")
    w = a[:, 20:24].astype(np.float64) / 1e3
    ml = w[:, :3].sum(1) > 0  # MMA-issuing (leader) CTAs
    if ml.any():
        print(f"   waits per leader CTA med (us): MMA on operands {np.median(w[ml, 0]):.2f}, MMA on free "
              f"accumulator {np.median(w[ml, 1]):.2f}, MMA on A region {np.median(w[ml, 2]):.2f}; epilogue on "
              f"accumulator (all CTAs) {np.median(w[:, 3]):.2f}")
    if lead.any():
        mm = (a[lead, 3] - a[lead, 2]) / 1e3
        print(f"   main loop per leader: med {np.median(mm):.2f} us, chunks med {np.median(chunks):.0f} "
              f"(min {chunks.min()}, max {chunks.max()}), us/chunk med {np.median(mm / np.maximum(chunks, 1)):.3f}")


def pointwise_inputs(torch, dev, level):
    import synthetic as syn
    h, c = [(72, 320), (36, 640), (18, 1280)][level]
    nf, b = 21, 8
    hb = -(-h // b)
    x = torch.from_numpy(syn.features_bf16((nf, h, h, c), "pwtrace").view(np.int16)).view(torch.bfloat16).to(dev)
    w = torch.from_numpy(syn.linear_weights_bf16(3 * c, c, "pwtrace").view(np.int16)).view(torch.bfloat16).to(dev)
    bias = torch.zeros(3 * c, dtype=torch.float32, device=dev)
    y = torch.zeros((nf, h, h, 3 * c), dtype=torch.bfloat16, device=dev)
    rg = syn.rng("pwtrace-mask", level)
    n_act = max(1, round(0.25 * hb * hb)) if level == 0 else max(1, round(0.4 * hb * hb))
    m = np.stack([syn.choose_cells(rg, hb, hb, n_act, "clustered") for _ in range(nf)])
    ids_np = np.flatnonzero(m.ravel()).astype(np.int32)
    ids = torch.from_numpy(ids_np).to(dev)
    cnt = torch.tensor([len(ids_np)], dtype=torch.int32, device=dev)
    px = sum(min(b, h - (i % (hb * hb)) // hb * b) * min(b, h - (i % hb) * b) for i in ids_np)
    return x, w, bias, y, ids, cnt, px, c


def run_pointwise(trace):
    import torch
    import paper_2511_18672_b200 as sp
    lib = sp.load(os.path.join(ROOT, "paper_2511_18672_b200", "libsphinx_trace.so" if trace else "libsphinx.so"))
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    launch = 0
    for level in range(3):
        x, w, bias, y, ids, cnt, px, c = pointwise_inputs(torch, dev, level)
        f = lambda: sp.sphinx_sparse_pointwise(x, w, bias, y, 8, ids, cnt)
        if trace:
            for _ in range(2):
                f()
                launch += 1
            torch.cuda.synchronize()
            lib.sphinx_debug_conv_trace_reset()
            os.environ["SPHINX_TRACE_LAUNCH"] = str(launch)
            f()
            launch += 1
            torch.cuda.synchronize()
            show(lib, sms, f"pointwise level {level} ({len(ids)} blocks, C {c} -> {3 * c})")
            if level == 0 and "SPHINX_DBG" not in os.environ:
                os.environ["SPHINX_DBG"] = "1"  # timing probe: no epilogue stores
                lib.sphinx_debug_conv_trace_reset()
                os.environ["SPHINX_TRACE_LAUNCH"] = str(launch)
                f()
                launch += 1
                torch.cuda.synchronize()
                show(lib, sms, f"pointwise level 0 WITHOUT epilogue stores (probe)")
                for dbg, what in (("4", "WITHOUT TMEM drain"), ("8", "with wait timers"),
                                  ("12", "WITHOUT TMEM drain, with wait timers"),
                                  ):
                    os.environ["SPHINX_DBG"] = dbg
                    lib.sphinx_debug_conv_trace_reset()
                    os.environ["SPHINX_TRACE_LAUNCH"] = str(launch)
                    f()
                    launch += 1
                    torch.cuda.synchronize()
                    show(lib, sms, f"pointwise level 0 {what} (probe)")
                del os.environ["SPHINX_DBG"]
                import bench
                os.environ["SPHINX_TRACE_LAUNCH"] = "-1"
                for bn in ("160", "256", "128"):  # dev build: C_out tile width A/B
                    for tmay in (True, False):
                        os.environ["SPHINX_BN"] = bn
                        if not tmay:
                            os.environ["SPHINX_NO_TMA_Y"] = "1"
                        t = bench.graph_time(torch, f)
                        print(json.dumps({"time": f"pointwise level 0, BN {bn}, TMA-store {tmay} (dev build)",
                                          "ms": round(t, 5)}))
                        os.environ.pop("SPHINX_NO_TMA_Y", None)
                        del os.environ["SPHINX_BN"]
        else:
            import bench
            t = bench.graph_time(torch, f)
            fl = px * 2 * c * 3 * c
            print(json.dumps({"time": f"pointwise level {level}", "blocks": int(cnt.item()), "ms": round(t, 5),
                              "tflops": round(fl / t / 1e9, 1)}), flush=True)


def run_single(trace, nf=1):
    """configs[1]: one 72x72x320 frame (nf = 21: the sweep's 21-frame variant), 3x3 conv, the
    density sweep's lists (default kernel choice; dev build: variant flags A/B)."""
    import torch
    import paper_2511_18672_b200 as sp
    import synthetic as syn
    import bench
    lib = sp.load(os.path.join(ROOT, "paper_2511_18672_b200", "libsphinx_trace.so" if trace else "libsphinx.so"))
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    h, c = 72, 320
    x = torch.from_numpy(syn.features_bf16((nf, h, h, c), "sweep").view(np.int16)).view(torch.bfloat16).to(dev)
    w = torch.from_numpy(syn.weights_bf16(c, c, "sweep").view(np.int16)).view(torch.bfloat16).to(dev)
    y = torch.zeros((nf, h, h, c), dtype=torch.bfloat16, device=dev)
    ws = torch.zeros(int(lib.sphinx_conv_workspace_size(nf, h, h, c, c, 8)), dtype=torch.uint8, device=dev)
    launch = 0
    for d in (0.05, 0.10, 0.25, 0.50, 1.0):
        rg = syn.rng("sweep-mask", nf, d)
        m = np.stack([syn.choose_cells(rg, 9, 9, round(d * 81), "clustered") for _ in range(nf)])
        ids_np = np.flatnonzero(m.ravel()).astype(np.int32)
        ids = torch.from_numpy(ids_np).to(dev)
        cnt = torch.tensor([len(ids_np)], dtype=torch.int32, device=dev)
        f = lambda: sp.sphinx_sparse_conv3x3(x, w, None, y, 8, ids, cnt, workspace=ws)
        if trace:
            f()
            launch += 1
            torch.cuda.synchronize()
            lib.sphinx_debug_conv_trace_reset()
            os.environ["SPHINX_TRACE_LAUNCH"] = str(launch)
            f()
            launch += 1
            torch.cuda.synchronize()
            show(lib, sms, f"{nf} frame(s), {len(ids_np)} blocks")
            os.environ["SPHINX_TRACE_LAUNCH"] = "-1"
            for name, fl in (("default", 0), ("no split", sp.CONV_NO_SPLIT), ("no stream-K", sp.CONV_NO_STREAMK),
                             ("force stream-K", sp.CONV_FORCE_STREAMK), ("per-tap", sp.CONV_FORCE_PERTAP),
                             ("halo", sp.CONV_FORCE_HALO), ("per-tap, direct stores", sp.CONV_FORCE_PERTAP)):
                if "direct" in name:
                    os.environ["SPHINX_NO_TMA_Y"] = "1"
                g_ = lambda: sp.sphinx_sparse_conv3x3(x, w, None, y, 8, ids, cnt, workspace=ws, variant=fl)
                t = bench.graph_time(torch, g_)
                os.environ.pop("SPHINX_NO_TMA_Y", None)
                print(json.dumps({"time": f"{nf} frame(s) {len(ids_np)} blocks, {name}", "ms": round(t, 5)}))
        else:
            t = bench.graph_time(torch, f)
            print(json.dumps({"time": f"single frame {len(ids_np)} blocks", "ms": round(t, 5)}), flush=True)


def run_step(name, trace):
    import torch
    import paper_2511_18672_b200 as sp
    from paper_2511_18672_b200.step import RefinementStep
    import bench
    lib = sp.load(os.path.join(ROOT, "paper_2511_18672_b200", "libsphinx_trace.so" if trace else "libsphinx.so"))
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    st = RefinementStep(bench.step_config(bench.WORKLOADS[name]["means"]), bench.make_batch(name), dev, sp)
    order = st.conv_order()
    # conv launches per step = len(order); the trace build counts conv_impl calls
    launch = 0
    for _ in range(3):
        st.run()
        launch += len(order)
    torch.cuda.synchronize()
    for j, (l, i) in enumerate(order):
        lib.sphinx_debug_conv_trace_reset()
        os.environ["SPHINX_TRACE_LAUNCH"] = str(launch + j)
        st.run()
        launch += len(order)
        torch.cuda.synchronize()
        show(lib, sms, f"{name} conv ({l},{i})")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "step"
    if what in ("single", "sweep21"):
        nf = 1 if what == "single" else 21
        if "--trace" in sys.argv:
            run_single(True, nf)
        else:
            run_single(False, nf)
            subprocess.check_call([sys.executable, __file__, what, "--trace"])
    elif what == "pointwise":
        if "--trace" in sys.argv:
            run_pointwise(True)
        else:
            run_pointwise(False)
            subprocess.check_call([sys.executable, __file__, "pointwise", "--trace"])
    else:
        run_step(sys.argv[2] if len(sys.argv) > 2 else "configs2", True)
