"""Benchmark of the Sphinx selective-refinement hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload configs3|configs2|configs4] [--no-extras] ...

A STEP is one pass of the whole hot path over one batch of requests
(paper_2511_18672_b200.step.RefinementStep): block masks + start steps from the 576x576
opacity and uncertainty maps -> compaction at 3 UNet levels (+ the inactive-frame list) ->
noise injection on the active latent blocks (start step k) and resampling of inactive frames
(u+1) -> per level two block-sparse 3x3 convs C->C in persistent-buffer mode (72x72x320,
36x36x640, 18x18x1280) -> cached scatter of the latent.  value = effective conv TFLOP/s of the
whole job: algorithmic FLOPs (2*9*Cin*Cout per REAL active output pixel, every frame of the
batch) / device step time (max over ranks).

Default workload = BASELINE configs[3]: 8 requests x 21 frames with request densities
[5,10,25,50,75,25,10,5]%, sharded across the N ranks by active-block cost (LPT) with NCCL
only for the mask/start-step all-gather and the owner gather of refined blocks;
total work is fixed, so scaling is "strong".  At N = 1 the line also carries configs[2]
(one request, round 1's headline workload), configs[4] (25% per request vs the same step
done densely with cuDNN), the configs[1] density sweep, the HBM-bound kernels, the NEXT rows,
the e2e serving loop and the CPU oracle baseline.

Launch: with --gpus N > 1 and no WORLD_SIZE in the environment, the script re-executes itself
under torch.distributed.run (one process per GPU, 127.0.0.1 rendezvous).
--impl reference times the CPU oracle (oracle/) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthetic as syn  # noqa: E402

METRIC = "block-sparse conv effective TFLOP/s & speedup vs dense at 10/25/50% density"
LEVELS = syn.UNET_LEVELS
CONVS_PER_LEVEL = 2
HP, F, B, U_STEP, GAMMA, FPR = 576, 8, 8, 25, 0.5, 21

WORKLOADS = {
    "configs3": dict(means=syn.CONFIG3_REQUEST_DENSITIES, tag="c3",
                     desc="configs[3]: 8 requests x 21 frames (168), request densities [5,10,25,50,75,25,10,5]% "
                          "(per-frame U-shape within each request), 3 UNet levels (72x72x320, 36x36x640, "
                          "18x18x1280), per-frame adaptive start steps, u=25; frames sharded across ranks by "
                          "active-block cost (LPT), refined blocks gathered to each request's owner"),
    "configs2": dict(means=(0.25,), tag="r0",
                     desc="configs[2]: 21-frame request, 3 UNet levels (72x72x320, 36x36x640, 18x18x1280), "
                          "per-frame adaptive start steps, mean level-0 density 25%"),
    "configs4": dict(means=(0.25,) * 8, tag="c4",
                     desc="configs[4]: full refinement step, 8 requests x 21 frames at 25% mean level-0 density "
                          "each, vs the same step done densely"),
}


def step_config(means):
    from paper_2511_18672_b200.step import StepConfig
    return StepConfig(hp=HP, f=F, b=B, levels=LEVELS, convs_per_level=CONVS_PER_LEVEL, frames_per_request=FPR,
                      n_requests=len(means), u=U_STEP, gamma=GAMMA)


def make_batch(name):
    w = WORKLOADS[name]
    return syn.make_batch(w["means"], tag=w["tag"], hp=HP, f=F, b=B, levels=LEVELS,
                          convs_per_level=CONVS_PER_LEVEL, frames_per_request=FPR)


# ----------------------------------------------------------------- measurement helpers

def ncu_tensor_pct(kernel_sig):
    """Mean ncu sm__pipe_tensor_cycles_active (% of peak, elapsed) of the conv launches whose name
    contains kernel_sig, from the newest committed `ncu --set full` capture of the configs[3] step
    (profiles/*_conv_full_raw.csv).  Returns (percent or None, source file)."""
    import csv
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_conv_full_raw.csv")))
    if not files:
        return None, None
    rows = list(csv.reader(open(files[-1])))
    if len(rows) < 3:
        return None, None
    idx = {h: i for i, h in enumerate(rows[0])}
    m = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
    if m not in idx:
        return None, os.path.basename(files[-1])
    vals = [float(r[idx[m]].replace(",", "")) for r in rows[2:] if kernel_sig in r[idx["Kernel Name"]]]
    return (round(sum(vals) / len(vals), 2) if vals else None), os.path.basename(files[-1])


def ncu_traffic(kernel_sig):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes) of the conv launches whose
    name contains kernel_sig, from the newest committed `ncu --set full` capture
    (profiles/*_conv_full_raw.csv).  Returns (bytes or None, source file)."""
    import csv
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_conv_full_raw.csv")))
    if not files:
        return None, None
    rows = list(csv.reader(open(files[-1])))
    if len(rows) < 3:
        return None, None
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    vals = []
    for r in rows[2:]:
        if kernel_sig not in r[idx["Kernel Name"]]:
            continue
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(r[idx[m]].replace(",", "")) * scale.get(units[idx[m]], 1)
        vals.append(tot)
    return (round(sum(vals) / len(vals)) if vals else None), os.path.basename(files[-1])


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained"), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def sample_clocks(stop, out, gpu_index):
    cmd = ["nvidia-smi", "-i", str(gpu_index),
           "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
           "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
           "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
           "--format=csv,noheader,nounits", "-lms", "100"]
    try:
        p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except FileNotFoundError:
        return

    def reader():
        for line in p.stdout:
            out.append(line.strip())
    th = threading.Thread(target=reader, daemon=True)
    th.start()
    stop.wait()
    p.terminate()
    th.join(timeout=2)


def summarize_clocks(lines):
    sm, mx, reasons = [], None, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for ln in lines:
        parts = [x.strip() for x in ln.split(",")]
        if len(parts) < 7:
            continue
        try:
            sm.append(float(parts[0]))
            mx = float(parts[1])
        except ValueError:
            continue
        for nm, v in zip(names, parts[3:7]):
            if v.lower() == "active":
                reasons.add(nm)
    if not sm:
        return None
    return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
            "samples": len(sm)}


def graph_time(torch, fn, reps=20):
    """Device time per call: `reps` calls captured in one CUDA graph and replayed (no host
    launch overhead in the measurement); median over 5 replays.  Warm-up runs on the capture
    stream, so per-stream workspaces exist before the capture."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):  # median of 5 replays
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    return sorted(ts)[2]


def capture_step(torch, st, with_conv_events):
    """Captures one single-rank step into a CUDA graph (a PDL chain of ~15 kernels).  Conv
    launches are bracketed by external event-record nodes so their device time is measured
    inside the replayed graph."""
    conv_ev = None
    L = st.cfg.L
    if with_conv_events:
        conv_ev = [[[torch.cuda.Event(enable_timing=True, external=True),
                     torch.cuda.Event(enable_timing=True, external=True)]
                    for _ in range(CONVS_PER_LEVEL)] for _ in range(L)]
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            st.run()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=side):
        st.run(conv_ev)
    torch.cuda.synchronize()
    return g, conv_ev


def timed_steps(torch, run_step, reps, flush, args, world, conv_events=None, conv_ms=None):
    """K steps, each bracketed by CUDA events on the launching stream, the L2 flushed between
    steps (256 MB write, outside the timed window), barrier + synchronize on both sides."""
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run_step()
        e1.record()
        if not args.no_flush:
            flush.fill_(1.0)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        if conv_events is not None:
            for l in range(len(conv_events)):
                for j in range(CONVS_PER_LEVEL):
                    conv_ms[l][j].append(conv_events[l][j][0].elapsed_time(conv_events[l][j][1]))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    return ms


def density_sweep(torch, sp, dev, frames_list=(1, 21, 168), dens=(0.05, 0.10, 0.25, 0.50, 0.75, 1.0)):
    """configs[1]: 72x72x320, block 8, density sweep 5-100% (1 frame, and the 21-frame and
    168-frame = configs[3]-sized batched variants): own sparse conv vs own dense launch (all
    blocks listed) vs cuDNN dense (torch conv2d, channels_last bf16, fp32 accumulate).  Graph-
    replay device time, L2-warm."""
    h, c = 72, 320
    hb = 9
    out = []
    for nf in frames_list:
        x = torch.from_numpy(syn.features_bf16((nf, h, h, c), "sweep").view(np.int16)).view(torch.bfloat16).to(dev)
        w = torch.from_numpy(syn.weights_bf16(c, c, "sweep").view(np.int16)).view(torch.bfloat16).to(dev)
        y = torch.zeros((nf, h, h, c), dtype=torch.bfloat16, device=dev)
        xn = x.permute(0, 3, 1, 2)
        wn = w.permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
        t_cudnn = graph_time(torch, lambda: torch.nn.functional.conv2d(xn, wn, padding=1))
        ws = torch.zeros(int(sp.load().sphinx_conv_workspace_size(nf, h, h, c, c, B)), dtype=torch.uint8, device=dev)
        rows = []
        for d in list(dens):
            rg = syn.rng("sweep-mask", nf, d)
            m = np.stack([syn.choose_cells(rg, hb, hb, round(d * 81), "clustered") for _ in range(nf)])
            ids_np = np.flatnonzero(m.ravel()).astype(np.int32)
            ids = torch.from_numpy(ids_np).to(dev)
            cnt = torch.tensor([len(ids_np)], dtype=torch.int32, device=dev)
            t = graph_time(torch, lambda: sp.sphinx_sparse_conv3x3(x, w, None, y, B, ids, cnt, workspace=ws))
            flops = len(ids_np) * 64 * 2 * 9 * c * c
            rows.append({"density": round(len(ids_np) / (nf * 81), 4), "active_blocks": int(len(ids_np)),
                         "sparse_ms": round(t, 5), "eff_tflops": round(flops / t / 1e9, 2)})
        t_own_dense = [r["sparse_ms"] for r in rows if r["active_blocks"] == nf * 81][0]
        t_dense = min(t_cudnn, t_own_dense)
        for r in rows:
            r["speedup_vs_dense"] = round(t_dense / r["sparse_ms"], 3)
            r["speedup_vs_cudnn"] = round(t_cudnn / r["sparse_ms"], 3)
            r["efficiency_S_times_d"] = round(r["speedup_vs_dense"] * r["density"], 3)
        out.append({"frames": nf, "shape": [nf, h, h, c], "dense_cudnn_ms": round(t_cudnn, 5),
                    "dense_cudnn_tflops": round(nf * h * h * 2 * 9 * c * c / t_cudnn / 1e9, 1),
                    "dense_own_ms": round(t_own_dense, 5), "rows": rows,
                    "timing": "CUDA-graph replay of 20 launches, L2-warm"})
    return out


def dense_step(torch, st, flush, reps):
    """configs[4]'s comparison: the same step done densely -- the six convs over every pixel
    (cuDNN via torch conv2d, channels_last bf16, fp32 accumulate) plus dense noise on the whole
    latent -- as a CUDA graph, same cold-L2 protocol as the sparse step."""
    d, cfg = st.d, st.cfg
    xs = [d[f"feat{l}"].permute(0, 3, 1, 2) for l in range(cfg.L)]
    ws = [[d[f"w{l}{j}"].permute(0, 3, 1, 2).contiguous(memory_format=torch.channels_last)
           for j in range(CONVS_PER_LEVEL)] for l in range(cfg.L)]
    bs = [[d[f"b{l}{j}"].to(torch.bfloat16) for j in range(CONVS_PER_LEVEL)] for l in range(cfg.L)]
    ab = d["abar"][cfg.u]
    a, sgm = ab.sqrt(), (1 - ab).sqrt()

    def run():
        zt = a * d["x0"] + sgm * d["eps"]
        outs = [zt]
        for l in range(cfg.L):
            src = xs[l]
            for j in range(CONVS_PER_LEVEL):
                src = torch.nn.functional.conv2d(src, ws[l][j], bs[l][j], padding=1)
            outs.append(src)
        return outs
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    ts = []
    for _ in range(max(reps, 3)):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.mean(ts)
    dense_flops = sum(cfg.n_frames * h * h * 2 * 9 * c * c * CONVS_PER_LEVEL for (h, c) in cfg.levels)
    return {"ms": round(ms, 5), "dense_tflops": round(dense_flops / (ms * 1e-3) / 1e12, 1),
            "what": "6 dense convs (cuDNN, channels_last bf16) + dense noise, CUDA graph, L2 flushed"}


def memory_kernels(torch, st, reps=10):
    """HBM-bound / latency-bound kernels timed one launch at a time after an L2 flush (cold),
    CUDA events on the launching stream; algorithmic bytes / time vs the measured HBM peak.
    The flush writes 256 MB and then reads another 256 MB, so L2 holds clean lines: a written-
    only flush leaves ~126 MB of dirty lines whose write-back lands inside a short kernel's
    window (the noise pass: 16.4 us after a write flush vs 12.2 us ncu-cold)
    Includes the NEXT rows (DDIM update, uncertainty producer) measured beside the step."""
    sp, d, dev, cfg = st.ops, st.d, st.dev, st.cfg
    hbm = peaks()[0]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_r = torch.zeros(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def timed(fn):
        # the launch is captured in a one-kernel CUDA graph and replayed right behind the flush:
        # a direct call's host time (ctypes marshalling, ~10 us) would otherwise sit between the
        # two events and be measured instead of the kernel (round-2 rows of 10.2 us for noise,
        # DDIM and compaction alike were that host gap)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        ts = []
        for i in range(reps + 2):
            flush.fill_(0.0)
            flush_r.amax()  # read pass: evicts the flush's dirty lines before the timed launch
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        warm.append(graph_time(torch, fn))  # warm as well (back-to-back launches, L2-warm)
        return statistics.median(ts)

    out = {}
    warm = []

    def row(name, ms, nbytes, note):
        out[name] = {"ms": round(ms, 5), "algorithmic_bytes": int(nbytes),
                     "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1),
                     "hbm_frac": round(nbytes / (ms * 1e-3) / 1e9 / hbm, 4), "bytes": note,
                     "warm_ms": round(warm[-1], 5), "warm_gbs": round(nbytes / (warm[-1] * 1e-3) / 1e9, 1)}
    n, hp = cfg.n_frames, cfg.hp
    ms = timed(lambda: sp.sphinx_block_mask(d["O"], d["U"], d["tau_u"], cfg.tau_o, cfg.f, cfg.b, st.masks,
                                            st.counts, st._start_args(), st.k))
    row("block_mask", ms, n * hp * hp * 8, "two fp32 maps read (8 B/px)")
    cnt = int(st.cnt[0].item())
    ms = timed(lambda: sp.sphinx_compact_blocks(st.masks[0], st.k, cfg.u, sp.SELECT_ACTIVE, st.ids[0], st.cnt[0]))
    out["compact_blocks"] = {"ms": round(ms, 5), "entries": n * cfg.hb[0] ** 2, "bound": "latency (one CTA)",
                             "warm_ms": round(warm[-1], 5)}
    ms = timed(lambda: sp.sphinx_noise_inject(d["x0"], d["eps"], st.zt, cfg.b, st.ids[0], st.cnt[0], st.k,
                                              d["abar"]))
    row("noise_inject", ms, cnt * 64 * cfg.c_lat * 12, "12 B per active latent element (x0, eps in; x_t out)")
    out0 = torch.empty_like(d["cache0"])
    ms = timed(lambda: sp.sphinx_scatter_cached(st.z[0], d["cache0"], out0, cfg.b, block_mask=st.masks[0],
                                                start_step=st.k, step_u=cfg.u))
    row("scatter_cached_level0_features", ms, 2 * out0.numel() * 2, f"2 x map bytes ({n}x72x72x320 bf16)")
    pay = torch.empty((max(cnt, 1), cfg.b, cfg.b, 320), dtype=torch.bfloat16, device=dev)
    ms = timed(lambda: sp.sphinx_gather_blocks(st.z[0], pay, cfg.b, st.ids[0], st.cnt[0]))
    row("gather_blocks_level0 (data plane pack)", ms, 2 * cnt * 64 * 320 * 2, "2 x listed block bytes")
    zo = torch.empty_like(st.zt)
    abar_h = d["abar"].cpu().numpy()  # host table (the step u is a loop scalar)
    ms = timed(lambda: sp.sphinx_ddim_step(st.zt, d["x0"], zo, cfg.b, st.ids[0], st.cnt[0], cfg.u, abar_h))
    row("ddim_step (NEXT-1)", ms, cnt * 64 * cfg.c_lat * 12, "12 B per active latent element (z, x0_hat in; z' out)")
    nu = min(n, 21)
    rgb = torch.from_numpy(syn.rgb_frames(nu, hp, hp, "bench")).to(dev)  # textured frames with flat patches
    U = torch.empty((nu, hp, hp), device=dev, dtype=torch.float32)
    tau = torch.empty((nu,), device=dev, dtype=torch.float32)
    ms = timed(lambda: sp.sphinx_uncertainty_map(rgb, U, tau))
    row("uncertainty_map (NEXT-2, 21 frames)", ms, nu * hp * hp * 16, "rgb read 12 B/px + U write 4 B/px")
    out["timing"] = ("ms: one launch per sample in a CUDA graph replayed behind a 256 MB write + 256 MB read "
                     "L2 flush (clean cold L2), median of 10; warm_ms: CUDA graph of 20 back-to-back launches "
                     "(L2-warm), per launch, median of 5 replays")
    return out


def resblock_levels(torch, st, reps=20):
    """NEXT-3: the block-sparse ResNet block (GN+SiLU -> conv -> GN+SiLU -> conv + skip) at each
    UNet level over the step's active list, after a full step (every block) filled the persistent
    h / y / statistics buffers.  Graph-replay device time per block (L2-warm) and its parts."""
    sp, d, dev, cfg = st.ops, st.d, st.dev, st.cfg
    out = []
    for l, (h, c) in enumerate(cfg.levels):
        n, hb = cfg.n_frames, cfg.hb[l]
        x = d[f"feat{l}"]
        g1, be1 = (torch.from_numpy(a).to(dev) for a in syn.gn_affine_f32(c, f"gn{l}1"))
        g2, be2 = (torch.from_numpy(a).to(dev) for a in syn.gn_affine_f32(c, f"gn{l}2"))
        hbuf = d[f"cache{l}"].clone()
        y = d[f"cache{l}"].clone()
        a = torch.empty_like(x)
        xs = sp.gn_stats_buffer(n, h, h, syn.GN_GROUPS, cfg.b, dev)
        hs = sp.gn_stats_buffer(n, h, h, syn.GN_GROUPS, cfg.b, dev)
        all_ids = torch.arange(n * hb * hb, dtype=torch.int32, device=dev)
        all_cnt = torch.tensor([n * hb * hb], dtype=torch.int32, device=dev)
        ids, cnt = st.ids[l], st.cnt[l]

        def block(i=ids, k=cnt):
            sp.sphinx_sparse_resblock(x, d[f"w{l}0"], d[f"b{l}0"], d[f"w{l}1"], d[f"b{l}1"], (g1, be1),
                                      (g2, be2), syn.GN_GROUPS, syn.GN_EPS, hbuf, xs, hs, y, a, cfg.b, i, k)
        block(all_ids, all_cnt)  # the full step: every block, fills h, y and both statistics
        t_block = graph_time(torch, block, reps)
        t_gn = graph_time(torch, lambda: (
            sp.sphinx_gn_block_stats(x, syn.GN_GROUPS, cfg.b, ids, cnt, xs),
            sp.sphinx_gn_silu(x, xs, g1, be1, syn.GN_EPS, syn.GN_GROUPS, cfg.b, ids, cnt, a)), reps)
        t_conv = graph_time(torch, lambda: sp.sphinx_sparse_conv3x3(a, d[f"w{l}0"], d[f"b{l}0"], hbuf, cfg.b,
                                                                    ids, cnt), reps)
        nb = int(cnt.item())
        idn = ids[:nb].cpu().numpy() % (hb * hb)
        by, bx = idn // hb, idn % hb
        px = int((np.minimum(cfg.b, h - by * cfg.b) * np.minimum(cfg.b, h - bx * cfg.b)).sum())
        ring = int(((np.minimum(by * cfg.b + cfg.b + 1, h) - np.maximum(by * cfg.b - 1, 0)) *
                    (np.minimum(bx * cfg.b + cfg.b + 1, h) - np.maximum(bx * cfg.b - 1, 0))).sum())
        flops = 2 * px * 2 * 9 * c * c
        gn_bytes = px * c * 2 + ring * c * 4  # stats read + activation read/write (ring incl.)
        out.append({"level": l, "shape": [n, h, h, c], "active_blocks": nb, "real_px": px,
                    "block_ms": round(t_block, 5), "block_tflops": round(flops / (t_block * 1e-3) / 1e12, 2),
                    "gn_silu_ms": round(t_gn, 5), "gn_silu_gbs": round(gn_bytes / (t_gn * 1e-3) / 1e9, 1),
                    "conv_ms": round(t_conv, 5), "gn_share_of_block": round(2 * t_gn / t_block, 4)})
    return {"levels": out, "timing": "CUDA-graph replay of 20 blocks, L2-warm; block = 6 launches "
            "(gn_block_stats, gn_silu, conv, gn_block_stats, gn_silu, conv+residual)",
            "block_tflops_note": "2 convs' algorithmic FLOPs (real active px) / whole-block time"}


def temporal_levels(torch, st, reps=20):
    """NEXT-4: the temporal-attention block with the K/V latent cache at each UNet level over the
    step's active list (T = 21 frames = one request), after a full step (every block) filled the
    persistent q|k|v cache and y.  Graph-replay device time (L2-warm) and its parts."""
    sp, d, dev, cfg = st.ops, st.d, st.dev, st.cfg
    out = []
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
    for l, (h, c) in enumerate(cfg.levels):
        n, hb = cfg.n_frames, cfg.hb[l]
        heads = c // syn.ATTN_HEAD_DIM
        x = d[f"feat{l}"]
        wq = bf(syn.linear_weights_bf16(3 * c, c, f"tq{l}", 0.5))
        wo = bf(syn.linear_weights_bf16(c, c, f"to{l}"))
        bq = torch.from_numpy(syn.bias_f32(3 * c, f"tq{l}")).to(dev)
        bo = torch.from_numpy(syn.bias_f32(c, f"to{l}")).to(dev)
        qkv = torch.zeros((n, h, h, 3 * c), dtype=torch.bfloat16, device=dev)
        o = torch.zeros_like(x)
        y = d[f"cache{l}"].clone()
        all_ids = torch.arange(n * hb * hb, dtype=torch.int32, device=dev)
        all_cnt = torch.tensor([n * hb * hb], dtype=torch.int32, device=dev)
        ids, cnt = st.ids[l], st.cnt[l]

        def block(i=ids, k=cnt):
            sp.sphinx_temporal_block(x, wq, bq, wo, bo, heads, cfg.frames_per_request, qkv, o, y, cfg.b, i, k)
        block(all_ids, all_cnt)  # the full step: every token's q|k|v cached, y filled
        t_block = graph_time(torch, block, reps)
        t_qkv = graph_time(torch, lambda: sp.sphinx_sparse_pointwise(x, wq, bq, qkv, cfg.b, ids, cnt), reps)
        t_att = graph_time(torch, lambda: sp.sphinx_temporal_attention(qkv, o, heads, cfg.frames_per_request, cfg.b,
                                                                       ids, cnt), reps)
        nb = int(cnt.item())
        idn = ids[:nb].cpu().numpy()
        pos = idn % (hb * hb)
        by, bx = pos // hb, pos % hb
        px = int((np.minimum(cfg.b, h - by * cfg.b) * np.minimum(cfg.b, h - bx * cfg.b)).sum())
        seq_pos = np.unique((idn // (hb * hb)) // cfg.frames_per_request * (hb * hb) + pos)
        sp_pos = seq_pos % (hb * hb)
        upx = int((np.minimum(cfg.b, h - (sp_pos // hb) * cfg.b) * np.minimum(cfg.b, h - (sp_pos % hb) * cfg.b)).sum())
        T = cfg.frames_per_request
        proj_flops = px * 2 * (3 * c * c + c * c)
        attn_flops = px * 4 * T * c
        staged = upx * T * 3 * c * 2
        out.append({"level": l, "shape": [n, h, h, c], "heads": heads, "frames_per_seq": T,
                    "active_blocks": nb, "real_px": px, "block_ms": round(t_block, 5),
                    "block_tflops": round((proj_flops + attn_flops) / (t_block * 1e-3) / 1e12, 2),
                    "qkv_proj_ms": round(t_qkv, 5),
                    "qkv_proj_tflops": round(px * 2 * 3 * c * c / (t_qkv * 1e-3) / 1e12, 2),
                    "attention_ms": round(t_att, 5),
                    "attention_staged_gbs": round(staged / (t_att * 1e-3) / 1e9, 1)})
    return {"levels": out, "timing": "CUDA-graph replay of 20 blocks, L2-warm; block = qkv pointwise "
            "(tcgen05) + plan + attention + output pointwise with residual",
            "flops_note": "projections 8 C^2 + attention 4 T C FLOP per listed token",
            "attention_bytes_note": "staged token bytes: T x 3C x 2 B per (sequence, pixel) with any listed frame"}


# ----------------------------------------------------------------- GPU arm

def conv_level_stats(st, conv_ms, px_l, blocks_l, tc_peak, tc_sust, ms_all, with_ncu=False):
    """Per-level conv times and rates; with_ncu (the configs[3] headline, the workload the committed
    ncu capture profiles): each level's ncu tensor-pipe activity from that capture."""
    cfg = st.cfg
    per_level = []
    for l, (h, c) in enumerate(cfg.levels):
        t_l = statistics.mean([statistics.mean(conv_ms[l][j]) for j in range(CONVS_PER_LEVEL)])
        f_l = px_l[l] * 2 * 9 * c * c
        per_level.append({"level": l, "shape": [cfg.n_frames, h, h, c], "active_blocks": blocks_l[l],
                          "real_px": px_l[l], "density": round(blocks_l[l] / (cfg.n_frames * cfg.hb[l] ** 2), 4),
                          "conv_ms": round(t_l, 5),
                          "conv_ms_each": [round(statistics.mean(conv_ms[l][j]), 5) for j in range(CONVS_PER_LEVEL)],
                          "tflops": round(f_l / (t_l * 1e-3) / 1e12, 2),
                          "frac_burst": round(f_l / (t_l * 1e-3) / 1e12 / tc_peak, 4)})
        if with_ncu:
            bn_l = 256 if c % 256 == 0 and c > 640 else 160
            pct, src = ncu_tensor_pct(f"<{bn_l}, 2, 8, 1, {1 if h % cfg.b else 0}, 0>")
            per_level[-1]["ncu_tensor_pipe_pct"] = pct
            per_level[-1]["ncu_source"] = src
    conv_total_ms = sum(p["conv_ms"] for p in per_level) * CONVS_PER_LEVEL
    dom = max(per_level, key=lambda p: p["conv_ms"])
    dom_flops = dom["real_px"] * 2 * 9 * cfg.levels[dom["level"]][1] ** 2
    achieved = dom_flops / (dom["conv_ms"] * 1e-3) / 1e12
    bn = 256 if cfg.levels[dom["level"]][1] % 256 == 0 and cfg.levels[dom["level"]][1] > 640 else 160
    edge = 1 if cfg.levels[dom["level"]][0] % cfg.b else 0
    sig = f"<{bn}, 2, 8, 1, {edge}, 0>"
    traffic, traffic_src = ncu_traffic(sig)
    flops = sum(p["real_px"] * 2 * 9 * c * c for p, (_, c) in zip(per_level, cfg.levels)) * CONVS_PER_LEVEL
    roof = {"bound": "tensor", "kernel": "sparse_conv3x3_tc_kernel%s (level %d)" % (sig, dom["level"]),
            "achieved": round(achieved, 2), "peak": tc_peak, "unit": "TFLOP/s",
            "frac": round(achieved / tc_peak, 4), "peak_kind": "measured bf16 burst (MEASURED_PEAKS.json)",
            "frac_sustained": round(achieved / tc_sust, 4) if tc_sust else None,
            "traffic": traffic, "traffic_unit": "bytes per launch (dram read+write)", "traffic_source": traffic_src,
            "all_convs_tflops": round(flops / (conv_total_ms * 1e-3) / 1e12, 2),
            "conv_share_of_step": round(conv_total_ms / ms_all, 4)}
    return per_level, roof


def single_rank_workload(torch, sp, name, dev, flush, args, tc_peak, tc_sust, with_dense=False):
    """A secondary workload at N = 1 (configs[2] or configs[4]): graph-replayed step, cold L2."""
    from paper_2511_18672_b200.step import RefinementStep
    cfg = step_config(WORKLOADS[name]["means"])
    st = RefinementStep(cfg, make_batch(name), dev, sp)
    g, _ = capture_step(torch, st, False)
    g_ev, conv_ev = capture_step(torch, st, True)
    for _ in range(3):
        g.replay()
    reps = max(3, min(args.steps, 10))
    ms = timed_steps(torch, g.replay, reps, flush, args, 1)
    conv_ms = [[[] for _ in range(CONVS_PER_LEVEL)] for _ in range(cfg.L)]
    timed_steps(torch, g_ev.replay, reps, flush, args, 1, conv_ev, conv_ms)
    flops, px_l, blocks_l = st.active_stats()
    step_ms = statistics.mean(ms)
    per_level, roof = conv_level_stats(st, conv_ms, px_l, blocks_l, tc_peak, tc_sust, step_ms)
    out = {"workload": WORKLOADS[name]["desc"], "frames": cfg.n_frames, "ms_per_step": round(step_ms, 5),
           "value_tflops": round(flops / (step_ms * 1e-3) / 1e12, 3), "conv_levels": per_level,
           "roofline": roof}
    if with_dense:
        dense = dense_step(torch, st, flush, reps)
        out["dense_step"] = dict(dense, speedup_of_step=round(dense["ms"] / step_ms, 3))
    del st, g, g_ev
    torch.cuda.empty_cache()
    return out


def warm_cold_conv(torch, st, flush, reps=10):
    """One conv per level on the step's lists, timed alone: warm (back-to-back graph replays,
    weights and features L2-resident) vs cold (256 MB L2 flush before each launch)."""
    out = []
    d, cfg, sp = st.d, st.cfg, st.ops
    for l, (h, c) in enumerate(cfg.levels):
        def fn():
            sp.sphinx_sparse_conv3x3(d[f"feat{l}"], d[f"w{l}0"], d[f"b{l}0"], st.y[l], cfg.b, st.ids[l], st.cnt[l],
                                     workspace=st.ws[l], reuse_plan=False)
        warm = graph_time(torch, fn)
        ts = []
        for i in range(reps + 2):
            flush.fill_(0.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        out.append({"level": l, "warm_ms": round(warm, 5), "cold_ms": round(statistics.median(ts), 5)})
    return out


def nccl_summary():
    """What NCCL's INIT log (NCCL_DEBUG=INFO -> NCCL_DEBUG_FILE) says on this rank."""
    import glob
    path = os.environ.get("NCCL_DEBUG_FILE", "")
    if not path:
        return None
    files = sorted(glob.glob(path.replace("%h", "*").replace("%p", str(os.getpid()))))
    lines = []
    for f in files:
        try:
            lines += open(f).read().splitlines()
        except OSError:
            pass
    pick = [ln.split("NCCL INFO", 1)[-1].strip() for ln in lines
            if "NCCL INFO" in ln and any(k in ln for k in ("NCCL version", "nRanks", "NVLS", "P2P", "Channel 00", "CollNet"))]
    return {"lines": pick[:12], "nvls": any("NVLS" in ln and "enabled" in ln.lower() for ln in lines),
            "log": path}


def run_gpu(args):
    import torch
    import torch.distributed as dist
    import paper_2511_18672_b200 as sp
    from paper_2511_18672_b200 import dist as sdist
    from paper_2511_18672_b200.step import RefinementStep
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.share_gpu:  # functional check of the N-rank path on a 1-GPU box (timings meaningless)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    sp.load()
    hbm, tc_peak, tc_sust, peak_kind = peaks()
    name = args.workload
    cfg = step_config(WORKLOADS[name]["means"])
    batch = make_batch(name)
    st = RefinementStep(cfg, batch, dev, sp, group=group, rank=rank, world=world)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    L = cfg.L
    if world == 1:
        # the step is timed on an event-free graph (event nodes would break the PDL chain between
        # kernels); a second graph with external event nodes around each conv gives per-conv times
        g, _ = capture_step(torch, st, with_conv_events=False)
        g_ev, conv_ev = capture_step(torch, st, with_conv_events=True)
        run_step, run_ev = g.replay, g_ev.replay
        timing_note = ("CUDA graph replay (event-free graph for the step; conv launches timed by captured external "
                       "events in a second graph)")
    else:
        conv_ev = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
                    for _ in range(CONVS_PER_LEVEL)] for _ in range(L)]
        run_step, run_ev = st.run, (lambda: st.run(conv_ev))
        timing_note = ("eager launches (the host LPT plan between the mask all-gather and the compaction makes "
                       "one D2H sync per step); per-conv CUDA events on the compute stream")
    for _ in range(max(args.warmup, 3)):
        run_step()
        flush.fill_(1.0)
    torch.cuda.synchronize()
    flops, px_l, blocks_l = st.active_stats()
    stop = threading.Event()
    clk_lines = []
    th = threading.Thread(target=sample_clocks, args=(stop, clk_lines, local), daemon=True)
    th.start()
    time.sleep(0.3)
    reps = max(1, args.steps)
    t_wall0 = time.time()
    step_ms = timed_steps(torch, run_step, reps, flush, args, world)
    wall_s = time.time() - t_wall0
    conv_ms = [[[] for _ in range(CONVS_PER_LEVEL)] for _ in range(L)]
    timed_steps(torch, run_ev, reps, flush, args, world, conv_ev, conv_ms)
    t_end = time.time() + 1.0
    while time.time() < t_end:  # a sustained stretch for the clock samples
        run_step()
        torch.cuda.synchronize()
    stop.set()
    th.join(timeout=3)
    ms = statistics.mean(step_ms)
    multi = None
    if world > 1:
        # whole-job throughput: the batch's work / max over ranks of the step time
        ms_all, _ = sdist.reduce_step(ms, 0.0, device=dev)
        ms_min = -sdist.reduce_step(-ms, 0.0, device=dev)[0]
        sent = torch.tensor([float(st.bytes_sent)], dtype=torch.float64, device=dev)
        dist.all_reduce(sent)
        comm_max, _ = sdist.reduce_step(st.comm_ms(), 0.0, device=dev)
        e2e_sh = None if args.no_e2e else run_e2e_sharded(torch, st, batch, dev, args, flops, world)
        p = st.plan
        multi = {"ranks": world, "partition": "LPT over frames by executed MMA work (sum_l count*C_l^2) at u",
                 "plan_imbalance_max_over_mean": round(p["imbalance"], 4),
                 "step_ms_max": round(ms_all, 5), "step_ms_min": round(ms_min, 5),
                 "bytes_moved_per_step": int(sent.item()),
                 "comm_ms_max": round(comm_max, 5),
                 "comm_note": "device time of the owner-gather sections (pack + grouped send/recv + unpack) "
                              "on the communication stream, summed over levels, max over ranks; it overlaps "
                              "the next level's convs",
                 "owner": "request j -> rank j*N//R", "nccl": nccl_summary() if rank == 0 else None}
    else:
        ms_all = ms
        e2e_sh = None
    value = flops / (ms_all * 1e-3) / 1e12
    if world > 1:  # the conv launches of THIS rank process its own lists (its share of the batch)
        my_px, my_blocks = [], []
        for l in range(L):
            ids = st.ids[l][: int(st.cnt[l].item())].cpu().numpy()
            my_px.append(cfg.real_px(l, ids))
            my_blocks.append(len(ids))
        per_level, roof = conv_level_stats(st, conv_ms, my_px, my_blocks, tc_peak, tc_sust, ms)
        roof["scope"] = "rank 0's own conv launches (its share of the batch)"
    else:
        per_level, roof = conv_level_stats(st, conv_ms, px_l, blocks_l, tc_peak, tc_sust, ms,
                                           with_ncu=(name == "configs3"))

    extras = {}
    if rank == 0 and world == 1 and not args.no_extras:
        extras["conv_warm_cold"] = warm_cold_conv(torch, st, flush)
        extras["e2e"] = None if args.no_e2e else run_e2e(torch, st, g, batch, dev, args, flops)
        extras["memory_kernels"] = memory_kernels(torch, st)
        extras["configs2"] = single_rank_workload(torch, sp, "configs2", dev, flush, args, tc_peak, tc_sust)
        del g, g_ev
        torch.cuda.empty_cache()
        extras["configs4"] = single_rank_workload(torch, sp, "configs4", dev, flush, args, tc_peak, tc_sust,
                                                  with_dense=True)
        if not args.no_resblock:
            st2 = RefinementStep(step_config(WORKLOADS["configs2"]["means"]), make_batch("configs2"), dev, sp)
            st2.run()
            torch.cuda.synchronize()
            extras["resblock (NEXT-3)"] = resblock_levels(torch, st2)
            extras["temporal_attention (NEXT-4)"] = temporal_levels(torch, st2)
            del st2
        if not args.no_sweep:
            extras["density_sweep"] = density_sweep(torch, sp, dev)
            # the metric's second half at a glance: speedup over the best dense launch (own or cuDNN)
            # at 10 / 25 / 50% density, per batch size of the sweep (configs[1] = 1 frame)
            extras["speedup_vs_dense"] = {
                f"{sw['frames']}_frames": {f"{int(round(r['density'] * 100 / 5) * 5)}%": r["speedup_vs_dense"]
                                           for r in sw["rows"] if 0.08 < r["density"] < 0.6}
                for sw in extras["density_sweep"]}

    if rank == 0:
        cpu = None if (world > 1 or args.no_cpu) else cpu_baseline(batch, cfg, bounded_s=args.cpu_seconds)
        if cpu is not None:
            fl_cfg = {name: flops}
            for k in ("configs2", "configs4"):
                if extras.get(k):
                    fl_cfg[k] = extras[k]["value_tflops"] * 1e12 * extras[k]["ms_per_step"] * 1e-3
            cpu["oracle_configs"] = oracle_record(fl_cfg, cpu["value"] * 1e12)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": reps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms_all, 5), "higher_is_better": True,
            "scaling": "strong" if name != "configs2" else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": WORKLOADS[name]["desc"], "frames": cfg.n_frames, "requests": cfg.n_requests,
                       "image": [HP, HP], "block": B, "u": U_STEP, "convs_per_level": CONVS_PER_LEVEL,
                       "active_blocks_per_level": blocks_l,
                       "density_per_level": [round(blocks_l[l] / (cfg.n_frames * cfg.hb[l] ** 2), 4) for l in range(L)],
                       "l2": ("NOT flushed (diagnostic --no-flush)" if args.no_flush else
                              "flushed between timed steps (256 MB write)"), "timing": timing_note,
                       "parallelism": f"dp{world} (frame sharding)"},
            "gpu_launches": (st.launches_per_step * reps if world == 1 else None),
            "roofline": roof,
            "conv_levels": per_level,
            "multi_gpu": multi,
            "wall_s_timed_steps": round(wall_s, 4),
            "paper_context": "1.8x average end-to-end speedup vs diffusion-only on 4x A40 (P:34, P:445); context "
                             "only, not this metric",
            "clocks": summarize_clocks(clk_lines),
            # the spread of the timed steps (this rank's), beside the mean above
            "step_ms_p10_p50_p90": [round(float(np.percentile(step_ms, q)), 5) for q in (10, 50, 90)],
        }
        if world > 1:
            # rank 0's own kernels in the timed steps (every rank launches its own share): the step's
            # kernels on its frames plus the owner-gather pack / unpack kernels of its exchanges
            line["gpu_launches"] = int((st.launches_per_step + st.exchange_launches) * reps)
            line["gpu_launches_note"] = ("rank 0: %d sphinx kernels per step (%d step + %d owner-gather pack/"
                                         "unpack), eager multi-rank step; NCCL kernels not counted" % (
                                             st.launches_per_step + st.exchange_launches, st.launches_per_step,
                                             st.exchange_launches))
        line.update(extras)
        line["e2e"] = extras.get("e2e") if world == 1 else e2e_sh
        line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_profile(args):
    """Minimal run for ncu: the captured step graph replayed twice; only the step's kernels
    (and the graph-capture warm-up's) appear in the launch list."""
    import torch
    import paper_2511_18672_b200 as sp
    from paper_2511_18672_b200.step import RefinementStep
    torch.cuda.set_device(0)
    cfg = step_config(WORKLOADS[args.workload]["means"])
    st = RefinementStep(cfg, make_batch(args.workload), torch.device("cuda", 0), sp)
    g, _ = capture_step(torch, st, with_conv_events=False)
    torch.cuda.synchronize()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    print(json.dumps({"profile": "done", "workload": args.workload, "launches_per_step": st.launches_per_step}))


def run_e2e(torch, st, g, batch, dev, args, flops):
    """Same step through the public API with HOST buffers: every step copies its inputs from
    pinned host memory (H2D) and reads its result back (D2H), all inside the timed region.  The
    level input features stay in pinned host memory and each step moves only the halo windows of its
    listed blocks (RefinementStep host_features: sphinx_gather_halo_windows reads them over PCIe);
    maps, scores and latents are copied whole."""
    from paper_2511_18672_b200.step import RefinementStep
    in_keys = ["O", "U", "tau_u", "q", "c0", "c1", "t", "x0", "eps", "lid", "lat_cache"]
    host = {k: torch.from_numpy(np.ascontiguousarray(batch[k].view(np.int16) if batch[k].dtype == np.uint16
                                                     else batch[k])).pin_memory() for k in in_keys}
    hfeat = {l: torch.from_numpy(np.ascontiguousarray(batch[f"feat{l}"]).view(np.int16)).pin_memory()
             .view(torch.bfloat16) for l in range(st.cfg.L)}
    out_host = torch.empty(st.lat_out.shape, dtype=st.lat_out.dtype).pin_memory()
    d2h = out_host.numel() * out_host.element_size()

    def copy_in(s_):
        for k, h in host.items():
            dst = s_.d[k]
            (dst.view(torch.int16) if dst.dtype == torch.bfloat16 else dst).copy_(h, non_blocking=True)

    # two input/output sets (one model state each), features read from the same pinned host maps
    sts = [RefinementStep(st.cfg, batch, dev, st.ops, host_features=hfeat) for _ in range(2)]
    graphs = [capture_step(torch, s_, with_conv_events=False)[0] for s_ in sts]
    torch.cuda.synchronize()
    h2d = sum(h.numel() * h.element_size() for h in host.values()) + sts[0].window_bytes()
    full_feat = sum(h.numel() * h.element_size() for h in hfeat.values())

    def step():
        copy_in(sts[0])
        graphs[0].replay()
        out_host.copy_(sts[0].lat_out, non_blocking=True)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(1, min(args.steps, 5))
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms_serial = e0.elapsed_time(e1) / reps

    # serving loop: step j's H2D runs on a copy stream while step j-1 computes (its feature windows
    # cross PCIe inside its compute), the result D2H on a third stream.  Every step still moves all
    # its inputs and reads its result.
    sets = [(sts[0], graphs[0], out_host), (sts[1], graphs[1], torch.empty_like(out_host).pin_memory())]
    main = torch.cuda.current_stream()
    cs, ds = torch.cuda.Stream(), torch.cuda.Stream()
    freed = [torch.cuda.Event(), torch.cuda.Event()]
    read = [torch.cuda.Event(), torch.cuda.Event()]
    start = torch.cuda.Event()

    def pipelined(n):
        start.record(main)
        cs.wait_event(start)
        for j in range(n):
            s_, g_, oh = sets[j % 2]
            cs.wait_event(freed[j % 2])
            with torch.cuda.stream(cs):
                copy_in(s_)
            landed = torch.cuda.Event()
            landed.record(cs)
            main.wait_event(landed)
            main.wait_event(read[j % 2])
            g_.replay()
            freed[j % 2].record(main)
            ds.wait_event(freed[j % 2])
            with torch.cuda.stream(ds):
                oh.copy_(s_.lat_out, non_blocking=True)
            read[j % 2].record(ds)
        main.wait_stream(ds)

    pipelined(4)
    torch.cuda.synchronize()
    n_pipe = max(4, min(args.steps, 10))
    e0.record(main)
    pipelined(n_pipe)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n_pipe
    del sts, graphs
    return {"value": round(flops / (ms * 1e-3) / 1e12, 4), "unit": "TFLOP/s", "ms_per_step": round(ms, 4),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "feature_bytes_moved_vs_whole_maps": [int(h2d - sum(h.numel() * h.element_size()
                                                               for h in host.values())), int(full_feat)],
            "steps_timed": n_pipe, "serial_ms_per_step": round(ms_serial, 4),
            "h2d_gbs": round(h2d / (ms * 1e-3) / 1e9, 1),
            "note": "serving loop, two input sets: step j's H2D (copy stream) overlaps step j-1's compute, the "
                    "result D2H on a third stream; serial_ms_per_step = copy, compute, read back one after the "
                    "other.  Conv weights resident (model state); per step: opacity/uncertainty maps, scores and "
                    "latents H2D whole, level input features as the halo windows of the listed blocks read from "
                    "pinned host memory by sphinx_gather_halo_windows; the refined latent (the step's result) D2H"}


def run_e2e_sharded(torch, st, batch, dev, args, flops, world):
    """e2e at N > 1 through the same public call: every step each rank copies from pinned host
    memory the maps of its mask slice and the latents of the frames the plan assigned to it (stable
    across steps: same masks, same u), gathers the halo windows of its listed blocks from the pinned
    host features, runs the sharded step, and reads back the refined latent of the frames it owns.
    Device time of the whole loop, max over ranks."""
    from paper_2511_18672_b200 import dist as sdist
    cfg = st.cfg
    mine = np.flatnonzero(st.plan["rank_of"] == st.rank)
    own = np.flatnonzero(st.owner == st.rank)
    sl = st.slice
    maps = ["O", "U", "tau_u", "q", "c0", "c1", "t", "lid"]
    frame_keys = ["x0", "eps", "lat_cache"]

    def pin(a):
        a = np.ascontiguousarray(a.view(np.int16) if a.dtype == np.uint16 else a)
        return torch.from_numpy(a).pin_memory()
    host_maps = {k: pin(batch[k][sl]) for k in maps}
    host_frames = {k: pin(batch[k][mine]) for k in frame_keys}
    # level features from pinned host memory: each step moves only the halo windows of this rank's
    # listed blocks (as the single-rank e2e, RefinementStep host_features)
    st.host_features = {l: pin(batch[f"feat{l}"]).view(torch.bfloat16) for l in range(cfg.L)}
    out_host = torch.empty((len(own),) + tuple(st.lat_out.shape[1:]), dtype=torch.float32).pin_memory()
    d2h = out_host.numel() * 4
    runs = [(int(a), int(b)) for a, b in _runs(mine)]

    def dev_view(k):
        t = st.d[k]
        return t.view(torch.int16) if t.dtype == torch.bfloat16 else t

    def step():
        for k, h in host_maps.items():
            dev_view(k)[sl].copy_(h, non_blocking=True)
        for k, h in host_frames.items():
            dv, off = dev_view(k), 0
            for a, b in runs:  # contiguous frame runs of this rank's assignment
                dv[a:b].copy_(h[off:off + b - a], non_blocking=True)
                off += b - a
        st.run()
        o0 = int(own[0])
        out_host.copy_(st.lat_out[o0:o0 + len(own)], non_blocking=True)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    reps = max(1, min(args.steps, 5))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms, _ = sdist.reduce_step(e0.elapsed_time(e1) / reps, 0.0, device=dev)
    h2d = sum(t.numel() * t.element_size() for t in list(host_maps.values()) + list(host_frames.values())) + \
        st.window_bytes()
    st.host_features = None
    tot = torch.tensor([float(h2d), float(d2h)], dtype=torch.float64, device=dev)
    import torch.distributed as dist
    dist.all_reduce(tot)
    return {"value": round(flops / (ms * 1e-3) / 1e12, 4), "unit": "TFLOP/s", "ms_per_step": round(ms, 4),
            "h2d_bytes_per_step": int(tot[0].item()), "d2h_bytes_per_step": int(tot[1].item()),
            "steps_timed": reps,
            "note": "serial loop per rank: H2D of the rank's mask-slice maps and its assigned frames' latents, "
                    "the halo windows of its listed blocks read from pinned host features, the sharded step, D2H "
                    "of the owned frames' refined latent; bytes summed over ranks, time max over ranks"}


def _runs(idx):
    """Contiguous runs [a, b) of a sorted index array."""
    idx = list(idx)
    out = []
    for i in idx:
        if out and out[-1][1] == i:
            out[-1][1] = i + 1
        else:
            out.append([i, i + 1])
    return out


# ----------------------------------------------------------------- CPU oracle arm

def oracle_step_sample(batch, cfg, max_blocks_per_level):
    """The same step on the CPU oracle, bounded: masks/start steps/compaction/noise/scatter on
    the whole batch, one conv per level on the first max_blocks_per_level active blocks.
    Returns (seconds, conv FLOPs computed)."""
    import oracle
    t0 = time.perf_counter()
    kl = batch["klogic"]
    lg = oracle.make_klogic(kl["thr"], kl["steps"], kl["fallback_k"], kl["k_max"])
    masks, counts = oracle.block_mask(batch["O"], batch["U"], batch["tau_u"], cfg.tau_o, cfg.f, cfg.b, cfg.L)
    k = oracle.start_step(batch["q"], batch["c0"], batch["c1"], batch["t"], cfg.gamma, [lg], logic_id=batch["lid"])
    ids = [oracle.compact(masks[l], k, cfg.u) for l in range(cfg.L)]
    inact = oracle.compact(None, k, cfg.u, oracle.SELECT_INACTIVE_FRAMES, shape=masks[0].shape)
    z = oracle.noise(batch["x0"], batch["eps"], batch["x0"], cfg.b, ids[0], k, batch["abar"])
    z = oracle.noise(batch["x0"], batch["eps"], z.astype(np.float32), cfg.b, inact,
                     np.full(cfg.n_frames, cfg.u + 1, np.int32), batch["abar"])
    oracle.scatter(z.astype(np.float32), batch["lat_cache"], cfg.b, mask=masks[0], k=k, u=cfg.u)
    flops = 0
    for l, (h, c) in enumerate(cfg.levels):
        sub = ids[l][:max_blocks_per_level]
        oracle.conv3x3_blocks(batch[f"feat{l}"], batch[f"w{l}0"], batch[f"b{l}0"], cfg.b, sub, n_threads=0)
        flops += cfg.real_px(l, sub) * 2 * 9 * c * c
    return time.perf_counter() - t0, flops


def calibrate_blocks(batch, cfg, seconds):
    """Blocks per level so that one oracle step sample takes about `seconds`."""
    t1, _ = oracle_step_sample(batch, cfg, 1)
    t3, _ = oracle_step_sample(batch, cfg, 3)
    slope = max((t3 - t1) / 2, 1e-3)
    return int(max(1, min(4000, 1 + (seconds - t1) / slope)))


def cpu_baseline(batch, cfg, bounded_s=15.0):
    cores = os.cpu_count()
    nb = calibrate_blocks(batch, cfg, bounded_s)
    t, f = oracle_step_sample(batch, cfg, nb)
    return {"value": round(f / t / 1e12, 8), "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
            "seconds": round(t, 2),
            "sample": f"the {cfg.n_frames}-frame batch: full mask/start-step/compaction/noise/scatter, one conv on "
                      f"the first {nb} active blocks of each level (fp64 direct conv, OpenMP {cores} threads)"}


def oracle_record(conv_flops_by_config, rate_all_cores, seconds_1core=8.0):
    """SURVEY 8(d) "oracle timing beside it": the oracle as it stands on this box's host cores.
    configs[0] (1 frame 16x16x32, b 4, 4 of 16 blocks): the whole path on one thread.
    configs[1] (1 frame 72x72x320, b 8): the conv at 10% (8 blocks) on one thread and on all
    cores (OpenMP over blocks, 16 per chunk: 8 blocks keep one thread busy).
    configs[2..4]: their full steps' conv FLOPs (from the GPU run) at the one-thread rate and at
    rate_all_cores (the cpu_baseline sample's measured all-core rate, FLOP/s), labelled
    extrapolated (the full runs are minutes to hours of CPU time)."""
    import oracle
    cores = os.cpu_count()
    out = {"cores": cores, "kind": "oracle"}
    # configs[0], everything on one thread (the conv's OpenMP pinned to 1)
    n, hp, b, c, S, u = 1, 16, 4, 32, 50, 25
    O, _ = syn.opacity_maps(n, hp, hp, b, [0.25], "scattered", tag="smoke")
    q, c0, c1, t = (np.float32([61.75]), np.float32([60]), np.float32([70]), np.float32([0.25]))
    lg = oracle.make_klogic(syn.SPEC_KLOGIC["thr"], syn.SPEC_KLOGIC["steps"])
    abar = syn.abar_cosine(S)
    x0 = syn.latents_f32((n, hp, hp, c), "smoke-x0")
    eps = syn.latents_f32((n, hp, hp, c), "smoke-eps")
    w = syn.weights_bf16(c, c, "smoke")
    bias = syn.bias_f32(c, "smoke")
    cache = syn.latents_f32((n, hp, hp, c), "smoke-cache")
    t0 = time.perf_counter()
    om, _ = oracle.block_mask(O, None, None, 0.5, 1, b, 1)
    ok = oracle.start_step(q, c0, c1, t, 0.5, [lg])
    oids = oracle.compact(om[0], ok, u)
    xt = oracle.noise(x0, eps, x0, b, oids, ok, abar).astype(np.float32)
    xbits = syn.to_bf16_bits(xt)
    oy, _ = oracle.conv3x3_blocks(xbits, w, bias, b, oids, n_threads=1, y_init=cache.astype(np.float64))
    oracle.scatter(oy.astype(np.float32), cache, b, mask=om[0], k=ok, u=u)
    t_c0 = time.perf_counter() - t0
    out["configs0_path_1thread_s"] = round(t_c0, 5)
    out["configs0_conv_flops"] = int(len(oids) * b * b * 2 * 9 * c * c)
    # configs[1]: 8 of 81 blocks of one 72x72x320 frame
    h, c = 72, 320
    x = syn.features_bf16((1, h, h, c), "sweep")
    w = syn.weights_bf16(c, c, "sweep")
    rg = syn.rng("sweep-mask", 1, 0.10)
    ids = np.flatnonzero(syn.choose_cells(rg, 9, 9, 8, "clustered").ravel()).astype(np.int32)
    fl = len(ids) * 64 * 2 * 9 * c * c
    t0 = time.perf_counter()
    oracle.conv3x3_blocks(x, w, None, 8, ids[:1], n_threads=1)
    t1 = time.perf_counter() - t0
    nb1 = int(max(1, min(len(ids), seconds_1core / max(t1, 1e-3))))
    t0 = time.perf_counter()
    oracle.conv3x3_blocks(x, w, None, 8, ids[:nb1], n_threads=1)
    t1 = time.perf_counter() - t0
    rate1 = nb1 * 64 * 2 * 9 * c * c / t1
    t0 = time.perf_counter()
    oracle.conv3x3_blocks(x, w, None, 8, ids, n_threads=cores)  # (also restores the thread count)
    tall = time.perf_counter() - t0
    out["configs1_conv_10pct"] = {"blocks": int(len(ids)), "gflop": round(fl / 1e9, 4),
                                  "s_1thread": round(t1 * len(ids) / nb1, 4),
                                  "s_1thread_note": f"measured on {nb1} of {len(ids)} blocks, scaled by block count",
                                  "s_all_cores": round(tall, 4),
                                  "gflops_1thread": round(rate1 / 1e9, 4)}
    out["extrapolated"] = {k: {"conv_gflop": round(v / 1e9, 1), "s_all_cores": round(v / rate_all_cores, 1),
                               "s_1thread": round(v / rate1, 1)}
                           for k, v in conv_flops_by_config.items()}
    out["extrapolated_note"] = ("full-step conv FLOPs from the GPU run / the measured fp64 direct-conv rate: one "
                                "thread (configs[1] above), all cores (the cpu_baseline sample's rate, "
                                f"{rate_all_cores / 1e9:.2f} GFLOP/s, mask/compaction/noise/scatter included)")
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.workload
    cfg = step_config(WORKLOADS[name]["means"])
    batch = make_batch(name)
    cores = os.cpu_count()
    nb = calibrate_blocks(batch, cfg, 150.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        oracle_step_sample(batch, cfg, nb)
    ts, fl = [], 0
    for _ in range(args.steps):
        t, f = oracle_step_sample(batch, cfg, nb)
        ts.append(t)
        fl = f
    ms = statistics.mean(ts) * 1e3
    value = fl / (ms * 1e-3) / 1e12
    sample = (f"bounded sample of {name}: full mask/start-step/compaction/noise/scatter over the {cfg.n_frames} "
              f"frames, conv on the first {nb} active blocks per level")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 8), "unit": "TFLOP/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[name]["desc"] + " (bounded oracle sample)", "frames": cfg.n_frames},
        "cpu_baseline": {"value": round(value, 8), "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(value, 8), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args):
    """--gpus N > 1 without a torchrun environment: re-execute under torch.distributed.run, one
    process per GPU on this node; rank 0 prints the JSON line."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
    env.setdefault("NCCL_DEBUG_FILE", "/tmp/sphinx_nccl.%h.%p.log")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="configs3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-extras", action="store_true", help="headline workload only")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-resblock", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo + --share-gpu: exercise the multi-rank path with every rank on cuda:0")
    ap.add_argument("--share-gpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-flush", action="store_true", help="diagnostic: keep L2 warm between steps")
    ap.add_argument("--profile", action="store_true",
                    help="ncu mode: capture the step graph, replay it twice (warm-up + profiled), exit")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.profile:
        run_profile(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    else:
        if int(os.environ.get("WORLD_SIZE", "1")) > 1:
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/sphinx_nccl.%h.%p.log")
        run_gpu(args)


if __name__ == "__main__":
    main()
