"""Dev A/B: the step's HBM-bound elementwise kernels (noise injection, DDIM update) of two
library builds, on configs[3]-sized latents (168 x 72x72x4 fp32, a 13 608-entry list).

    SPHINX_LIB=<path> python tools/mem_ab.py

warm: CUDA-graph replay of 20 launches (L2-warm); cold: one launch in a graph replayed right
behind a 256 MB write + 256 MB read L2 flush (bench.py memory_kernels' protocol)."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18672_b200 as sp  # noqa: E402
import synthetic as syn  # noqa: E402


def cold(fn, flush, reps=12, flush_r=[]):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    ts = []
    for i in range(reps):
        flush.fill_(0.0)
        if not flush_r:
            flush_r.append(torch.zeros_like(flush))
        flush_r[0].amax()  # clean L2 (bench.py memory_kernels' protocol)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    sp.load(os.environ["SPHINX_LIB"]) if os.environ.get("SPHINX_LIB") else sp.load()
    dev = torch.device("cuda", 0)
    n, h, c, b, S = 168, 72, 4, 8, 50
    hb = h // b
    x0 = torch.from_numpy(syn.latents_f32((n, h, h, c), "memab-x0")).to(dev)
    eps = torch.from_numpy(syn.latents_f32((n, h, h, c), "memab-eps")).to(dev)
    xt = torch.empty_like(x0)
    zo = torch.empty_like(x0)
    rg = np.random.default_rng(5)
    ids_np = np.flatnonzero(rg.random(n * hb * hb) < 1.0).astype(np.int32)  # every block (13 608)
    ids = torch.from_numpy(ids_np).to(dev)
    cnt = torch.tensor([len(ids_np)], dtype=torch.int32, device=dev)
    k = torch.from_numpy(rg.integers(0, 40, n).astype(np.int32)).to(dev)
    abar = torch.from_numpy(syn.abar_cosine(S)).to(dev)
    abar_h = abar.cpu().numpy()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    nbytes = len(ids_np) * 64 * c * 12
    out = {"lib": os.path.basename(os.environ.get("SPHINX_LIB", "libsphinx.so")), "mbytes": round(nbytes / 1e6, 2)}
    f_noise = lambda: sp.sphinx_noise_inject_step(x0, eps, xt, b, ids, cnt, k, 25, abar)
    f_ddim = lambda: sp.sphinx_ddim_step(xt, x0, zo, b, ids, cnt, 25, abar_h)
    for name, f in (("noise", f_noise), ("ddim", f_ddim)):
        out[name + "_warm_us"] = round(bench.graph_time(torch, f) * 1e3, 2)
        out[name + "_cold_us"] = round(cold(f, flush) * 1e3, 2)
    # step 1 (block mask + counts + start steps) at the configs[2] and configs[3] frame counts
    for nf in (21, 168):
        O, cells = syn.opacity_maps(nf, 576, 576, 64, list(syn.request_densities(nf)), "clustered", tag="memab")
        U, tau = syn.uncertainty_maps(nf, 576, 576, 64, cells, tag="memab")
        Od, Ud, taud = (torch.from_numpy(a).to(dev) for a in (O, U, tau))
        masks = [torch.empty((nf, 9 >> l if l == 0 else -(-9 // (1 << l)), 9 if l == 0 else -(-9 // (1 << l))),
                             dtype=torch.uint8, device=dev) for l in range(3)]
        counts = torch.empty((nf, 3), dtype=torch.int32, device=dev)
        f_mask = lambda: sp.sphinx_block_mask(Od, Ud, taud, 0.5, 8, 8, masks, counts, None, None)
        out[f"mask{nf}_mbytes"] = round(nf * 576 * 576 * 8 / 1e6, 1)
        out[f"mask{nf}_warm_us"] = round(bench.graph_time(torch, f_mask) * 1e3, 2)
        out[f"mask{nf}_cold_us"] = round(cold(f_mask, flush) * 1e3, 2)
        # step 2: the step's batched compaction (3 ACTIVE lists + the NOISE list) over these masks
        kk = torch.from_numpy(rg.integers(0, 40, nf).astype(np.int32)).to(dev)
        f_mask()
        lists = [(torch.empty((nf * m.shape[1] * m.shape[2],), dtype=torch.int32, device=dev),
                  torch.empty((1,), dtype=torch.int32, device=dev)) for m in masks + masks[:1]]
        jobs = [dict(block_mask=masks[l], start_step=kk, step_u=25, select=sp.SELECT_ACTIVE, block_ids=lists[l][0],
                     count=lists[l][1]) for l in range(3)] + \
               [dict(block_mask=masks[0], start_step=kk, step_u=25, select=sp.SELECT_NOISE, block_ids=lists[3][0],
                     count=lists[3][1])]
        f_comp = lambda: sp.sphinx_compact_blocks_batch(jobs)
        out[f"compact{nf}_warm_us"] = round(bench.graph_time(torch, f_comp) * 1e3, 2)
        out[f"compact{nf}_cold_us"] = round(cold(f_comp, flush) * 1e3, 2)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
