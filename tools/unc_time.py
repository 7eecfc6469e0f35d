import sys, os, json, torch
sys.path.insert(0, os.getcwd())
import bench, synthetic as syn, paper_2511_18672_b200 as sp
sp.load(os.environ["SPHINX_LIB"]) if os.environ.get("SPHINX_LIB") else sp.load(); dev = torch.device("cuda", 0)
for src in ("rand", "frames"):
    rgb = torch.rand((21, 576, 576, 3), device=dev) if src == "rand" else torch.from_numpy(syn.rgb_frames(21, 576, 576, "bench")).to(dev)
    U = torch.empty((21, 576, 576), device=dev); tau = torch.empty((21,), device=dev)
    t = bench.graph_time(torch, lambda: sp.sphinx_uncertainty_map(rgb, U, tau))
    print(json.dumps({"lib": os.environ.get("SPHINX_LIB", "default"), "uncertainty": src, "ms": round(t, 5)}))
