"""Summarise tools/next_profile.sh launch lists (NEXT-3 / NEXT-4) as markdown (CPU box).
    python tools/next_summary.py <tag> >> profiles/<tag>_ncu_summary.md"""
import csv
import io
import os
import sys

tag = sys.argv[1]
d0 = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
out = ["", "## NEXT-3 / NEXT-4 kernels (ncu launch lists, `tools/next_profile.sh`)", "",
       "One level, 21 frames, 25% clustered blocks; the last partial step after a full step. Cold, "
       "serialised per-launch metrics (ncu): compare shares, not absolutes.", ""]
for kind, title, last in (("rbprof", "ResNet block (NEXT-3): 2 x (stats, finalize, gn_silu, [plan], conv)", 8),
                          ("taprof", "Temporal block (NEXT-4): qkv pointwise, plan, attention, out pointwise", 4)):
    for l in (0, 2):
        path = os.path.join(d0, f"{tag}_{kind}_l{l}.csv")
        if not os.path.exists(path):
            continue
        txt = open(path).read()
        txt = txt[txt.index('"ID"'):]
        byid = {}
        for r in csv.DictReader(io.StringIO(txt)):
            byid.setdefault(r["ID"], {"k": r["Kernel Name"].split("(")[0].replace("void ", "")[:48]})[
                r["Metric Name"]] = r["Metric Value"]
        ids = sorted(byid, key=int)
        n = last + (2 if (kind == "rbprof" and l > 0) else 0)
        out += [f"{title}, level {l}:", "", "| kernel | us | dram read MB | dram write MB | grid | SM thr % |",
                "|---|---|---|---|---|---|"]
        for i in ids[-n:]:
            d = byid[i]
            out.append(f"| `{d['k']}` | {float(d['gpu__time_duration.sum']) / 1000:.1f} | "
                       f"{float(d['dram__bytes_read.sum']) / 1e6:.1f} | {float(d['dram__bytes_write.sum']) / 1e6:.1f} | "
                       f"{d['launch__grid_size']} | {d['sm__throughput.avg.pct_of_peak_sustained_elapsed']} |")
        out.append("")
print("\n".join(out))
