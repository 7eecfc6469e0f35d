"""Summarise ncu output for profiles/ (runs on the CPU box).

    python tools/ncu_summary.py <tag> [--launches X.csv] [--rep X.ncu-rep] [--bench X.json] > profiles/<tag>.md

Launch list: per-kernel count, mean/total device time and share of the step (cold, serialised
by ncu: compare SHARES, not absolutes).  Full capture: per-launch duration, tensor-pipe and
DRAM metrics, dram bytes (the `traffic` figure), achieved TMA ingress.
"""
import argparse
import csv
import json
import subprocess
import sys
from collections import OrderedDict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0].replace("void ", "")
            v = float(d["Metric Value"].replace(",", ""))
            unit = d.get("Metric Unit", "ns")
            v = v / 1000.0 if unit == "ns" else v  # -> us
            agg.setdefault(name, []).append(v)
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: (v + (" " + u if u else "")) for h, v, u in zip(hdr, r, units)}
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--bench")
    ap.add_argument("--mem", help="ncu --set full capture of the HBM-bound kernels")
    a = ap.parse_args()
    print(f"# ncu summary — {a.tag}\n")
    if a.bench:
        b = json.load(open(a.bench))
        print("## bench line (same build)\n")
        print(f"- value: **{b['value']} {b['unit']}**, ms_per_step {b['ms_per_step']}, clocks {b.get('clocks')}")
        print(f"- roofline: `{json.dumps(b['roofline'])}`")
        for lv in b.get("conv_levels", []):
            print(f"- conv level {lv['level']} {lv['shape']}: {lv['active_blocks']} blocks, {lv['conv_ms']} ms, "
                  f"{lv['tflops']} TFLOP/s")
        print()
    if a.launches:
        agg = launches(a.launches)
        tot = sum(sum(v) for v in agg.values())
        print("## launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, `bench.py --profile`)\n")
        print("Cold-cache, serialised per-launch times of 4 steps (2 eager capture warm-ups, 2 graph "
              "replays): compare shares, not absolutes.\n")
        print("| kernel | launches | mean us | total us | share |")
        print("|---|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            print(f"| `{k[:70]}` | {len(v)} | {sum(v)/len(v):.1f} | {sum(v):.1f} | {sum(v)/tot:.1%} |")
        print()
    if a.rep:
        rows = full(a.rep)
        keys = [("gpu__time_duration.sum", "us"), ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "%"),
                ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "%"),
                ("dram__bytes_read.sum", "B"), ("dram__bytes_write.sum", "B"),
                ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum.per_second", "B/s"),
                ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
                ("sm__cycles_elapsed.avg.per_second", "Hz")]
        print("## full capture (`ncu --set full --clock-control none`)\n")
        print("| kernel | grid | " + " | ".join(k.split('.')[0].replace('__', ' ') for k, _ in keys) + " |")
        print("|---" * (len(keys) + 2) + "|")
        for d in rows:
            vals = [d.get(k, "") for k, _ in keys]
            print(f"| `{d.get('Kernel Name','')[:60]}` | {d.get('Grid Size','')} | " + " | ".join(vals) + " |")
        print("\n(dram bytes in the unit ncu reports; `traffic` = read + write per launch)")
    if a.mem:
        rows = full(a.mem)
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "launch__grid_size"]
        print("\n## HBM-bound kernels of the step (`ncu --set full --clock-control none`)\n")
        print("| kernel | " + " | ".join(k.split('.')[0].replace('__', ' ') for k in keys) + " | achieved GB/s |")
        print("|---" * (len(keys) + 2) + "|")
        for d in rows:
            def num(k):
                v = d.get(k, "0 ").split()
                x = float(v[0].replace(",", ""))
                u = v[1] if len(v) > 1 else ""
                return x * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9}.get(u, 1)
            gbs = (num("dram__bytes_read.sum") + num("dram__bytes_write.sum")) / max(num("gpu__time_duration.sum"), 1e-12) / 1e9
            print(f"| `{d.get('Kernel Name','')[:50]}` | " + " | ".join(d.get(k, "") for k in keys) + f" | {gbs:.0f} |")


if __name__ == "__main__":
    main()
