"""bench.py's driver contract on the GPU: the JSON line of a 1-GPU run, and the N-rank path
(self-launch under torch.distributed.run, frame sharding, owner gather) with 2 ranks sharing the
test GPU over gloo (functional: its timings mean nothing).  The round-end driver runs the same
script with NCCL on N GPUs; this is the closest check one GPU allows."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=1200):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_one_gpu():
    d = _run(["--steps", "2", "--warmup", "3", "--no-sweep", "--no-resblock", "--cpu-seconds", "2"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "gpu_launches", "roofline", "clocks", "e2e",
              "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] >= 3 and d["value"] > 0
    assert d["unit"] == "TFLOP/s" and d["higher_is_better"] is True and d["data"] == "synthetic"
    assert "workload" in d["config"] and d["config"]["workload"].startswith("configs[3]")
    assert isinstance(d["gpu_launches"], int) and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_bench_two_ranks_self_launch():
    d = _run(["--gpus", "2", "--dist-backend", "gloo", "--share-gpu", "--steps", "2", "--warmup", "3"])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    m = d["multi_gpu"]
    assert m["ranks"] == 2 and m["plan_imbalance_max_over_mean"] >= 1.0 and m["bytes_moved_per_step"] > 0
    assert isinstance(d["gpu_launches"], int) and d["gpu_launches"] > 0
