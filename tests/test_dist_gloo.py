"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU host logic."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_18672_b200 import dist as sdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, counts, channels, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = counts.shape[0]
        mine = sdist.round_robin(n, world, rank)
        local = torch.from_numpy(counts[mine].astype(np.int32))
        full = sdist.gather_counts(local, mine, n)
        assign, load = sdist.lpt_assign(sdist.frame_costs(full, channels), world)
        ms, work = sdist.reduce_step(1.0 + rank, 10.0 * (rank + 1))
        q.put((rank, full, [a.tolist() for a in assign], load.tolist(), ms, work))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_counts_plan_and_reduction():
    rg = np.random.default_rng(7)
    counts = rg.integers(0, 82, size=(21, 3))
    counts[:, 1] = np.minimum(counts[:, 1], 25)
    counts[:, 2] = np.minimum(counts[:, 2], 9)
    channels = [320, 640, 1280]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, counts, channels, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    (_, full0, asg0, load0, ms0, w0), (_, full1, asg1, load1, ms1, w1) = res
    # the all-gather reconstructs the full count table on both ranks
    assert np.array_equal(full0, counts) and np.array_equal(full1, counts)
    # both ranks derive the same plan; every frame exactly once
    assert asg0 == asg1 and load0 == load1
    assert sorted(asg0[0] + asg0[1]) == list(range(21))
    # timing: max of the per-rank step times, sum of the work
    assert ms0 == ms1 == 2.0 and w0 == w1 == 30.0


def test_lpt_balance_and_determinism():
    rg = np.random.default_rng(11)
    for world in (2, 4, 8):
        costs = rg.integers(0, 10_000, size=168)
        assign, load = sdist.lpt_assign(costs, world)
        assert sorted(np.concatenate(assign).tolist()) == list(range(168))
        assert np.array_equal(load, [costs[a].sum() for a in assign])
        # Graham's LPT bound: max load <= mean + max single cost
        assert load.max() <= costs.sum() / world + costs.max()
        assign2, _ = sdist.lpt_assign(costs, world)
        assert all(np.array_equal(a, b) for a, b in zip(assign, assign2))
    # ties: equal costs go round-robin from rank 0 in frame order
    a, _ = sdist.lpt_assign([5, 5, 5, 5], 2)
    assert a[0].tolist() == [0, 2] and a[1].tolist() == [1, 3]


def test_frame_costs_weighting():
    # a level-2 block (1280 ch) costs 16x a level-0 block (320 ch)
    c = sdist.frame_costs([[1, 0, 0], [0, 0, 1]], [320, 640, 1280])
    assert c[1] == 16 * c[0]
