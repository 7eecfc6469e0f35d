"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU host logic."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys_path_tests = os.path.dirname(os.path.abspath(__file__))

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


def _lpt_reference(costs, world):
    """The LPT rule written out literally (the definition dist.lpt_assign implements): frames by
    cost descending, ties by lower frame id; each goes to the least-loaded rank, ties lowest rank."""
    costs = [int(c) for c in costs]
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0] * world
    assign = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda j: (load[j], j))
        assign[r].append(i)
        load[r] += costs[i]
    return [sorted(a) for a in assign], load


def test_lpt_matches_the_rule():
    rg = np.random.default_rng(3)
    cases = [rg.integers(0, 10_000, size=168), rg.integers(0, 4, size=168),  # tie-heavy
             np.zeros(21, np.int64), rg.integers(0, 2**40, size=200), np.array([7]), np.array([], np.int64)]
    for costs in cases:
        for world in (1, 2, 3, 4, 8):
            assign, load = sdist.lpt_assign(costs, world)
            want_a, want_l = _lpt_reference(costs, world)
            assert [a.tolist() for a in assign] == want_a
            assert load.tolist() == want_l


def test_frame_costs_weighting():
    # a level-2 block (1280 ch) costs 16x a level-0 block (320 ch)
    c = sdist.frame_costs([[1, 0, 0], [0, 0, 1]], [320, 640, 1280])
    assert c[1] == 16 * c[0]


# ------------------------------------------------------------------ the sharded step

def _small_cfg():
    from paper_2511_18672_b200.step import StepConfig
    # 4 requests x 6 frames of 48x48 images, f=4 -> 12x12 latent; levels 12/6/3 with 4x4 blocks
    # (ragged edge blocks at 6 and 3)
    return StepConfig(hp=48, f=4, b=4, levels=((12, 16), (6, 32), (3, 32)), convs_per_level=2,
                      frames_per_request=6, n_requests=4, u=25, gamma=0.5)


def _small_batch():
    import synthetic as syn
    cfg = _small_cfg()
    return syn.make_batch([0.3, 0.9, 0.1, 0.6], tag="gloo-step", hp=cfg.hp, f=cfg.f, b=cfg.b, levels=cfg.levels,
                          convs_per_level=cfg.convs_per_level, frames_per_request=cfg.frames_per_request)


def _step_outputs(st):
    cfg = st.cfg
    outs = [st.out(l).view(torch.int16).numpy().copy() for l in range(cfg.L)]
    return outs, st.lat_out.numpy().copy()


def _step_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, sys_path_tests)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle_ops
        from paper_2511_18672_b200.step import RefinementStep
        cfg = _small_cfg()
        st = RefinementStep(cfg, _small_batch(), "cpu", oracle_ops, rank=rank, world=world)
        for _ in range(2):  # two steps: persistent buffers and the plan are reused across steps
            st.run()
        outs, lat = _step_outputs(st)
        q.put((rank, outs, lat, st.plan["rank_of"].tolist(), st.bytes_sent, st.k_mine.numpy().tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_sharded_step_matches_single_rank(world):
    """The whole data plane at world 2 and 4 (gloo, CPU, oracle compute): mask slices, the
    mask/start-step all-gather, the LPT plan, compaction over assigned frames and the owner
    gather of refined blocks.  Every owner's buffers (the last conv of every level and the
    latent) equal a single-rank step over the whole batch bit for bit, for its requests' frames."""
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import oracle_ops
    from paper_2511_18672_b200.step import RefinementStep
    cfg = _small_cfg()
    ref = RefinementStep(cfg, _small_batch(), "cpu", oracle_ops)
    ref.run()
    ref.run()
    want_outs, want_lat = _step_outputs(ref)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    owner = cfg.owner_of_frame(world)
    plans = [r[3] for r in res]
    assert all(p == plans[0] for p in plans)              # every rank derived the same plan
    rank_of = np.array(plans[0])
    assert (rank_of != owner).any()                       # some frames are computed off-owner
    assert sum(r[4] for r in res) > 0                     # ... so refined blocks moved
    for rank, outs, lat, _, _, kmine in res:
        mine = owner == rank
        for l in range(cfg.L):
            assert np.array_equal(outs[l][mine], want_outs[l][mine]), (rank, l)
        assert np.array_equal(lat[mine].view(np.uint32), want_lat[mine].view(np.uint32)), rank
        # this rank compacted exactly the frames assigned to it
        assert all((kmine[n] == -1) == (rank_of[n] != rank or ref.k[n].item() == -1) for n in range(cfg.n_frames))
