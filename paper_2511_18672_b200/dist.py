"""Multi-GPU host logic (one process per GPU, torch.distributed) — plumbing, no compute.

The hot path shards naturally by frame: spatial ResNet/conv layers act per frame,
so frames (and whole requests) are independent units.  Two schemes are supported:

* weak scaling (bench.py default): every rank runs its own request; the only collectives
  are the timing reductions (max over ranks of the step time, sum of the work).
* frame sharding of a request batch (BASELINE configs[3]: 8 requests x 21 frames): ranks
  all-gather the per-frame, per-level active-block counts produced by sphinx_block_mask
  (one NCCL all_gather of N x L int32 -- the only exchange the partition needs) and every
  rank computes the SAME deterministic LPT assignment of frames to ranks, weighted by the
  executed MMA work cost_n = sum_l count[n,l] * C_l^2 (a level-l block costs (C_l/C_0)^2
  level-0 blocks of work).
"""
import heapq

import numpy as np


def frame_costs(counts, channels):
    """counts: int [N, L] active blocks per frame and level; channels: [L] C_l.
    Returns int64 [N] cost in units of (block x C^2)."""
    counts = np.asarray(counts, dtype=np.int64)
    c2 = np.asarray(channels, dtype=np.int64) ** 2
    return (counts * c2[None, :]).sum(axis=1)


def lpt_assign(costs, world):
    """Longest-processing-time-first: frames sorted by cost descending (ties: lower frame id
    first) go to the currently least-loaded rank (ties: lowest rank).  Deterministic, so
    every rank computes the same plan from the same gathered counts.
    Returns (list of frame-id arrays per rank, int64 load per rank).
    (Runs once per sharded step on every rank, between the mask all-gather and the compaction:
    plain Python ints and a (load, rank) heap -- the heap order is exactly "least loaded, then
    lowest rank" -- keep it at ~0.1 ms for 168 frames; a numpy-scalar loop took ~0.9 ms.)"""
    costs = np.asarray(costs, dtype=np.int64)
    order = np.lexsort((np.arange(len(costs)), -costs)).tolist()  # cost desc, then frame id
    cl = costs.tolist()
    heap = [(0, r) for r in range(world)]  # already a heap
    rank_of = [0] * len(cl)
    for i in order:
        ld, r = heap[0]
        rank_of[i] = r
        heapq.heapreplace(heap, (ld + cl[i], r))
    rank_of = np.asarray(rank_of, dtype=np.int64)
    load = np.bincount(rank_of, weights=costs, minlength=world).astype(np.int64) if len(cl) else \
        np.zeros(world, dtype=np.int64)
    idx = np.arange(len(cl), dtype=np.int64)
    return [idx[rank_of == r] for r in range(world)], load


def round_robin(n, world, rank):
    """Frames whose masks this rank computes before the counts all-gather."""
    return np.arange(rank, n, world, dtype=np.int64)


def gather_counts(local_counts, frame_ids, n_frames, group=None):
    """All-gathers per-frame counts computed on round-robin slices.  local_counts: int32
    tensor [len(frame_ids), L] on this rank's device (or CPU for gloo).  Returns the full
    [n_frames, L] int64 numpy array, identical on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    L = local_counts.shape[1]
    per = -(-n_frames // world)
    pad = torch.zeros((per, L), dtype=torch.int32, device=local_counts.device)
    pad[: local_counts.shape[0]] = local_counts
    out = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    full = np.zeros((n_frames, L), dtype=np.int64)
    for r in range(world):
        ids = round_robin(n_frames, world, r)
        full[ids] = out[r][: len(ids)].cpu().numpy()
    return full


def reduce_step(ms, work, device=None, group=None):
    """Max over ranks of the device step time and sum of the work: the whole-job throughput
    is sum(work) / max(ms).  Returns (ms_max, work_sum)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    w = torch.tensor([float(work)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(w, op=dist.ReduceOp.SUM, group=group)
    return float(t.item()), float(w.item())
