"""One refinement step of the Sphinx hot path over a batch of requests, on one rank or sharded
across the ranks of a process group.

This is the public call a serving loop makes once per denoising step u (Alg1 lines 13-19,
P:396).  Argument marshalling and orchestration only: every step of the path runs in the
kernels behind the C ABI (include/sphinx.h), reached through ``ops`` (the
``paper_2511_18672_b200`` binding).  PyTorch supplies device memory, streams and
``torch.distributed``.

Single rank (world = 1): one stream, every launch PDL-chained, CUDA-graph capturable:
    sphinx_block_mask (a1 + a2) -> sphinx_compact_blocks_batch (a3: the L levels' ACTIVE lists at
    u + the NOISE list) -> sphinx_conv_edge_plan (ragged levels) -> sphinx_noise_inject_step
    (a4: active latent blocks to their start step k, Alg1 line 12, and inactive frames resampled
    to u+1, line 19, in one pass) -> per level `convs_per_level` x sphinx_sparse_conv3x3 C->C in persistent-
    buffer mode (a5; the feature-level scatter a6 fused into the epilogue, R-17) ->
    sphinx_scatter_cached of the latent (a6 at latent resolution, P:352 latent reuse).

Sharded (world = N > 1; "spatial ResNet layers ... per frame"):
    1. every rank runs sphinx_block_mask on its contiguous slice of F/N frames;
    2. C1: NCCL all-gather of the slices' block masks and start steps (the per-frame active
       counts follow from them), so every rank holds the whole batch's masks;
    3. every rank computes the SAME deterministic LPT plan ON THE DEVICE (sphinx_shard_plan, frames
       weighted by executed MMA work sum_l count[n,l] C_l^2 at this u; the host twin is make_plan /
       dist.lpt_assign); the host reads the exchange sizes back only when it issues the exchange,
       after the convs are queued;
    4. compaction over the frames assigned to this rank (k of other frames masked to -1), then
       noise, convs and the latent scatter exactly as on one rank;
    5. C2: after each level, the refined blocks of frames owned by another rank (request j is
       owned by rank j*N // R, a contiguous frame range) are packed in list order
       (sphinx_gather_blocks), sent with one grouped NCCL send/recv (sizes known from the plan),
       and unpacked into the owner's persistent buffers (sphinx_scatter_blocks), on a
       communication stream that overlaps the next level's convs.  The latent's refined blocks
       travel the same way with the level-0 list.
After a step, each owner's buffers hold exactly what a single-rank step over the whole batch
leaves in them for its requests' frames (bit for bit: every block is computed by exactly one
rank with the same kernels, and the copies are bit copies).

Inputs are replicated on every rank (the request data, generated from the same seeds: the
synthetic-benchmark equivalent of broadcasting a request's inputs once when it arrives,
amortised over its denoising steps); nothing of them moves per step.
"""
import contextlib

import numpy as np

from . import dist as sdist


class StepConfig:
    """Geometry of a batch: n_requests x frames_per_request frames of hp x hp images (f image
    pixels per level-0 cell), UNet `levels` [(H_l, C_l)], b x b blocks, step u."""

    def __init__(self, hp=576, f=8, b=8, levels=((72, 320), (36, 640), (18, 1280)), convs_per_level=2,
                 frames_per_request=21, n_requests=1, u=25, gamma=0.5, tau_o=0.5, c_lat=4,
                 interleave_levels=True, conv_variant=None):
        self.hp, self.f, self.b = hp, f, b
        # per-level kernel-variant flags of sphinx_sparse_conv3x3_ex (A/B and tests; None = the
        # library's default choice)
        self.conv_variant = conv_variant
        self.interleave_levels = interleave_levels  # conv launch order (RefinementStep.conv_order)
        self.levels = [tuple(x) for x in levels]
        self.convs_per_level = convs_per_level
        self.frames_per_request, self.n_requests = frames_per_request, n_requests
        self.n_frames = frames_per_request * n_requests
        self.u, self.gamma, self.tau_o, self.c_lat = u, gamma, tau_o, c_lat
        self.h0 = hp // f
        self.hb = [-(-h // b) for (h, _) in self.levels]
        self.L = len(self.levels)

    def owner_of_frame(self, world):
        """Rank owning each frame's request: request j -> j * world // R (contiguous ranges)."""
        req = np.arange(self.n_frames) // self.frames_per_request
        return (req * world) // self.n_requests

    def real_px(self, l, ids):
        """Real (in-image) pixels of the listed level-l blocks (truncated edge blocks, R-2)."""
        h, hb, b = self.levels[l][0], self.hb[l], self.b
        r = np.asarray(ids) % (hb * hb)
        by, bx = r // hb, r % hb
        return int((np.minimum(b, h - by * b) * np.minimum(b, h - bx * b)).sum())


class _Transport:
    """Point-to-point and all-gather over a torch.distributed group.  NCCL moves device tensors
    directly; gloo (CPU tests, or several ranks sharing one GPU in the GPU tests) stages through
    host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.backend = dist.get_backend(group)

    def _host(self, t):
        return t if (self.backend == "nccl" or not t.is_cuda) else None

    def all_gather_into(self, out, inp):
        """out: [world * m, ...] contiguous; inp: [m, ...] (the rank's slice)."""
        dist = self.dist
        if self.backend == "nccl":
            dist.all_gather_into_tensor(out, inp, group=self.group)
            return
        world = dist.get_world_size(self.group)
        src = inp.detach().to("cpu", copy=True).contiguous()
        parts = [torch_empty_like_cpu(src) for _ in range(world)]
        dist.all_gather(parts, src, group=self.group)
        out.copy_(torch_cat(parts))

    def exchange(self, sends, recvs):
        """sends: [(dst_rank, tensor)], recvs: [(src_rank, tensor)], byte-typed contiguous
        tensors; one grouped batch of isend/irecv, waited on the current stream."""
        dist = self.dist
        if not sends and not recvs:
            return
        if self.backend == "nccl":
            ops = [dist.P2POp(dist.isend, t, r, self.group) for r, t in sends] + \
                  [dist.P2POp(dist.irecv, t, r, self.group) for r, t in recvs]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            return
        stage_s = [(r, t.cpu() if t.is_cuda else t) for r, t in sends]
        stage_r = [(r, t, torch_empty_like_cpu(t) if t.is_cuda else t) for r, t in recvs]
        ops = [dist.P2POp(dist.isend, t, r, self.group) for r, t in stage_s] + \
              [dist.P2POp(dist.irecv, h, r, self.group) for r, _, h in stage_r]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        for _, t, h in stage_r:
            if t is not h:
                t.copy_(h)


def torch_int32():
    import torch
    return torch.int32


def torch_cat(parts):
    import torch
    return torch.cat(parts)


def torch_empty_like_cpu(t):
    import torch
    return torch.empty(t.shape, dtype=t.dtype, device="cpu")


def _bytes(t):
    import torch
    return t.reshape(-1).view(torch.uint8)


class RefinementStep:
    """Device state of one batch of requests on this rank + the step.

    inputs: host numpy arrays (bench.make_batch / the tests' generators): O, U, tau_u [F,Hp,Wp]
    / [F]; q, c0, c1, t [F] fp32; lid [F] int32 (-1 = conditioning frame, R-14); abar [S+1];
    x0, eps, lat_cache [F,H0,H0,C_lat] fp32; feat{l}, cache{l} [F,H_l,H_l,C_l] bf16 bits (uint16);
    w{l}{j} [C_l,3,3,C_l] bf16 bits, b{l}{j} [C_l] fp32; klogic dict(thr, steps, fallback_k, k_max).
    ops: the binding module (or a stand-in exposing the same calls).  group: torch.distributed
    process group or None (single rank)."""

    def __init__(self, cfg, inputs, device, ops, group=None, rank=0, world=1, host_features=None):
        """host_features: None (the level input features feat{l} are device-resident step inputs) or
        {l: pinned host bf16 tensor [F,H_l,H_l,C_l]}: each step then moves only the halo windows of
        its listed blocks over PCIe into the device maps (sphinx_gather_halo_windows), i.e. exactly
        what the level's first conv reads."""
        import torch
        self.cfg, self.ops, self.torch = cfg, ops, torch
        self.host_features = host_features
        self.dev = torch.device(device)
        self.rank, self.world = rank, world
        self.cuda = self.dev.type == "cuda"
        F, L, b = cfg.n_frames, cfg.L, cfg.b
        if F % world:
            raise ValueError(f"{F} frames do not split evenly over {world} ranks")
        if world > 1 and cfg.n_requests < world:
            raise ValueError("fewer requests than ranks")

        def put(a):
            a = np.ascontiguousarray(a)
            if a.dtype == np.uint16:  # bf16 bit patterns
                return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).to(self.dev)
            return torch.from_numpy(a).to(self.dev)
        self.d = {k: put(v) for k, v in inputs.items() if isinstance(v, np.ndarray)}
        kl = inputs["klogic"]
        self.logics = [ops.make_klogic(kl["thr"], kl["steps"], kl.get("fallback_k", 0), kl.get("k_max", 40))]
        i32, u8 = torch.int32, torch.uint8
        self.masks = [torch.zeros((F, hb, hb), dtype=u8, device=self.dev) for hb in cfg.hb]
        self.counts = torch.zeros((F, L), dtype=i32, device=self.dev)
        self.k = torch.full((F,), -1, dtype=i32, device=self.dev)
        self.k_mine = self.k if world == 1 else torch.full((F,), -1, dtype=i32, device=self.dev)
        self.ids = [torch.zeros((F * hb * hb,), dtype=i32, device=self.dev) for hb in cfg.hb]
        self.cnt = [torch.zeros((1,), dtype=i32, device=self.dev) for _ in range(L)]
        # the noise pass's list: active blocks of active frames + every block of inactive frames
        self.ids_noise = torch.zeros((F * cfg.hb[0] ** 2,), dtype=i32, device=self.dev)
        self.cnt_noise = torch.zeros((1,), dtype=i32, device=self.dev)
        self.zt = self.d["x0"].clone()
        # persistent buffers (R-17): pre-filled with the cache once (the full step's job); the conv
        # epilogue then writes only listed blocks, i.e. the feature-level scatter is fused
        self.y = [self.d[f"cache{l}"].clone() for l in range(L)]
        self.z = [self.d[f"cache{l}"].clone() for l in range(L)]
        self.lat_out = self.d["lat_cache"].clone()
        # one conv workspace per level, owned here (one per stream, sphinx.h), zeroed once
        self.ws = []
        for (h, c) in cfg.levels:
            nb = int(ops.load().sphinx_conv_workspace_size(F, h, h, c, c, b)) if self.cuda else 0
            self.ws.append(torch.zeros(max(nb, 256), dtype=u8, device=self.dev))
        # launches per step (single rank): mask 2 + compaction 1 + edge plans + noise 1 + convs + scatter 1
        n_edge = sum(1 for (h, _) in cfg.levels if h % b)
        self.launches_per_step = 2 + 1 + n_edge + 1 + L * cfg.convs_per_level + 1 + \
            (L if host_features is not None else 0)
        self.conv_events = None
        self.comm = None
        self._plan, self._plan_pending = None, False
        if world > 1:
            self.tp = _Transport(group)
            self.slice = slice(rank * F // world, (rank + 1) * F // world)
            self.owner = cfg.owner_of_frame(world)
            self.comm_stream = torch.cuda.Stream(device=self.dev) if self.cuda else None
            # the frame -> rank plan lives on the device (sphinx_shard_plan); the host reads back only
            # what sizes the owner gather, when it issues it
            self.owner_d = torch.from_numpy(self.owner.astype(np.int32)).to(self.dev)
            self.rank_of_d = torch.zeros((F,), dtype=i32, device=self.dev)
            self.load_d = torch.zeros((world,), dtype=torch.int64, device=self.dev)
            self.pair_d = torch.zeros((L, world, world), dtype=i32, device=self.dev)
            pin = dict(pin_memory=True) if self.cuda else {}
            self.h_rank_of = torch.zeros((F,), dtype=i32, **pin)
            self.h_load = torch.zeros((world,), dtype=torch.int64, **pin)
            self.h_pair = torch.zeros((L, world, world), dtype=i32, **pin)
            self.plan_ev = torch.cuda.Event() if self.cuda else None
            self._plan, self._plan_pending = None, False
            # packed C1 buffer: row r = rank r's slice [mask level 0 | ... | mask level L-1 | k (int32)]
            fs = F // world
            off, self.gath_lv = 0, []
            for hb in cfg.hb:
                self.gath_lv.append((off, fs * hb * hb, (fs, hb, hb)))
                off += fs * hb * hb
            off = (off + 15) // 16 * 16
            self.gath_k = (off, 4 * fs)
            self.gath = torch.zeros((world, (off + 4 * fs + 15) // 16 * 16), dtype=u8, device=self.dev)
            self.recv_ids = [torch.zeros((F * hb * hb,), dtype=i32, device=self.dev) for hb in cfg.hb]
            self.recv_cnt = torch.zeros((L,), dtype=i32, device=self.dev)
            self._pay = {}

    # ------------------------------------------------------------------ pieces of the step
    def _start_args(self, sl=slice(None)):
        d = self.d
        return dict(q_reg=d["q"][sl], c0=d["c0"][sl], c1=d["c1"][sl], t=d["t"][sl], gamma=self.cfg.gamma,
                    logics=self.logics, logic_id=d["lid"][sl])

    def _masks(self):
        cfg, ops, d = self.cfg, self.ops, self.d
        if self.world == 1:
            ops.sphinx_block_mask(d["O"], d["U"], d["tau_u"], cfg.tau_o, cfg.f, cfg.b, self.masks, self.counts,
                                  self._start_args(), self.k)
            return
        sl = self.slice
        # the slice's masks and start steps are written straight into this rank's row of one packed
        # buffer [world][level masks | k], so C1 is ONE all-gather (not one per level + one for k)
        mine = self.gath[self.rank]
        views = [mine[o:o + n].view(shp) for (o, n, shp) in self.gath_lv]
        ko, kn = self.gath_k
        kv = mine[ko:ko + kn].view(torch_int32())
        ops.sphinx_block_mask(d["O"][sl], d["U"][sl], d["tau_u"][sl], cfg.tau_o, cfg.f, cfg.b, views,
                              self.counts[sl], self._start_args(sl), kv)
        # C1: every rank gets the whole batch's masks and start steps
        self.tp.all_gather_into(self.gath.view(-1), mine)
        w = self.world
        for m, (o, n, _) in zip(self.masks, self.gath_lv):
            m.view(w, n).copy_(self.gath[:, o:o + n])
        self.k.view(w, kn // 4).copy_(self.gath[:, ko:ko + kn].view(torch_int32()))

    def make_plan(self, masks, k):
        """Host plan from the batch's masks [L][F,Hb,Wb] and start steps k [F] (numpy): LPT
        assignment of frames to ranks by executed MMA work at this u, and the exchange sizes.
        Deterministic: every rank derives the same plan."""
        cfg, world = self.cfg, self.world
        F, L = cfg.n_frames, cfg.L
        active = (k >= 0) & (k <= cfg.u)
        cnt = np.stack([masks[l].reshape(F, -1).sum(1) * active for l in range(L)], 1).astype(np.int64)
        cost = sdist.frame_costs(cnt, [c for (_, c) in cfg.levels])
        assign, load = sdist.lpt_assign(cost, world)
        rank_of = np.zeros(F, np.int64)
        for r, fr in enumerate(assign):
            rank_of[fr] = r
        # blocks of level l computed by s for frames owned by o: pair[l][s, o]
        cell = rank_of * world + self.owner
        pair = np.stack([np.bincount(cell, weights=cnt[:, l], minlength=world * world)
                         for l in range(L)]).astype(np.int64).reshape(L, world, world)
        return dict(rank_of=rank_of, load=load, cnt=cnt, pair=pair,
                    imbalance=float(load.max() / max(load.mean(), 1e-9)))

    def _plan_device(self):
        """The LPT plan on the device from the gathered masks and k (sphinx_shard_plan: the same rule
        as make_plan, on every rank): this rank's k_mine and the receive counts stay on the device;
        the exchange sizes, loads and assignment are copied back asynchronously."""
        cfg = self.cfg
        self.ops.sphinx_shard_plan(self.masks, [c for (_, c) in cfg.levels], self.k, cfg.u, self.owner_d,
                                   self.world, self.rank, self.k_mine, self.rank_of_d, self.load_d, self.pair_d,
                                   self.recv_cnt)
        for h, t in ((self.h_pair, self.pair_d), (self.h_load, self.load_d), (self.h_rank_of, self.rank_of_d)):
            h.copy_(t, non_blocking=self.cuda)
        if self.cuda:
            self.plan_ev.record()
        self._plan, self._plan_pending = None, True

    @property
    def plan(self):
        """The step's plan on the host (rank_of, load, pair [L][sender][owner], imbalance); waits for
        the read-back of sphinx_shard_plan's outputs the first time it is needed in a step."""
        if self._plan_pending:
            if self.cuda:
                self.plan_ev.synchronize()
            load = self.h_load.numpy().astype(np.int64)
            self._plan = dict(rank_of=self.h_rank_of.numpy().astype(np.int64), load=load,
                              pair=self.h_pair.numpy().astype(np.int64),
                              imbalance=float(load.max() / max(load.mean(), 1e-9)))
            self._plan_pending = False
        return self._plan

    def _compute(self, conv_events=None):
        cfg, ops, d = self.cfg, self.ops, self.d
        kk = self.k_mine
        L = cfg.L
        ops.sphinx_compact_blocks_batch(
            [dict(block_mask=self.masks[l], start_step=kk, step_u=cfg.u, select=ops.SELECT_ACTIVE,
                  block_ids=self.ids[l], count=self.cnt[l]) for l in range(L)] +
            [dict(block_mask=self.masks[0], start_step=kk, step_u=cfg.u, select=ops.SELECT_NOISE,
                  block_ids=self.ids_noise, count=self.cnt_noise)])
        if self.host_features is not None:
            # features from the host: only the listed blocks' halo windows cross PCIe (well ahead of the
            # convs, so each conv may still start INPUT_READY)
            for l in range(L):
                ops.sphinx_gather_halo_windows(self.host_features[l], d[f"feat{l}"], cfg.b, self.ids[l], self.cnt[l])
        # edge-class plans of the ragged levels right after compaction, so every conv of the step
        # reuses its level's plan and may start before its predecessor ends
        for l, (h, c) in enumerate(cfg.levels):
            if h % cfg.b:
                ops.sphinx_conv_edge_plan(self.ids[l], self.cnt[l], cfg.n_frames, h, h, cfg.b, c,
                                          workspace=self.ws[l])
        # Alg1 line 12 (active latent blocks noised to their start step k) and line 19 (inactive
        # frames resampled to u+1) in one pass over the NOISE list
        ops.sphinx_noise_inject_step(d["x0"], d["eps"], self.zt, cfg.b, self.ids_noise, self.cnt_noise, kk, cfg.u,
                                     d["abar"])
        # step 5 at latent resolution: refined latent blocks from this step, the latent cache of
        # the last full step everywhere else (P:352 spatial latent reuse); depends on the noise
        # pass only, so it runs before the convs and does not drain the conv chain
        ops.sphinx_scatter_cached(self.zt, d["lat_cache"], self.lat_out, cfg.b, block_mask=self.masks[0],
                                  start_step=kk, step_u=cfg.u)
        src = [d[f"feat{l}"] for l in range(L)]
        prev = None
        for (l, j) in self.conv_order():
            dst = self.y[l] if j % 2 == 0 else self.z[l]
            if conv_events is not None:
                conv_events[l][j][0].record()
            # INPUT_READY unless the input was written by the kernel right before: a level's input
            # features are step inputs, and with several levels conv j's input (conv j-1's output)
            # is at least two launches back in conv_order(), so the loads and MMAs may overlap the
            # preceding conv's tail
            ops.sphinx_sparse_conv3x3(src[l], d[f"w{l}{j}"], d[f"b{l}{j}"], dst, cfg.b, self.ids[l], self.cnt[l],
                                      workspace=self.ws[l], reuse_plan=True, list_ready=True,
                                      input_ready=(j == 0 or prev != (l, j - 1)),
                                      variant=(cfg.conv_variant[l] if cfg.conv_variant else 0))
            if conv_events is not None:
                conv_events[l][j][1].record()
            src[l] = dst
            prev = (l, j)
            if self.world > 1 and j == cfg.convs_per_level - 1:
                self._exchange_level(l, dst)

    def conv_order(self):
        """Launch order of the step's convs (level l, index j): anti-diagonals d = l + j, levels
        descending within one, e.g. (0,0) (1,0) (0,1) (2,0) (1,1) (2,1).  Consecutive convs are
        of different levels, so no conv's input was written by the kernel right before it: each
        conv is launched with INPUT_READY and its main loop fills its predecessor's tail (the
        predecessor does not feed it).  A single level runs in order (its convs are dependent)."""
        L, C = self.cfg.L, self.cfg.convs_per_level
        if not self.cfg.interleave_levels:  # level by level (A/B reference)
            return [(l, j) for l in range(L) for j in range(C)]
        order = [(l, dd - l) for dd in range(L + C - 1) for l in range(L - 1, -1, -1) if 0 <= dd - l < C]
        return order

    def out(self, l):
        """The level-l output map of the step (the last conv's persistent buffer)."""
        return self.y[l] if self.cfg.convs_per_level % 2 == 1 else self.z[l]

    def _payload(self, key, shape, dtype):
        t = self._pay.get(key)
        n = int(np.prod(shape))
        if t is None or t.numel() < n:
            t = self._pay[key] = self.torch.empty(max(n, 16), dtype=dtype, device=self.dev)
        return t[:n].view(shape)

    def _exchange_level(self, l, z_l):
        """C2 for level l: pack my refined blocks of frames owned by others (one segment per owner,
        contiguous in my ascending list), grouped send/recv, unpack what others computed for my
        frames.  Runs on the communication stream after the level's last conv."""
        torch, cfg, ops, p = self.torch, self.cfg, self.ops, self.plan
        me, world, b = self.rank, self.world, cfg.b
        h, c = cfg.levels[l]
        pair = p["pair"][l]
        sends_n = [(o, int(pair[me, o])) for o in range(world)]
        recv_from = [(s, int(pair[s, me])) for s in range(world) if s != me and pair[s, me] > 0]
        n_send = sum(n for o, n in sends_n if o != me)
        if n_send == 0 and not recv_from:
            return
        ctx = contextlib.nullcontext()
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record()
            self.comm_stream.wait_event(ev)
            ctx = torch.cuda.stream(self.comm_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.comm_stream)
        with ctx:
            n_mine = int(pair[me].sum())
            items = [(self.out(l), c, torch.bfloat16, "f")]
            if l == 0:
                items.append((self.lat_out, cfg.c_lat, torch.float32, "lat"))
            sends, recvs, unpack = [], [], []
            n_recv = sum(n for _, n in recv_from)
            for mp, ch, dt, tag in items:
                pay = self._payload((tag, l, "s"), (n_mine, b, b, ch), dt)
                ops.sphinx_gather_blocks(mp, pay, b, self.ids[l], self.cnt[l])
                self.exchange_launches += 1
                rpay = self._payload((tag, l, "r"), (n_recv, b, b, ch), dt)
                off = 0
                for o, n in sends_n:
                    if o != me and n > 0:
                        sends.append((o, _bytes(pay[off:off + n])))
                    off += n
                off = 0
                for s, n in recv_from:
                    recvs.append((s, _bytes(rpay[off:off + n])))
                    off += n
                unpack.append((rpay, mp))
            off = 0
            for o, n in sends_n:  # the ids of each segment travel with it
                if o != me and n > 0:
                    sends.append((o, _bytes(self.ids[l][off:off + n])))
                off += n
            off = 0
            for s, n in recv_from:
                recvs.append((s, _bytes(self.recv_ids[l][off:off + n])))
                off += n
            self.tp.exchange(sends, recvs)
            if n_recv:
                for rpay, mp in unpack:
                    ops.sphinx_scatter_blocks(rpay, mp, b, self.recv_ids[l], self.recv_cnt[l:l + 1],
                                              capacity=n_recv)
                    self.exchange_launches += 1
            self.bytes_sent += sum(t.numel() for _, t in sends)
        if self.cuda:
            e1.record(self.comm_stream)
            self.comm_events.append((e0, e1))

    # ------------------------------------------------------------------ the step
    def run(self, conv_events=None):
        """One refinement step (all of SURVEY 8(a)) on this rank's share of the batch."""
        self.bytes_sent = 0
        self.exchange_launches = 0  # pack / unpack kernels of the owner gather this step (N > 1)
        self.comm_events = []
        self._masks()
        if self.world > 1:
            self._plan_device()
        self._compute(conv_events)
        if self.world > 1 and self.cuda:
            self.torch.cuda.current_stream().wait_stream(self.comm_stream)

    def comm_ms(self):
        """Device time of the last step's owner-gather sections (pack, grouped send/recv, unpack)
        on the communication stream, summed over levels (call after synchronising)."""
        return sum(a.elapsed_time(b) for a, b in getattr(self, "comm_events", []))

    def window_bytes(self):
        """Bytes the halo-window gathers of the last step moved (host features): each listed block's
        own pixels plus the parts of its 1-pixel ring owned by UNLISTED neighbour blocks (the rule of
        sphinx_gather_halo_windows)."""
        cfg, out = self.cfg, 0
        for l, (h, c) in enumerate(cfg.levels):
            hb, b = cfg.hb[l], cfg.b
            ids = self.ids[l][: int(self.cnt[l].item())].cpu().numpy().astype(np.int64)
            is_listed = np.zeros(cfg.n_frames * hb * hb, bool)
            is_listed[ids] = True
            n, r = ids // (hb * hb), ids % (hb * hb)
            by, bx = r // hb, r % hb
            for rr in range(b + 2):
                y = by * b - 1 + rr
                oy = by - 1 if rr == 0 else (by + 1 if rr == b + 1 else by)
                yok = (y >= 0) & (y < h)
                for part, (xs, xe) in enumerate(((bx * b - 1, bx * b), (bx * b, np.minimum(bx * b + b, h)),
                                                 (bx * b + b, bx * b + b + 1))):
                    ox = bx - 1 + part
                    inside = (ox >= 0) & (ox < hb) & (oy >= 0) & (oy < hb)
                    own = (oy == by) & (ox == bx)
                    nb = (n * hb + np.clip(oy, 0, hb - 1)) * hb + np.clip(ox, 0, hb - 1)
                    keep = inside & (own | ~is_listed[nb])
                    width = np.clip(np.minimum(xe, h) - np.maximum(xs, 0), 0, None)
                    out += int((width * (keep & yok)).sum()) * c * 2
        return out

    def active_stats(self):
        """Algorithmic conv FLOPs of the step over the WHOLE batch (real active pixels of every
        level x 2*9*C^2 x convs per level), per-level real pixels and blocks.  Computed on the host
        from the batch's masks and start steps (identical on every rank)."""
        cfg = self.cfg
        masks = [m.cpu().numpy() for m in self.masks]
        k = self.k.cpu().numpy()
        active = (k >= 0) & (k <= cfg.u)
        flops, px_l, blocks = 0, [], []
        for l, (h, c) in enumerate(cfg.levels):
            m = masks[l] * active[:, None, None]
            ids = np.flatnonzero(m.ravel())
            px = cfg.real_px(l, ids)
            px_l.append(px)
            blocks.append(len(ids))
            flops += cfg.convs_per_level * px * 2 * 9 * c * c
        return flops, px_l, blocks
