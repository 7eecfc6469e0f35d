"""Python binding of libsphinx.so — the B200-native Sphinx selective-refinement hot path.

Argument marshalling only: every step runs in the CUDA kernels behind the C ABI
(include/sphinx.h).  PyTorch supplies device memory and streams.  There is no
CPU or PyTorch fallback: if the library is missing or the device is not sm_100,
every call raises.

Functions carry the C names:
    sphinx_block_mask       step 1  (Alg1 lines 4-10; Eq. 2)
    sphinx_compact_blocks   step 2  (Alg1 lines 17, 19)
    sphinx_noise_inject     step 3  (Alg1 lines 12, 19)
    sphinx_sparse_conv3x3   step 4
    sphinx_scatter_cached   step 5
    sphinx_ddim_step        NEXT-1  (Alg1 line 18)
    sphinx_uncertainty_map  NEXT-2  (Alg1 lines 7-8)
    sphinx_gn_block_stats / sphinx_gn_silu / sphinx_sparse_conv3x3_residual /
    sphinx_sparse_resblock  NEXT-3  (block-sparse ResNet block)
    sphinx_sparse_pointwise / sphinx_temporal_attention / sphinx_temporal_block
                            NEXT-4  (temporal-attention latent cache)
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libsphinx.so")

OK, ERR_INVALID_ARGUMENT, ERR_UNSUPPORTED, ERR_CUDA, ERR_DEVICE = 0, 1, 2, 3, 4
BF16, F32 = 0, 1
SELECT_ACTIVE, SELECT_INACTIVE_FRAMES, SELECT_ALL, SELECT_NOISE = 0, 1, 2, 3
SRC_FULL, SRC_COMPACT = 0, 1
MAX_LOGICS = 8
ABI_VERSION = 10
EXPORTS = ("sphinx_abi_version", "sphinx_last_cuda_error", "sphinx_block_mask",
           "sphinx_compact_blocks", "sphinx_noise_inject", "sphinx_sparse_conv3x3",
           "sphinx_conv_workspace_size", "sphinx_scatter_cached", "sphinx_ddim_step",
           "sphinx_uncertainty_map", "sphinx_uncertainty_workspace_size",
           "sphinx_gn_stats_size", "sphinx_gn_block_stats", "sphinx_gn_silu",
           "sphinx_sparse_conv3x3_residual", "sphinx_sparse_resblock",
           "sphinx_sparse_pointwise", "sphinx_temporal_attention_workspace_size",
           "sphinx_temporal_attention", "sphinx_temporal_block", "sphinx_gn_scale_shift",
           "sphinx_sparse_conv3x3_gn_silu", "sphinx_compact_blocks_batch", "sphinx_sparse_conv3x3_ex",
           "sphinx_sparse_resblock_ex", "sphinx_temporal_attention_ex", "sphinx_gather_blocks",
           "sphinx_scatter_blocks", "sphinx_noise_inject_step",
           "sphinx_conv_edge_plan", "sphinx_shard_plan", "sphinx_gather_halo_windows")

_lib = None


class SphinxError(RuntimeError):
    def __init__(self, fn, status, cuda_err=0):
        names = {1: "INVALID_ARGUMENT", 2: "UNSUPPORTED", 3: "CUDA", 4: "DEVICE"}
        super().__init__(f"{fn}: SPHINX_ERR_{names.get(status, status)}"
                         + (f" (cudaError {cuda_err})" if status == ERR_CUDA else ""))
        self.status = status


class KLogic(ctypes.Structure):
    """sphinx_klogic."""
    _fields_ = [("m", ctypes.c_int32), ("thr", ctypes.c_double * 16),
                ("step", ctypes.c_int32 * 16), ("fallback_k", ctypes.c_int32),
                ("k_max", ctypes.c_int32)]


class CompactJob(ctypes.Structure):
    """sphinx_compact_job (one list of a batched compaction)."""
    _fields_ = [("block_mask", ctypes.c_void_p), ("n", ctypes.c_int32), ("hb", ctypes.c_int32),
                ("wb", ctypes.c_int32), ("start_step", ctypes.c_void_p), ("step_u", ctypes.c_int32),
                ("select", ctypes.c_int32), ("block_ids", ctypes.c_void_p), ("count", ctypes.c_void_p)]


MAX_COMPACT_JOBS = 8
CONV_REUSE_PLAN = 1
CONV_LIST_READY = 2
CONV_INPUT_READY = 4
RB_FUSED_GN = 1
CONV_FORCE_CG1 = 1 << 8
CONV_FORCE_HALO = 1 << 9
CONV_FORCE_PERTAP = 1 << 10
CONV_NO_SPLIT = 1 << 11
CONV_NO_EDGE = 1 << 12
CONV_NO_STREAMK = 1 << 13
CONV_FORCE_STREAMK = 1 << 14


class StartArgs(ctypes.Structure):
    """sphinx_start_args (Alg1 lines 3-6)."""
    _fields_ = [("q_reg", ctypes.c_void_p), ("c0", ctypes.c_void_p), ("c1", ctypes.c_void_p),
                ("t", ctypes.c_void_p), ("logic_id", ctypes.c_void_p), ("gamma", ctypes.c_float),
                ("logics", ctypes.c_void_p), ("n_logics", ctypes.c_int32)]


def make_klogic(thr, steps, fallback_k=0, k_max=40):
    lg = KLogic()
    lg.m = len(thr)
    for i, (t, s) in enumerate(zip(thr, steps)):
        lg.thr[i] = float(t)
        lg.step[i] = int(s)
    lg.fallback_k = int(fallback_k)
    lg.k_max = int(k_max)
    return lg


def load(path=SO_PATH):
    """Loads libsphinx.so (raises if absent: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libsphinx.so not built at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    P, I, F, Z = ctypes.c_void_p, ctypes.c_int32, ctypes.c_float, ctypes.c_size_t
    sig = {
        "sphinx_abi_version": ([], I),
        "sphinx_last_cuda_error": ([], I),
        "sphinx_block_mask": ([P, P, P, F, I, I, I, I, I, I, P, P, P, P, P], I),
        "sphinx_compact_blocks": ([P, I, I, I, P, I, I, P, P, P], I),
        "sphinx_shard_plan": ([P, P, P, I, I, P, I, P, I, I, P, P, P, P, P, P], I),
        "sphinx_gather_halo_windows": ([P, P, I, I, I, I, I, I, P, P, I, P], I),
        "sphinx_noise_inject": ([P, P, P, I, I, I, I, I, P, P, I, P, P, I, P], I),
        "sphinx_sparse_conv3x3": ([P, P, P, P, I, I, I, I, I, I, I, P, P, I, P, Z, P], I),
        "sphinx_conv_workspace_size": ([I, I, I, I, I, I], Z),
        "sphinx_scatter_cached": ([P, I, P, P, I, I, I, I, I, I, P, P, I, P, P, P], I),
        "sphinx_ddim_step": ([P, P, P, I, I, I, I, I, P, P, I, I, P, I, P], I),
        "sphinx_uncertainty_map": ([P, I, I, I, I, I, P, P, P, Z, P], I),
        "sphinx_uncertainty_workspace_size": ([I], Z),
        "sphinx_gn_stats_size": ([I, I, I, I, I], Z),
        "sphinx_gn_block_stats": ([P, I, I, I, I, I, I, P, P, I, P, P], I),
        "sphinx_gn_silu": ([P, P, P, P, F, I, I, I, I, I, I, P, P, I, P, P], I),
        "sphinx_sparse_conv3x3_residual": ([P, P, P, P, P, I, I, I, I, I, I, I, P, P, I, P, Z, P], I),
        "sphinx_sparse_resblock": ([P, P, P, P, P, P, P, P, P, I, F, P, P, P, P, I, P,
                                    I, I, I, I, I, P, P, I, P, Z, P], I),
        "sphinx_sparse_resblock_ex": ([P, P, P, P, P, P, P, P, P, I, F, P, P, P, P, I, P,
                                       I, I, I, I, I, P, P, I, P, Z, I, P], I),
        "sphinx_sparse_pointwise": ([P, P, P, P, P, I, I, I, I, I, I, I, P, P, I, P, Z, P], I),
        "sphinx_gather_blocks": ([P, P, I, I, I, I, I, I, P, P, I, P], I),
        "sphinx_noise_inject_step": ([P, P, P, I, I, I, I, I, P, P, I, P, I, P, I, P], I),
        "sphinx_scatter_blocks": ([P, P, I, I, I, I, I, I, P, P, I, P], I),
        "sphinx_gn_scale_shift": ([P, P, P, F, I, I, I, I, I, I, P, P], I),
        "sphinx_compact_blocks_batch": ([P, I, P], I),
        "sphinx_conv_edge_plan": ([P, P, I, I, I, I, I, P, Z, P], I),
        "sphinx_sparse_conv3x3_ex": ([P, P, P, P, P, I, I, I, I, I, I, I, P, P, I, P, Z, I, P], I),
        "sphinx_sparse_conv3x3_gn_silu": ([P, P, P, P, P, P, I, I, I, I, I, I, I, P, P, I, P, Z, P], I),
        "sphinx_temporal_attention_workspace_size": ([I, I, I, I, I], Z),
        "sphinx_temporal_attention": ([P, P, I, I, I, I, I, I, I, P, P, I, P, Z, P], I),
        "sphinx_temporal_attention_ex": ([P, P, I, I, I, I, I, I, I, P, P, I, P, Z, I, P], I),
        "sphinx_temporal_block": ([P, P, P, P, P, I, I, P, P, P, I, I, I, I, I, I, P, P, I,
                                   P, Z, P, Z, P], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.sphinx_abi_version() != ABI_VERSION:
        raise RuntimeError("libsphinx ABI version mismatch")
    _lib = lib
    return lib


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _chk(fn, rc):
    if rc != OK:
        raise SphinxError(fn, rc, load().sphinx_last_cuda_error() if rc == ERR_CUDA else 0)


def _dev(t, dtype, name):
    import torch
    if t is None:
        return
    if not (t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise ValueError(f"{name}: expected a contiguous CUDA {dtype} tensor")


def sphinx_block_mask(opacity, uncertainty, tau_u, tau_o, px_per_cell, block, block_masks,
                      active_count=None, start=None, start_step=None, stream=None):
    """Step 1.  opacity/uncertainty [N,Hp,Wp] fp32; block_masks: list of u8 [N,Hb_l,Wb_l]
    (one per level); start: dict(q_reg, c0, c1, t, gamma, logics=[KLogic], logic_id=None)."""
    import torch
    _dev(opacity, torch.float32, "opacity")
    _dev(uncertainty, torch.float32, "uncertainty")
    _dev(tau_u, torch.float32, "tau_u")
    for m in block_masks:
        _dev(m, torch.uint8, "block_mask")
    _dev(active_count, torch.int32, "active_count")
    n, hp, wp = opacity.shape
    L = len(block_masks)
    masks = (ctypes.c_void_p * L)(*[m.data_ptr() for m in block_masks])
    ss = None
    keep = []
    if start is not None:
        logics = (KLogic * len(start["logics"]))(*start["logics"])
        keep.append(logics)
        for k in ("q_reg", "c0", "c1", "t"):
            _dev(start[k], torch.float32, k)
        _dev(start.get("logic_id"), torch.int32, "logic_id")
        _dev(start_step, torch.int32, "start_step")
        ss = StartArgs(start["q_reg"].data_ptr(), start["c0"].data_ptr(), start["c1"].data_ptr(),
                       start["t"].data_ptr(),
                       start["logic_id"].data_ptr() if start.get("logic_id") is not None else None,
                       float(start["gamma"]), ctypes.cast(logics, ctypes.c_void_p), len(start["logics"]))
        keep.append(ss)
    rc = load().sphinx_block_mask(_ptr(opacity), _ptr(uncertainty), _ptr(tau_u), float(tau_o),
                                  n, hp, wp, int(px_per_cell), int(block), L,
                                  ctypes.cast(masks, ctypes.c_void_p), _ptr(active_count),
                                  ctypes.byref(ss) if ss is not None else None, _ptr(start_step),
                                  _stream(stream))
    _chk("sphinx_block_mask", rc)


def sphinx_compact_blocks(block_mask, start_step, step_u, select, block_ids, count, shape=None,
                          stream=None):
    """Step 2.  block_mask u8 [N,Hb,Wb] (or None with shape=(N,Hb,Wb)); block_ids int32 [N*Hb*Wb];
    count int32 [1] (stays on the device)."""
    import torch
    _dev(block_mask, torch.uint8, "block_mask")
    _dev(start_step, torch.int32, "start_step")
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    n, hb, wb = block_mask.shape if block_mask is not None else shape
    if block_ids.numel() < n * hb * wb:
        raise ValueError("block_ids capacity < N*Hb*Wb")
    rc = load().sphinx_compact_blocks(_ptr(block_mask), n, hb, wb, _ptr(start_step), int(step_u),
                                      int(select), _ptr(block_ids), _ptr(count), _stream(stream))
    _chk("sphinx_compact_blocks", rc)


def sphinx_compact_blocks_batch(jobs, stream=None):
    """Several compactions in one launch.  jobs: list of dicts with the arguments of
    sphinx_compact_blocks (block_mask, start_step, step_u, select, block_ids, count, shape)."""
    import torch
    if not 0 < len(jobs) <= MAX_COMPACT_JOBS:
        raise ValueError("1..8 jobs")
    arr = (CompactJob * len(jobs))()
    for i, jb in enumerate(jobs):
        m = jb.get("block_mask")
        _dev(m, torch.uint8, "block_mask")
        _dev(jb.get("start_step"), torch.int32, "start_step")
        _dev(jb["block_ids"], torch.int32, "block_ids")
        _dev(jb["count"], torch.int32, "count")
        n, hb, wb = m.shape if m is not None else jb["shape"]
        arr[i] = CompactJob(None if m is None else m.data_ptr(), n, hb, wb,
                            None if jb.get("start_step") is None else jb["start_step"].data_ptr(),
                            int(jb.get("step_u", 0)), int(jb["select"]), jb["block_ids"].data_ptr(),
                            jb["count"].data_ptr())
    rc = load().sphinx_compact_blocks_batch(ctypes.cast(arr, ctypes.c_void_p), len(jobs), _stream(stream))
    _chk("sphinx_compact_blocks_batch", rc)


def sphinx_shard_plan(block_masks, channels, start_step, step_u, owner, world, rank, k_mine, rank_of, rank_load,
                      pair, recv, stream=None):
    """§8(e) frame -> rank LPT plan on the device (sphinx.h).  block_masks: list of u8 [N,Hb_l,Wb_l];
    channels: host ints C_l; start_step/owner/k_mine/rank_of int32 [N]; rank_load int64 [world];
    pair int32 [L,world,world]; recv int32 [L]."""
    import torch
    L = len(block_masks)
    for m in block_masks:
        _dev(m, torch.uint8, "block_mask")
    for t, nm in ((start_step, "start_step"), (owner, "owner"), (k_mine, "k_mine"), (rank_of, "rank_of"),
                  (pair, "pair"), (recv, "recv")):
        _dev(t, torch.int32, nm)
    _dev(rank_load, torch.int64, "rank_load")
    n = block_masks[0].shape[0]
    masks = (ctypes.c_void_p * L)(*[m.data_ptr() for m in block_masks])
    bpf = (ctypes.c_int32 * L)(*[int(m.shape[1] * m.shape[2]) for m in block_masks])
    ch = (ctypes.c_int32 * L)(*[int(c) for c in channels])
    rc = load().sphinx_shard_plan(ctypes.cast(masks, ctypes.c_void_p), ctypes.cast(bpf, ctypes.c_void_p),
                                      ctypes.cast(ch, ctypes.c_void_p), L, int(n), _ptr(start_step), int(step_u),
                                      _ptr(owner), int(world), int(rank), _ptr(k_mine), _ptr(rank_of), _ptr(rank_load),
                                      _ptr(pair), _ptr(recv), _stream(stream))
    _chk("sphinx_shard_plan", rc)


def sphinx_noise_inject(x0, eps, x_t, block, block_ids, count, step, abar, capacity=None,
                        stream=None):
    """Step 3.  x0/eps/x_t NHWC fp32 [N,H,W,C]; step int32 [N]; abar fp32 [S+1]."""
    import torch
    for t, nm in ((x0, "x0"), (eps, "eps"), (x_t, "x_t"), (abar, "abar")):
        _dev(t, torch.float32, nm)
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    _dev(step, torch.int32, "step")
    n, h, w, c = x0.shape
    cap = block_ids.numel() if capacity is None else capacity
    rc = load().sphinx_noise_inject(_ptr(x0), _ptr(eps), _ptr(x_t), n, h, w, c, int(block),
                                    _ptr(block_ids), _ptr(count), int(cap), _ptr(step), _ptr(abar),
                                    abar.numel() - 1, _stream(stream))
    _chk("sphinx_noise_inject", rc)


def sphinx_noise_inject_step(x0, eps, x_t, block, block_ids, count, start_step, step_u, abar, capacity=None,
                             stream=None):
    """Step 3, the step's whole noise pass (Alg1 lines 12 + 19): listed blocks of frames with
    0 <= k <= u to their start step k, of frames with k > u to u + 1 (SELECT_NOISE list)."""
    import torch
    for t, nm in ((x0, "x0"), (eps, "eps"), (x_t, "x_t"), (abar, "abar")):
        _dev(t, torch.float32, nm)
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    _dev(start_step, torch.int32, "start_step")
    n, h, w, c = x0.shape
    cap = block_ids.numel() if capacity is None else capacity
    rc = load().sphinx_noise_inject_step(_ptr(x0), _ptr(eps), _ptr(x_t), n, h, w, c, int(block),
                                         _ptr(block_ids), _ptr(count), int(cap), _ptr(start_step), int(step_u),
                                         _ptr(abar), abar.numel() - 1, _stream(stream))
    _chk("sphinx_noise_inject_step", rc)


_ws_cache = {}


def _stream_key(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def conv_workspace(c_out, device, n=1, h=1, w=1, block=8, stream=None):
    """Zero-initialised workspace (split-K counters + partial tiles, edge-class plan) for a conv
    of this geometry on `device` and STREAM (sphinx.h: one workspace per stream), allocated once
    and cached (the kernel leaves its counters zeroed).  Memory only: no computation happens
    here.  CUDA-graph users warm up on the capture stream (so the workspace exists before the
    capture) or pass their own workspace."""
    key = (device, c_out, n, h, w, block, _stream_key(stream))
    ws = _ws_cache.get(key)
    if ws is None:
        import torch
        nbytes = int(load().sphinx_conv_workspace_size(int(n), int(h), int(w), 8, int(c_out), int(block)))
        ws = _ws_cache[key] = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    return ws


def sphinx_sparse_conv3x3(x, w, bias, y, block, block_ids, count, capacity=None, stream=None,
                          workspace=None, residual=None, reuse_plan=False, list_ready=False,
                          input_ready=False, variant=0):
    """Step 4.  x bf16 NHWC [N,H,W,Cin]; w bf16 [Cout,3,3,Cin]; bias fp32 [Cout] or None;
    y NHWC [N,H,W,Cout] bf16 or fp32 (only listed blocks are written).
    workspace: None = a cached zeroed split-K workspace for this device and stream, False = no
    split-K, or a caller-owned zero-initialised uint8 CUDA tensor (one per stream).
    variant: CONV_FORCE_* / CONV_NO_* kernel-variant flags (tests and tuning; 0 = default)."""
    import torch
    _dev(x, torch.bfloat16, "x")
    _dev(w, torch.bfloat16, "w")
    _dev(bias, torch.float32, "bias")
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    if y.dtype not in (torch.bfloat16, torch.float32) or not (y.is_cuda and y.is_contiguous()):
        raise ValueError("y: contiguous CUDA bf16/fp32")
    n, h, wd, cin = x.shape
    cout = w.shape[0]
    cap = block_ids.numel() if capacity is None else capacity
    if workspace is None:
        workspace = conv_workspace(cout, y.device, n, h, wd, block, stream)
    ws_ptr, ws_bytes = (None, 0) if workspace is False else (_ptr(workspace), workspace.numel())
    if reuse_plan or list_ready or input_ready or variant:
        _dev(residual, torch.bfloat16, "residual")
        flags = ((CONV_REUSE_PLAN if reuse_plan else 0) | (CONV_LIST_READY if list_ready else 0) |
                 (CONV_INPUT_READY if input_ready else 0) | int(variant))
        rc = load().sphinx_sparse_conv3x3_ex(
            _ptr(x), _ptr(w), _ptr(bias), _ptr(residual), _ptr(y), F32 if y.dtype == torch.float32 else BF16,
            n, h, wd, cin, cout, int(block), _ptr(block_ids), _ptr(count), int(cap), ws_ptr, ws_bytes,
            flags, _stream(stream))
        _chk("sphinx_sparse_conv3x3_ex", rc)
        return
    if residual is not None:
        _dev(residual, torch.bfloat16, "residual")
        rc = load().sphinx_sparse_conv3x3_residual(
            _ptr(x), _ptr(w), _ptr(bias), _ptr(residual), _ptr(y),
            F32 if y.dtype == torch.float32 else BF16, n, h, wd, cin, cout, int(block),
            _ptr(block_ids), _ptr(count), int(cap), ws_ptr, ws_bytes, _stream(stream))
        _chk("sphinx_sparse_conv3x3_residual", rc)
        return
    rc = load().sphinx_sparse_conv3x3(_ptr(x), _ptr(w), _ptr(bias), _ptr(y),
                                      F32 if y.dtype == torch.float32 else BF16,
                                      n, h, wd, cin, cout, int(block), _ptr(block_ids), _ptr(count),
                                      int(cap), ws_ptr, ws_bytes, _stream(stream))
    _chk("sphinx_sparse_conv3x3", rc)


def sphinx_conv_edge_plan(block_ids, count, n, h, w, block, c_out, capacity=None, workspace=None,
                          stream=None):
    """Edge-class plan of a list into the (cached) conv workspace of this geometry, so the convs
    over the list can pass reuse_plan=True (and list_ready=True)."""
    import torch
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    cap = block_ids.numel() if capacity is None else capacity
    if workspace is None:
        workspace = conv_workspace(c_out, block_ids.device, n, h, w, block, stream)
    rc = load().sphinx_conv_edge_plan(_ptr(block_ids), _ptr(count), int(n), int(h), int(w), int(block), int(cap),
                                      _ptr(workspace), workspace.numel(), _stream(stream))
    _chk("sphinx_conv_edge_plan", rc)


def _block_copy(fn, src, dst, block, block_ids, count, capacity, stream, map_side):
    import torch
    if src.dtype not in (torch.bfloat16, torch.float32) or dst.dtype != src.dtype:
        raise ValueError("src/dst: same dtype, bf16 or fp32")
    for t, nm in ((src, "src"), (dst, "dst")):
        if not (t.is_cuda and t.is_contiguous()):
            raise ValueError(f"{nm}: contiguous CUDA tensor")
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    n, h, w, c = map_side.shape
    cap = block_ids.numel() if capacity is None else capacity
    rc = getattr(load(), fn)(_ptr(src), _ptr(dst), F32 if src.dtype == torch.float32 else BF16, n, h, w, c,
                             int(block), _ptr(block_ids), _ptr(count), int(cap), _stream(stream))
    _chk(fn, rc)


def sphinx_gather_halo_windows(src, dst, block, block_ids, count, capacity=None, stream=None):
    """dst [N,H,W,C] <- the halo windows of the listed blocks of src (same shape and dtype); src may
    be a PINNED host tensor, read by the GPU over PCIe (sphinx.h)."""
    import torch
    if src.dtype not in (torch.bfloat16, torch.float32) or dst.dtype != src.dtype or src.shape != dst.shape:
        raise ValueError("src/dst: same shape and dtype, bf16 or fp32")
    if not (src.is_contiguous() and (src.is_cuda or src.is_pinned())):
        raise ValueError("src: contiguous CUDA or pinned host tensor")
    if not (dst.is_cuda and dst.is_contiguous()):
        raise ValueError("dst: contiguous CUDA tensor")
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    n, h, w, c = dst.shape
    cap = block_ids.numel() if capacity is None else capacity
    rc = load().sphinx_gather_halo_windows(_ptr(src), _ptr(dst), F32 if src.dtype == torch.float32 else BF16, n, h,
                                           w, c, int(block), _ptr(block_ids), _ptr(count), int(cap), _stream(stream))
    _chk("sphinx_gather_halo_windows", rc)


def sphinx_gather_blocks(src, dst, block, block_ids, count, capacity=None, stream=None):
    """Data plane pack: dst [cap,b,b,C] <- listed blocks of the NHWC map src [N,H,W,C]."""
    _block_copy("sphinx_gather_blocks", src, dst, block, block_ids, count, capacity, stream, src)


def sphinx_scatter_blocks(src, out, block, block_ids, count, capacity=None, stream=None):
    """Data plane unpack: listed blocks of the NHWC map out [N,H,W,C] <- compact src [cap,b,b,C]."""
    _block_copy("sphinx_scatter_blocks", src, out, block, block_ids, count, capacity, stream, out)


def sphinx_scatter_cached(src, cache, out, block, block_mask=None, start_step=None, step_u=0,
                          block_ids=None, count=None, src_layout=SRC_FULL, stream=None):
    """Step 5.  out = active ? src : cache (bit copy); NHWC bf16 or fp32."""
    import torch
    if cache.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("cache: bf16/fp32")
    for t, nm in ((src, "src"), (cache, "cache"), (out, "out")):
        _dev(t, cache.dtype, nm)
    _dev(block_mask, torch.uint8, "block_mask")
    _dev(start_step, torch.int32, "start_step")
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    n, h, w, c = cache.shape
    rc = load().sphinx_scatter_cached(_ptr(src), int(src_layout), _ptr(cache), _ptr(out),
                                      F32 if cache.dtype == torch.float32 else BF16,
                                      n, h, w, c, int(block), _ptr(block_mask), _ptr(start_step),
                                      int(step_u), _ptr(block_ids), _ptr(count), _stream(stream))
    _chk("sphinx_scatter_cached", rc)


def sphinx_ddim_step(z, x0_hat, z_out, block, block_ids, count, step_u, abar_host, capacity=None,
                     stream=None):
    """NEXT-1 (Alg1 line 18).  z/x0_hat/z_out NHWC fp32 [N,H,W,C] on the device;
    abar_host: numpy fp32 [S+1] (host: the step u is a loop scalar)."""
    import numpy as np
    import torch
    for t, nm in ((z, "z"), (x0_hat, "x0_hat"), (z_out, "z_out")):
        _dev(t, torch.float32, nm)
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    ab = np.ascontiguousarray(abar_host, dtype=np.float32)
    n, h, w, c = z.shape
    cap = block_ids.numel() if capacity is None else capacity
    rc = load().sphinx_ddim_step(_ptr(z), _ptr(x0_hat), _ptr(z_out), n, h, w, c, int(block),
                                 _ptr(block_ids), _ptr(count), int(cap), int(step_u),
                                 ab.ctypes.data_as(ctypes.c_void_p), len(ab) - 1, _stream(stream))
    _chk("sphinx_ddim_step", rc)


def sphinx_uncertainty_map(rgb, uncertainty, tau_u, window=7, smooth=5, workspace=None, stream=None):
    """NEXT-2 (Alg1 lines 7-8).  rgb NHWC fp32 [N,H,W,3] -> uncertainty fp32 [N,H,W],
    tau_u fp32 [N] (the inputs of sphinx_block_mask).  workspace: uint8 CUDA tensor or None
    (a cached one per device is used)."""
    import torch
    _dev(rgb, torch.float32, "rgb")
    _dev(uncertainty, torch.float32, "uncertainty")
    _dev(tau_u, torch.float32, "tau_u")
    n, h, w, c = rgb.shape
    if c != 3:
        raise ValueError("rgb: [N,H,W,3]")
    if workspace is None:
        key = ("unc", rgb.device, n, _stream_key(stream))
        workspace = _ws_cache.get(key)
        if workspace is None:
            nbytes = int(load().sphinx_uncertainty_workspace_size(int(n)))
            workspace = _ws_cache[key] = torch.zeros(nbytes, dtype=torch.uint8, device=rgb.device)
    rc = load().sphinx_uncertainty_map(_ptr(rgb), n, h, w, int(window), int(smooth), _ptr(uncertainty),
                                       _ptr(tau_u), _ptr(workspace), workspace.numel(), _stream(stream))
    _chk("sphinx_uncertainty_map", rc)


def gn_stats_buffer(n, h, w, groups, block, device):
    """A GroupNorm statistics buffer for NEXT-3 (flat fp32: block entries [N,Hb,Wb,G,2] then
    frame entries [N,G,2]); memory only."""
    import torch
    nbytes = int(load().sphinx_gn_stats_size(int(n), int(h), int(w), int(groups), int(block)))
    return torch.zeros(nbytes // 4, dtype=torch.float32, device=device)


def gn_block_entries(stats, n, h, w, groups, block):
    """View of the per-block (mean, M2) entries of a statistics buffer: [N,Hb,Wb,G,2]."""
    hb, wb = -(-h // block), -(-w // block)
    return stats[: n * hb * wb * groups * 2].view(n, hb, wb, groups, 2)


def sphinx_gn_block_stats(x, groups, block, block_ids, count, stats, capacity=None, stream=None):
    """NEXT-3: rewrite the per-block (mean, M2) entries of the listed blocks of bf16 NHWC x."""
    import torch
    _dev(x, torch.bfloat16, "x")
    _dev(stats, torch.float32, "stats")
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    n, h, w, c = x.shape
    if stats.numel() * 4 != load().sphinx_gn_stats_size(n, h, w, int(groups), int(block)):
        raise ValueError("stats: expected a gn_stats_buffer(...) of this geometry")
    cap = block_ids.numel() if capacity is None else capacity
    rc = load().sphinx_gn_block_stats(_ptr(x), n, h, w, c, int(groups), int(block), _ptr(block_ids),
                                      _ptr(count), int(cap), _ptr(stats), _stream(stream))
    _chk("sphinx_gn_block_stats", rc)


def sphinx_gn_silu(x, stats, gamma, beta, eps, groups, block, block_ids, count, a, capacity=None,
                   stream=None):
    """NEXT-3: a = bf16(SiLU(GroupNorm(x))) on listed blocks + their 1-pixel ring."""
    import torch
    _dev(x, torch.bfloat16, "x")
    _dev(a, torch.bfloat16, "a")
    _dev(stats, torch.float32, "stats")
    _dev(gamma, torch.float32, "gamma")
    _dev(beta, torch.float32, "beta")
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    n, h, w, c = x.shape
    cap = block_ids.numel() if capacity is None else capacity
    rc = load().sphinx_gn_silu(_ptr(x), _ptr(stats), _ptr(gamma), _ptr(beta), float(eps), n, h, w, c,
                               int(groups), int(block), _ptr(block_ids), _ptr(count), int(cap), _ptr(a),
                               _stream(stream))
    _chk("sphinx_gn_silu", rc)


def sphinx_sparse_resblock(x, w1, b1, w2, b2, gn1, gn2, groups, eps, h_buf, x_stats, h_stats, y,
                           a_scratch, block, block_ids, count, capacity=None, workspace=None,
                           stream=None, fused=False):
    """NEXT-3 block-sparse ResNet block (R-26, R-27).  gn1/gn2 = (gamma, beta)
    fp32 [C]; h_buf bf16 / y bf16-or-fp32 / x_stats / h_stats persistent (see sphinx.h)."""
    import torch
    for t, nm in ((x, "x"), (w1, "w1"), (w2, "w2"), (h_buf, "h_buf"), (a_scratch, "a_scratch")):
        _dev(t, torch.bfloat16, nm)
    for t, nm in ((b1, "b1"), (b2, "b2"), (gn1[0], "gn1.gamma"), (gn1[1], "gn1.beta"),
                  (gn2[0], "gn2.gamma"), (gn2[1], "gn2.beta"), (x_stats, "x_stats"),
                  (h_stats, "h_stats")):
        _dev(t, torch.float32, nm)
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    if y.dtype not in (torch.bfloat16, torch.float32) or not (y.is_cuda and y.is_contiguous()):
        raise ValueError("y: contiguous CUDA bf16/fp32")
    n, h, wd, c = x.shape
    cap = block_ids.numel() if capacity is None else capacity
    if workspace is None:
        workspace = conv_workspace(c, y.device, n, h, wd, block, stream)
    ws_ptr, ws_bytes = (None, 0) if workspace is False else (_ptr(workspace), workspace.numel())
    rc = load().sphinx_sparse_resblock_ex(
        _ptr(x), _ptr(w1), _ptr(b1), _ptr(w2), _ptr(b2), _ptr(gn1[0]), _ptr(gn1[1]), _ptr(gn2[0]),
        _ptr(gn2[1]), int(groups), float(eps), _ptr(h_buf), _ptr(x_stats), _ptr(h_stats), _ptr(y),
        F32 if y.dtype == torch.float32 else BF16, _ptr(a_scratch), n, h, wd, c, int(block),
        _ptr(block_ids), _ptr(count), int(cap), ws_ptr, ws_bytes, RB_FUSED_GN if fused else 0,
        _stream(stream))
    _chk("sphinx_sparse_resblock_ex", rc)


def attn_workspace(n, h, w, frames_per_seq, block, device, stream=None):
    """Workspace of sphinx_temporal_attention (listed-frame bitmasks), cached per stream; memory
    only."""
    key = ("attn", device, n, h, w, frames_per_seq, block, _stream_key(stream))
    ws = _ws_cache.get(key)
    if ws is None:
        import torch
        nbytes = int(load().sphinx_temporal_attention_workspace_size(int(n), int(h), int(w),
                                                                     int(frames_per_seq), int(block)))
        ws = _ws_cache[key] = torch.zeros(max(nbytes, 4), dtype=torch.uint8, device=device)
    return ws


def sphinx_sparse_pointwise(x, w, bias, y, block, block_ids, count, residual=None, capacity=None,
                            workspace=None, stream=None):
    """NEXT-4 pointwise projection on listed blocks: y = (residual) + bias + W x.
    x bf16 NHWC [N,H,W,Cin]; w bf16 [Cout, Cin]; y NHWC bf16/fp32 [N,H,W,Cout]."""
    import torch
    _dev(x, torch.bfloat16, "x")
    _dev(w, torch.bfloat16, "w")
    _dev(bias, torch.float32, "bias")
    _dev(residual, torch.bfloat16, "residual")
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    if y.dtype not in (torch.bfloat16, torch.float32) or not (y.is_cuda and y.is_contiguous()):
        raise ValueError("y: contiguous CUDA bf16/fp32")
    n, h, wd, cin = x.shape
    cout = w.shape[0]
    cap = block_ids.numel() if capacity is None else capacity
    if workspace is None:
        workspace = conv_workspace(cout, y.device, n, h, wd, block, stream)
    ws_ptr, ws_bytes = (None, 0) if workspace is False else (_ptr(workspace), workspace.numel())
    rc = load().sphinx_sparse_pointwise(_ptr(x), _ptr(w), _ptr(bias), _ptr(residual), _ptr(y),
                                        F32 if y.dtype == torch.float32 else BF16, n, h, wd, cin, cout,
                                        int(block), _ptr(block_ids), _ptr(count), int(cap), ws_ptr,
                                        ws_bytes, _stream(stream))
    _chk("sphinx_sparse_pointwise", rc)


def sphinx_temporal_attention(qkv, o, heads, frames_per_seq, block, block_ids, count, capacity=None,
                              workspace=None, stream=None, head_group=0):
    """NEXT-4 attention of listed tokens over their sequence's frames (K/V cache in qkv).
    head_group: k > 0 stages (pixel, k heads) units (tests); 0 = the library's choice."""
    import torch
    _dev(qkv, torch.bfloat16, "qkv")
    _dev(o, torch.bfloat16, "o")
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    n, h, w, c = o.shape
    cap = block_ids.numel() if capacity is None else capacity
    if workspace is None:
        workspace = attn_workspace(n, h, w, frames_per_seq, block, o.device, stream)
    rc = load().sphinx_temporal_attention_ex(_ptr(qkv), _ptr(o), n, h, w, c, int(heads),
                                             int(frames_per_seq), int(block), _ptr(block_ids), _ptr(count),
                                             int(cap), _ptr(workspace), workspace.numel(), int(head_group),
                                             _stream(stream))
    _chk("sphinx_temporal_attention_ex", rc)


def sphinx_temporal_block(x, wqkv, bqkv, wo, bo, heads, frames_per_seq, qkv_buf, o_scratch, y, block,
                          block_ids, count, capacity=None, workspace=None, attn_ws=None, stream=None):
    """NEXT-4 temporal block (R-28): y[listed] = x + Wo attn(qkv) + bo with the
    persistent q|k|v buffer as the latent cache of unlisted tokens."""
    import torch
    for t, nm in ((x, "x"), (wqkv, "wqkv"), (wo, "wo"), (qkv_buf, "qkv_buf"), (o_scratch, "o_scratch")):
        _dev(t, torch.bfloat16, nm)
    _dev(bqkv, torch.float32, "bqkv")
    _dev(bo, torch.float32, "bo")
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    if y.dtype not in (torch.bfloat16, torch.float32) or not (y.is_cuda and y.is_contiguous()):
        raise ValueError("y: contiguous CUDA bf16/fp32")
    n, h, wd, c = x.shape
    cap = block_ids.numel() if capacity is None else capacity
    if workspace is None:
        workspace = conv_workspace(3 * c, y.device, n, h, wd, block, stream)
    if attn_ws is None:
        attn_ws = attn_workspace(n, h, wd, frames_per_seq, block, y.device, stream)
    ws_ptr, ws_bytes = (None, 0) if workspace is False else (_ptr(workspace), workspace.numel())
    rc = load().sphinx_temporal_block(
        _ptr(x), _ptr(wqkv), _ptr(bqkv), _ptr(wo), _ptr(bo), int(heads), int(frames_per_seq),
        _ptr(qkv_buf), _ptr(o_scratch), _ptr(y), F32 if y.dtype == torch.float32 else BF16,
        n, h, wd, c, int(block), _ptr(block_ids), _ptr(count), int(cap), ws_ptr, ws_bytes,
        _ptr(attn_ws), attn_ws.numel(), _stream(stream))
    _chk("sphinx_temporal_block", rc)


def sphinx_gn_scale_shift(stats, gamma, beta, eps, n, h, w, c, groups, block, table, stream=None):
    """NEXT-3 fused-conv table [N,C,2] = (gamma*rstd, beta - mean*gamma*rstd) from the statistics."""
    import torch
    for t, nm in ((stats, "stats"), (gamma, "gamma"), (beta, "beta"), (table, "table")):
        _dev(t, torch.float32, nm)
    rc = load().sphinx_gn_scale_shift(_ptr(stats), _ptr(gamma), _ptr(beta), float(eps), int(n), int(h), int(w),
                                      int(c), int(groups), int(block), _ptr(table), _stream(stream))
    _chk("sphinx_gn_scale_shift", rc)


def sphinx_sparse_conv3x3_gn_silu(x, scale_shift, w, bias, y, block, block_ids, count, residual=None,
                                  capacity=None, workspace=None, stream=None):
    """NEXT-3: conv3x3 of SiLU(x*scale+shift) with the normalisation fused into the conv's halo
    path (x raw bf16 NHWC; scale_shift fp32 [N,Cin,2])."""
    import torch
    _dev(x, torch.bfloat16, "x")
    _dev(w, torch.bfloat16, "w")
    _dev(scale_shift, torch.float32, "scale_shift")
    _dev(bias, torch.float32, "bias")
    _dev(residual, torch.bfloat16, "residual")
    _dev(block_ids, torch.int32, "block_ids")
    _dev(count, torch.int32, "count")
    n, h, wd, cin = x.shape
    cout = w.shape[0]
    cap = block_ids.numel() if capacity is None else capacity
    if workspace is None:
        workspace = conv_workspace(cout, y.device, n, h, wd, block, stream)
    ws_ptr, ws_bytes = (None, 0) if workspace is False else (_ptr(workspace), workspace.numel())
    rc = load().sphinx_sparse_conv3x3_gn_silu(
        _ptr(x), _ptr(scale_shift), _ptr(w), _ptr(bias), _ptr(residual), _ptr(y),
        F32 if y.dtype == torch.float32 else BF16, n, h, wd, cin, cout, int(block), _ptr(block_ids),
        _ptr(count), int(cap), ws_ptr, ws_bytes, _stream(stream))
    _chk("sphinx_sparse_conv3x3_gn_silu", rc)
