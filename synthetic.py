"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws random
tensors with the shapes, value distributions and spatial structure of the
paper's workloads (DESIGN.md §5 "input recipe").  Both the oracle and the CUDA
path receive exactly these arrays.

Workload shapes: SEVA 576x576 images -> 72x72 latent (/8),
21 frames = 2 inputs + 19 targets, UNet levels 72x72x320,
36x36x640, 18x18x1280 (BASELINE configs[2]).  Opacity follows SPEC's toy
disocclusion recipe: background U(0.8,1.0), low-opacity ellipses
U(0,0.4).
"""
import hashlib
import math

import numpy as np

BASE_SEED = 7  # SPEC's example seed


def rng(*names):
    """Independent PCG64 stream per (BASE_SEED, names...)."""
    h = hashlib.sha256(repr((BASE_SEED,) + tuple(names)).encode()).digest()
    return np.random.Generator(np.random.PCG64(int.from_bytes(h[:8], "little")))


def to_bf16_bits(a):
    """float32 -> bf16 bit patterns (round to nearest even), as uint16."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32)
    r = (u >> 16) & 1                 # uint32 arithmetic: no finite value overflows 2^32
    r += 0x7FFF
    r += u
    r >>= 16
    out = r.astype(np.uint16)
    out[np.isnan(a)] = 0x7FC0
    return out


def bf16_bits_to_f32(b):
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# ------------------------------------------------------------ block choice ---

def choose_cells(rg, hb, wb, n_active, pattern="clustered"):
    """Pick n_active cells of an hb x wb grid. 'clustered' grows 4-connected blobs from
    random seeds (disocclusions are contiguous regions); 'scattered' is uniform;
    'checker' is a checkerboard (halo worst case)."""
    n_active = int(max(0, min(n_active, hb * wb)))
    sel = np.zeros((hb, wb), bool)
    if n_active == 0:
        return sel
    if pattern == "scattered":
        idx = rg.choice(hb * wb, n_active, replace=False)
        sel.flat[idx] = True
        return sel
    if pattern == "checker":
        cand = [(y, x) for y in range(hb) for x in range(wb) if (y + x) % 2 == 0]
        cand += [(y, x) for y in range(hb) for x in range(wb) if (y + x) % 2 == 1]
        for (y, x) in cand[:n_active]:
            sel[y, x] = True
        return sel
    # clustered
    frontier = []
    n_blobs = max(1, n_active // 12)
    while sel.sum() < n_active:
        if not frontier or len(frontier) == 0 or rg.random() < 1.0 / (4 * n_blobs):
            free = np.flatnonzero(~sel.ravel())
            c = free[rg.integers(len(free))]
            y, x = divmod(int(c), wb)
        else:
            y, x = frontier.pop(rg.integers(len(frontier)))
            if sel[y, x]:
                continue
        sel[y, x] = True
        for dy, dx in ((1, 0), (-1, 0), (0, 1), (0, -1)):
            yy, xx = y + dy, x + dx
            if 0 <= yy < hb and 0 <= xx < wb and not sel[yy, xx]:
                frontier.append((yy, xx))
    return sel


def opacity_maps(n, hp, wp, cell_px, densities, pattern="clustered", tag="opacity"):
    """Opacity O [n,hp,wp] fp32.  For frame i, round(densities[i]*cells) cells of
    cell_px x cell_px pixels (cell_px = b*f, one level-0 block footprint) receive one
    low-opacity ellipse U(0,0.4) strictly inside them; everything else U(0.8,1.0)."""
    rg = rng(tag, n, hp, wp, cell_px, pattern)
    O = rg.uniform(0.8, 1.0, size=(n, hp, wp)).astype(np.float32)
    hb, wb = -(-hp // cell_px), -(-wp // cell_px)
    cells = []
    for i in range(n):
        d = float(densities[i] if np.ndim(densities) else densities)
        sel = choose_cells(rg, hb, wb, round(d * hb * wb), pattern)
        cells.append(sel)
        for (cy, cx) in zip(*np.nonzero(sel)):
            y0, x0 = cy * cell_px, cx * cell_px
            hh, ww = min(cell_px, hp - y0), min(cell_px, wp - x0)
            ry = max(0.5, rg.uniform(0.15, 0.5) * hh)
            rx = max(0.5, rg.uniform(0.15, 0.5) * ww)
            my = rg.uniform(ry, max(ry, hh - ry)) if hh > 1 else 0.0
            mx = rg.uniform(rx, max(rx, ww - rx)) if ww > 1 else 0.0
            yy, xx = np.mgrid[0:hh, 0:ww]
            inside = ((yy + 0.5 - my) / ry) ** 2 + ((xx + 0.5 - mx) / rx) ** 2 <= 1.0
            if not inside.any():
                inside[min(int(my), hh - 1), min(int(mx), ww - 1)] = True
            patch = O[i, y0:y0 + hh, x0:x0 + ww]
            patch[inside] = rg.uniform(0.0, 0.4, size=int(inside.sum())).astype(np.float32)
    return O, np.stack(cells)


def uncertainty_maps(n, hp, wp, cell_px, cells, frac_blobs=0.3, tag="uncert"):
    """Uncertainty U [n,hp,wp] in U(0,0.6) with a 0.9 blob inside a fraction of the
    already-chosen cells, plus per-frame threshold tau_u = 0.7 (reading R-10: the
    Otsu producer is NEXT-2, so tau_u is an input)."""
    rg = rng(tag, n, hp, wp, cell_px)
    U = rg.uniform(0.0, 0.6, size=(n, hp, wp)).astype(np.float32)
    for i in range(n):
        for (cy, cx) in zip(*np.nonzero(cells[i])):
            if rg.random() < frac_blobs:
                y = cy * cell_px + rg.integers(min(cell_px, hp - cy * cell_px))
                x = cx * cell_px + rg.integers(min(cell_px, wp - cx * cell_px))
                U[i, y, x] = 0.9
    tau_u = np.full(n, 0.7, np.float32)
    return U, tau_u


# ------------------------------------------------------------ tensors -------

def _chunked_bf16_normal(shape, names, frames_per_chunk=8):
    """N(0,1) -> bf16 bits for a large frame-major tensor: frame chunks drawn from independent
    streams rng(*names, chunk) on a thread pool (numpy releases the GIL), same values whatever
    the thread count."""
    from concurrent.futures import ThreadPoolExecutor
    out = np.empty(shape, np.uint16)
    starts = list(range(0, shape[0], frames_per_chunk))

    def one(i):
        s0 = starts[i]
        sub = (min(frames_per_chunk, shape[0] - s0),) + tuple(shape[1:])
        out[s0:s0 + sub[0]] = to_bf16_bits(rng(*names, i).standard_normal(sub, dtype=np.float32))
    with ThreadPoolExecutor(8) as ex:
        list(ex.map(one, range(len(starts))))
    return out


def features_bf16(shape, tag):
    """x ~ N(0,1) rounded to bf16 (bit patterns).  Batches of more than one request (> 21
    frames) are drawn in independent 8-frame chunks in parallel."""
    if len(shape) == 4 and shape[0] > 21:
        return _chunked_bf16_normal(shape, ("feat-chunk", tag, shape))
    return to_bf16_bits(rng("feat", tag, shape).standard_normal(shape, dtype=np.float32))


def weights_bf16(cout, cin, tag):
    """W ~ N(0, 1/(9 cin)) in OHWI [cout][3][3][cin] (reading R-19), bf16 bits."""
    w = rng("w", tag, cout, cin).standard_normal((cout, 3, 3, cin), dtype=np.float32)
    return to_bf16_bits(w * np.float32(1.0 / math.sqrt(9 * cin)))


def bias_f32(cout, tag):
    return (rng("bias", tag, cout).standard_normal(cout, dtype=np.float32) * np.float32(0.01))


def resblock_features_bf16(shape, tag):
    """NEXT-3 ResNet-block input: per-channel offset U(-1,1) and scale U(0.5,2) on N(0,1)
    (so the GroupNorm statistics are far from (0,1)), rounded to bf16 bits."""
    g = rng("rbfeat", tag, shape)
    c = shape[-1]
    off = g.uniform(-1.0, 1.0, c).astype(np.float32)
    sc = g.uniform(0.5, 2.0, c).astype(np.float32)
    return to_bf16_bits(g.standard_normal(shape, dtype=np.float32) * sc + off)


def gn_affine_f32(c, tag):
    """GroupNorm affine parameters: gamma ~ 1 + 0.2 N(0,1), beta ~ 0.2 N(0,1), fp32 [c]."""
    g = rng("gn", tag, c)
    return ((1.0 + 0.2 * g.standard_normal(c)).astype(np.float32),
            (0.2 * g.standard_normal(c)).astype(np.float32))


def linear_weights_bf16(cout, cin, tag, gain=1.0):
    """Pointwise (1x1) projection W ~ N(0, gain^2/cin), [cout][cin] bf16 bits (NEXT-4 Wqkv, Wo)."""
    w = rng("lin", tag, cout, cin).standard_normal((cout, cin), dtype=np.float32)
    return to_bf16_bits(w * np.float32(gain / math.sqrt(cin)))


ATTN_HEAD_DIM = 64  # SD/SVD attention head width (reading R-28)
GN_GROUPS = 32     # torch/SD UNet Normalize(): GroupNorm(32, C, eps=1e-6) (reading R-26)
GN_EPS = 1e-6


def latents_f32(shape, tag):
    return rng("lat", tag, shape).standard_normal(shape, dtype=np.float32)


def abar_cosine(S=50):
    """S:43 cosine table abar[u] = cos^2((pi/2)(1-u/S)*0.98), u=0 noisiest.
    abar[S] = cos^2(0) = 1, so SPEC's renormalisation is a no-op (reading R-5)."""
    u = np.arange(S + 1, dtype=np.float64)
    a = np.cos((math.pi / 2) * (1.0 - u / S) * 0.98) ** 2
    return a.astype(np.float32)


def abar_linear(S=50):
    """S:43 linear table abar[0] = 0.01 -> abar[S] = 1."""
    return np.linspace(0.01, 1.0, S + 1).astype(np.float32)


def request_scores(n_frames=21, c0=62.0, c1=66.0, tag="req"):
    """Per-frame (q, c0, c1, t) for one request: frames 0 and n-1 are the input views
    (2 inputs), targets t_i = i/(n-1).  q follows a U-shaped quality dip
    toward the middle (Fig. avg_k): q_i = mean(c0,c1)(1 - 0.2 sin(pi t)) + noise."""
    rg = rng("scores", tag, n_frames)
    t = np.arange(n_frames, dtype=np.float64) / (n_frames - 1)
    base = 0.5 * (c0 + c1)
    q = base * (1.0 - 0.2 * np.sin(math.pi * t)) + 0.6 * rg.standard_normal(n_frames)
    return (q.astype(np.float32), np.full(n_frames, c0, np.float32),
            np.full(n_frames, c1, np.float32), t.astype(np.float32))


def request_densities(n_frames=21, mean=0.25, lo=0.05, hi=0.60):
    """Per-frame level-0 block density, proportional to sin(pi t), clipped, rescaled to
    the requested mean (frames far from the inputs have more disocclusion)."""
    t = np.arange(n_frames) / (n_frames - 1)
    d = np.sin(math.pi * t) + 0.05
    for _ in range(50):
        d = np.clip(d * (mean / max(d.mean(), 1e-9)), lo, hi)
    return d


SPEC_KLOGIC = dict(thr=[0.85, 0.92, 0.97], steps=[10, 25, 40], fallback_k=0, k_max=40)


def exhaustive_block_patterns(grid=4, cell=4, tag="exhaustive"):
    """Every one of the 2^(grid*grid) block patterns of a grid x grid block map (configs[0]
    geometry: 16x16 pixels, f=1, b=4): frame p paints one flagged pixel U(0, 0.4999) at a
    random spot of every block whose bit is set in p; everything else U(0.5, 1.0) (0.5 itself
    is not flagged, R-8).  Returns (O [2^(g*g), g*cell, g*cell] fp32, pattern bool [n, g*g])."""
    nb = grid * grid
    n = 1 << nb
    pat = ((np.arange(n)[:, None] >> np.arange(nb)[None, :]) & 1).astype(bool)
    rg = rng("pin-exhaustive", grid, cell) if tag == "exhaustive" else rng(tag, grid, cell)
    side = grid * cell
    O = rg.uniform(0.5, 1.0, size=(n, side, side)).astype(np.float32)
    oy = rg.integers(0, cell, size=(n, nb))
    ox = rg.integers(0, cell, size=(n, nb))
    fi, bi = np.nonzero(pat)
    by, bx = bi // grid, bi % grid
    O[fi, by * cell + oy[fi, bi], bx * cell + ox[fi, bi]] = rg.uniform(0, 0.4999, size=len(fi))
    return O, pat


def sparse_pixel_maps(n, hp, wp, cell_px, n_px, tag="sparse-px"):
    """Opacity + uncertainty maps with UNIFORMLY RANDOM isolated flagged pixels (no cell
    structure): per frame n_px opacity pixels drawn U(0, 0.5) and n_px uncertainty spikes, half
    of each placed on a row AND/OR column adjacent to a multiple of cell_px (block-footprint
    boundaries, where an off-by-one in the footprint arithmetic shows), plus per frame one
    opacity pixel exactly at tau_o = 0.5 and one uncertainty pixel exactly at tau_u (equality:
    not flagged, R-8) and one NaN pixel (flagged, R-9).  Background opacity U(0.5+, 1.0),
    uncertainty U(0, 0.6), tau_u = 0.7.  Returns (O, U, tau_u)."""
    rg = rng(tag, n, hp, wp, cell_px, n_px)
    O = rg.uniform(0.5000001, 1.0, size=(n, hp, wp)).astype(np.float32)
    U = rg.uniform(0.0, 0.6, size=(n, hp, wp)).astype(np.float32)
    tau_u = np.full(n, 0.7, np.float32)

    def coords(k):
        y = rg.integers(0, hp, size=k)
        x = rg.integers(0, wp, size=k)
        half = k // 2
        # boundary rows/cols: c*cell_px - 1 or c*cell_px (the last / first pixel of a footprint)
        by = rg.integers(0, -(-hp // cell_px), size=half) * cell_px - rg.integers(0, 2, size=half)
        bx = rg.integers(0, -(-wp // cell_px), size=half) * cell_px - rg.integers(0, 2, size=half)
        which = rg.integers(0, 3, size=half)  # 0: row only, 1: column only, 2: both
        y[:half] = np.where(which != 1, np.clip(by, 0, hp - 1), y[:half])
        x[:half] = np.where(which != 0, np.clip(bx, 0, wp - 1), x[:half])
        return y, x

    for i in range(n):
        y, x = coords(n_px)
        O[i, y, x] = rg.uniform(0.0, 0.5, size=n_px).astype(np.float32)
        y, x = coords(n_px)
        U[i, y, x] = rg.uniform(0.71, 1.0, size=n_px).astype(np.float32)
        y, x = coords(3)
        O[i, y[0], x[0]] = np.float32(0.5)
        U[i, y[1], x[1]] = tau_u[i]
        if i % 2 == 0:
            O[i, y[2], x[2]] = np.nan
        else:
            U[i, y[2], x[2]] = np.nan
    return O, U, tau_u


# ------------------------------------------------------------ request batches ---

UNET_LEVELS = ((72, 320), (36, 640), (18, 1280))     # BASELINE configs[2]
CONFIG3_REQUEST_DENSITIES = (0.05, 0.10, 0.25, 0.50, 0.75, 0.25, 0.10, 0.05)  # BASELINE configs[3]


def make_batch(request_means, tag="r0", hp=576, f=8, b=8, levels=UNET_LEVELS, convs_per_level=2,
               frames_per_request=21, pattern="clustered", c_lat=4, S=50, lo=None, hi=None):
    """Host inputs of a batch of requests (DESIGN.md input recipe): per request, per-frame
    level-0 densities U-shaped around the request's mean (request_densities), toy-disocclusion
    opacity + uncertainty maps, U-shaped scores; frames 0 and n-1 of every request are its
    conditioning inputs (logic_id -1, R-14); latents, level features, caches, conv weights.
    With one request and tag 'r0' this is exactly the round-1 configs[2] request."""
    n_req = len(request_means)
    fpr = frames_per_request
    one = n_req == 1
    O, U, tau, q, c0, c1, t, lid = [], [], [], [], [], [], [], []
    for r, mean in enumerate(request_means):
        rt = tag if one else f"{tag}.{r}"
        kw = {}
        if lo is not None or not one:
            kw["lo"] = lo if lo is not None else 1.0 / ((hp // f // b) ** 2)
        if hi is not None or not one:
            kw["hi"] = hi if hi is not None else 1.0
        dens = request_densities(fpr, mean, **kw)
        o, cells = opacity_maps(fpr, hp, hp, b * f, dens, pattern, tag=f"O{rt}")
        uu, tu = uncertainty_maps(fpr, hp, hp, b * f, cells, tag=f"U{rt}")
        qq, a0, a1, tt = request_scores(fpr, tag=f"q{rt}")
        li = np.zeros(fpr, np.int32)
        li[0] = li[-1] = -1
        for lst, v in ((O, o), (U, uu), (tau, tu), (q, qq), (c0, a0), (c1, a1), (t, tt), (lid, li)):
            lst.append(v)
    cat = np.concatenate
    F = n_req * fpr
    h0 = hp // f
    batch = dict(O=cat(O), U=cat(U), tau_u=cat(tau), q=cat(q), c0=cat(c0), c1=cat(c1), t=cat(t), lid=cat(lid),
                 abar=abar_cosine(S), klogic=dict(SPEC_KLOGIC))
    batch["x0"] = latents_f32((F, h0, h0, c_lat), f"x0{tag}")
    batch["eps"] = latents_f32((F, h0, h0, c_lat), f"eps{tag}")
    batch["lat_cache"] = latents_f32((F, h0, h0, c_lat), f"lc{tag}")
    for l, (h, c) in enumerate(levels):
        batch[f"feat{l}"] = features_bf16((F, h, h, c), f"x{l}{tag}")
        batch[f"cache{l}"] = features_bf16((F, h, h, c), f"c{l}{tag}")
        for j in range(convs_per_level):
            batch[f"w{l}{j}"] = weights_bf16(c, c, f"w{l}{j}")
            batch[f"b{l}{j}"] = bias_f32(c, f"b{l}{j}")
    return batch


def rgb_frames(n, h, w, tag):
    """Regression-output-like RGB frames in [0,1] (NEXT-2 input): smooth gradients with sharp
    texture everywhere except a few flat disc-shaped patches (the blurry regions Otsu separates)."""
    rg = rng("gpu-rgb", tag, n, h, w)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float32)
    out = np.empty((n, h, w, 3), np.float32)
    for i in range(n):
        base = 0.5 + 0.3 * np.sin(yy / (7 + i)) * np.cos(xx / (11 + i))
        tex = rg.random((h, w)).astype(np.float32) * 0.4
        blur = np.zeros((h, w), bool)
        for _ in range(3):
            cy, cx, r = rg.integers(0, h), rg.integers(0, w), rg.integers(h // 10 + 2, h // 4 + 3)
            blur |= (yy - cy) ** 2 + (xx - cx) ** 2 < r * r
        img = np.where(blur, base, base + tex - 0.2)
        out[i] = np.clip(np.stack([img, img * 0.9, img * 1.1], -1), 0, 1)
    return out
