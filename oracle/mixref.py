"""numpy float64 restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.

Follows `/root/reference/pkg/src/mixserve/{csp,kernels,patched,cache,model}.py`
(cited per function).  Arithmetic order is kept identical to the reference
wherever the reference pins bits (channel-ordered contractions, numpy reductions
over the same axes, 256-row attention chunks) so the golden vectors recorded
from the reference compare bit-exactly where the reference is deterministic.

Only tests, `__graft_entry__.smoke()` and bench.py's CPU legs use this module.

BLAS mode (`blas_contractions()` / `DENSE_BLAS`): the channel contractions (linear, FF, 1x1
and 3x3 conv) run as fp64 matrix products instead of the reference's channel-ordered axpy
loops.  Same fp64 arithmetic, different summation order: results differ from the reference
by fp64 rounding only (~1e-15 relative; tests/test_oracle_golden.py checks the mode against
the golden vectors at 1e-10).  It makes the C = 320 parity checks at the benchmark's shapes
(tests/test_gpu_parity_c320.py) run in seconds instead of minutes; bit-exact comparisons
(masks, copies) never depend on it.
"""

from __future__ import annotations

import contextlib
import math
import zlib
from dataclasses import dataclass, field, replace
from typing import Sequence

import numpy as np

from .pairwise import np_mean_sq_diff

# ----------------------------------------------------------------- errors
# errors.py:4-9


class InputError(ValueError):
    pass


class IntegrityError(RuntimeError):
    pass


# ------------------------------------------------------------------- CSP
# csp.py:20-23 — neighbour directions clockwise from north
DIRECTIONS = ("N", "NE", "E", "SE", "S", "SW", "W", "NW")
DIR_STEPS = ((-1, 0), (-1, 1), (0, 1), (1, 1), (1, 0), (1, -1), (0, -1), (-1, -1))
STANDARD_LATENTS = {"low": 64, "med": 96, "high": 128}  # csp.py:42-46 (pixel/8)


def choose_patch_size(dims) -> int:
    """csp.py:49-56 — gcd of the latent dims."""
    dims = list(dims)
    if not dims or any(d <= 0 for d in dims):
        raise InputError("bad latent dims")
    return math.gcd(*dims)


@dataclass
class Req:
    request_id: str
    latent: int
    side: int
    patch_start: int
    patch_count: int


@dataclass
class Batch:
    """csp.py:68-114 (CSPBatch) restated."""

    patch_size: int
    data: np.ndarray
    requests: list
    request_offset: np.ndarray
    resolution_dims: list
    resolution_offset: np.ndarray
    request_index: np.ndarray
    ordinal: np.ndarray
    row: np.ndarray
    col: np.ndarray
    neighbors: np.ndarray

    @property
    def n_patches(self):
        return self.data.shape[0]

    @property
    def n_requests(self):
        return len(self.requests)

    def slot(self, rid):
        for i, e in enumerate(self.requests):
            if e.request_id == rid:
                return i
        raise InputError(rid)

    def patches_of_request(self, rid) -> slice:
        r = self.slot(rid)
        return slice(int(self.request_offset[r]), int(self.request_offset[r + 1]))

    def patch_key(self, p):
        return (self.requests[int(self.request_index[p])].request_id, int(self.ordinal[p]))


def csp_metadata(dims: Sequence[int], ps: int):
    """Integer half of split (csp.py:142-179): order, offsets, per-patch tables."""
    order = sorted(range(len(dims)), key=lambda i: dims[i])  # stable, csp.py:143
    sides = [dims[i] // ps for i in order]
    counts = [s * s for s in sides]
    request_offset = np.zeros(len(order) + 1, dtype=np.int64)
    request_offset[1:] = np.cumsum(counts)
    total = int(request_offset[-1])
    request_index = np.empty(total, dtype=np.int64)
    ordinal = np.empty(total, dtype=np.int64)
    row = np.empty(total, dtype=np.int64)
    col = np.empty(total, dtype=np.int64)
    nbr = np.full((total, 8), -1, dtype=np.int64)
    for slot, side in enumerate(sides):
        base = int(request_offset[slot])
        k = np.arange(side * side)
        request_index[base:base + side * side] = slot
        ordinal[base:base + side * side] = k
        row[base:base + side * side] = k // side
        col[base:base + side * side] = k % side
        for d, (dr, dc) in enumerate(DIR_STEPS):
            rr, cc = k // side + dr, k % side + dc
            ok = (rr >= 0) & (rr < side) & (cc >= 0) & (cc < side)
            nbr[base + k[ok], d] = base + rr[ok] * side + cc[ok]
    res_dims = sorted(set(dims))
    resolution_offset = np.zeros(len(res_dims) + 1, dtype=np.int64)
    for g, d in enumerate(res_dims):
        resolution_offset[g + 1] = resolution_offset[g] + sum(
            c for c, i in zip(counts, order) if dims[i] == d)
    return order, sides, request_offset, res_dims, resolution_offset, request_index, ordinal, row, col, nbr


def split(requests, patch_size=None) -> Batch:
    """csp.py:117-193."""
    if not requests:
        raise InputError("empty batch")
    ids = [r for r, _ in requests]
    if len(set(ids)) != len(ids):
        raise InputError("duplicate ids")
    arrs = [np.asarray(a, dtype=np.float64) for _, a in requests]
    for a in arrs:
        if a.ndim != 3 or a.shape[1] != a.shape[2]:
            raise InputError("latent must be (C,H,H)")
    if any(a.shape[0] != arrs[0].shape[0] for a in arrs):
        raise InputError("channel mismatch")
    dims = [a.shape[1] for a in arrs]
    ps = choose_patch_size(dims) if patch_size is None else patch_size
    if any(d % ps for d in dims):
        raise InputError("patch size does not tile")
    order, sides, ro, rd, so, ri, od, rw, cl, nb = csp_metadata(dims, ps)
    c = arrs[0].shape[0]
    data = np.empty((int(ro[-1]), c, ps, ps))
    reqs = []
    for slot, src in enumerate(order):
        s = sides[slot]
        base = int(ro[slot])
        # (C, s*ps, s*ps) -> (s, s, C, ps, ps) pure copy (csp.py:161-167)
        tiles = arrs[src].reshape(c, s, ps, s, ps).transpose(1, 3, 0, 2, 4)
        data[base:base + s * s] = tiles.reshape(s * s, c, ps, ps)
        reqs.append(Req(ids[src], dims[src], s, base, s * s))
    return Batch(ps, data, reqs, ro, rd, so, ri, od, rw, cl, nb)


def reassemble(batch: Batch, data=None) -> dict:
    """csp.py:196-214."""
    src = batch.data if data is None else np.asarray(data)
    if src.shape != batch.data.shape:
        raise InputError("shape mismatch")
    ps = batch.patch_size
    out = {}
    for e in batch.requests:
        s = e.side
        t = src[e.patch_start:e.patch_start + e.patch_count].reshape(s, s, src.shape[1], ps, ps)
        out[e.request_id] = np.ascontiguousarray(t.transpose(2, 0, 3, 1, 4).reshape(src.shape[1], s * ps, s * ps))
    return out


# --------------------------------------------------------------- params
# kernels.py:27-96


@dataclass(frozen=True)
class ConvParams:
    weights: np.ndarray  # (C_out, C_in, k, k)
    bias: np.ndarray

    @property
    def kernel_size(self):
        return self.weights.shape[2]


@dataclass(frozen=True)
class GroupNormParams:
    groups: int
    gamma: np.ndarray
    beta: np.ndarray
    eps: float = 1e-5


@dataclass(frozen=True)
class LayerNormParams:
    gamma: np.ndarray
    beta: np.ndarray
    eps: float = 1e-5


@dataclass(frozen=True)
class LinearParams:
    weights: np.ndarray  # (C_out, C_in)
    bias: np.ndarray


@dataclass(frozen=True)
class FeedForwardParams:
    w1: np.ndarray  # (H, C)
    b1: np.ndarray
    w2: np.ndarray  # (C, H)
    b2: np.ndarray


@dataclass(frozen=True)
class AttentionParams:
    wq: np.ndarray  # (D_in, D_out); used as x @ w (kernels.py:264-267)
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray


# -------------------------------------------------------- dense kernels


def _f64(x):
    a = np.asarray(x, dtype=np.float64)
    if not np.all(np.isfinite(a)):
        raise InputError("non-finite")
    return a


DENSE_BLAS = False


@contextlib.contextmanager
def blas_contractions():
    """Evaluate the channel contractions as fp64 BLAS products inside the block."""
    global DENSE_BLAS
    prev, DENSE_BLAS = DENSE_BLAS, True
    try:
        yield
    finally:
        DENSE_BLAS = prev


def channel_contract(w, b, x):
    """kernels.py:99-111 — per output channel, accumulate input channels in order."""
    w, b, x = _f64(w), _f64(b), _f64(x)
    if DENSE_BLAS:
        xm = np.moveaxis(x, 1, -1)  # (N, ..., C_in)
        return np.moveaxis(xm @ w.T + b, -1, 1)
    out = np.empty((x.shape[0], w.shape[0]) + x.shape[2:])
    for o in range(w.shape[0]):
        acc = np.full(x.shape[:1] + x.shape[2:], b[o])
        for c in range(w.shape[1]):
            acc += w[o, c] * x[:, c]
        out[:, o] = acc
    return out


def gelu(x):
    """kernels.py:118-121 (tanh form)."""
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * x * (1.0 + np.tanh(0.7978845608028654 * (x + 0.044715 * x * x * x)))


def feed_forward(x, p: FeedForwardParams):
    """kernels.py:124-127."""
    return channel_contract(p.w2, p.b2, gelu(channel_contract(p.w1, p.b1, x)))


def linear(x, p: LinearParams):
    """kernels.py:114-115."""
    return channel_contract(p.weights, p.bias, x)


def conv_valid(xpad, w, b):
    """kernels.py:148-161 — channel, then tap order accumulation over a padded input."""
    xpad, w, b = _f64(xpad), _f64(w), _f64(b)
    n, _, hp, wp = xpad.shape
    k = w.shape[2]
    h, wd = hp - k + 1, wp - k + 1
    if DENSE_BLAS:
        # im2col per chunk of patches: (N, C*k*k, h*w) columns, one (C_out, C*k*k) product
        out = np.empty((n, w.shape[0], h, wd))
        wm = w.reshape(w.shape[0], -1)
        for n0 in range(0, n, 8):
            xs = xpad[n0:n0 + 8]
            cols = np.empty((xs.shape[0], xs.shape[1], k, k, h, wd))
            for ki in range(k):
                for kj in range(k):
                    cols[:, :, ki, kj] = xs[:, :, ki:ki + h, kj:kj + wd]
            out[n0:n0 + 8] = (wm @ cols.reshape(xs.shape[0], -1, h * wd)).reshape(xs.shape[0], -1, h, wd)
        return out + b[None, :, None, None]
    out = np.empty((n, w.shape[0], h, wd))
    for o in range(w.shape[0]):
        acc = np.full((n, h, wd), b[o])
        for c in range(w.shape[1]):
            for ki in range(k):
                for kj in range(k):
                    acc += w[o, c, ki, kj] * xpad[:, c, ki:ki + h, kj:kj + wd]
        out[:, o] = acc
    return out


def conv2d(x, p: ConvParams):
    """kernels.py:164-178 — zero padding at image borders."""
    x = _f64(x)
    pad = p.kernel_size // 2
    if pad:
        xp = np.zeros((x.shape[0], x.shape[1], x.shape[2] + 2 * pad, x.shape[3] + 2 * pad))
        xp[:, :, pad:-pad, pad:-pad] = x
    else:
        xp = x
    return conv_valid(xp, p.weights, p.bias)


def group_norm(x, p: GroupNormParams):
    """kernels.py:181-206 — statistics per (image, group)."""
    x = _f64(x)
    n, c, h, w = x.shape
    xg = x.reshape(n, p.groups, (c // p.groups) * h * w)
    mean = xg.mean(axis=2)
    var = ((xg - mean[:, :, None]) ** 2).mean(axis=2)
    cg = c // p.groups
    xn = (x.reshape(n, p.groups, cg, h, w) - mean[:, :, None, None, None]) / np.sqrt(
        var[:, :, None, None, None] + p.eps)
    return xn.reshape(n, c, h, w) * _f64(p.gamma)[None, :, None, None] + _f64(p.beta)[None, :, None, None]


def layer_norm(x, p: LayerNormParams):
    """kernels.py:209-227 — channel-ordered mean/var per position."""
    x = _f64(x)
    c = x.shape[1]
    s = x[:, 0].copy()
    for ci in range(1, c):
        s += x[:, ci]
    mean = s / c
    v = (x[:, 0] - mean) ** 2
    for ci in range(1, c):
        v += (x[:, ci] - mean) ** 2
    inv = 1.0 / np.sqrt(v / c + p.eps)
    out = np.empty_like(x)
    g, bt = _f64(p.gamma), _f64(p.beta)
    for ci in range(c):
        out[:, ci] = (x[:, ci] - mean) * inv * g[ci] + bt[ci]
    return out


ATTN_CHUNK = 256  # kernels.py:17


def attend(q, k, v):
    """kernels.py:230-243 — 256-row chunked softmax(q k^T / sqrt(D)) v."""
    t, d = q.shape
    scale = 1.0 / np.sqrt(d)
    kt = np.ascontiguousarray(k.T)
    out = np.empty_like(v)
    for i in range(0, t, ATTN_CHUNK):
        s = (q[i:i + ATTN_CHUNK] @ kt) * scale
        s -= s.max(axis=1, keepdims=True)
        np.exp(s, out=s)
        s /= s.sum(axis=1, keepdims=True)
        out[i:i + ATTN_CHUNK] = s @ v
    return out


def attend_tokens(tokens, p: AttentionParams):
    """kernels.py:257-267."""
    tokens = _f64(tokens)
    return attend(tokens @ p.wq, tokens @ p.wk, tokens @ p.wv) @ p.wo


def image_to_tokens(img):
    """kernels.py:270-273 — (C,H,W) -> (H*W, C) row-major."""
    return img.reshape(img.shape[0], -1).T.copy()


def tokens_to_image(t, h, w):
    """kernels.py:276-277."""
    return t.T.reshape(t.shape[1], h, w).copy()


def pixelwise(kind, x, params):
    """kernels.py:137-145."""
    if kind == "linear":
        return linear(x, params)
    if kind == "feed_forward":
        return feed_forward(x, params)
    raise InputError(kind)


# ------------------------------------------------------- patched ops
LAUNCHES: dict = {}


def _launch(kind):
    LAUNCHES[kind] = LAUNCHES.get(kind, 0) + 1


def exchange_halos(batch: Batch, data):
    """patched.py:57-89 — (P,C,ps+2,ps+2) frames, zero where no neighbour."""
    data = _f64(data)
    pn, c, ps, _ = data.shape
    fr = np.zeros((pn, c, ps + 2, ps + 2))
    fr[:, :, 1:-1, 1:-1] = data
    nb = batch.neighbors
    # (direction, frame rows, frame cols, source rows, source cols)
    pieces = (
        (0, 0, slice(1, -1), -1, slice(None)),
        (4, -1, slice(1, -1), 0, slice(None)),
        (6, slice(1, -1), 0, slice(None), -1),
        (2, slice(1, -1), -1, slice(None), 0),
        (7, 0, 0, -1, -1),
        (1, 0, -1, -1, 0),
        (5, -1, 0, 0, -1),
        (3, -1, -1, 0, 0),
    )
    for p in range(pn):
        for d, fr_r, fr_c, sr, sc in pieces:
            q = nb[p, d]
            if q >= 0:
                fr[p, :, fr_r, fr_c] = data[q, :, sr, sc]
    return fr


def patched_conv(batch, data, p: ConvParams, frames=None):
    """patched.py:92-113."""
    data = _f64(data)
    if p.kernel_size == 1:
        _launch("conv")
        return conv_valid(data, p.weights, p.bias)
    if frames is None:
        frames = exchange_halos(batch, data)
        _launch("halo_exchange")
    _launch("conv")
    return conv_valid(frames, p.weights, p.bias)


def stitched_group_norm(batch, data, p: GroupNormParams, emit_halos=False):
    """patched.py:116-144 — stats pooled over each request's patches (axes 0,2,3,4)."""
    data = _f64(data)
    c = data.shape[1]
    cg = c // p.groups
    ps = batch.patch_size
    out = np.empty_like(data)
    g, b = _f64(p.gamma), _f64(p.beta)
    for e in batch.requests:
        sl = slice(e.patch_start, e.patch_start + e.patch_count)
        v = data[sl].reshape(e.patch_count, p.groups, cg, ps, ps)
        mean = v.mean(axis=(0, 2, 3, 4))
        var = ((v - mean[None, :, None, None, None]) ** 2).mean(axis=(0, 2, 3, 4))
        xn = (v - mean[None, :, None, None, None]) / np.sqrt(var[None, :, None, None, None] + p.eps)
        out[sl] = xn.reshape(e.patch_count, c, ps, ps) * g[None, :, None, None] + b[None, :, None, None]
    _launch("group_norm")
    if emit_halos:
        return out, exchange_halos(batch, out)
    return out


def patched_layer_norm(batch, data, p: LayerNormParams):
    """patched.py:147-151."""
    _launch("layer_norm")
    return layer_norm(data, p)


def stitch(batch, data, e: Req):
    ps = batch.patch_size
    s = e.side
    t = data[e.patch_start:e.patch_start + e.patch_count].reshape(s, s, data.shape[1], ps, ps)
    return np.ascontiguousarray(t.transpose(2, 0, 3, 1, 4).reshape(data.shape[1], s * ps, s * ps))


def unstitch(img, ps):
    c, h, _ = img.shape
    s = h // ps
    return img.reshape(c, s, ps, s, ps).transpose(1, 3, 0, 2, 4).reshape(s * s, c, ps, ps)


def patched_self_attention(batch, data, p: AttentionParams):
    """patched.py:154-176 — stitch each image, attend, re-split."""
    data = _f64(data)
    out = np.empty_like(data)
    for e in batch.requests:
        img = stitch(batch, data, e)
        res = tokens_to_image(attend_tokens(image_to_tokens(img), p), e.latent, e.latent)
        out[e.patch_start:e.patch_start + e.patch_count] = unstitch(res, batch.patch_size)
    _launch("attention")
    return out


# precision-emulation hook (tools/drift_emulation.py only): when set, applied to every stage's
# output inside run_block (e.g. bf16 rounding of the intra-block activations); None = exact
STAGE_ROUND = None


def run_block(batch, x, ops):
    """patched.py:179-221 — stage interpreter; GN followed by conv k3 emits halos."""
    x = _f64(x)
    cur, frames = x, None
    rnd = STAGE_ROUND
    for i, (kind, prm) in enumerate(ops):
        if rnd is not None and i > 0:
            cur = rnd(cur)
            if frames is not None:
                frames = rnd(frames)
        nxt = ops[i + 1] if i + 1 < len(ops) else None
        if kind == "group_norm":
            if nxt is not None and nxt[0] == "conv" and nxt[1].kernel_size == 3:
                cur, frames = stitched_group_norm(batch, cur, prm, emit_halos=True)
            else:
                cur, frames = stitched_group_norm(batch, cur, prm), None
            continue
        if kind == "conv":
            cur = patched_conv(batch, cur, prm, frames=frames)
        elif kind == "layer_norm":
            cur = patched_layer_norm(batch, cur, prm)
        elif kind == "attention":
            cur = patched_self_attention(batch, cur, prm)
        elif kind in ("feed_forward", "linear"):
            cur = pixelwise(kind, cur, prm)
            _launch(kind)
        elif kind == "residual":
            cur = cur + x
            _launch("residual")
        else:
            raise InputError(kind)
        frames = None
    return cur


def masked_block_forward(batch, x, mask, ops, cached_inputs, cached_outputs):
    """patched.py:224-246 — substitute cached inputs, run, splice cached outputs."""
    x = _f64(x)
    mask = np.asarray(mask)
    if mask.shape != (batch.n_patches,) or mask.dtype != np.bool_:
        raise InputError("bad mask")
    if mask.all():
        return np.array(cached_outputs, dtype=np.float64, copy=True)
    if not mask.any():
        return run_block(batch, x, ops)
    sel = mask[:, None, None, None]
    y = run_block(batch, np.where(sel, _f64(cached_inputs), x), ops)
    return np.where(sel, _f64(cached_outputs), y)


def run_block_whole(img, ops):
    """model.py:106-126 — dense interpreter on one (C,H,W) image."""
    x = np.asarray(img, dtype=np.float64)[None]
    cur = x
    for kind, prm in ops:
        if kind == "group_norm":
            cur = group_norm(cur, prm)
        elif kind == "layer_norm":
            cur = layer_norm(cur, prm)
        elif kind == "conv":
            cur = conv2d(cur, prm)
        elif kind == "attention":
            h, w = cur.shape[2], cur.shape[3]
            cur = tokens_to_image(attend_tokens(image_to_tokens(cur[0]), prm), h, w)[None]
        elif kind in ("feed_forward", "linear"):
            cur = pixelwise(kind, cur, prm)
        elif kind == "residual":
            cur = cur + x
        else:
            raise InputError(kind)
    return cur[0]


# ------------------------------------------------------------- cache
# cache.py:23-192


def mse(a, b) -> float:
    """cache.py:54-55 (numpy pairwise mean, restated in pairwise.py)."""
    return np_mean_sq_diff(a, b)


def partition_sets(prev_keys, cur_keys):
    """cache.py:58-70."""
    ps_, cs = set(prev_keys), set(cur_keys)
    if len(ps_) != len(prev_keys) or len(cs) != len(cur_keys):
        raise InputError("duplicate keys")
    return ([k for k in cur_keys if k in ps_], [k for k in cur_keys if k not in ps_],
            [k for k in prev_keys if k not in cs])


@dataclass(frozen=True)
class Entry:
    input_snapshot: np.ndarray
    output_snapshot: np.ndarray
    reuse_streak: int = 0


@dataclass
class Stats:
    predicted_reuse: int = 0
    fresh_compute: int = 0
    inserted: int = 0
    refreshed: int = 0
    evicted: int = 0


class Cache:
    """cache.py:73-181 — per-block dict stores with batched ops."""

    def __init__(self, n_blocks, sigma=0.1, max_streak=3):
        self.sigma, self.max_streak = sigma, max_streak
        self.stores = [dict() for _ in range(n_blocks)]
        self.stats = Stats()

    def predict_reuse(self, b, keys, inputs):
        st = self.stores[b]
        mask = np.zeros(len(keys), dtype=bool)
        for i, k in enumerate(keys):
            e = st.get(k)
            mask[i] = (e is not None and mse(inputs[i], e.input_snapshot) < self.sigma
                       and e.reuse_streak < self.max_streak)
        self.stats.predicted_reuse += int(mask.sum())
        self.stats.fresh_compute += int((~mask).sum())
        return mask

    def gather(self, b, keys, mask, shape):
        st = self.stores[b]
        ins = np.zeros((len(keys),) + tuple(shape))
        outs = np.zeros_like(ins)
        for i, k in enumerate(keys):
            if mask[i]:
                e = st.get(k)
                if e is None:
                    raise IntegrityError(k)
                ins[i], outs[i] = e.input_snapshot, e.output_snapshot
        return ins, outs

    def batched_fill(self, b, keys, mask, out=None):
        st = self.stores[b]
        for i, k in enumerate(keys):
            if mask[i]:
                e = st.get(k)
                if e is None:
                    raise IntegrityError(k)
                if out is not None:
                    out[i] = e.output_snapshot
                st[k] = replace(e, reuse_streak=e.reuse_streak + 1)
        return out

    def batched_update(self, b, keys, mask, inputs, outputs):
        st = self.stores[b]
        for i, k in enumerate(keys):
            if not mask[i]:
                if k in st:
                    self.stats.refreshed += 1
                else:
                    self.stats.inserted += 1
                st[k] = Entry(np.array(inputs[i], copy=True), np.array(outputs[i], copy=True), 0)

    def evict_expired(self, live_keys):
        live = set(live_keys)
        n = 0
        for st in self.stores:
            dead = [k for k in st if k not in live]
            for k in dead:
                del st[k]
            n += len(dead)
        self.stats.evicted += n
        return n


# ------------------------------------------------------------- model
# model.py:28-166

RATE_START, RATE_END = 0.15, 0.05


@dataclass(frozen=True)
class ModelConfig:
    arch: str = "dit_like"
    channels: int = 4
    hidden: int = 8
    n_blocks: int = 2
    groups: int = 2
    seed: int = 0


def rate_schedule(step_idx, total_steps):
    """model.py:56-63."""
    if not 0 <= step_idx < total_steps:
        raise InputError("step out of range")
    if total_steps == 1:
        return RATE_START
    return RATE_START + (RATE_END - RATE_START) * (step_idx / (total_steps - 1))


def init_weights(cfg: ModelConfig):
    """model.py:66-94 — identical draw order from default_rng(seed)."""
    rng = np.random.default_rng(cfg.seed)
    c, h = cfg.channels, cfg.hidden
    blocks = []
    for _ in range(cfg.n_blocks):
        gamma = 1.0 + 0.05 * rng.normal(size=c)
        beta = 0.05 * rng.normal(size=c)
        at = AttentionParams(*(rng.normal(size=(c, c)) * (0.8 / np.sqrt(c)) for _ in range(4)))
        ff = FeedForwardParams(
            w1=rng.normal(size=(h, c)) * (0.8 / np.sqrt(c)),
            b1=0.01 * rng.normal(size=h),
            w2=rng.normal(size=(c, h)) * (0.8 / np.sqrt(h)),
            b2=0.01 * rng.normal(size=c),
        )
        if cfg.arch == "unet_like":
            gn = GroupNormParams(cfg.groups, gamma, beta)
            c3 = ConvParams(rng.normal(size=(c, c, 3, 3)) * (0.8 / np.sqrt(9 * c)), 0.01 * rng.normal(size=c))
            blocks.append([("group_norm", gn), ("conv", c3), ("attention", at),
                           ("feed_forward", ff), ("residual", None)])
        else:
            blocks.append([("layer_norm", LayerNormParams(gamma, beta)), ("attention", at),
                           ("feed_forward", ff), ("residual", None)])
    return blocks


def make_prompt(cfg: ModelConfig, request_id: str):
    """model.py:97-103."""
    digest = (zlib.crc32(request_id.encode()) ^ (cfg.seed * 0x9E3779B9)) & 0xFFFFFFFF
    return 0.1 * np.random.default_rng(digest).normal(size=cfg.channels)


def blend(x, h, rate):
    """model.py:129-131."""
    return (1.0 - rate) * x + rate * np.tanh(h)


def denoise_image(cfg, weights, img, prompt, step_idx, total_steps):
    """model.py:134-143."""
    img = np.asarray(img, dtype=np.float64)
    h = img + np.asarray(prompt, dtype=np.float64)[:, None, None]
    for ops in weights:
        h = run_block_whole(h, ops)
    return blend(img, h, rate_schedule(step_idx, total_steps))


def denoise_batch(cfg, weights, batch, prompts, step_idx, total_steps, round_fn=None):
    """model.py:146-166.  `round_fn` (optional) rounds after every block, to emulate
    a reduced-precision residual stream when checking tolerance budgets."""
    bias = np.stack([np.asarray(prompts[e.request_id], dtype=np.float64) for e in batch.requests])
    rate = np.array([rate_schedule(step_idx[e.request_id], total_steps[e.request_id]) for e in batch.requests])
    h = batch.data + bias[batch.request_index][:, :, None, None]
    if round_fn is not None:
        h = round_fn(h)
    for ops in weights:
        h = run_block(batch, h, ops)
        if round_fn is not None:
            h = round_fn(h)
    return blend(batch.data, h, rate[batch.request_index][:, None, None, None])


def latent_for(seed: int, idx: int, channels: int, dim: int):
    """engine.py:231-235 — seeded N(0,1) latent of request #idx."""
    return np.random.default_rng([seed, idx]).normal(size=(channels, dim, dim))
