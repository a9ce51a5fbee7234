"""Compressed sparse patch (CSP) batch format — drop-in for mixserve/csp.py.

`split` builds the integer metadata on the host through the C ABI
(`ps_csp_build`, csp.py:142-179) and copies pixels on the device
(`ps_csp_split`, csp.py:161-167); `reassemble` is the device inverse
(csp.py:196-214).  `CSPBatch.data` is a CUDA tensor with the reference's
logical layout (P, C, ps, ps), C-contiguous; metadata stays available as host
int64 arrays (the reference's types) plus cached int32 device copies.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _lib
from ._dev import i32, ptr, require_cuda, stream, to_device
from .errors import InputError

DIRECTIONS = ("N", "NE", "E", "SE", "S", "SW", "W", "NW")  # csp.py:21
OPPOSITE = {d: DIRECTIONS[(i + 4) % 8] for i, d in enumerate(DIRECTIONS)}


@dataclass(frozen=True)
class ResolutionClass:
    """csp.py:26-39."""

    name: str
    pixel: int

    def __post_init__(self):
        if self.pixel % 8 != 0:
            raise InputError(f"pixel size must be divisible by 8, got {self.pixel}")

    @property
    def latent(self) -> int:
        return self.pixel // 8


STANDARD_CLASSES = {
    "low": ResolutionClass("low", 512),
    "med": ResolutionClass("med", 768),
    "high": ResolutionClass("high", 1024),
    # beyond csp.py:42-46: the BASELINE configs' other sizes -- config 1's 256 / 384 px and config
    # 5's 2048 px -- so those requests can enter the serving plane
    "tiny": ResolutionClass("tiny", 256),
    "small": ResolutionClass("small", 384),
    "ultra": ResolutionClass("ultra", 2048),
}


def choose_patch_size(latent_dims: Iterable[int]) -> int:
    """csp.py:49-56."""
    dims = list(latent_dims)
    if not dims:
        raise InputError("no latent dims given")
    if any(d <= 0 for d in dims):
        raise InputError(f"latent dims must be positive, got {dims}")
    return math.gcd(*dims)


@dataclass(frozen=True)
class RequestEntry:
    request_id: str
    latent: int
    side: int
    patch_start: int
    patch_count: int


@dataclass
class CSPBatch:
    """csp.py:68-114; `data` is a CUDA tensor (P, C, ps, ps)."""

    patch_size: int
    data: torch.Tensor
    requests: list
    request_offset: np.ndarray
    resolution_dims: list
    resolution_offset: np.ndarray
    request_index: np.ndarray
    ordinal: np.ndarray
    row: np.ndarray
    col: np.ndarray
    neighbors: np.ndarray
    _slot: dict = field(default_factory=dict, repr=False)
    _dev: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        if not self._slot:
            self._slot = {e.request_id: i for i, e in enumerate(self.requests)}

    @property
    def n_patches(self) -> int:
        return int(self.request_offset[-1])

    @property
    def n_requests(self) -> int:
        return len(self.requests)

    def request_slot(self, request_id: str) -> int:
        try:
            return self._slot[request_id]
        except KeyError:
            raise InputError(f"unknown request {request_id!r}") from None

    def patches_of_request(self, request_id: str) -> slice:
        r = self.request_slot(request_id)
        return slice(int(self.request_offset[r]), int(self.request_offset[r + 1]))

    def group_by_resolution(self) -> list:
        return [(d, slice(int(self.resolution_offset[g]), int(self.resolution_offset[g + 1])))
                for g, d in enumerate(self.resolution_dims)]

    def patch_key(self, p: int) -> tuple:
        return (self.requests[int(self.request_index[p])].request_id, int(self.ordinal[p]))

    def patch_keys(self) -> list:
        ids = [e.request_id for e in self.requests]
        return [(ids[r], int(o)) for r, o in zip(self.request_index.tolist(), self.ordinal.tolist())]

    # ------------------------------------------------ device-side metadata
    def device(self) -> dict:
        """int32 device copies of the metadata plus attention tiles (cached)."""
        if not self._dev:
            dev = require_cuda()
            ps = self.patch_size
            hw = ps * ps
            tok0 = (self.request_offset * hw).astype(np.int64)
            # attention tiles: (q0, image) per 128 queries, longest images first (LPT)
            order = sorted(range(self.n_requests), key=lambda r: -(tok0[r + 1] - tok0[r]))
            q0s, imgs, pq0, pimg = [], [], [], []
            for r in order:
                for q in range(int(tok0[r]), int(tok0[r + 1]), 128):
                    q0s.append(q)
                    imgs.append(r)
                for q in range(int(tok0[r]), int(tok0[r + 1]), 256):  # CTA-pair tiles
                    pq0.append(q)
                    pimg.append(r)
            self._dev.update(
                request_offset=i32(self.request_offset, dev),
                request_index=i32(self.request_index, dev),
                neighbors=i32(self.neighbors.reshape(-1), dev),
                sides=i32([e.side for e in self.requests], dev),
                img_tok0=i32(tok0, dev),
                tile_q0=i32(q0s, dev),
                tile_q0_host=np.asarray(q0s, dtype=np.int64),
                tile_img_host=np.asarray(imgs, dtype=np.int64),
                tile_img=i32(imgs, dev),
                n_tiles=len(q0s),
                pair_q0=i32(pq0, dev),
                pair_img=i32(pimg, dev),
                n_pairs=len(pq0),
            )
        return self._dev


def _plan(dims: list, ps: int):
    lib = _lib.load()
    n = len(dims)
    d = (C.c_int32 * n)(*dims)
    P, nres = C.c_int32(), C.c_int32()
    _lib.check(lib.ps_csp_count(n, d, ps, C.byref(P), C.byref(nres)))
    P, nres = P.value, nres.value
    arr = lambda k: np.zeros(k, dtype=np.int32)
    order, ro, rd, so = arr(n), arr(n + 1), arr(nres), arr(nres + 1)
    ri, od, rw, cl, nb = arr(P), arr(P), arr(P), arr(P), arr(P * 8)
    ptrs = [a.ctypes.data_as(C.c_void_p) for a in (order, ro, rd, so, ri, od, rw, cl, nb)]
    _lib.check(lib.ps_csp_build(n, d, ps, *ptrs))
    return order, ro, rd, so, ri, od, rw, cl, nb.reshape(P, 8)


def split(requests: Sequence, patch_size: int | None = None) -> CSPBatch:
    """Cut (request_id, latent) pairs into a CSP batch (csp.py:117-193).

    Latents are (C, H, H) CUDA tensors (numpy / CPU tensors are copied to the
    device first); the patch array keeps their dtype (float32, bfloat16 or float64 -- numpy
    float64 latents stay exact, as csp.py:167 copies them).
    """
    if not requests:
        raise InputError("empty batch")
    ids = [rid for rid, _ in requests]
    if len(set(ids)) != len(ids):
        raise InputError("duplicate request ids in batch")
    lats = []
    for rid, lat in requests:
        t = to_device(lat)
        if t.dtype not in (torch.float32, torch.bfloat16, torch.float64):
            t = t.to(torch.float32)
        if t.dim() != 3 or t.shape[1] != t.shape[2]:
            raise InputError(f"latent for {rid!r} must be (C,H,H), got {tuple(t.shape)}")
        lats.append(t)
    channels = lats[0].shape[0]
    if any(t.shape[0] != channels for t in lats):
        raise InputError("all latents in a batch must share a channel count")
    dtype = lats[0].dtype
    if any(t.dtype != dtype for t in lats):
        dtype = torch.float64 if any(t.dtype == torch.float64 for t in lats) else torch.float32
        lats = [t.to(dtype) for t in lats]
    dims = [int(t.shape[1]) for t in lats]
    ps = choose_patch_size(dims) if patch_size is None else int(patch_size)
    if any(d % ps for d in dims):
        raise InputError(f"patch size {ps} does not tile latent dims {sorted(set(dims))}")
    order, ro, rd, so, ri, od, rw, cl, nb = _plan(dims, ps)
    entries = [RequestEntry(ids[src], dims[src], dims[src] // ps, int(ro[s]), int(ro[s + 1] - ro[s]))
               for s, src in enumerate(order.tolist())]
    P = int(ro[-1])
    dev = require_cuda()
    data = torch.empty((P, channels, ps, ps), dtype=dtype, device=dev)
    batch = CSPBatch(ps, data, entries, ro.astype(np.int64), [int(x) for x in rd], so.astype(np.int64),
                     ri.astype(np.int64), od.astype(np.int64), rw.astype(np.int64), cl.astype(np.int64),
                     nb.astype(np.int64))
    src_ptrs = torch.tensor([lats[s].data_ptr() for s in order.tolist()], dtype=torch.int64, device=dev)
    md = batch.device()
    _lib.call("ps_csp_split", stream(), src_ptrs.data_ptr(), md["request_offset"].data_ptr(), md["sides"].data_ptr(),
              len(order), channels, ps, _dtype_code(dtype), data.data_ptr(), P)
    return batch


def _dtype_code(dt) -> int:
    if dt == torch.float32:
        return _lib.DTYPE_F32
    if dt == torch.bfloat16:
        return _lib.DTYPE_BF16
    if dt == torch.float64:
        return _lib.DTYPE_F64
    raise InputError(f"unsupported dtype {dt}")


def reassemble(batch: CSPBatch, data=None) -> dict:
    """Stitch patches back into full latents keyed by request id (csp.py:196-214)."""
    src = batch.data if data is None else to_device(data)
    if tuple(src.shape) != tuple(batch.data.shape):
        raise InputError(f"data shape {tuple(src.shape)} does not match batch {tuple(batch.data.shape)}")
    if src.dtype not in (torch.float32, torch.bfloat16, torch.float64):
        src = src.to(torch.float32)
    src = src.contiguous()
    c, ps = src.shape[1], batch.patch_size
    out = {e.request_id: torch.empty((c, e.latent, e.latent), dtype=src.dtype, device=src.device)
           for e in batch.requests}
    dev = batch.device()
    dst_ptrs = torch.tensor([out[e.request_id].data_ptr() for e in batch.requests], dtype=torch.int64,
                            device=src.device)
    _lib.call("ps_csp_reassemble", stream(), src.data_ptr(), dst_ptrs.data_ptr(), dev["request_offset"].data_ptr(),
              dev["sides"].data_ptr(), batch.n_requests, c, ps, _dtype_code(src.dtype), batch.n_patches)
    # dst_ptrs / temporaries may be freed now: the caching allocator only hands
    # their memory to later work on this stream, after the copy kernel ran
    return out
