"""Patch sharding across GPUs with images split between GPUs.

Request ownership (shard.py) never splits an image.  When one image carries
more work than a GPU's share (config 5: one 2048 px image next to 512 px ones)
the CSP patch list itself is cut into `world` contiguous ranges (csp.py:143
order: stable sort by latent size), balanced by per-patch work; a cut may fall
inside an image.  Rank r then holds every request its range touches, with the
full CSP geometry of those images (so neighbour tables, token offsets and
GroupNorm pooling ranges are the single-GPU ones), but only computes the
patches it OWNS.  The patches of a split image it does not own are GHOSTS: their
slots are filled by three exchanges per block, and only with what the owned
patches read:

1. GroupNorm partials (patched.py:132-140): the per-(patch, group) (mean, M2)
   of every owned patch of a split image is all-gathered, so each rank pools
   exactly the single-GPU partials in the single-GPU order (bit-identical
   statistics).
2. Halo strips (patched.py:57-89 across a cut): for every owned patch whose
   neighbour q is owned elsewhere, the one pixel row / column of q the 3x3
   stencil reads (all channels) is sent point-to-point by q's owner.
3. Attention K / V (patched.py:164-176): every owned token range of a split
   image is all-gathered as K rows and V^T columns, so attention over the whole
   image runs for the owned query tiles.

Everything else (conv, GEMMs, attention queries, blend) runs on owned rows
only.  Given identical inputs the owned rows are bit-identical to the
single-GPU run (tests/test_gpu_split.py).

The plan is pure host arithmetic, identical on every rank (no negotiation).
"""

from __future__ import annotations

import bisect  # noqa: F401
import threading
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from .errors import InputError

# neighbour directions as in csp.py:21-23, with the pixel strip of the
# neighbour that the 3x3 stencil of the centre patch reads (patched.py:64-88):
# code < ps -> pixel row `code`; code >= ps -> pixel column `code - ps`
_DIRS = ((-1, 0), (-1, 1), (0, 1), (1, 1), (1, 0), (1, -1), (0, -1), (-1, -1))  # N NE E SE S SW W NW


def _strip_code(d: int, ps: int) -> int:
    dr, dc = _DIRS[d]
    if dr < 0:
        return ps - 1      # N, NE, NW: bottom row of the neighbour
    if dr > 0:
        return 0           # S, SE, SW: top row
    return ps + (0 if dc > 0 else ps - 1)  # E: left column, W: right column


def patch_cost(latent: int, patch_size: int, channels: int = 320, hidden: int = 1280) -> float:
    """Per-patch FLOPs of one unet_like block (attention queries see the whole image)."""
    t = latent * latent
    hw = patch_size * patch_size
    return hw * (4.0 * t * channels + 8.0 * channels * channels + 18.0 * channels * channels
                 + 4.0 * channels * hidden)


def linear_partition(w: Sequence[float], parts: int) -> list[int]:
    """Cut points c_0 = 0 <= ... <= c_parts = n minimising the largest range sum.

    Binary search on the bottleneck with a greedy feasibility test, then the
    greedy cut at the optimum; ranges left empty are filled by halving the
    largest range so every part gets work when n >= parts.
    """
    n = len(w)
    if parts < 1:
        raise InputError("world must be >= 1")
    pre = np.concatenate([[0.0], np.cumsum(np.asarray(w, dtype=np.float64))])

    def greedy(cap):
        cuts, start = [0], 0
        while start < n:
            end = int(np.searchsorted(pre, pre[start] + cap * (1 + 1e-12), side="right")) - 1
            end = max(end, start + 1)
            cuts.append(min(end, n))
            start = cuts[-1]
        return cuts

    lo, hi = max(w) if n else 0.0, float(pre[-1])
    for _ in range(100):
        if hi - lo <= 1e-9 * max(hi, 1.0):
            break
        mid = 0.5 * (lo + hi)
        if len(greedy(mid)) - 1 <= parts:
            hi = mid
        else:
            lo = mid
    cuts = greedy(hi) if n else [0]
    while len(cuts) - 1 < parts:
        sizes = [cuts[i + 1] - cuts[i] for i in range(len(cuts) - 1)]
        i = int(np.argmax(sizes)) if sizes else 0
        if not sizes or sizes[i] < 2:
            cuts.append(cuts[-1])  # fewer patches than ranks: trailing empty ranges
            continue
        cuts.insert(i + 1, cuts[i] + sizes[i] // 2)
    return cuts


@dataclass(frozen=True)
class _Req:
    index: int      # position in the caller's request list
    request_id: str
    latent: int
    side: int
    g0: int         # first global patch (CSP order)

    @property
    def count(self) -> int:
        return self.side * self.side


class SplitPlan:
    """Global CSP order, per-rank patch ranges and the exchange tables."""

    def __init__(self, requests: Sequence[tuple], patch_size: int, world: int,
                 cost: Callable[[int], float] | None = None, mode: str = "balanced"):
        """`requests`: (request_id, latent_dim) in arrival order.

        mode "contiguous": the CSP patch list is cut into `world` contiguous ranges (optimal
        linear partition of per-patch cost).  mode "balanced" (default): only requests that
        cost more than a GPU's share are split -- their patches, in CSP order, are cut into
        contiguous ranges over all ranks by the same linear partition -- and every other
        request stays whole, placed longest-first on the least loaded rank (the
        reference's lowest-load dispatch, engine.py:228).  Config 5 then gives every GPU
        two patches of the 2048 px image and one 512 px image."""
        if mode not in ("balanced", "contiguous"):
            raise InputError(f"unknown split mode {mode!r}")
        if world < 1:
            raise InputError("world must be >= 1")
        ps = int(patch_size)
        self.ps, self.world = ps, world
        dims = [int(r[1]) for r in requests]
        if any(d % ps for d in dims):
            raise InputError(f"patch size {ps} does not tile latent dims {sorted(set(dims))}")
        order = sorted(range(len(dims)), key=lambda i: dims[i])  # csp.py:143 (stable)
        self.reqs: list[_Req] = []
        g = 0
        for i in order:
            s = dims[i] // ps
            self.reqs.append(_Req(i, str(requests[i][0]), dims[i], s, g))
            g += s * s
        self.n_patches = g
        cost = cost or (lambda lat: patch_cost(lat, ps))
        w = [cost(r.latent) for r in self.reqs for _ in range(r.count)]
        self.mode = mode
        self._g0 = [r.g0 for r in self.reqs]
        self._shards: dict = {}
        owner = np.zeros(g, dtype=np.int32)
        if mode == "contiguous" or world == 1:
            self.cuts = linear_partition(w, world)
            for k in range(world):
                owner[self.cuts[k]:self.cuts[k + 1]] = k
        else:
            self.cuts = None
            share = sum(w) / world
            req_cost = [sum(w[r.g0:r.g0 + r.count]) for r in self.reqs]
            big = [k for k, c in enumerate(req_cost) if c > share * (1 + 1e-9) and self.reqs[k].count > 1]
            loads = np.zeros(world)
            if big:
                pats = [gg for k in big for gg in range(self.reqs[k].g0, self.reqs[k].g0 + self.reqs[k].count)]
                cuts = linear_partition([w[gg] for gg in pats], world)
                for r_ in range(world):
                    for i in range(cuts[r_], cuts[r_ + 1]):
                        owner[pats[i]] = r_
                        loads[r_] += w[pats[i]]
            bigset = set(big)
            for k in sorted((k for k in range(len(self.reqs)) if k not in bigset), key=lambda k: -req_cost[k]):
                r_ = int(np.argmin(loads))
                rq = self.reqs[k]
                owner[rq.g0:rq.g0 + rq.count] = r_
                loads[r_] += req_cost[k]
        self.owner_tab = owner
        self._owned = [np.flatnonzero(owner == r_).tolist() for r_ in range(world)]
        self.load = [float(sum(w[gg] for gg in self._owned[r_])) for r_ in range(world)]

    # ---------------------------------------------------------- geometry
    def owner(self, g: int) -> int:
        return int(self.owner_tab[g])

    def owned_by(self, r: int) -> list:
        """Global patches owned by rank r, ascending."""
        return self._owned[r]

    def req_of(self, g: int) -> int:
        return bisect.bisect_right(self._g0, g) - 1

    def ranks_of(self, k: int) -> list[int]:
        r = self.reqs[k]
        return sorted({self.owner(g) for g in range(r.g0, r.g0 + r.count)})

    def split_requests(self) -> list[int]:
        """CSP slots of requests whose patches are owned by more than one rank."""
        return [k for k in range(len(self.reqs)) if len(self.ranks_of(k)) > 1]

    def neighbour(self, g: int, d: int) -> int:
        k = self.req_of(g)
        r = self.reqs[k]
        o = g - r.g0
        row, col = divmod(o, r.side)
        rr, cc = row + _DIRS[d][0], col + _DIRS[d][1]
        if not (0 <= rr < r.side and 0 <= cc < r.side):
            return -1
        return r.g0 + rr * r.side + cc

    def halo_strips(self, src: int, dst: int) -> list[tuple[int, int]]:
        """Sorted (global patch, strip code) that rank `src` sends to rank `dst`."""
        if src == dst:
            return []
        need = set()
        for g in self.owned_by(dst):
            for d in range(8):
                q = self.neighbour(g, d)
                if q >= 0 and self.owner(q) == src:
                    need.add((q, _strip_code(d, self.ps)))
        return sorted(need)

    def shard(self, rank: int) -> "LocalShard":
        if not 0 <= rank < self.world:
            raise InputError(f"rank {rank} outside world {self.world}")
        if rank not in self._shards:
            self._shards[rank] = LocalShard(self, rank)
        return self._shards[rank]


@dataclass
class LocalShard:
    """Rank-local view: the local CSP batch layout and this rank's exchange lists."""

    plan: SplitPlan
    rank: int
    _dev: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        pl, r = self.plan, self.rank
        mine = pl.owned_by(r)
        ks = sorted({pl.req_of(g) for g in mine})
        self.slots = ks                                   # global CSP slots held, in CSP order
        self.local_slot = {k: i for i, k in enumerate(ks)}
        off = [0]
        for k in ks:
            off.append(off[-1] + pl.reqs[k].count)
        self.request_offset = np.asarray(off, dtype=np.int64)
        self.n_patches = off[-1]
        self.requests = [(pl.reqs[k].request_id, pl.reqs[k].latent) for k in ks]
        self.owned = np.asarray([self.local(g) for g in mine], dtype=np.int64)
        split = set(pl.split_requests())
        self.split_slots = [k for k in ks if k in split]

        # GroupNorm partials: every rank's owned patches of split images, global order
        self.gn_lists = []
        for s in range(pl.world):
            self.gn_lists.append([g for g in pl.owned_by(s) if pl.req_of(g) in split])
        self.gn_max = max((len(x) for x in self.gn_lists), default=0)
        self.gn_send = [self.local(g) for g in self.gn_lists[r]]
        self.gn_recv = []  # (src rank, slot in src's list, local patch)
        for s in range(pl.world):
            if s == r:
                continue
            for i, g in enumerate(self.gn_lists[s]):
                if pl.req_of(g) in self.local_slot:
                    self.gn_recv.append((s, i, self.local(g)))

        # halo strips: point-to-point lists, local patch indices
        self.halo_send = {d: [(self.local(g), c) for g, c in pl.halo_strips(r, d)] for d in range(pl.world)}
        self.halo_recv = {s: [(self.local(g), c) for g, c in pl.halo_strips(s, r)] for s in range(pl.world)}
        self.halo_send = {d: v for d, v in self.halo_send.items() if v}
        self.halo_recv = {s: v for s, v in self.halo_recv.items() if v}

        # attention K / V: per rank, (global slot, first ordinal, n patches) owned of split images
        self.kv_segs = []
        for s in range(pl.world):
            segs = []
            for k in sorted(split):
                rq = pl.reqs[k]
                mine_k = [g for g in pl.owned_by(s) if rq.g0 <= g < rq.g0 + rq.count]
                if mine_k:
                    a, b = mine_k[0], mine_k[-1] + 1
                    if b - a != len(mine_k):
                        raise InputError("split image ranges must be contiguous per rank")
                    segs.append((k, a - rq.g0, b - a))
            self.kv_segs.append(segs)
        hw = pl.ps * pl.ps
        self.kv_max_tokens = max((sum(n for _, _, n in segs) * hw for segs in self.kv_segs), default=0)

    def local(self, g: int) -> int:
        pl = self.plan
        k = pl.req_of(g)
        return int(self.request_offset[self.local_slot[k]]) + g - pl.reqs[k].g0


    # --------------------------------------------------- offsets (host)
    def gn_offsets(self, G: int):
        """(pack src, pack dst, unpack src, unpack dst) byte offsets for fp32 [*, G, 2] rows."""
        row = G * 2 * 4
        ps_ = np.asarray(self.gn_send, dtype=np.int64) * row
        pd = np.arange(len(self.gn_send), dtype=np.int64) * row
        us = np.asarray([(s * self.gn_max + i) * row for s, i, _ in self.gn_recv], dtype=np.int64)
        ud = np.asarray([p * row for _, _, p in self.gn_recv], dtype=np.int64)
        return ps_, pd, us, ud, row

    def kv_offsets(self, dpp: int, ldv: int):
        """Byte offsets for K rows (qk [T, 2Dp], K at column Dp) and V^T rows ([Dp, ldv]).

        Send-buffer layout per segment: K [ntok][Dp] then V^T [Dp][ntok] (bf16).
        Returns (k_pack_src, k_pack_dst, v_pack_src, v_pack_dst, pack V seg bytes per segment,
        and the same four for unpack) grouped per segment size; see `kv_plan`.
        """
        return kv_plan(self, dpp, ldv)


def kv_plan(sh: LocalShard, dpp: int, ldv: int) -> dict:
    """Segment-copy lists for the K / V^T pack (own segments) and unpack (others')."""
    pl = sh.plan
    hw = pl.ps * pl.ps
    kb = dpp * 2                       # one K row (bytes)
    qk_row = 2 * dpp * 2               # qk row pitch (bytes)
    k_src, k_dst = [], []              # K rows: one segment of kb bytes per token
    v_jobs = []                        # V^T: (src list, dst list, seg bytes) per token-run length
    ku_src, ku_dst = [], []
    vu_jobs = []
    maxb = sh.kv_max_tokens * 2 * dpp * 2

    def seg_layout(segs):
        pos, out = 0, []
        for k, o0, n in segs:
            ntok = n * hw
            out.append((k, o0, n, pos, pos + ntok * kb))
            pos += ntok * 2 * kb
        return out

    for k, o0, n, kpos, vpos in seg_layout(sh.kv_segs[sh.rank]):
        t0 = (int(sh.request_offset[sh.local_slot[k]]) + o0) * hw
        ntok = n * hw
        k_src.extend((t0 + i) * qk_row + kb for i in range(ntok))
        k_dst.extend(kpos + i * kb for i in range(ntok))
        v_jobs.append(([d * ldv * 2 + t0 * 2 for d in range(dpp)],
                       [vpos + d * ntok * 2 for d in range(dpp)], ntok * 2))
    for s in range(pl.world):
        if s == sh.rank:
            continue
        for k, o0, n, kpos, vpos in seg_layout(sh.kv_segs[s]):
            if k not in sh.local_slot:
                continue
            t0 = (int(sh.request_offset[sh.local_slot[k]]) + o0) * hw
            ntok = n * hw
            base = s * maxb
            ku_src.extend(base + kpos + i * kb for i in range(ntok))
            ku_dst.extend((t0 + i) * qk_row + kb for i in range(ntok))
            vu_jobs.append(([base + vpos + d * ntok * 2 for d in range(dpp)],
                            [d * ldv * 2 + t0 * 2 for d in range(dpp)], ntok * 2))
    def merged(jobs):  # one variable-length segment list per direction (ps_copy_segments_var)
        return ([o for js, _, _ in jobs for o in js], [o for _, jd, _ in jobs for o in jd],
                [nb for js, _, nb in jobs for _ in js])
    return dict(k_pack=(k_src, k_dst, kb), v_pack=v_jobs, k_unpack=(ku_src, ku_dst, kb), v_unpack=vu_jobs,
                v_pack_var=merged(v_jobs), v_unpack_var=merged(vu_jobs), buf_bytes=maxb)


class VirtualGroup:
    """In-process stand-in for a process group: `world` threads, one per virtual
    rank, on one device.  Collectives meet at a barrier; the last arriving thread
    moves the data (device copies on the shared stream), so kernel order is
    pack (all ranks) -> move -> unpack (all ranks)."""

    def __init__(self, world: int):
        self.world = world
        self._bar = threading.Barrier(world)
        self._slots: list = [None] * world
        self._out: list = [None] * world
        self._lock = threading.Lock()

    def _meet(self, rank: int, payload, combine):
        self._slots[rank] = payload
        i = self._bar.wait()
        if i == 0:
            self._out = combine(list(self._slots))
        self._bar.wait()
        res = self._out[rank]
        self._bar.wait()
        return res

    def all_gather(self, rank: int, t):
        import torch

        def comb(xs):
            g = torch.stack(xs)
            return [g] * self.world
        return self._meet(rank, t, comb)

    def peer_buffers(self, rank: int, shape, dtype, device):
        """Each virtual rank's buffer of `shape` and every rank's device pointer (one GPU:
        plain allocations, addressed directly)."""
        import torch
        t = torch.empty(shape, dtype=dtype, device=device)
        ptrs = self._meet(rank, t.data_ptr(), lambda xs: [list(xs)] * self.world)
        return t, ptrs

    def device_barrier(self, rank: int) -> None:
        """All ranks' preceding work is enqueued (shared stream on one GPU: also ordered)."""
        self._meet(rank, None, lambda xs: [None] * self.world)

    def exchange(self, rank: int, sends: dict, recv_like: dict | None = None):
        """sends: {dst: tensor}; returns {src: tensor} addressed to `rank`."""
        def comb(xs):
            return [{s: xs[s][d] for s in range(self.world) if xs[s] and d in xs[s]} for d in range(self.world)]
        return self._meet(rank, sends, comb)


# ------------------------------------------------------------------ device side


class DistComm:
    """torch.distributed adapter.  NCCL moves device buffers directly over
    NVLink; any other backend (gloo, for the CPU / shared-GPU tests) stages
    through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.stage = dist.get_backend(group) != "nccl"

    def all_gather(self, rank: int, t):
        import torch

        src = t.cpu() if self.stage else t
        if self.stage:
            parts = [torch.empty_like(src) for _ in range(self.world)]
            self.dist.all_gather(parts, src, group=self.group)
            return torch.stack(parts).to(t.device)
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, src, group=self.group)
        return out

    def all_gather_async(self, rank: int, t):
        """(gathered, wait): NCCL runs the gather on its own stream, so kernels enqueued
        before wait() overlap it; wait() makes the current stream wait for it."""
        if self.stage:
            return self.all_gather(rank, t), (lambda: None)
        import torch
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        work = self.dist.all_gather_into_tensor(out, t, group=self.group, async_op=True)
        return out, work.wait

    def peer_buffers(self, rank: int, shape, dtype, device):
        """Symmetric-memory buffer mapped into every rank's address space over NVLink
        (torch.distributed._symmetric_memory); returns (local tensor, peer pointers)."""
        import torch.distributed._symmetric_memory as symm_mem
        t = symm_mem.empty(shape, dtype=dtype, device=device)
        name = self.group.group_name if self.group is not None else self.dist.group.WORLD.group_name
        hdl = symm_mem.rendezvous(t, name)
        self._handles = getattr(self, "_handles", []) + [hdl]
        return t, list(hdl.buffer_ptrs)

    def device_barrier(self, rank: int) -> None:
        """Stream-ordered cross-GPU barrier: a 1-element all-reduce after this rank's
        producer kernels; later kernels see every rank's writes."""
        import torch
        if not hasattr(self, "_bar"):
            self._bar = torch.zeros(1, dtype=torch.int32, device="cuda")
        if self.stage:
            self.dist.barrier(group=self.group)
        else:
            self.dist.all_reduce(self._bar, group=self.group)

    def exchange(self, rank: int, sends: dict, recv_like: dict) -> dict:
        """Point-to-point: sends {dst: tensor}, recv_like {src: (shape, dtype, device)}."""
        import torch

        dist = self.dist
        ops, recvs = [], {}
        for s, (shape, dtype, device) in sorted(recv_like.items()):
            recvs[s] = torch.empty(shape, dtype=dtype, device="cpu" if self.stage else device)
            ops.append(dist.P2POp(dist.irecv, recvs[s], s, self.group))
        for d, t in sorted(sends.items()):
            ops.append(dist.P2POp(dist.isend, t.cpu() if self.stage else t, d, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if self.stage:
            recvs = {s: t.to(recv_like[s][2]) for s, t in recvs.items()}
        return recvs


class ShardExchange:
    """The three per-block exchanges of one rank (module docstring), as library
    pack / unpack kernels around `comm` collectives."""

    def __init__(self, shard: LocalShard, comm, peer_kv: bool = False):
        """peer_kv: attention reads the split images' remote K / V directly from the owners'
        buffers over NVLink (ps_attention_peer) instead of all-gathering them."""
        self.sh, self.comm = shard, comm
        self.rank = shard.rank
        self.peer_kv = peer_kv and bool(shard.plan.split_requests())
        self.bytes_moved = 0  # payload bytes this rank sent (telemetry)
        self._cache: dict = {}
        self._parity = 0

    def _dev_i64(self, key, values):
        import torch

        from ._dev import require_cuda
        if key not in self._cache:
            self._cache[key] = torch.as_tensor(np.asarray(values, dtype=np.int64), device=require_cuda())
        return self._cache[key]

    def _copy(self, src, dst, key, src_off, dst_off, seg_bytes):
        from . import _lib
        from ._dev import stream
        n = len(src_off)
        if n == 0:
            return
        so = self._dev_i64(key + ("s",), src_off)
        do = self._dev_i64(key + ("d",), dst_off)
        _lib.call("ps_copy_segments", stream(), src.data_ptr(), dst.data_ptr(), n, so.data_ptr(), do.data_ptr(),
                  int(seg_bytes))

    def _copy_var(self, src, dst, key, segs):
        from . import _lib
        from ._dev import stream
        src_off, dst_off, nbytes = segs
        if not src_off:
            return
        so = self._dev_i64(key + ("s",), src_off)
        do = self._dev_i64(key + ("d",), dst_off)
        nb = self._dev_i64(key + ("n",), nbytes)
        _lib.call("ps_copy_segments_var", stream(), src.data_ptr(), dst.data_ptr(), len(src_off), so.data_ptr(),
                  do.data_ptr(), nb.data_ptr())

    # 1. GroupNorm partials ----------------------------------------------
    def gn(self, partials, G: int) -> None:
        import torch
        sh = self.sh
        if sh.gn_max == 0:
            return
        ps_, pd, us, ud, row = sh.gn_offsets(G)
        send = torch.zeros(sh.gn_max * G * 2, dtype=torch.float32, device=partials.device)
        self._copy(partials, send, ("gnp", G), ps_, pd, row)
        got = self.comm.all_gather(self.rank, send)
        self._copy(got, partials, ("gnu", G), us, ud, row)
        self.bytes_moved += send.numel() * 4

    # 2. halo strips -------------------------------------------------------
    def _desc(self, key, strips):
        import torch

        from ._dev import require_cuda
        if key not in self._cache:
            self._cache[key] = torch.as_tensor(np.asarray(strips, dtype=np.int32).reshape(-1, 2),
                                               device=require_cuda())
        return self._cache[key]

    def halo(self, x, C: int) -> None:
        import torch

        from . import _lib
        from ._dev import stream
        sh = self.sh
        ps = sh.plan.ps
        sends = {}
        for d, strips in sh.halo_send.items():
            buf = torch.empty((len(strips), C, ps), dtype=x.dtype, device=x.device)
            _lib.call("ps_halo_strips", stream(), x.data_ptr(), C, ps, len(strips),
                      self._desc(("hs", d), strips).data_ptr(), buf.data_ptr(), 0)
            sends[d] = buf
            self.bytes_moved += buf.numel() * buf.element_size()
        like = {s: ((len(strips), C, ps), x.dtype, x.device) for s, strips in sh.halo_recv.items()}
        got = self.comm.exchange(self.rank, sends, like)
        for s, strips in sh.halo_recv.items():
            _lib.call("ps_halo_strips", stream(), x.data_ptr(), C, ps, len(strips),
                      self._desc(("hr", s), strips).data_ptr(), got[s].contiguous().data_ptr(), 1)

    # 3. attention K / V^T -------------------------------------------------
    def kv_start(self, qk, vt, ldv: int, dpp: int):
        """Pack this rank's K / V^T of split images and start their all-gather; returns the
        finish() that waits for it and unpacks the peers' segments into the ghost rows.
        Kernels enqueued between the two (attention over the owned keys) overlap the gather
        when the backend runs it asynchronously (NCCL)."""
        import torch
        sh = self.sh
        if sh.kv_max_tokens == 0:
            return lambda: None
        key = ("kv", dpp, ldv)
        if key not in self._cache:
            self._cache[key] = kv_plan(sh, dpp, ldv)
        pl = self._cache[key]
        send = torch.empty(pl["buf_bytes"], dtype=torch.uint8, device=qk.device)
        ks, kd, kb = pl["k_pack"]
        self._copy(qk, send, key + ("kp",), ks, kd, kb)
        self._copy_var(vt, send, key + ("vp",), pl["v_pack_var"])
        self.bytes_moved += send.numel()
        if hasattr(self.comm, "all_gather_async"):
            got, wait = self.comm.all_gather_async(self.rank, send)
        else:
            got, wait = self.comm.all_gather(self.rank, send), (lambda: None)

        def finish():
            wait()
            ks_, kd_, kb_ = pl["k_unpack"]
            self._copy(got, qk, key + ("ku",), ks_, kd_, kb_)
            self._copy_var(got, vt, key + ("vu",), pl["v_unpack_var"])
        return finish

    def kv(self, qk, vt, ldv: int, dpp: int) -> None:
        import torch
        sh = self.sh
        if sh.kv_max_tokens == 0:
            return
        key = ("kv", dpp, ldv)
        if key not in self._cache:
            self._cache[key] = kv_plan(sh, dpp, ldv)
        pl = self._cache[key]
        send = torch.empty(pl["buf_bytes"], dtype=torch.uint8, device=qk.device)
        ks, kd, kb = pl["k_pack"]
        self._copy(qk, send, key + ("kp",), ks, kd, kb)
        self._copy_var(vt, send, key + ("vp",), pl["v_pack_var"])
        got = self.comm.all_gather(self.rank, send)
        ks, kd, kb = pl["k_unpack"]
        self._copy(got, qk, key + ("ku",), ks, kd, kb)
        self._copy_var(got, vt, key + ("vu",), pl["v_unpack_var"])
        self.bytes_moved += send.numel()

    # 3'. attention K / V read in place from the owners (peer_kv) ----------
    def kv_buffers(self, dpp: int, T: int, device):
        """Persistent, peer-visible qk [T, 2 Dp] and V^T [Dp, ldv] of this call's parity
        (double-buffered: a peer may still read block j's buffers while block j+1 writes)."""
        from ._dev import round_up
        import torch
        par = self._parity
        self._parity ^= 1
        key = ("pkv", dpp, par)
        if key not in self._cache:
            ldv = round_up(T, 64)
            qk, qk_ptrs = self.comm.peer_buffers(self.rank, (T, 2 * dpp), torch.bfloat16, device)
            vt, vt_ptrs = self.comm.peer_buffers(self.rank, (dpp, ldv), torch.bfloat16, device)
            self._cache[key] = (qk, vt, ldv, qk_ptrs, vt_ptrs, None)
        return par, self._cache[key]

    def kv_tables(self, dpp: int, par: int):
        """(kb_src, kb_row, device tensor maps) for ps_attention_peer, built once per parity."""
        import ctypes as C
        import torch

        from . import _lib
        from ._dev import require_cuda, round_up
        key = ("pkv", dpp, par)
        qk, vt, ldv, qk_ptrs, vt_ptrs, tabs = self._cache[key]
        if tabs is None:
            sh, pl = self.sh, self.sh.plan
            hw = pl.ps * pl.ps
            world = pl.world
            shards = [pl.shard(r) for r in range(world)]
            T = [int(x.n_patches) * hw for x in shards]
            ldvs = [round_up(t, 64) for t in T]
            split = set(pl.split_requests())
            nblk = (sh.n_patches * hw + 127) // 128
            src = np.full(nblk, -1, dtype=np.int32)
            row = np.zeros(nblk, dtype=np.int32)
            owned = set(int(x) for x in sh.owned)
            for k in sh.slots:
                if k not in split:
                    continue
                rq = pl.reqs[k]
                for g in range(rq.g0, rq.g0 + rq.count):
                    lp = sh.local(g)
                    if lp in owned:
                        continue
                    s_ = pl.owner(g)
                    rp = shards[s_].local(g)
                    for t in range(0, hw, 128):
                        src[(lp * hw + t) // 128] = s_
                        row[(lp * hw + t) // 128] = rp * hw + t
            dev = require_cuda()
            maps = torch.empty(2 * world * 128, dtype=torch.uint8, device=dev)  # 2 x 128-B CUtensorMap per rank
            arr64 = lambda v: (C.c_uint64 * world)(*[int(x) for x in v])
            arr32 = lambda v: (C.c_int32 * world)(*[int(x) for x in v])
            _lib.call("ps_kv_peer_maps", maps.data_ptr(), world, arr64(qk_ptrs), arr32(T), arr64(vt_ptrs),
                      arr32(ldvs), dpp)
            tabs = (torch.as_tensor(src, device=dev), torch.as_tensor(row, device=dev), maps)
            self._cache[key] = (qk, vt, ldv, qk_ptrs, vt_ptrs, tabs)
        return tabs

    def kv_sync(self) -> None:
        """Every rank's QKV projection of this block is done (and visible) before any
        rank's attention reads it."""
        self.comm.device_barrier(self.rank)
