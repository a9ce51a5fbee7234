"""Patch-level reuse cache on the device — drop-in for mixserve/cache.py.

Per block the cache is a slab: input snapshots and output snapshots (bf16,
(capacity, C*ps*ps), NCHW patch order) plus per-slot `exists` and `streak`
arrays.  Keys (request_id, ordinal) map to slots on the host; a key keeps its
slot across steps and re-splits (cache.py:81, csp.py:112-114), so the batch ops
only upload one int32 slot vector per call.

predict_reuse runs the bit-exact fp64 pairwise MSE (K8, csrc/cache.cu) and
returns a device bool mask; gather / batched_fill / batched_update /
evict_expired are device kernels (K9).  `stats` and `size()` read device
counters back (one small D2H each).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Hashable, Sequence

import numpy as np
import torch

from . import _lib
from ._dev import require_cuda, stream, to_device
from .errors import InputError, IntegrityError

Key = Hashable


@dataclass(frozen=True)
class PredictorConfig:
    """cache.py:23-32."""

    mse_threshold: float = 0.1
    max_streak: int = 3

    def __post_init__(self):
        if self.mse_threshold <= 0:
            raise InputError("mse_threshold must be positive")
        if self.max_streak < 1:
            raise InputError("max_streak must be >= 1")


@dataclass(frozen=True)
class CacheEntry:
    input_snapshot: torch.Tensor
    output_snapshot: torch.Tensor
    reuse_streak: int = 0


@dataclass
class CacheStats:
    predicted_reuse: int = 0
    fresh_compute: int = 0
    inserted: int = 0
    refreshed: int = 0
    evicted: int = 0

    def as_dict(self) -> dict:
        return dict(self.__dict__)


class PairwisePlan:
    """Device copy of numpy's pairwise-summation tree for n elements (ps_pairwise_plan)."""

    _cache: dict = {}

    def __init__(self, n: int):
        lib = _lib.load()
        L, I, H = C.c_int32(), C.c_int32(), C.c_int32()
        _lib.check(lib.ps_pairwise_plan(n, C.byref(L), C.byref(I), C.byref(H), None, None, None))
        self.n, self.L, self.I, self.H = n, L.value, I.value, H.value
        leaves = np.zeros(2 * self.L, dtype=np.int32)
        nodes = np.zeros(max(1, 2 * self.I), dtype=np.int32)
        lvl = np.zeros(self.H + 1, dtype=np.int32)
        _lib.check(lib.ps_pairwise_plan(n, C.byref(L), C.byref(I), C.byref(H), leaves.ctypes.data_as(C.c_void_p),
                                        nodes.ctypes.data_as(C.c_void_p), lvl.ctypes.data_as(C.c_void_p)))
        dev = require_cuda()
        self.leaves = torch.as_tensor(leaves, device=dev)
        self.nodes = torch.as_tensor(nodes, device=dev)
        self.level_off = torch.as_tensor(lvl, device=dev)
        self.host = (leaves, nodes, lvl)

    @classmethod
    def get(cls, n: int) -> "PairwisePlan":
        p = cls._cache.get(n)
        if p is None:
            p = cls._cache[n] = PairwisePlan(n)
        return p


_LIB_DTYPE = {torch.bfloat16: _lib.DTYPE_BF16, torch.float32: _lib.DTYPE_F32, torch.float64: _lib.DTYPE_F64}


def _patches(x, dtype: torch.dtype) -> torch.Tensor:
    """Device copy of x in the slab dtype (bf16 on the hot path: fp32 inputs are rounded the way
    the block inputs are; fp32 / fp64 slabs keep numpy inputs exact)."""
    t = to_device(x)
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def scratch_doubles(P: int, plan: "PairwisePlan") -> int:
    """fp64 scratch of ps_cache_predict: per-patch tree values + P int32 tickets."""
    return P * (plan.L + plan.I) + (P + 1) // 2


def mse(a, b) -> float:
    """float(np.mean((a - b) ** 2)) (cache.py:54-55) on the device, bit-exact in fp64.

    The operands keep their precision: bf16 / fp32 tensors are widened exactly, anything else
    (numpy float64 arrays, fp64 tensors) is evaluated in fp64 -- no rounding before the
    subtraction, so the result equals numpy's for every input."""
    ta, tb = to_device(a), to_device(b)
    if ta.shape != tb.shape:
        raise InputError("mse: shape mismatch")
    dt = ta.dtype if (ta.dtype == tb.dtype and ta.dtype in _LIB_DTYPE) else torch.float64
    ta, tb = _patches(ta, dt), _patches(tb, dt)
    n = ta.numel()
    if n == 0:
        return float("nan")  # np.mean of an empty array
    plan = PairwisePlan.get(n)
    dev = ta.device
    slots = torch.zeros(1, dtype=torch.int32, device=dev)
    exists = torch.ones(1, dtype=torch.uint8, device=dev)
    streak = torch.zeros(1, dtype=torch.int32, device=dev)
    scratch = torch.empty(scratch_doubles(1, plan), dtype=torch.float64, device=dev)
    mask = torch.empty(1, dtype=torch.uint8, device=dev)
    # sigma = +inf makes the mask always true; the fp64 root is read from scratch
    _lib.call("ps_cache_predict", stream(), ta.data_ptr(), _LIB_DTYPE[dt], 1, n, slots.data_ptr(), tb.data_ptr(),
              exists.data_ptr(), streak.data_ptr(), float("inf"), 1, plan.leaves.data_ptr(), plan.L,
              plan.nodes.data_ptr(), plan.I, plan.level_off.data_ptr(), plan.H, scratch.data_ptr(), mask.data_ptr(),
              None)
    root = scratch[plan.L + plan.I - 1] if plan.I > 0 else scratch[0]
    return (0.0 + float(root)) / n


def partition_sets(prev_keys: Sequence[Key], cur_keys: Sequence[Key]):
    """Common / New / Expired key lists (cache.py:58-70); host-side set algebra."""
    prev_set, cur_set = set(prev_keys), set(cur_keys)
    if len(prev_set) != len(prev_keys) or len(cur_set) != len(cur_keys):
        raise InputError("duplicate keys in partition input")
    return ([k for k in cur_keys if k in prev_set], [k for k in cur_keys if k not in prev_set],
            [k for k in prev_keys if k not in cur_set])


class BlockCache:
    """Per-block patch cache with batched predict / gather / fill / update / evict."""

    def __init__(self, n_blocks: int, cfg: PredictorConfig | None = None,
                 predictor: Callable | None = None, capacity: int = 256, dtype: torch.dtype = torch.bfloat16):
        if n_blocks < 1:
            raise InputError("n_blocks must be >= 1")
        self.cfg = cfg or PredictorConfig()
        self._predictor = predictor
        self._n_blocks = n_blocks
        self._dev = require_cuda()
        if dtype not in _LIB_DTYPE:
            raise InputError(f"cache dtype must be bf16, fp32 or fp64, got {dtype}")
        # snapshot precision: bf16 on the hot path (the block inputs / outputs are bf16); fp64
        # keeps numpy inputs exact for the numpy-interface drop-in (dropin.py)
        self.dtype = dtype
        self._dt = _LIB_DTYPE[dtype]
        self._slot_of: dict = {}
        self._free: list = []
        self._cap = 0
        self._shape = None  # per-patch shape (C, ps, ps)
        self._n = 0
        self._snap_in: list = []
        self._snap_out: list = []
        self._exists = None  # (n_blocks, cap) uint8
        self._streak = None  # (n_blocks, cap) int32
        self._ctr = torch.zeros((n_blocks, 4), dtype=torch.int64, device=self._dev)  # reuse, fresh, refreshed, inserted
        self._err = torch.zeros(1, dtype=torch.int32, device=self._dev)
        self._evicted = 0
        self._want_cap = capacity
        # storage generation: bumped whenever the slab tensors are replaced (_grow, restore), so
        # holders of raw pointers into them (engine_step.CachedStepGraph) know to re-capture
        self.storage_gen = 0

    # --------------------------------------------------------- storage
    @property
    def n_blocks(self) -> int:
        return self._n_blocks

    def _ensure_shape(self, shape) -> None:
        shape = tuple(int(s) for s in shape)
        if self._shape is None:
            self._shape = shape
            self._n = int(np.prod(shape))
            self._grow(max(self._want_cap, 1))
        elif shape != self._shape:
            raise InputError(f"patch shape {shape} differs from the cache's {self._shape}")

    def _grow(self, cap: int) -> None:
        old = self._cap
        if cap <= old:
            return
        dev = self._dev
        ni = [torch.zeros((cap, self._n), dtype=self.dtype, device=dev) for _ in range(self._n_blocks)]
        no = [torch.zeros((cap, self._n), dtype=self.dtype, device=dev) for _ in range(self._n_blocks)]
        ex = torch.zeros((self._n_blocks, cap), dtype=torch.uint8, device=dev)
        st = torch.zeros((self._n_blocks, cap), dtype=torch.int32, device=dev)
        if old:
            for b in range(self._n_blocks):
                ni[b][:old].copy_(self._snap_in[b])
                no[b][:old].copy_(self._snap_out[b])
            ex[:, :old].copy_(self._exists)
            st[:, :old].copy_(self._streak)
        self._snap_in, self._snap_out, self._exists, self._streak = ni, no, ex, st
        self.storage_gen += 1
        self._free.extend(range(cap - 1, old - 1, -1))
        self._cap = cap

    def _check_block(self, block_id: int) -> None:
        if not 0 <= block_id < self._n_blocks:
            raise InputError(f"block_id {block_id} out of range [0, {self._n_blocks})")

    def slots_for(self, keys: Sequence[Key], allocate: bool) -> torch.Tensor:
        out = np.empty(len(keys), dtype=np.int32)
        for i, k in enumerate(keys):
            s = self._slot_of.get(k)
            if s is None:
                if allocate:
                    if not self._free:
                        self._grow(max(2 * self._cap, self._cap + len(keys)))
                    s = self._free.pop()
                    self._slot_of[k] = s
                else:
                    s = -1
            out[i] = s
        return torch.as_tensor(out, device=self._dev)

    def _mask_u8(self, mask, n: int) -> torch.Tensor:
        m = mask if isinstance(mask, torch.Tensor) else torch.as_tensor(np.asarray(mask, dtype=bool))
        if tuple(m.shape) != (n,):
            raise InputError(f"mask must have shape ({n},)")
        return m.to(device=self._dev, dtype=torch.bool).contiguous().view(torch.uint8)

    def _raise_if_missing(self, block_id: int) -> None:
        if int(self._err.item()):
            self._err.zero_()
            raise IntegrityError(f"masked patch missing from block {block_id}")

    # ------------------------------------------------------- inspection
    def entry(self, block_id: int, key: Key) -> CacheEntry | None:
        self._check_block(block_id)
        s = self._slot_of.get(key)
        if s is None or self._exists is None or not int(self._exists[block_id, s]):
            return None
        return CacheEntry(self._snap_in[block_id][s].view(self._shape).clone(),
                          self._snap_out[block_id][s].view(self._shape).clone(),
                          int(self._streak[block_id, s]))

    def size(self) -> int:
        return 0 if self._exists is None else int(self._exists.sum())

    @property
    def stats(self) -> CacheStats:
        c = self._ctr.sum(dim=0).tolist()
        return CacheStats(predicted_reuse=c[0], fresh_compute=c[1], refreshed=c[2], inserted=c[3],
                          evicted=self._evicted)

    # ---------------------------------------------------------- batch ops
    def predict_reuse(self, block_id: int, keys: Sequence[Key], inputs, slots: torch.Tensor | None = None):
        """Device bool mask: entry exists, mse < sigma, streak < R (cache.py:107-122)."""
        self._check_block(block_id)
        x = _patches(inputs, self.dtype)
        if len(keys) != x.shape[0]:
            raise InputError("keys and inputs length mismatch")
        P = x.shape[0]
        if P == 0:
            return torch.zeros(0, dtype=torch.bool, device=self._dev)
        self._ensure_shape(x.shape[1:])
        if slots is None:
            slots = self.slots_for(keys, allocate=False)
        if self._predictor is not None:
            return self._predict_custom(block_id, keys, x)
        plan = PairwisePlan.get(self._n)
        mask = torch.empty(P, dtype=torch.bool, device=self._dev)
        scratch = torch.empty(scratch_doubles(P, plan), dtype=torch.float64, device=self._dev)
        _lib.call("ps_cache_predict", stream(), x.data_ptr(), self._dt, P, self._n, slots.data_ptr(),
                  self._snap_in[block_id].data_ptr(), self._exists[block_id].data_ptr(),
                  self._streak[block_id].data_ptr(), float(self.cfg.mse_threshold), int(self.cfg.max_streak),
                  plan.leaves.data_ptr(), plan.L, plan.nodes.data_ptr(), plan.I, plan.level_off.data_ptr(), plan.H,
                  scratch.data_ptr(), mask.view(torch.uint8).data_ptr(), self._ctr[block_id].data_ptr())
        return mask

    def _predict_custom(self, block_id, keys, x):
        # user-supplied predictor (cache.py:76-82): called per live entry, as the reference does
        out = np.zeros(len(keys), dtype=bool)
        for i, k in enumerate(keys):
            e = self.entry(block_id, k)
            out[i] = e is not None and bool(self._predictor(e, x[i])) and e.reuse_streak < self.cfg.max_streak
        n_re = int(out.sum())
        self._ctr[block_id, 0] += n_re
        self._ctr[block_id, 1] += len(keys) - n_re
        return torch.as_tensor(out, device=self._dev)

    def gather(self, block_id: int, keys: Sequence[Key], mask, shape):
        """Cached (inputs, outputs) for masked rows, zeros elsewhere (cache.py:124-137)."""
        self._check_block(block_id)
        P = len(keys)
        shape = tuple(int(s) for s in shape)
        ins = torch.zeros((P,) + shape, dtype=self.dtype, device=self._dev)
        outs = torch.zeros_like(ins)
        m = self._mask_u8(mask, P)
        if P == 0:
            return ins, outs
        if self._shape is None:
            if bool(m.any()):
                raise IntegrityError(f"masked patch missing from block {block_id}")
            return ins, outs
        self._ensure_shape(shape)
        slots = self.slots_for(keys, allocate=False)
        _lib.call("ps_cache_gather", stream(), m.data_ptr(), slots.data_ptr(), self._exists[block_id].data_ptr(), P,
                  self._n, self._dt, self._snap_in[block_id].data_ptr(), self._snap_out[block_id].data_ptr(), ins.data_ptr(),
                  outs.data_ptr(), self._err.data_ptr())
        self._raise_if_missing(block_id)
        return ins, outs

    def batched_fill(self, block_id: int, keys: Sequence[Key], mask, out=None):
        """Serve masked rows from output snapshots and advance their streaks (cache.py:139-151)."""
        self._check_block(block_id)
        P = len(keys)
        m = self._mask_u8(mask, P)
        if P == 0:
            return out
        if self._shape is None:
            if bool(m.any()):
                raise IntegrityError(f"masked patch missing from block {block_id}")
            return out
        slots = self.slots_for(keys, allocate=False)
        dst = None
        if out is not None:
            dst = out if (isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == self.dtype
                          and out.is_contiguous()) else torch.empty((P, self._n), dtype=self.dtype,
                                                                    device=self._dev)
        _lib.call("ps_cache_fill", stream(), m.data_ptr(), slots.data_ptr(), self._exists[block_id].data_ptr(),
                  self._streak[block_id].data_ptr(), P, self._n, self._dt, self._snap_out[block_id].data_ptr(),
                  None if dst is None else dst.data_ptr(), self._err.data_ptr())
        self._raise_if_missing(block_id)
        if out is not None and dst is not out:
            mb = m.view(torch.bool).cpu().numpy() if not isinstance(out, torch.Tensor) else m.view(torch.bool)
            src = dst.view((P,) + self._shape)
            if isinstance(out, torch.Tensor):
                out[mb] = src[mb].to(out.dtype).to(out.device)
            else:
                out[mb] = src.double().cpu().numpy()[mb]
        return out

    def batched_update(self, block_id: int, keys: Sequence[Key], mask, inputs, outputs,
                       slots: torch.Tensor | None = None) -> None:
        """Fresh snapshots with streak 0 for every unmasked row (cache.py:153-169)."""
        self._check_block(block_id)
        x, y = _patches(inputs, self.dtype), _patches(outputs, self.dtype)
        if not (len(keys) == x.shape[0] == y.shape[0]):
            raise InputError("keys/inputs/outputs length mismatch")
        P = len(keys)
        m = self._mask_u8(mask, P)
        if P == 0:
            return
        self._ensure_shape(x.shape[1:])
        if slots is None:
            slots = self.slots_for(keys, allocate=True)
        _lib.call("ps_cache_update", stream(), m.data_ptr(), slots.data_ptr(), self._exists[block_id].data_ptr(),
                  self._streak[block_id].data_ptr(), P, self._n, self._dt, x.data_ptr(), y.data_ptr(),
                  self._snap_in[block_id].data_ptr(), self._snap_out[block_id].data_ptr(),
                  self._ctr[block_id, 2:].data_ptr())

    def evict_expired(self, live_keys: Sequence[Key]) -> int:
        """Drop entries whose key is not live (cache.py:171-181); returns the count."""
        live = set(live_keys)
        dead = [(k, s) for k, s in self._slot_of.items() if k not in live]
        if not dead or self._exists is None:
            for k, _ in dead:
                self._slot_of.pop(k)
            return 0
        ds = np.array([s for _, s in dead], dtype=np.int32)
        n = int(self._exists[:, torch.as_tensor(ds, device=self._dev).long()].sum())
        slots = torch.as_tensor(ds, device=self._dev)
        for b in range(self._n_blocks):
            _lib.call("ps_cache_evict", stream(), self._exists[b].data_ptr(), self._streak[b].data_ptr(),
                      slots.data_ptr(), len(ds))
        for k, s in dead:
            self._slot_of.pop(k)
            self._free.append(s)
        self._evicted += n
        return n

    # ------------------------------------------------ fused block path
    def block_substitute(self, block_id: int, slots: torch.Tensor, mask: torch.Tensor, x: torch.Tensor,
                         patches=None):
        """x_sub = mask ? snap_in : x (gather + np.where of patched.py:243-244, fused).
        patches: optional (device list, length bound, device length) -- only those rows are
        written (the others are left unspecified)."""
        out = torch.empty_like(x)
        plist, n_ub, n_dev = patches if patches is not None else (None, 0, None)
        _lib.call("ps_cache_substitute", stream(), mask.view(torch.uint8).data_ptr(), slots.data_ptr(), x.shape[0],
                  self._n, self._dt, x.data_ptr(), self._snap_in[block_id].data_ptr(), out.data_ptr(),
                  None if plist is None else plist.data_ptr(), n_ub, None if n_dev is None else n_dev.data_ptr())
        return out

    def block_finish(self, block_id: int, slots: torch.Tensor, mask: torch.Tensor, x: torch.Tensor,
                     y: torch.Tensor) -> None:
        """Splice cached outputs into masked rows of y, bump their streaks, and store fresh
        snapshots for the rest (patched.py:246 + cache.py:139-169, fused)."""
        _lib.call("ps_cache_finish", stream(), mask.view(torch.uint8).data_ptr(), slots.data_ptr(),
                  self._exists[block_id].data_ptr(), self._streak[block_id].data_ptr(), x.shape[0], self._n,
                  self._dt, x.data_ptr(), y.data_ptr(), self._snap_in[block_id].data_ptr(),
                  self._snap_out[block_id].data_ptr(), self._ctr[block_id, 2:].data_ptr())

    # ------------------------------------------------------ atomic steps
    def snapshot(self) -> "CacheSnapshot":
        """Copy of the device store for step rollback (cache.py:185-187): a list with one
        element per block, like the reference's list of per-block dicts (a slice of it is no
        longer a valid snapshot, cache.py:189-190)."""
        snap = CacheSnapshot({"block": b} for b in range(self._n_blocks))
        snap.slots, snap.free, snap.cap = dict(self._slot_of), list(self._free), self._cap
        if self._exists is not None:
            snap.exists, snap.streak = self._exists.clone(), self._streak.clone()
            snap.snap_in = [t.clone() for t in self._snap_in]
            snap.snap_out = [t.clone() for t in self._snap_out]
        return snap

    def restore(self, snap: "CacheSnapshot") -> None:
        """cache.py:189-192."""
        if not isinstance(snap, CacheSnapshot) or len(snap) != self._n_blocks:
            raise IntegrityError("snapshot block count mismatch")
        self._slot_of, self._free = dict(snap.slots), list(snap.free)
        if snap.exists is None:
            if self._exists is not None:
                self._exists.zero_()
                self._streak.zero_()
            self.storage_gen += 1
            return
        self._cap = snap.cap
        self._exists, self._streak = snap.exists.clone(), snap.streak.clone()
        self._snap_in = [t.clone() for t in snap.snap_in]
        self._snap_out = [t.clone() for t in snap.snap_out]
        self.storage_gen += 1


class CacheSnapshot(list):
    """BlockCache.snapshot(): one element per block; the device copies ride along."""

    slots: dict = {}
    free: list = []
    cap: int = 0
    exists = None
    streak = None
    snap_in: list = []
    snap_out: list = []
