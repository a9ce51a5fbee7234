"""numpy-interface drop-in for the reference's hot-path modules.

The reference (`mixserve`) passes numpy float64 arrays between its engine and the patch path
(engine.py:126-160).  This module gives the same functions with the same signatures, argument
meaning, error types and return TYPES (numpy arrays, a CSPBatch whose `.data` is numpy), so the
reference's Engine, verify code and tests run unchanged with their imports pointed here
(INTEGRATION.md §1).  Every computation still runs in libpatchserve.so on the GPU: arrays cross
to the device at each call and come back as numpy float64.

Precision contract (what differs from the fp64 reference):
* exact: split / reassemble / exchange_halos (fp64 copies on the device), patch keys and all
  metadata, partition_sets, the cache (fp64 slab: snapshots are exact copies, masks bit-exact
  because `mse` is numpy's fp64 pairwise tree), streaks and stats;
* tolerance: the compute stages (GroupNorm, conv, attention, LayerNorm, FF, blocks, the denoise
  step) run on bf16 tensor cores with fp32 accumulation (tests state the bounds).

This adapter is for drop-in compatibility and verification; the throughput path keeps tensors on
the device (pipeline.DenoisePipeline, engine_step) instead of round-tripping through numpy.
"""

from __future__ import annotations

from collections.abc import Mapping
from typing import Sequence

import numpy as np
import torch

from . import cache as _cache
from . import csp as _csp
from . import model as _model
from . import patched as _patched
from .cache import CacheEntry, CacheStats, PredictorConfig, partition_sets  # noqa: F401
from .csp import CSPBatch, RequestEntry, STANDARD_CLASSES, choose_patch_size  # noqa: F401
from .errors import InputError, IntegrityError  # noqa: F401
from .model import ModelConfig, init_weights, make_prompt, rate_schedule  # noqa: F401
from .patched import launch_counters, reset_launch_counters  # noqa: F401


def _np(t) -> np.ndarray:
    if isinstance(t, torch.Tensor):
        return t.detach().to(torch.float64).cpu().numpy()
    return np.asarray(t, dtype=np.float64)


def _dev64(x) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(x, np.float64)))
    return t.to(device="cuda", dtype=torch.float64 if t.dtype == torch.float64 or not isinstance(x, torch.Tensor)
                else t.dtype).contiguous()


# ------------------------------------------------------------------ csp.py


def split(requests: Sequence, patch_size: int | None = None) -> CSPBatch:
    """csp.py:117-193; `.data` is a numpy float64 (P, C, ps, ps) array (exact copies)."""
    reqs = []
    for rid, lat in requests:
        a = np.asarray(lat, dtype=np.float64)
        reqs.append((rid, torch.from_numpy(np.ascontiguousarray(a)).cuda()))
    batch = _csp.split(reqs, patch_size=patch_size)
    batch.data = _np(batch.data)
    return batch


def reassemble(batch: CSPBatch, data=None) -> dict:
    """csp.py:196-214 -> {request_id: numpy (C, L, L)}."""
    src = batch.data if data is None else data
    out = _csp.reassemble(batch, _dev64(src))
    return {k: _np(v) for k, v in out.items()}


# --------------------------------------------------------------- patched.py


def exchange_halos(batch: CSPBatch, data) -> np.ndarray:
    return _np(_patched.exchange_halos(batch, _dev64(data)))


def patched_conv(batch: CSPBatch, data, p, frames=None) -> np.ndarray:
    return _np(_patched.patched_conv(batch, _dev64(data), p, None if frames is None else _dev64(frames)))


def stitched_group_norm(batch: CSPBatch, data, p, emit_halos: bool = False):
    out = _patched.stitched_group_norm(batch, _dev64(data), p, emit_halos=emit_halos)
    if emit_halos:
        return _np(out[0]), _np(out[1])
    return _np(out)


def patched_layer_norm(batch: CSPBatch, data, p) -> np.ndarray:
    return _np(_patched.patched_layer_norm(batch, _dev64(data), p))


def patched_self_attention(batch: CSPBatch, data, p) -> np.ndarray:
    return _np(_patched.patched_self_attention(batch, _dev64(data), p))


def run_block(batch: CSPBatch, x, ops) -> np.ndarray:
    return _np(_patched.run_block(batch, _dev64(x), ops))


def masked_block_forward(batch: CSPBatch, x, mask, ops, cached_inputs, cached_outputs) -> np.ndarray:
    m = mask if isinstance(mask, np.ndarray) else np.asarray(mask)
    return _np(_patched.masked_block_forward(batch, _dev64(x), m, ops, _dev64(cached_inputs),
                                             _dev64(cached_outputs)))


# ----------------------------------------------------------------- model.py


def denoise_batch(cfg, weights, batch: CSPBatch, prompts: dict, step_idx: dict, total_steps: dict) -> np.ndarray:
    """model.py:146-166; batch.data may be numpy (this module's split) or a tensor."""
    data = batch.data
    batch.data = _dev64(data).to(torch.float32)
    try:
        return _np(_model.denoise_batch(cfg, weights, batch, prompts, step_idx, total_steps))
    finally:
        batch.data = data


def blend(x, h, rate) -> np.ndarray:
    """model.py:129-131 on the device (fp32); rate scalar or one per leading row."""
    return _np(_model.blend(np.asarray(x, np.float64), np.asarray(h, np.float64), rate))


# ----------------------------------------------------------------- cache.py


def mse(a, b) -> float:
    """cache.py:54-55, bit-exact (fp64 operands stay fp64)."""
    return _cache.mse(np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64))


class _StoreView(Mapping):
    """Read-only per-block key -> CacheEntry view (the reference's `BlockCache._stores[b]` dict,
    which its test helpers inspect, pkg/tests/helpers_cache.py:71-72)."""

    def __init__(self, cache: "BlockCache", b: int):
        self._c, self._b = cache, b

    def _live(self):
        c = self._c
        if c._exists is None:
            return []
        ex = c._exists[self._b].cpu().numpy()
        return [k for k, s in c._slot_of.items() if ex[s]]

    def __len__(self):
        return len(self._live())

    def __iter__(self):
        return iter(self._live())

    def __getitem__(self, key):
        e = self._c.entry(self._b, key)
        if e is None:
            raise KeyError(key)
        return e


class BlockCache(_cache.BlockCache):
    """cache.py:73-192 with numpy in/out: an fp64 device slab, so snapshots are exact and masks
    equal the reference's bit for bit; predict_reuse returns a numpy bool mask, gather numpy
    arrays, entry() numpy snapshots.  Entries keep the reference's immutability contract
    (cache.py:6-8): entry() returns the same object until that entry changes, and
    snapshot() / restore() bring the objects back with the state."""

    def __init__(self, n_blocks: int, cfg=None, predictor=None):
        super().__init__(n_blocks, cfg, predictor=predictor, dtype=torch.float64)
        self._memo: dict = {}

    @property
    def _stores(self):
        return [_StoreView(self, b) for b in range(self.n_blocks)]

    def predict_reuse(self, block_id, keys, inputs):
        if self._predictor is not None:
            self._check_block(block_id)
            x = np.asarray(inputs, dtype=np.float64)
            if len(keys) != len(x):
                raise InputError("keys and inputs length mismatch")
            out = np.zeros(len(keys), dtype=bool)
            for i, k in enumerate(keys):
                e = self.entry(block_id, k)
                out[i] = (e is not None and bool(self._predictor(e, x[i]))
                          and e.reuse_streak < self.cfg.max_streak)
            n_re = int(out.sum())
            self._ctr[block_id, 0] += n_re
            self._ctr[block_id, 1] += len(keys) - n_re
            return out
        return super().predict_reuse(block_id, keys, _dev64(inputs)).cpu().numpy()

    def gather(self, block_id, keys, mask, shape):
        ins, outs = super().gather(block_id, keys, np.asarray(mask, dtype=bool), shape)
        return _np(ins), _np(outs)

    def batched_fill(self, block_id, keys, mask, out=None):
        return super().batched_fill(block_id, keys, np.asarray(mask, dtype=bool), out=out)

    def batched_update(self, block_id, keys, mask, inputs, outputs):
        super().batched_update(block_id, keys, np.asarray(mask, dtype=bool), _dev64(inputs), _dev64(outputs))

    def entry(self, block_id, key):
        e = super().entry(block_id, key)
        if e is None:
            return None
        new = CacheEntry(_np(e.input_snapshot), _np(e.output_snapshot), e.reuse_streak)
        seen = self._memo.setdefault((block_id, key), [])
        for old in seen:  # the object handed out earlier for this exact state (immutability)
            if (old.reuse_streak == new.reuse_streak and np.array_equal(old.input_snapshot, new.input_snapshot)
                    and np.array_equal(old.output_snapshot, new.output_snapshot)):
                return old
        seen.insert(0, new)
        del seen[4:]
        return new

    def snapshot(self):
        snap = super().snapshot()
        snap.memo = {k: list(v) for k, v in self._memo.items()}
        return snap

    def restore(self, snap):
        super().restore(snap)
        for k, v in getattr(snap, "memo", {}).items():
            cur = self._memo.setdefault(k, [])
            cur[:0] = [o for o in v if all(o is not c for c in cur)]
            del cur[8:]


# names a reference module exposes -> this module's replacement (used to point the
# reference's own engine / tests at the drop-in, tests/refswap.py)
SWAP = {
    "errors": ("InputError", "IntegrityError"),
    "csp": ("split", "reassemble"),
    "patched": ("exchange_halos", "patched_conv", "stitched_group_norm", "patched_layer_norm",
                "patched_self_attention", "run_block", "masked_block_forward", "launch_counters",
                "reset_launch_counters"),
    "cache": ("BlockCache", "mse", "partition_sets"),
    "model": ("denoise_batch", "blend"),
}
