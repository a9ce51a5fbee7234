"""One serving step with the patch cache in the loop — engine.py:126-160 on the device.

Per block the reference does (engine.py:137-148):

    mask = cache.predict_reuse(b, keys, h)                    # cache.py:107-122
    cached_in, cached_out = cache.gather(b, keys, mask, ...)  # cache.py:124-137
    y = masked_block_forward(batch, h, mask, ops, cached_in, cached_out)   # patched.py:224-246
    cache.batched_fill(b, keys, mask)                          # cache.py:139-151
    cache.batched_update(b, keys, mask, h, y)                  # cache.py:153-169

Here that is: the bit-exact reuse test (K8); one mask read-back (the reference
also reads `mask.sum()` on the host, engine.py:143-144); then
* all patches reusable -> no block compute at all (patched.py:237-238);
* none reusable       -> run_block;
* otherwise           -> substitute cached inputs at masked patches (K9) and run
  the block compacted to the patches that need fresh outputs (run_block_active);
and one fused kernel that splices cached outputs, bumps streaks and stores
fresh snapshots (K9).  The results equal the reference sequence's: the
compacted rows are bit-identical to an uncompacted run.

Where the kernels cover the geometry (patched.device_compaction_ok) the read-back is
gone: the mask stays on the device, ps_compact_lists builds the compaction lists there
and every kernel of the block reads its work count from device memory
(patched.run_block_masked), so the host never waits inside a step; the per-block counts
are read once at the end of the step for StepStats.  PS_DEVICE_COMPACTION=0 restores the
per-block read-back.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from ._dev import check_finite, trusted_inputs
from .cache import BlockCache
from .csp import CSPBatch
from .model import blend_batch, prompt_bias
from .patched import _bf16_nchw, device_compaction_ok, masked_context, run_block, run_block_active, run_block_ctx

# eager steps: per-block mask read-back (default) or device-built compaction lists; the
# device form pays off inside a CUDA graph (CachedStepGraph), where no host work is left --
# eagerly its ~15 launches per block cost more host time than the read-back's bubble when
# whole blocks are reused
DEVICE_COMPACTION = os.environ.get("PS_DEVICE_COMPACTION", "0") == "1"


def _device_blocks(batch, weights, cache, keys, slots, lat, h, rates):
    """The blocks of a cached step with every decision on the device (no host round trip):
    returns (new latents, device int32 [n_blocks] of recomputed patches per block)."""
    counts = []
    for b, ops in enumerate(weights):
        mask = cache.predict_reuse(b, keys, h, slots=slots)
        ctx, cnt = masked_context(batch, mask)
        # the block reads its input only at the patches of live images
        x_sub = cache.block_substitute(b, slots, mask, h, patches=ctx.gn_live)
        y = _bf16_nchw(run_block_ctx(ctx, x_sub, ops))
        cache.block_finish(b, slots, mask, h, y)
        counts.append(cnt[4:5])
        h = y
    return blend_batch(batch, lat, h, rates), torch.cat(counts)


class CachedStepGraph:
    """numeric_step with the patch cache in the loop for a FIXED batch composition, captured
    as one CUDA graph: reuse test, compaction lists, compacted blocks, cache splice / streak
    / snapshot and blend all replay without the host (engine.py:126-160 on the device).

    The first run() is an eager step (it also allocates the cache storage and warms every
    plan); the graph is captured on the second call and replayed from then on.  Inputs are
    copied into static buffers; the returned latents are a static buffer overwritten by the
    next run().  Results equal numeric_step's bit for bit.  Needs the default predictor and
    patched.device_compaction_ok(batch)."""

    def __init__(self, batch: CSPBatch, weights, cache: BlockCache, keys=None):
        if not device_compaction_ok(batch) or batch.n_patches == 0:
            raise ValueError("CachedStepGraph: batch geometry not covered by the device compaction path")
        if cache._predictor is not None:
            raise ValueError("CachedStepGraph: a custom predictor runs on the host")
        self.batch, self.weights, self.cache = batch, weights, cache
        self.keys = batch.patch_keys() if keys is None else keys
        self.lat = batch.data.float().clone()
        self.bias = None
        self.rates = None
        self.slots = None
        self.graph = None
        self._gen = None  # cache.storage_gen the graph was captured against
        self._out = self._counts = None

    def _body(self):
        self.batch.data = self.lat
        with trusted_inputs():
            h = prompt_bias(self.batch, self.lat, self.bias)
            return _device_blocks(self.batch, self.weights, self.cache, self.keys, self.slots, self.lat, h,
                                  self.rates)

    def run(self, lat: torch.Tensor, bias: torch.Tensor, rates: torch.Tensor):
        """One step; returns (new latents [static buffer], StepStats)."""
        self.lat.copy_(lat)
        if self.bias is None:
            self.bias, self.rates = bias.clone(), rates.clone()
            self.cache._ensure_shape(self.lat.shape[1:])
            self.slots = self.cache.slots_for(self.keys, allocate=True)
            out, counts = self._body()           # eager first step
        else:
            self.bias.copy_(bias)
            self.rates.copy_(rates)
            if self.graph is not None and self._gen != self.cache.storage_gen:
                # the cache slab was re-allocated (grown by another batch, or restored): the graph's
                # baked pointers are stale -- capture again against the current storage
                self.graph = None
            if self.graph is None:
                self.slots = self.cache.slots_for(self.keys, allocate=True)
                self._gen = self.cache.storage_gen
                g = torch.cuda.CUDAGraph()
                # thread-local capture: another thread driving the same GPU (a second virtual rank,
                # a copy stream) does not invalidate this capture
                with torch.cuda.graph(g, capture_error_mode="thread_local"):
                    self._out, self._counts = self._body()
                self.graph = g
            self.graph.replay()
            out, counts = self._out, self._counts
        st = StepStats()
        st.computed = st.rows_run = int(counts.sum().item())
        st.skipped = self.batch.n_patches * len(self.weights) - st.computed
        return out, st


@dataclass
class StepStats:
    skipped: int = 0      # patch-blocks served from the cache
    computed: int = 0     # patch-blocks recomputed (reference telemetry, engine.py:143-147)
    rows_run: int = 0     # patch-blocks whose pixel-wise stages actually ran (after compaction)


def numeric_step(batch: CSPBatch, weights, cache: BlockCache | None, bias: torch.Tensor, rates: torch.Tensor,
                 keys=None, slots: torch.Tensor | None = None, compact: bool = True):
    """Denoise one step of `batch` (fp32 latents in batch.data); returns (new latents, StepStats)."""
    check_finite(batch.data)  # once per step (kernels.py:20-24); the blocks run trusted
    with trusted_inputs():
        return _numeric_step(batch, weights, cache, bias, rates, keys, slots, compact)


def _numeric_step(batch, weights, cache, bias, rates, keys, slots, compact):
    P = batch.n_patches
    lat = batch.data if batch.data.dtype == torch.float32 else batch.data.float()
    h = prompt_bias(batch, lat.contiguous(), bias)
    st = StepStats()
    if cache is not None and keys is None:
        keys = batch.patch_keys()
    if cache is not None and slots is None:
        cache._ensure_shape(h.shape[1:])
        slots = cache.slots_for(keys, allocate=True)
    if cache is not None and compact and DEVICE_COMPACTION and P and device_compaction_ok(batch):
        out, counts = _device_blocks(batch, weights, cache, keys, slots, lat, h, rates)
        computed = int(counts.sum().item())  # the step's only read-back
        st.computed = st.rows_run = computed
        st.skipped = P * len(weights) - computed
        return out, st
    for b, ops in enumerate(weights):
        if cache is None:
            h = run_block(batch, h, ops)
            st.computed += P
            st.rows_run += P
            continue
        mask = cache.predict_reuse(b, keys, h, slots=slots)
        m = mask.cpu().numpy()
        n_masked = int(m.sum())
        if n_masked == P:
            y = torch.empty_like(h)          # every row is spliced from the cache below
        elif n_masked == 0:
            y = run_block(batch, h, ops)
            st.rows_run += P
        else:
            x_sub = cache.block_substitute(b, slots, mask, h)
            y = run_block_active(batch, x_sub, ops, ~m) if compact else run_block(batch, x_sub, ops)
            st.rows_run += (P - n_masked) if compact else P
        y = _bf16_nchw(y)
        cache.block_finish(b, slots, mask, h, y)
        st.skipped += n_masked
        st.computed += P - n_masked
        h = y
    return blend_batch(batch, lat, h, rates), st
