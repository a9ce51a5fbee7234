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
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .cache import BlockCache
from .csp import CSPBatch
from .model import blend_batch, prompt_bias
from .patched import _bf16_nchw, run_block, run_block_active


@dataclass
class StepStats:
    skipped: int = 0      # patch-blocks served from the cache
    computed: int = 0     # patch-blocks recomputed (reference telemetry, engine.py:143-147)
    rows_run: int = 0     # patch-blocks whose pixel-wise stages actually ran (after compaction)


def numeric_step(batch: CSPBatch, weights, cache: BlockCache | None, bias: torch.Tensor, rates: torch.Tensor,
                 keys=None, slots: torch.Tensor | None = None, compact: bool = True):
    """Denoise one step of `batch` (fp32 latents in batch.data); returns (new latents, StepStats)."""
    P = batch.n_patches
    lat = batch.data if batch.data.dtype == torch.float32 else batch.data.float()
    h = prompt_bias(batch, lat.contiguous(), bias)
    st = StepStats()
    if cache is not None and keys is None:
        keys = batch.patch_keys()
    if cache is not None and slots is None:
        cache._ensure_shape(h.shape[1:])
        slots = cache.slots_for(keys, allocate=True)
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
