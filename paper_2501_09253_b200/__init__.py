"""B200-native PatchedServe patch-execution path (arXiv 2501.09253).

Drop-in for the hot-path subset of the reference `mixserve` package: CSP
split/merge with halos, per-image GroupNorm, per-image attention, the pixel-wise
stages, the block interpreter, the patch cache and the denoise step.  All
compute runs in libpatchserve.so (hand-written sm_100a CUDA: tcgen05/TMEM/TMA)
through its C ABI (include/patchserve.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .errors import InputError, IntegrityError  # noqa: F401
from .csp import (CSPBatch, DIRECTIONS, OPPOSITE, RequestEntry, ResolutionClass, STANDARD_CLASSES,  # noqa: F401
                  choose_patch_size, reassemble, split)
from .params import (AttentionParams, ConvParams, FeedForwardParams, GroupNormParams,  # noqa: F401
                     LayerNormParams, LinearParams)
from .patched import (exchange_halos, launch_counters, masked_block_forward, patched_conv,  # noqa: F401
                      patched_layer_norm, patched_self_attention, reset_launch_counters, run_block,
                      stitched_group_norm)
from .cache import BlockCache, CacheEntry, CacheStats, PredictorConfig, mse, partition_sets  # noqa: F401
from .model import (ModelConfig, SDXL_SHAPED, blend, denoise_batch, init_weights, make_prompt,  # noqa: F401
                    rate_schedule)

__all__ = [
    "AttentionParams", "BlockCache", "CSPBatch", "CacheEntry", "CacheStats", "ConvParams", "FeedForwardParams",
    "GroupNormParams", "InputError", "IntegrityError", "LayerNormParams", "LinearParams", "ModelConfig",
    "PredictorConfig", "STANDARD_CLASSES", "blend", "choose_patch_size", "denoise_batch", "exchange_halos",
    "init_weights", "launch_counters", "make_prompt", "masked_block_forward", "mse", "partition_sets",
    "patched_conv", "patched_layer_norm", "patched_self_attention", "rate_schedule", "reassemble",
    "reset_launch_counters", "run_block", "split", "stitched_group_norm",
]
