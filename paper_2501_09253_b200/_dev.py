"""Small torch plumbing shared by the facade: device checks, streams, pointers."""

from __future__ import annotations

import numpy as np
import torch

from .errors import InputError


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2501_09253_b200 needs a CUDA device (B200); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, dtype=None) -> torch.Tensor:
    """CUDA tensor view/copy of x (torch tensor or numpy array)."""
    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    if t.device.type != "cuda":
        t = t.to(dev, non_blocking=True)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


# Input validation of the public eager API (kernels.py:20-24 rejects non-finite inputs with
# InputError).  Internal drivers whose inputs were validated once at their own entry
# (engine_step.numeric_step, pipeline.DenoisePipeline -- its split kernel flags non-finite
# latents on the device -- and CachedStepGraph) run inside `trusted_inputs()`, so their blocks
# neither synchronise nor break stream capture; checks are also skipped while capturing.
_TRUSTED = [0]


class trusted_inputs:
    def __enter__(self):
        _TRUSTED[0] += 1

    def __exit__(self, *exc):
        _TRUSTED[0] -= 1


def check_finite(t: torch.Tensor) -> None:
    if _TRUSTED[0] or not t.is_floating_point() or torch.cuda.is_current_stream_capturing():
        return
    if not bool(torch.isfinite(t).all()):
        raise InputError("non-finite values in input")


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def i32(a, dev=None) -> torch.Tensor:
    return torch.as_tensor(np.asarray(a, dtype=np.int32), device=dev or require_cuda())


def checksum(t: torch.Tensor) -> int:
    """XOR fold of a CUDA tensor's 32-byte words (ps_checksum): an order-independent u32 over the
    raw bytes, for checking resident latents / snapshots after a copy.  Needs a contiguous tensor
    whose byte size is a multiple of 32 and whose storage is 32-byte aligned."""
    from . import _lib
    if t.device.type != "cuda" or not t.is_contiguous():
        raise InputError("checksum: needs a contiguous CUDA tensor")
    out = torch.zeros(1, dtype=torch.int32, device=t.device)
    _lib.call("ps_checksum", stream(), t.data_ptr(), t.numel() * t.element_size(), out.data_ptr())
    return int(out.item()) & 0xFFFFFFFF
