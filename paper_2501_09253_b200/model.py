"""Denoiser step over a CSP batch — drop-in for mixserve/model.py.

`init_weights` draws exactly the reference's parameters (model.py:66-94, same
default_rng(seed) draw order) so parity runs use identical weights; the
SDXL-shaped bench model is `ModelConfig("unet_like", channels=320,
hidden=1280, groups=32, n_blocks=7)`.  `denoise_batch` is the patched step
(model.py:146-166): prompt bias into the first block input (one kernel),
the blocks, then `blend` with fp32 master latents (one kernel).
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._dev import check_finite, require_cuda, stream, to_device, trusted_inputs
from .csp import CSPBatch
from .errors import InputError
from .params import (AttentionParams, ConvParams, FeedForwardParams, GroupNormParams, LayerNormParams)
from .patched import run_block, run_block_shard, shard_context

ARCHS = ("unet_like", "dit_like")
RATE_START = 0.15
RATE_END = 0.05


@dataclass(frozen=True)
class ModelConfig:
    """model.py:40-53."""

    arch: str = "dit_like"
    channels: int = 4
    hidden: int = 8
    n_blocks: int = 2
    groups: int = 2
    seed: int = 0

    def __post_init__(self):
        if self.arch not in ARCHS:
            raise InputError(f"arch must be one of {ARCHS}, got {self.arch!r}")
        if self.channels % self.groups != 0:
            raise InputError("groups must divide channels")


SDXL_SHAPED = ModelConfig(arch="unet_like", channels=320, hidden=1280, groups=32, n_blocks=7, seed=0)


def rate_schedule(step_idx: int, total_steps: int) -> float:
    """model.py:56-63."""
    if not 0 <= step_idx < total_steps:
        raise InputError(f"step {step_idx} outside [0, {total_steps})")
    if total_steps == 1:
        return RATE_START
    return RATE_START + (RATE_END - RATE_START) * (step_idx / (total_steps - 1))


def init_weights(cfg: ModelConfig) -> list:
    """Per-block (kind, params) stage lists, deterministic in cfg.seed (model.py:66-94)."""
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
            gn = GroupNormParams(groups=cfg.groups, gamma=gamma, beta=beta)
            c3 = ConvParams(weights=rng.normal(size=(c, c, 3, 3)) * (0.8 / np.sqrt(9 * c)),
                            bias=0.01 * rng.normal(size=c))
            ops = [("group_norm", gn), ("conv", c3), ("attention", at), ("feed_forward", ff), ("residual", None)]
        else:
            ops = [("layer_norm", LayerNormParams(gamma=gamma, beta=beta)), ("attention", at),
                   ("feed_forward", ff), ("residual", None)]
        blocks.append(ops)
    return blocks


def make_prompt(cfg: ModelConfig, request_id: str) -> np.ndarray:
    """Deterministic per-request conditioning vector (model.py:97-103)."""
    digest = (zlib.crc32(request_id.encode()) ^ (cfg.seed * 0x9E3779B9)) & 0xFFFFFFFF
    return 0.1 * np.random.default_rng(digest).normal(size=cfg.channels)


def prompt_bias(batch: CSPBatch, latents: torch.Tensor, bias: torch.Tensor) -> torch.Tensor:
    """h = bf16(latent + prompt[request]) — the first block input (model.py:163)."""
    P, c, ps = latents.shape[0], latents.shape[1], batch.patch_size
    h = torch.empty((P, c, ps, ps), dtype=torch.bfloat16, device=latents.device)
    _lib.call("ps_prompt_bias", stream(), latents.data_ptr(), bias.data_ptr(),
              batch.device()["request_index"].data_ptr(), P, c, ps, h.data_ptr())
    return h


def blend_batch(batch: CSPBatch, latents: torch.Tensor, h: torch.Tensor, rates: torch.Tensor) -> torch.Tensor:
    """(1 - r) * x + r * tanh(h) per request rate, fp32 out (model.py:129-131, 166)."""
    P, c, ps = latents.shape[0], latents.shape[1], batch.patch_size
    out = torch.empty_like(latents)
    _lib.call("ps_blend", stream(), latents.data_ptr(), h.data_ptr(), rates.data_ptr(),
              batch.device()["request_index"].data_ptr(), P, c, ps, out.data_ptr())
    return out


def blend(x, h, rate) -> torch.Tensor:
    """model.py:129-131 on the device: (1 - rate) x + rate tanh(h), fp32 out.  `rate` is a scalar
    or one rate per leading row of x (e.g. the engine's rate[request_index][:, None, None, None],
    engine.py:158)."""
    xt = to_device(x, torch.float32)
    ht = to_device(h)
    if ht.shape != xt.shape:
        raise InputError("blend: shape mismatch")
    r = np.asarray(rate.detach().cpu() if isinstance(rate, torch.Tensor) else rate, dtype=np.float64)
    if r.size == 1:
        rows = 1
    elif xt.dim() >= 1 and r.size == xt.shape[0] and all(d == 1 for d in r.shape[1:]):
        rows = xt.shape[0]
    else:
        raise InputError(f"blend: rate must be a scalar or one value per row, got shape {r.shape}")
    n = xt.numel() // max(1, rows)
    if n % 4:
        raise InputError("blend: elements per row must be a multiple of 4")
    flat = xt.reshape(rows, n // 4, 2, 2).contiguous()
    hb = ht.to(torch.bfloat16).reshape(rows, n // 4, 2, 2).contiguous()
    out = torch.empty_like(flat)
    rates = torch.as_tensor(r.reshape(-1), dtype=torch.float32, device=xt.device)
    ri = torch.arange(rows, dtype=torch.int32, device=xt.device)
    # view each row as one "patch" of n/4 channels of 2x2 pixels with its own rate
    _lib.call("ps_blend", stream(), flat.data_ptr(), hb.data_ptr(), rates.data_ptr(), ri.data_ptr(), rows, n // 4, 2,
              out.data_ptr())
    return out.reshape(xt.shape)


def step_inputs(cfg: ModelConfig, batch: CSPBatch, prompts: dict, step_idx: dict, total_steps: dict):
    """Device prompt-bias matrix [R, C] and per-request rates [R] (model.py:156-162)."""
    bias = np.empty((batch.n_requests, cfg.channels))
    rate = np.empty(batch.n_requests)
    for slot, e in enumerate(batch.requests):
        if e.request_id not in prompts:
            raise InputError(f"missing prompt for request {e.request_id!r}")
        bias[slot] = np.asarray(prompts[e.request_id], dtype=np.float64)
        rate[slot] = rate_schedule(step_idx[e.request_id], total_steps[e.request_id])
    dev = require_cuda()
    return (torch.as_tensor(bias, dtype=torch.float32, device=dev),
            torch.as_tensor(rate, dtype=torch.float32, device=dev))


def denoise_batch(cfg: ModelConfig, weights, batch: CSPBatch, prompts: dict, step_idx: dict,
                  total_steps: dict) -> torch.Tensor:
    """Patched step over a mixed batch; returns the updated (P, C, ps, ps) fp32 latents."""
    if batch.data.shape[1] != cfg.channels:
        raise InputError(f"batch has {batch.data.shape[1]} channels, model expects {cfg.channels}")
    bias, rates = step_inputs(cfg, batch, prompts, step_idx, total_steps)
    lat = batch.data if batch.data.dtype == torch.float32 else batch.data.float()
    lat = lat.contiguous()
    check_finite(lat)  # kernels.py:20-24, once per step
    h = prompt_bias(batch, lat, bias)
    with trusted_inputs():
        for ops in weights:
            h = run_block(batch, h, ops)
    return blend_batch(batch, lat, h, rates)


def denoise_batch_shard(cfg: ModelConfig, weights, batch: CSPBatch, shard, exch, prompts: dict, step_idx: dict,
                        total_steps: dict, inputs=None, ctx=None) -> torch.Tensor:
    """denoise_batch for one rank of the split-image path (patchshard.py).

    `batch` is the rank's local CSP batch (the requests its patch range touches,
    `shard.requests`); rows of the owned patches (`shard.owned`) of the result
    equal the single-GPU denoise_batch rows of the same patches; ghost rows are
    unspecified.  `inputs` = precomputed (bias, rates) device tensors and `ctx` = a
    shard_context reused across steps make the call free of host->device copies, so a
    fixed-composition step can be captured in a CUDA graph.
    """
    if batch.data.shape[1] != cfg.channels:
        raise InputError(f"batch has {batch.data.shape[1]} channels, model expects {cfg.channels}")
    bias, rates = inputs if inputs is not None else step_inputs(cfg, batch, prompts, step_idx, total_steps)
    lat = batch.data if batch.data.dtype == torch.float32 else batch.data.float()
    lat = lat.contiguous()
    h = prompt_bias(batch, lat, bias)
    ctx = ctx or shard_context(batch, shard, exch)
    for ops in weights:
        h = run_block_shard(batch, h, ops, shard, exch, ctx=ctx)
    return blend_batch(batch, lat, h, rates)
