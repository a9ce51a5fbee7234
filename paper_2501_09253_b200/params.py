"""Parameter types (mirror mixserve/kernels.py:27-96) and their device images.

Parameters stay host numpy arrays in the reference's layouts so user code and
`init_weights` are unchanged; `device_params(p, C)` uploads each parameter set
once (cached by identity) into the layouts the sm_100a kernels consume:

* conv k=3 : B [Cp_out, 9*Cp_in] bf16, K index tap*Cp_in + c, tap = ky*3 + kx
* conv k=1 / linear : B [Cp_out, Cp_in]
* feed_forward : W1 [Hp, Cp], W2 [Cp, Hp] (+ fp32 biases, zero padded)
* attention : Wqkv^T [3*Dp, Dp] (rows: q, k, v output features; the reference
  applies x @ W, kernels.py:264-267, hence the transpose), Wo^T [Dp, Dp]
* norms : fp32 gamma / beta
Padding channels carry zero weights, so they stay exactly zero end to end.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._dev import require_cuda, round_up
from .errors import InputError


@dataclass(frozen=True)
class ConvParams:
    weights: np.ndarray  # (C_out, C_in, k, k)
    bias: np.ndarray

    def __post_init__(self):
        w = np.asarray(self.weights)
        if w.ndim != 4 or w.shape[2] != w.shape[3]:
            raise InputError(f"conv weights must be (C_out,C_in,k,k), got {w.shape}")
        if w.shape[2] not in (1, 3):
            raise InputError(f"kernel size must be 1 or 3, got {w.shape[2]}")
        if np.asarray(self.bias).shape != (w.shape[0],):
            raise InputError("conv bias must be (C_out,)")

    @property
    def kernel_size(self) -> int:
        return int(np.asarray(self.weights).shape[2])

    @property
    def padding(self) -> int:
        return self.kernel_size // 2


@dataclass(frozen=True)
class GroupNormParams:
    groups: int
    gamma: np.ndarray
    beta: np.ndarray
    eps: float = 1e-5

    def __post_init__(self):
        if self.groups < 1:
            raise InputError("groups must be >= 1")
        if self.eps <= 0:
            raise InputError("eps must be positive")


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
    w1: np.ndarray  # (hidden, C)
    b1: np.ndarray
    w2: np.ndarray  # (C, hidden)
    b2: np.ndarray


@dataclass(frozen=True)
class AttentionParams:
    wq: np.ndarray  # (D, D), applied as x @ wq
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray


_CACHE: dict = {}


def _bf16(a, dev) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device=dev).to(torch.bfloat16).contiguous()


def _f32(a, dev) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device=dev).contiguous()


def _pad2(w: np.ndarray, rows: int, cols: int) -> np.ndarray:
    out = np.zeros((rows, cols), dtype=np.float64)
    out[: w.shape[0], : w.shape[1]] = w
    return out


def _pad1(b: np.ndarray, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.float64)
    out[: b.shape[0]] = b
    return out


def _kind_of(prm) -> str:
    # duck-typed so the reference's own parameter objects work unchanged
    if hasattr(prm, "wq"):
        return "attention"
    if hasattr(prm, "w1"):
        return "feed_forward"
    if hasattr(prm, "weights"):
        return "conv" if np.asarray(prm.weights).ndim == 4 else "linear"
    if hasattr(prm, "groups"):
        return "group_norm"
    if hasattr(prm, "gamma"):
        return "layer_norm"
    raise InputError(f"unsupported parameter type {type(prm).__name__}")


def device_params(prm, channels: int) -> dict:
    """Device image of a parameter set for an input with `channels` channels."""
    key = (id(prm), channels)
    hit = _CACHE.get(key)
    if hit is not None and hit[0] is prm:
        return hit[1]
    dev = require_cuda()
    d: dict = {}
    kind = _kind_of(prm)
    if kind == "conv":
        w = np.asarray(prm.weights, dtype=np.float64)
        co, ci, k, _ = w.shape
        if ci != channels:
            raise InputError(f"conv channel mismatch: {channels} vs {ci}")
        cpi, cpo = round_up(ci, 64), round_up(co, 64)
        if k == 3:
            wt = np.zeros((cpo, 9, cpi))
            wt[:co, :, :ci] = w.transpose(0, 2, 3, 1).reshape(co, 9, ci)
            d["w"] = _bf16(wt.reshape(cpo, 9 * cpi), dev)
        else:
            d["w"] = _bf16(_pad2(w[:, :, 0, 0], cpo, cpi), dev)
        d.update(b=_f32(_pad1(np.asarray(prm.bias, dtype=np.float64), cpo), dev), c_out=co, cp_out=cpo, cp_in=cpi, k=k)
    elif kind == "linear":
        w = np.asarray(prm.weights, dtype=np.float64)
        co, ci = w.shape
        if ci != channels:
            raise InputError(f"channel mismatch: weights expect {ci}, input has {channels}")
        cpi, cpo = round_up(ci, 64), round_up(co, 64)
        d.update(w=_bf16(_pad2(w, cpo, cpi), dev), b=_f32(_pad1(np.asarray(prm.bias, dtype=np.float64), cpo), dev),
                 c_out=co, cp_out=cpo, cp_in=cpi)
    elif kind == "feed_forward":
        w1 = np.asarray(prm.w1, dtype=np.float64)
        w2 = np.asarray(prm.w2, dtype=np.float64)
        h, ci = w1.shape
        if ci != channels or w2.shape != (ci, h):
            raise InputError(f"feed_forward shape mismatch for {channels} channels")
        cp, hp = round_up(ci, 64), round_up(h, 64)
        d.update(w1=_bf16(_pad2(w1, hp, cp), dev), b1=_f32(_pad1(np.asarray(prm.b1, dtype=np.float64), hp), dev),
                 w2=_bf16(_pad2(w2, cp, hp), dev), b2=_f32(_pad1(np.asarray(prm.b2, dtype=np.float64), cp), dev),
                 hidden=h, hp=hp, cp=cp, c_out=ci)
    elif kind == "attention":
        ws = [np.asarray(getattr(prm, k), dtype=np.float64) for k in ("wq", "wk", "wv", "wo")]
        dd = ws[0].shape[0]
        if dd != channels or any(w.shape != (dd, dd) for w in ws):
            raise InputError(f"attention weights must be ({channels},{channels})")
        dp = round_up(dd, 64)
        if dp > 320:
            raise InputError(f"attention head dim {dd} > 320 is not supported by the sm_100a kernel")
        qkv = np.concatenate([_pad2(w.T, dp, dp) for w in ws[:3]], axis=0)
        d.update(wqkv=_bf16(qkv, dev), wo=_bf16(_pad2(ws[3].T, dp, dp), dev), d=dd, dp=dp)
    elif kind in ("group_norm", "layer_norm"):
        g = np.asarray(prm.gamma, dtype=np.float64)
        if g.shape != (channels,):
            raise InputError("norm affine parameters must be (C,)")
        d.update(gamma=_f32(g, dev), beta=_f32(np.asarray(prm.beta, dtype=np.float64), dev), eps=float(prm.eps))
        if kind == "group_norm":
            if channels % prm.groups:
                raise InputError(f"groups={prm.groups} does not divide channels={channels}")
            d["groups"] = prm.groups
    else:
        raise InputError(f"unsupported parameter type {type(prm).__name__}")
    _CACHE[key] = (prm, d)
    return d
