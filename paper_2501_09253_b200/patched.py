"""Patched operators over CSP batches — drop-in for mixserve/patched.py.

Every stage runs on the sm_100a library through the C ABI.  Inside a block the
activations live channels-last ("CL": tokens x Cp, bf16, Cp = C rounded up to
64) so every contraction is a K-major tcgen05 GEMM; block inputs/outputs (the
residual stream) are NCHW (P, C, ps, ps) bf16, the reference's logical layout.

Fusions (each still counts one stage launch, as the reference does,
patched.py:33-45):
* group_norm followed by a k=3 conv emits channels-last halo frames directly
  (the stitcher, patched.py:191-201);
* a GEMM stage followed by `residual` writes the NCHW block output with the
  residual added in its epilogue (patched.py:215-217);
* attention = QKV GEMM (V written transposed) -> per-image flash attention ->
  output projection (patched.py:154-176, kernels.py:257-267).
"""

from __future__ import annotations

import ctypes as C
import os
from collections import Counter

import numpy as np
import torch

from . import _lib
from ._dev import check_finite, require_cuda, round_up, stream, to_device
from .csp import CSPBatch
from .errors import InputError
from .params import device_params

_launches: Counter = Counter()
BF16 = torch.bfloat16
# attention on CTA pairs (tcgen05 cta_group::2, 256-query tiles): the default since the pair's
# remote barrier arrives dropped their cluster-scope fences and the MMAs got two issuer warps
# (config-2 step 15.9 -> 15.4 ms); PS_ATTN_PAIRS=0 selects the single-CTA kernel
USE_PAIRS = os.environ.get("PS_ATTN_PAIRS", "1") == "1"
# bench hook: when a list, (start, end) CUDA events are recorded around every
# attention-kernel launch on the launching stream
ATTN_TIMER = None


def reset_launch_counters() -> None:
    _launches.clear()


def launch_counters() -> dict:
    return dict(_launches)


def _launch(kind: str) -> None:
    _launches[kind] += 1


# ---------------------------------------------------------------- helpers


def _check_data(batch: CSPBatch, data, finite: bool = True) -> torch.Tensor:
    t = to_device(data)
    if t.dim() != 4 or t.shape[0] != batch.n_patches or tuple(t.shape[2:]) != (batch.patch_size,) * 2:
        raise InputError(
            f"patch data must be ({batch.n_patches},C,{batch.patch_size},{batch.patch_size}), got {tuple(t.shape)}")
    if finite:
        check_finite(t)  # kernels.py:20-24 (skipped under trusted_inputs / stream capture)
    return t


def _bf16_nchw(t: torch.Tensor) -> torch.Tensor:
    if t.dtype == BF16:
        return t.contiguous()
    if t.dtype != torch.float32:
        t = t.to(torch.float32)
    out = torch.empty(t.shape, dtype=BF16, device=t.device)
    _lib.call("ps_convert", stream(), t.contiguous().data_ptr(), _lib.DTYPE_F32, out.data_ptr(), _lib.DTYPE_BF16,
              t.numel())
    return out


class Act:
    """An activation: NCHW bf16 (P, C, ps, ps) or CL bf16 (T, Cp)."""

    __slots__ = ("layout", "t", "C")

    def __init__(self, layout: str, t: torch.Tensor, c: int):
        self.layout, self.t, self.C = layout, t, c

    @property
    def Cp(self) -> int:
        return round_up(self.C, 64)


class Ctx:
    """Per-call geometry and device metadata for one batch."""

    def __init__(self, batch: CSPBatch):
        self.b = batch
        self.ps = batch.patch_size
        self.P = batch.n_patches
        self.hw = self.ps * self.ps
        self.T = self.P * self.hw
        self.dev = batch.device()
        self.device = require_cuda()
        # active-patch compaction (None = every 128-row tile): (device tile map, count)
        self.rows_live = None   # tiles of images with >= 1 patch to recompute (context for conv3/attention/GN)
        self.rows_act = None    # tiles of the patches to recompute
        self.attn_live = None   # attention query tiles (tile_q0, tile_img, n) of live images / active patches
        self.attn_act = None
        self.rows = None        # row set of the stage being run (set by _run_ops)
        self.attn_tiles = None
        # split-image multi-GPU path (patchshard.py): the owned patches and the exchanger
        self.owned = None       # device int32 list of owned patches
        self.owned_host = None
        self.exch = None
        # device-decided compaction (run_block_masked): live patch list, upper bound, device count
        self.gn_live = None

    def _attention_overlapped(self, qk, vt, ldv, dpp, d, host, finish, o):
        """Two-phase attention on the split-image path: phase A (owned keys of split images,
        all keys of whole images) runs while the K / V^T all-gather is in flight; phase B
        (remote keys) after finish(); partials merged by the combine kernel."""
        plan = self._overlap_plan(host)
        a_tiles, b_tiles, n_slots, comb = plan
        part_o = torch.empty((max(1, n_slots), 128, dpp), dtype=torch.float32, device=self.device)
        part_ml = torch.empty((max(1, n_slots), 128, 2), dtype=torch.float32, device=self.device)

        def launch(t):
            q0, img, kb0, nkb, slot, n = t
            if n:
                _lib.call("ps_attention_splitkv", stream(), qk.data_ptr(), vt.data_ptr(), ldv, self.T, dpp, d,
                          self.dev["img_tok0"].data_ptr(), q0.data_ptr(), img.data_ptr(), kb0.data_ptr(),
                          nkb.data_ptr(), slot.data_ptr(), n, part_o.data_ptr(), part_ml.data_ptr(), o.data_ptr())
        launch(a_tiles)
        finish()
        launch(b_tiles)
        cq0, cs0, cns, cimg, n_q = comb
        if n_q:
            _lib.call("ps_attention_combine", stream(), part_o.data_ptr(), part_ml.data_ptr(), cq0.data_ptr(),
                      cs0.data_ptr(), cns.data_ptr(), cimg.data_ptr(), self.dev["img_tok0"].data_ptr(), n_q, dpp,
                      o.data_ptr())

    def _overlap_plan(self, host):
        key = ("ovl", np.asarray(host[0]).tobytes(), np.asarray(host[1]).tobytes(),
               np.asarray(self.owned_host).tobytes(), sm_count(), str(self.device))
        if key not in _SKV_CACHE:
            _SKV_CACHE[key] = overlap_plan(host[0], host[1], self.b.request_offset, self.hw,
                                           np.asarray(self.owned_host), sm_count(), self.device)
        return _SKV_CACHE[key]

    def _tiles128(self, host):
        """Device copies of 128-query tile lists (cached by content)."""
        key = ("t128", np.asarray(host[0]).tobytes(), np.asarray(host[1]).tobytes(), str(self.device))
        if key not in _SKV_CACHE:
            _SKV_CACHE[key] = (torch.as_tensor(np.asarray(host[0], np.int32), device=self.device),
                               torch.as_tensor(np.asarray(host[1], np.int32), device=self.device))
        return _SKV_CACHE[key]

    def _splitkv(self, q0_host, img_host):
        """Split-KV plan when the query tiles cannot fill the SMs (cached per tile list)."""
        tok0 = self.b.request_offset * self.hw
        key = (np.asarray(q0_host).tobytes(), np.asarray(img_host).tobytes(), np.asarray(tok0).tobytes(),
               sm_count(), SPLITKV_MIN_BLOCKS, str(self.device))
        if key not in _SKV_CACHE:
            if len(_SKV_CACHE) > 64:
                _SKV_CACHE.clear()
            _SKV_CACHE[key] = splitkv_plan(q0_host, img_host, tok0, sm_count(), self.device)
        return _SKV_CACHE[key]

    def _splitkv_pairs(self, q0_host, img_host, min_base: int = 0):
        """Pair split-KV plan over the 256-query pair tiles of these 128-query tiles (every
        other one: a patch's 128-query tiles are consecutive and hw % 256 == 0)."""
        tok0 = self.b.request_offset * self.hw
        pq0, pimg = np.asarray(q0_host)[0::2], np.asarray(img_host)[0::2]
        key = ("pairs", pq0.tobytes(), pimg.tobytes(), np.asarray(tok0).tobytes(), sm_count(), SPLITKV_MIN_BLOCKS,
               min_base, str(self.device))
        if key not in _SKV_CACHE:
            if len(_SKV_CACHE) > 64:
                _SKV_CACHE.clear()
            _SKV_CACHE[key] = splitkv_plan_pairs(pq0, pimg, tok0, sm_count(), self.device, min_base)
        return _SKV_CACHE[key]

    def empty_cl(self, cp: int) -> torch.Tensor:
        return torch.empty((self.T, cp), dtype=BF16, device=self.device)

    def empty_nchw(self, c: int) -> torch.Tensor:
        return torch.empty((self.P, c, self.ps, self.ps), dtype=BF16, device=self.device)

    # layout conversions --------------------------------------------------
    def as_cl(self, a: Act) -> torch.Tensor:
        if a.layout == "cl":
            return a.t
        out = self.empty_cl(a.Cp)
        _lib.call("ps_to_cl", stream(), a.t.data_ptr(), self.P, a.C, self.ps, a.Cp, 0, None, None, 0, None, None,
                  C.c_float(0.0), out.data_ptr())
        return out

    def as_nchw(self, a: Act, resid: torch.Tensor | None = None) -> torch.Tensor:
        if a.layout == "nchw" and resid is None:
            return a.t
        src = self.as_cl(a) if a.layout == "nchw" else a.t
        out = self.empty_nchw(a.C)
        _lib.call("ps_from_cl", stream(), src.data_ptr(), self.P, a.C, self.ps, a.Cp,
                  None if resid is None else resid.data_ptr(), out.data_ptr())
        return out

    # GEMM ------------------------------------------------------------------
    def gemm(self, a, lda, b, n, k, bias, epi, out, ldo=0, out2=None, ldo2=0, n_split=0, resid=None, c_real=0,
             conv=False, cp_in=0, a_tiled=False, out_tiled=False, rows=None):
        g = _lib.GemmArgs()
        if rows is not None:
            g.m_map, g.m_count = rows[0].data_ptr(), rows[1]
            if len(rows) > 2:  # device-decided count (rows[1] is then an upper bound)
                g.m_count_dev = rows[2].data_ptr()
        g.a, g.lda, g.M = a.data_ptr(), lda, self.T
        g.a_mode, g.P, g.ps, g.Cp = (1 if conv else 2 if a_tiled else 0), self.P, self.ps, cp_in
        g.out_tiled = 1 if out_tiled else 0
        g.b, g.N, g.K = b.data_ptr(), n, k
        g.bias = None if bias is None else bias.data_ptr()
        g.epi, g.out, g.ldo = epi, out.data_ptr(), ldo
        g.out2, g.ldo2, g.n_split = (None if out2 is None else out2.data_ptr()), ldo2, n_split
        g.resid, g.c_real = (None if resid is None else resid.data_ptr()), c_real
        g.bn = 0  # library picks the tile width (gemm_pick_bn)
        _lib.check(_lib.load().ps_gemm(stream(), C.byref(g)))

    def gemm_out(self, a_cl, lda, w, n, k, bias, c_out, resid_nchw, gelu=False, a_tiled=False, rows=None):
        """Plain GEMM; NCHW output with residual when `resid_nchw` is given."""
        if resid_nchw is not None:
            out = self.empty_nchw(c_out)
            self.gemm(a_cl, lda, w, n, k, bias, 2, out, resid=resid_nchw, c_real=c_out, a_tiled=a_tiled, rows=rows)
            return Act("nchw", out, c_out)
        out = self.empty_cl(n)
        self.gemm(a_cl, lda, w, n, k, bias, 1 if gelu else 0, out, ldo=n, a_tiled=a_tiled, rows=rows)
        return Act("cl", out, c_out)

    # stages ---------------------------------------------------------------
    def gn_stats(self, x_nchw: torch.Tensor, c: int, dp: dict) -> torch.Tensor:
        g = dp["groups"]
        part = torch.empty((self.P, g, 2), dtype=torch.float32, device=self.device)
        if self.owned is not None:
            # owned patches here; the split images' other partials arrive from their owners
            _lib.call("ps_gn_partials_sub", stream(), x_nchw.data_ptr(), self.P, c, self.ps, g,
                      self.owned[0].data_ptr(), self.owned[1], part.data_ptr(), None)
            self.exch.gn(part, g)
        elif self.gn_live is not None:
            # device-decided compaction: the patches of images with a patch to recompute
            lp, n_ub, n_dev = self.gn_live
            _lib.call("ps_gn_partials_sub", stream(), x_nchw.data_ptr(), self.P, c, self.ps, g, lp.data_ptr(), n_ub,
                      part.data_ptr(), n_dev.data_ptr())
        else:
            _lib.call("ps_gn_partials", stream(), x_nchw.data_ptr(), self.P, c, self.ps, g, part.data_ptr())
        stats = torch.empty((self.b.n_requests, g, 2), dtype=torch.float32, device=self.device)
        _lib.call("ps_gn_finalize", stream(), part.data_ptr(), self.dev["request_offset"].data_ptr(),
                  self.b.n_requests, g, (c // g) * self.hw, C.c_float(dp["eps"]), stats.data_ptr())
        return stats

    def group_norm(self, a: Act, prm, frames: bool):
        dp = device_params(prm, a.C)
        x = self.as_nchw(a)
        stats = self.gn_stats(x, a.C, dp)
        if frames:
            return None, self._frames(x, a.C, a.Cp, 1, stats, dp["groups"], dp["gamma"], dp["beta"])
        out = self.empty_cl(a.Cp)
        _lib.call("ps_to_cl", stream(), x.data_ptr(), self.P, a.C, self.ps, a.Cp, 1, stats.data_ptr(),
                  self.dev["request_index"].data_ptr(), dp["groups"], dp["gamma"].data_ptr(), dp["beta"].data_ptr(),
                  C.c_float(dp["eps"]), out.data_ptr())
        return Act("cl", out, a.C), None

    def _frames(self, x, c, cp, mode, stats, groups, gamma, beta) -> torch.Tensor:
        fr = torch.empty((self.P, self.ps + 2, self.ps + 2, cp), dtype=BF16, device=self.device)
        args = (x.data_ptr(), self.P, c, self.ps, cp, mode, None if stats is None else stats.data_ptr(),
                self.dev["request_index"].data_ptr(), self.dev["neighbors"].data_ptr(), groups,
                None if gamma is None else gamma.data_ptr(), None if beta is None else beta.data_ptr())
        if self.owned is not None:
            # the stencil rows / columns of neighbours owned by other GPUs land in their ghost slots of x
            self.exch.halo(x, c)
            _lib.call("ps_frames_cl_sub", stream(), *args, self.owned[0].data_ptr(), self.owned[1], fr.data_ptr(),
                      None)
        elif self.gn_live is not None:
            lp, n_ub, n_dev = self.gn_live
            _lib.call("ps_frames_cl_sub", stream(), *args, lp.data_ptr(), n_ub, fr.data_ptr(), n_dev.data_ptr())
        else:
            _lib.call("ps_frames_cl", stream(), *args, fr.data_ptr())
        return fr

    def frames_of(self, a: Act) -> torch.Tensor:
        return self._frames(self.as_nchw(a), a.C, a.Cp, 0, None, 1, None, None)

    def conv(self, a: Act, prm, frames, resid):
        dp = device_params(prm, a.C)
        if dp["k"] == 3:
            if frames is None:
                frames = self.frames_of(a)
                _launch("halo_exchange")
            if resid is not None:
                out = self.empty_nchw(dp["c_out"])
                self.gemm(frames, 0, dp["w"], dp["cp_out"], 9 * dp["cp_in"], dp["b"], 2, out, resid=resid,
                          c_real=dp["c_out"], conv=True, cp_in=dp["cp_in"], rows=self.rows)
                return Act("nchw", out, dp["c_out"])
            out = self.empty_cl(dp["cp_out"])
            self.gemm(frames, 0, dp["w"], dp["cp_out"], 9 * dp["cp_in"], dp["b"], 0, out, ldo=dp["cp_out"],
                      conv=True, cp_in=dp["cp_in"], rows=self.rows)
            return Act("cl", out, dp["c_out"])
        x = self.as_cl(a)
        return self.gemm_out(x, a.Cp, dp["w"], dp["cp_out"], dp["cp_in"], dp["b"], dp["c_out"], resid,
                             rows=self.rows)

    def linear(self, a: Act, prm, resid):
        dp = device_params(prm, a.C)
        x = self.as_cl(a)
        return self.gemm_out(x, a.Cp, dp["w"], dp["cp_out"], dp["cp_in"], dp["b"], dp["c_out"], resid,
                             rows=self.rows)

    def feed_forward(self, a: Act, prm, resid):
        dp = device_params(prm, a.C)
        x = self.as_cl(a)
        if (resid is not None and FF_FUSED and dp["cp"] in (128, 192, 256, 320) and dp["hp"] % 128 == 0
                and self.hw % 128 == 0 and self.T % 128 == 0):
            # one fused kernel: the hidden activations stay on chip (ffused.cu)
            out = self.empty_nchw(dp["c_out"])
            rows = self.rows
            _lib.call("ps_feed_forward", stream(), x.data_ptr(), self.T, dp["cp"], dp["w1"].data_ptr(),
                      dp["b1"].data_ptr(), dp["w2"].data_ptr(), dp["b2"].data_ptr(), dp["hp"], dp["c_out"], self.ps,
                      resid.data_ptr(), out.data_ptr(), None if rows is None else rows[0].data_ptr(),
                      0 if rows is None else rows[1], None if rows is None or len(rows) < 3 else rows[2].data_ptr())
            return Act("nchw", out, dp["c_out"])
        # hidden activations in 128x64 tile-major order: the second GEMM streams
        # each of its A boxes as one contiguous 16 KB block from HBM
        h = torch.empty((round_up(self.T, 128), dp["hp"]), dtype=BF16, device=self.device)
        self.gemm(x, a.Cp, dp["w1"], dp["hp"], dp["cp"], dp["b1"], 1, h, ldo=dp["hp"], out_tiled=True,
                  rows=self.rows)
        return self.gemm_out(h, dp["hp"], dp["w2"], dp["cp"], dp["hp"], dp["b2"], dp["c_out"], resid, a_tiled=True,
                             rows=self.rows)

    def layer_norm(self, a: Act, prm):
        dp = device_params(prm, a.C)
        x = self.as_nchw(a)
        out = self.empty_cl(a.Cp)
        _lib.call("ps_to_cl", stream(), x.data_ptr(), self.P, a.C, self.ps, a.Cp, 2, None, None, 0,
                  dp["gamma"].data_ptr(), dp["beta"].data_ptr(), C.c_float(dp["eps"]), out.data_ptr())
        return Act("cl", out, a.C)

    def attention(self, a: Act, prm, resid):
        dp = device_params(prm, a.C)
        x = self.as_cl(a)
        d, dpp = dp["d"], dp["dp"]
        peer = self.owned is not None and getattr(self.exch, "peer_kv", False)
        if peer:
            # persistent peer-visible operand buffers: peers read our K / V^T in place
            par, (qk, vt, ldv, _, _, _) = self.exch.kv_buffers(dpp, self.T, self.device)
        else:
            qk = torch.empty((self.T, 2 * dpp), dtype=BF16, device=self.device)
            ldv = round_up(self.T, 64)
            vt = torch.empty((dpp, ldv), dtype=BF16, device=self.device)
        self.gemm(x, a.Cp, dp["wqkv"], 3 * dpp, dpp, None, 3, qk, ldo=2 * dpp, out2=vt, ldo2=ldv, n_split=2 * dpp,
                  rows=self.rows_live)
        finish = None
        if peer:
            self.exch.kv_sync()
            kb_src, kb_row, maps = self.exch.kv_tables(dpp, par)
        elif self.owned is not None and OVERLAP_KV and self.attn_tiles is not None:
            # start the K / V^T all-gather; attention over keys already here runs meanwhile
            finish = self.exch.kv_start(qk, vt, ldv, dpp)
        elif self.owned is not None:
            self.exch.kv(qk, vt, ldv, dpp)  # K rows / V^T columns of split images from their owners
        o = self.empty_cl(dpp)
        timer = ATTN_TIMER
        if timer is not None:
            ext = torch.cuda.is_current_stream_capturing()  # event nodes inside a captured graph
            ev = (torch.cuda.Event(enable_timing=True, external=ext), torch.cuda.Event(enable_timing=True, external=ext))
            ev[0].record()
        host = None
        if self.attn_tiles is not None:
            tq0, timg, nt, pairs = self.attn_tiles[:4]
            host = self.attn_tiles[4:]
        elif USE_PAIRS and self.hw % 256 == 0:
            tq0, timg, nt, pairs = self.dev["pair_q0"], self.dev["pair_img"], self.dev["n_pairs"], True
            host = (self.dev["tile_q0_host"], self.dev["tile_img_host"])
        else:
            tq0, timg, nt, pairs = self.dev["tile_q0"], self.dev["tile_img"], self.dev["n_tiles"], False
            host = (self.dev["tile_q0_host"], self.dev["tile_img_host"])
        # split-KV on the split-image path (few long query tiles per GPU); single-GPU batches keep
        # the one-pass kernels so compacted and full runs stay bit-identical
        use_skv = SPLITKV and (self.owned is not None or SPLITKV_ALL)
        skv = pskv = None
        if host is not None and host[0] is None:
            host = None  # device-decided tile lists (no host copy): one-pass kernels
        if host is not None and SPLITKV and pairs and SPLITKV_PAIRS and not peer and finish is None:
            # single-GPU batches: only long attentions (SPLITKV_SINGLE_MIN_BLOCKS)
            min_base = 0 if use_skv else SPLITKV_SINGLE_MIN_BLOCKS
            pskv = self._splitkv_pairs(host[0], host[1], min_base=min_base)
        elif host is not None and use_skv:
            skv = self._splitkv(host[0], host[1])
        if pskv is not None:
            # few long pair tiles for the SM pairs: keys split over several pairs, partials merged
            kb0, nkb, s0, s1, n_rows, cq0, cslot0, cns, cimg, n_q, pq0, pimg, n_slots = pskv
            part_o = torch.empty((n_slots, 128, dpp), dtype=torch.float32, device=self.device)
            part_ml = torch.empty((n_slots, 128, 2), dtype=torch.float32, device=self.device)
            _lib.call("ps_attention_pairs_splitkv", stream(), qk.data_ptr(), vt.data_ptr(), ldv, self.T, dpp, d,
                      self.dev["img_tok0"].data_ptr(), pq0.data_ptr(), pimg.data_ptr(), kb0.data_ptr(),
                      nkb.data_ptr(), s0.data_ptr(), s1.data_ptr(), n_rows, part_o.data_ptr(), part_ml.data_ptr(),
                      o.data_ptr())
            _lib.call("ps_attention_combine", stream(), part_o.data_ptr(), part_ml.data_ptr(), cq0.data_ptr(),
                      cslot0.data_ptr(), cns.data_ptr(), cimg.data_ptr(), self.dev["img_tok0"].data_ptr(), n_q, dpp,
                      o.data_ptr())
        elif finish is not None:
            self._attention_overlapped(qk, vt, ldv, dpp, d, host, finish, o)
        elif peer and skv is None:
            # one-pass kernel over 128-query tiles, remote key blocks read from their owners
            q0d, imgd = self._tiles128(host)
            _lib.call("ps_attention_peer", stream(), qk.data_ptr(), vt.data_ptr(), ldv, self.T, dpp, d,
                      self.dev["img_tok0"].data_ptr(), q0d.data_ptr(), imgd.data_ptr(), None, None, None,
                      len(host[0]), None, None, kb_src.data_ptr(), kb_row.data_ptr(), maps.data_ptr(), o.data_ptr())
        elif skv is not None:
            # few query tiles for the SMs: keys split over several CTAs per tile, partials merged
            kb0, nkb, slot, n_split_tiles, cq0, cslot0, cns, cimg, n_q = skv[:9]
            part_o = torch.empty((n_split_tiles, 128, dpp), dtype=torch.float32, device=self.device)
            part_ml = torch.empty((n_split_tiles, 128, 2), dtype=torch.float32, device=self.device)
            if peer:
                _lib.call("ps_attention_peer", stream(), qk.data_ptr(), vt.data_ptr(), ldv, self.T, dpp, d,
                          self.dev["img_tok0"].data_ptr(), skv_q0(skv).data_ptr(), skv_img(skv).data_ptr(),
                          kb0.data_ptr(), nkb.data_ptr(), slot.data_ptr(), n_split_tiles, part_o.data_ptr(),
                          part_ml.data_ptr(), kb_src.data_ptr(), kb_row.data_ptr(), maps.data_ptr(), o.data_ptr())
            else:
                _lib.call("ps_attention_splitkv", stream(), qk.data_ptr(), vt.data_ptr(), ldv, self.T, dpp, d,
                          self.dev["img_tok0"].data_ptr(), skv_q0(skv).data_ptr(), skv_img(skv).data_ptr(),
                          kb0.data_ptr(), nkb.data_ptr(), slot.data_ptr(), n_split_tiles, part_o.data_ptr(),
                          part_ml.data_ptr(), o.data_ptr())
            _lib.call("ps_attention_combine", stream(), part_o.data_ptr(), part_ml.data_ptr(), cq0.data_ptr(),
                      cslot0.data_ptr(), cns.data_ptr(), cimg.data_ptr(), self.dev["img_tok0"].data_ptr(), n_q, dpp,
                      o.data_ptr())
        elif pairs:
            n_dev = self.attn_tiles[6] if self.attn_tiles is not None and len(self.attn_tiles) > 6 else None
            _lib.call("ps_attention_pairs", stream(), qk.data_ptr(), vt.data_ptr(), ldv, self.T, dpp, d,
                      self.dev["img_tok0"].data_ptr(), tq0.data_ptr(), timg.data_ptr(), nt, o.data_ptr(),
                      None if n_dev is None else n_dev.data_ptr())
        else:
            _lib.call("ps_attention", stream(), qk.data_ptr(), vt.data_ptr(), ldv, self.T, dpp, d,
                      self.dev["img_tok0"].data_ptr(), tq0.data_ptr(), timg.data_ptr(), nt, o.data_ptr())
        if timer is not None:
            ev[1].record()
            timer.append(ev)
        return self.gemm_out(o, dpp, dp["wo"], dpp, dpp, None, d, resid, rows=self.rows)


# ------------------------------------------------------- public operators


def exchange_halos(batch: CSPBatch, data) -> torch.Tensor:
    """(P, C, ps+2, ps+2) frames: patch pixels plus a 1-pixel neighbour ring (patched.py:57-89)."""
    data = _check_data(batch, data, finite=False)  # a pure copy: the reference does not validate values
    if data.dtype not in (torch.float32, BF16, torch.float64):
        data = data.to(torch.float32)
    p_n, c, ps = data.shape[0], data.shape[1], batch.patch_size
    out = torch.empty((p_n, c, ps + 2, ps + 2), dtype=data.dtype, device=data.device)
    code = {torch.float32: _lib.DTYPE_F32, BF16: _lib.DTYPE_BF16, torch.float64: _lib.DTYPE_F64}[data.dtype]
    _lib.call("ps_halo_frames_nchw", stream(), data.data_ptr(), code,
              batch.device()["neighbors"].data_ptr(), p_n, c, ps, out.data_ptr())
    return out


def _frames_nchw_to_cl(ctx: Ctx, frames: torch.Tensor, c: int) -> torch.Tensor:
    f = _bf16_nchw(frames)
    cp = round_up(c, 64)
    out = torch.empty((ctx.P, ctx.ps + 2, ctx.ps + 2, cp), dtype=BF16, device=ctx.device)
    _lib.call("ps_to_cl", stream(), f.data_ptr(), ctx.P, c, ctx.ps + 2, cp, 0, None, None, 0, None, None,
              C.c_float(0.0), out.data_ptr())
    return out


def patched_conv(batch: CSPBatch, data, p, frames=None) -> torch.Tensor:
    """Convolution over patches; k=3 reads context from halo frames (patched.py:92-113)."""
    data = _check_data(batch, data)
    c = data.shape[1]
    k = int(np.asarray(p.weights).shape[2])
    ctx = Ctx(batch)
    a = Act("nchw", _bf16_nchw(data), c)
    fr = None
    if k == 3 and frames is not None:
        frames = to_device(frames)
        if tuple(frames.shape) != (batch.n_patches, c, batch.patch_size + 2, batch.patch_size + 2):
            raise InputError(f"bad halo frame shape {tuple(frames.shape)}")
        fr = _frames_nchw_to_cl(ctx, frames, c)
    out = ctx.conv(a, p, fr, None)
    _launch("conv")
    return ctx.as_nchw(out)


def stitched_group_norm(batch: CSPBatch, data, p, emit_halos: bool = False):
    """Group norm pooled over each request's patches (patched.py:116-144)."""
    data = _check_data(batch, data)
    c = data.shape[1]
    if c % p.groups != 0:
        raise InputError(f"groups={p.groups} does not divide channels={c}")
    ctx = Ctx(batch)
    out_cl, _ = ctx.group_norm(Act("nchw", _bf16_nchw(data), c), p, frames=False)
    out = ctx.as_nchw(out_cl)
    _launch("group_norm")
    if emit_halos:
        return out, exchange_halos(batch, out)
    return out


def patched_layer_norm(batch: CSPBatch, data, p) -> torch.Tensor:
    """Per-position layer norm (patched.py:147-151)."""
    data = _check_data(batch, data)
    ctx = Ctx(batch)
    out = ctx.as_nchw(ctx.layer_norm(Act("nchw", _bf16_nchw(data), data.shape[1]), p))
    _launch("layer_norm")
    return out


def patched_self_attention(batch: CSPBatch, data, p) -> torch.Tensor:
    """Global self-attention per image (patched.py:154-176)."""
    data = _check_data(batch, data)
    ctx = Ctx(batch)
    out = ctx.as_nchw(ctx.attention(Act("nchw", _bf16_nchw(data), data.shape[1]), p, None))
    _launch("attention")
    return out


def feed_forward(batch: CSPBatch, data, p) -> torch.Tensor:
    """Pixel-wise MLP (kernels.py:124-127) over the patch array."""
    data = _check_data(batch, data)
    ctx = Ctx(batch)
    return ctx.as_nchw(ctx.feed_forward(Act("nchw", _bf16_nchw(data), data.shape[1]), p, None))


_GEMM_STAGES = ("conv", "feed_forward", "linear", "attention")


def run_block(batch: CSPBatch, x, ops) -> torch.Tensor:
    """Execute one block of (kind, params) stages (patched.py:179-221); returns NCHW bf16."""
    x = _check_data(batch, x)
    return _run_ops(Ctx(batch), x, ops)


def run_block_active(batch: CSPBatch, x, ops, active) -> torch.Tensor:
    """run_block whose outputs are only needed for the `active` patches.

    Active-patch compaction: pixel-wise stages and attention query
    rows run on the active patches only; the context stages (conv3 halo
    neighbours, attention keys/values) run on every patch of an image that has at
    least one active patch.  Rows of inactive patches in the result are
    unspecified (the cache splices their cached outputs, patched.py:246).  The
    active rows are bit-identical to run_block's.
    """
    x = _check_data(batch, x, finite=False)  # inactive rows may be unspecified
    active = np.asarray(active, dtype=bool)
    ctx = Ctx(batch)
    if ctx.hw % 128 or active.all():
        return _run_ops(ctx, x, ops)  # tiles would span patches: no compaction
    act = np.flatnonzero(active)
    live_img = np.unique(batch.request_index[act])
    live = np.flatnonzero(np.isin(batch.request_index, live_img))
    ctx.rows_live, ctx.rows_act = _row_tiles(ctx, live), _row_tiles(ctx, act)
    ctx.attn_live, ctx.attn_act = _attn_tiles(ctx, live), _attn_tiles(ctx, act)
    return _run_ops(ctx, x, ops)


def device_compaction_ok(batch: CSPBatch) -> bool:
    """run_block_masked's kernels cover this geometry: 256-query attention pairs per patch,
    8-pixel stitcher units, 8-channel groups."""
    ps_ = batch.patch_size
    return USE_PAIRS and (ps_ * ps_) % 256 == 0 and ps_ % 8 == 0 and batch.data.shape[1] % 8 == 0


def run_block_masked(batch: CSPBatch, x, ops, mask: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """run_block_active with the reuse decision left on the device: `mask` is the cache's
    DEVICE bool mask (True = reused).  ps_compact_lists turns it into the GEMM row tiles,
    attention query tiles and GroupNorm / stitcher patch lists of the active and live sets,
    and every kernel reads its own work count from device memory -- no host round trip, so
    the host enqueues the next block while this one runs.  The active rows are bit-identical
    to run_block_active's (same kernels and tile contents; only the tile counts move).
    Returns (output, counts) with counts the device int32 [6] of ps_compact_lists."""
    x = _check_data(batch, x, finite=False)  # inactive rows may be unspecified
    if not device_compaction_ok(batch):
        raise InputError("run_block_masked: geometry not covered (see device_compaction_ok)")
    m = mask.to(device=require_cuda(), dtype=torch.bool).contiguous()
    if tuple(m.shape) != (batch.n_patches,):
        raise InputError(f"mask must be ({batch.n_patches},) bool")
    ctx, counts = masked_context(batch, m)
    return _run_ops(ctx, x, ops), counts


def masked_context(batch: CSPBatch, mask: torch.Tensor) -> tuple["Ctx", torch.Tensor]:
    """The Ctx of run_block_masked (device-built compaction lists from the DEVICE mask) and
    its counts; ctx.gn_live lists the patches whose block input is read."""
    ctx = Ctx(batch)
    return ctx, _device_lists(ctx, mask)


def run_block_ctx(ctx: "Ctx", x, ops) -> torch.Tensor:
    """The block stages of `ops` on a prepared Ctx (masked_context)."""
    return _run_ops(ctx, _check_data(ctx.b, x, finite=False), ops)  # rows off the live set: unspecified


def _attn_order(ctx: "Ctx") -> torch.Tensor:
    """Device copy of the attention patch order of _attn_tiles (longest images first, stable)."""
    b = ctx.b
    sizes = b.request_offset[1:] - b.request_offset[:-1]
    key = ("order", np.asarray(b.request_index).tobytes(), np.asarray(sizes).tobytes(), str(ctx.device))
    if key not in _SKV_CACHE:
        order = sorted(range(ctx.P), key=lambda p: -int(sizes[b.request_index[p]]))
        _SKV_CACHE[key] = torch.as_tensor(np.asarray(order, np.int32), device=ctx.device)
    return _SKV_CACHE[key]


def _device_lists(ctx: "Ctx", mask: torch.Tensor) -> torch.Tensor:
    P, R, hw = ctx.P, ctx.b.n_requests, ctx.hw
    tpp, tq = hw // 128, 256
    qpp = hw // tq
    sizes = [R, P * tpp, P * tpp, P, P * qpp, P * qpp, P * qpp, P * qpp, 6]
    buf = torch.empty(sum(sizes), dtype=torch.int32, device=ctx.device)
    live, rows_act, rows_live, live_p, aq_a, ai_a, aq_l, ai_l, counts = torch.split(buf, sizes)
    _lib.call("ps_compact_lists", stream(), mask.view(torch.uint8).data_ptr(), P, ctx.dev["request_index"].data_ptr(),
              R, _attn_order(ctx).data_ptr(), tpp, qpp, tq, hw, live.data_ptr(), rows_act.data_ptr(),
              rows_live.data_ptr(), live_p.data_ptr(), aq_a.data_ptr(), ai_a.data_ptr(), aq_l.data_ptr(),
              ai_l.data_ptr(), counts.data_ptr())
    ctx.rows_act = (rows_act, P * tpp, counts[0:1])
    ctx.rows_live = (rows_live, P * tpp, counts[1:2])
    ctx.attn_act = (aq_a, ai_a, P * qpp, True, None, None, counts[2:3])
    ctx.attn_live = (aq_l, ai_l, P * qpp, True, None, None, counts[3:4])
    ctx.gn_live = (live_p, P, counts[5:6])
    return counts


def _row_tiles(ctx: "Ctx", pats: np.ndarray):
    """Device list of the 128-row GEMM tiles of these patches (ps*ps % 128 == 0)."""
    tpp = ctx.hw // 128
    m = (np.asarray(pats, dtype=np.int64)[:, None] * tpp + np.arange(tpp)[None, :]).ravel().astype(np.int32)
    return torch.as_tensor(m, device=ctx.device), int(m.size)


_SMS = None


def sm_count() -> int:
    global _SMS
    if _SMS is None:
        _SMS = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return _SMS


# fused FF1 + GELU + FF2 + residual on CTA pairs (ffused.cu); PS_FF_FUSED=0 -> two GEMMs
FF_FUSED = os.environ.get("PS_FF_FUSED", "1") == "1"
# split-KV planning (splitkv_plan); PS_SPLITKV=0 disables it
SPLITKV = os.environ.get("PS_SPLITKV", "1") != "0"
SPLITKV_ALL = os.environ.get("PS_SPLITKV_ALL", "0") == "1"  # also outside the split-image path
# split-image path: overlap the K / V^T all-gather with attention over the keys already local
# (opt-in: at config 5 the second phase costs more than the ~0.1 ms/block gather it hides)
OVERLAP_KV = os.environ.get("PS_OVERLAP_KV", "0") == "1"
_SKV_CACHE: dict = {}
SPLITKV_MIN_BLOCKS = 8  # key blocks (of 128) per split
# split-KV on the persistent CTA-pair kernel when the query tiles pair up (PS_SPLITKV_PAIRS=0: the
# single-CTA split-KV kernel)
SPLITKV_PAIRS = os.environ.get("PS_SPLITKV_PAIRS", "1") != "0"
# single-GPU batches (no split images) use the pair split-KV only when the longest-first makespan
# of the unsplit pair tiles is at least this many key blocks: long attentions (config 5's 2048 px
# image: 4 waves of 512-block tiles, 29.8 -> ~27.5 ms/step) gain more from a balanced last wave
# than the partials cost; short ones (config 2, every test shape) keep the one-pass kernel, so
# their compacted and full runs stay bit-identical
SPLITKV_SINGLE_MIN_BLOCKS = int(os.environ.get("PS_SPLITKV_SINGLE_MIN_BLOCKS", "1536"))


def _lpt_makespan(pieces, sms: int) -> int:
    """Greedy longest-first makespan of `pieces` (key blocks) on `sms` SMs (one CTA per SM)."""
    import heapq
    loads = [0] * min(sms, max(1, len(pieces)))
    heapq.heapify(loads)
    for w in sorted(pieces, reverse=True):
        heapq.heappush(loads, heapq.heappop(loads) + w)
    return max(loads)


def splitkv_plan(q0_host, img_host, img_tok0_host, sms: int, device):
    """Split long query tiles' keys over several CTAs when that shortens the kernel.

    The attention kernel is one CTA per (query tile, key range); a tile costs its
    number of 128-key blocks.  When few long tiles (a large image split across GPUs)
    cannot keep `sms` SMs busy, every tile longer than a target is cut into equal key
    ranges; the target is chosen to minimise the simulated longest-first makespan plus
    a small charge per partial (fp32 O write + combine read).  Returns None when no
    split helps; else device arrays for ps_attention_splitkv (kb0, nkb, slot per split
    tile, longest first) and ps_attention_combine (q0, first slot, splits, image per
    query tile), plus counts and the split tiles' (q0, image)."""
    n = len(q0_host)
    if n == 0:
        return None
    nkb_img = [(int(img_tok0_host[i + 1] - img_tok0_host[i]) + 127) // 128 for i in range(len(img_tok0_host) - 1)]
    units = [nkb_img[int(i)] for i in img_host]
    base = _lpt_makespan(units, sms)
    best, best_cost = None, base
    for k in range(2, 17):
        target = max(SPLITKV_MIN_BLOCKS, -(-max(units) // k))
        pieces, n_part = [], 0
        for nb in units:
            ns = -(-nb // target) if nb > target else 1
            q, r = divmod(nb, ns)
            pieces.extend([q + 1] * r + [q] * (ns - r))
            n_part += ns if ns > 1 else 0
        # a partial costs its fp32 O write + combine read (~320 KB/128 rows at Dp=320) ~ 4 key blocks of SM time
        cost = _lpt_makespan(pieces, sms) + 4.0 * n_part / max(1, sms)
        if cost < 0.97 * best_cost:
            best, best_cost = target, cost
    if best is None:
        return None
    rows = []  # (q0, img, kb0, nkb, slot)
    cq0, cs0, cns, cimg = [], [], [], []
    slot = 0
    for q0, img, nb in zip(q0_host, img_host, units):
        ns = -(-nb // best) if nb > best else 1
        q, r = divmod(nb, ns)
        cq0.append(int(q0)); cs0.append(slot); cns.append(ns); cimg.append(int(img))
        k = 0
        for s_ in range(ns):
            m = q + (1 if s_ < r else 0)
            rows.append((int(q0), int(img), k, m, slot))
            k += m
            slot += 1
    rows.sort(key=lambda r_: -r_[3])  # longest ranges first
    t = lambda v: torch.as_tensor(np.asarray(v, dtype=np.int32), device=device)
    cols = list(zip(*rows))
    return (t(cols[2]), t(cols[3]), t(cols[4]), len(rows), t(cq0), t(cs0), t(cns), t(cimg), len(cq0),
            t(cols[0]), t(cols[1]))


def splitkv_plan_pairs(q0_host, img_host, img_tok0_host, sms: int, device, min_base: int = 0):
    """splitkv_plan for the persistent CTA-pair kernel (ps_attention_pairs_splitkv): units are
    256-query pair tiles (q0_host / img_host) on sms // 2 SM pairs.  A pair tile whose keys are
    not split writes bf16 O directly (slots -1); a split one writes its two 128-row halves to
    slots [base, base + ns) and [base + ns, base + 2 ns), merged by ps_attention_combine over
    128-query tiles.  Returns None when no split helps; else device arrays (kb0, nkb, slot0,
    slot1 per pair tile, longest first), the number of pair tiles, the combine lists (q0, first
    slot, splits, image per 128-query tile), their count, the pair tiles' (q0, image), and the
    number of partial slots."""
    n = len(q0_host)
    if n == 0:
        return None
    pairs = max(1, sms // 2)
    nkb_img = [(int(img_tok0_host[i + 1] - img_tok0_host[i]) + 127) // 128 for i in range(len(img_tok0_host) - 1)]
    units = [nkb_img[int(i)] for i in img_host]
    base = _lpt_makespan(units, pairs)
    if base < min_base:
        return None
    best, best_cost = None, base
    for k in range(2, 17):
        target = max(SPLITKV_MIN_BLOCKS, -(-max(units) // k))
        pieces, n_part = [], 0
        for nb in units:
            ns = -(-nb // target) if nb > target else 1
            q, r = divmod(nb, ns)
            pieces.extend([q + 1] * r + [q] * (ns - r))
            n_part += ns if ns > 1 else 0
        # a pair partial: two fp32 halves written + read by the combine ~ 4 key blocks of pair time
        cost = _lpt_makespan(pieces, pairs) + 4.0 * n_part / pairs
        if cost < 0.97 * best_cost:
            best, best_cost = target, cost
    if best is None:
        return None
    rows = []  # (q0, img, kb0, nkb, slot0, slot1)
    cq0, cs0, cns, cimg = [], [], [], []
    slot = 0
    for q0, img, nb in zip(q0_host, img_host, units):
        ns = -(-nb // best) if nb > best else 1
        if ns == 1:
            rows.append((int(q0), int(img), 0, nb, -1, -1))
            continue
        q, r = divmod(nb, ns)
        for h in range(2):
            cq0.append(int(q0) + 128 * h); cs0.append(slot + h * ns); cns.append(ns); cimg.append(int(img))
        k = 0
        for s_ in range(ns):
            m = q + (1 if s_ < r else 0)
            rows.append((int(q0), int(img), k, m, slot + s_, slot + ns + s_))
            k += m
        slot += 2 * ns
    if not cq0:
        return None
    rows.sort(key=lambda r_: -r_[3])  # longest ranges first
    t = lambda v: torch.as_tensor(np.asarray(v, dtype=np.int32), device=device)
    cols = list(zip(*rows))
    return (t(cols[2]), t(cols[3]), t(cols[4]), t(cols[5]), len(rows), t(cq0), t(cs0), t(cns), t(cimg), len(cq0),
            t(cols[0]), t(cols[1]), slot)


def overlap_plan(q0_host, img_host, req_off, hw: int, owned, sms: int, device):
    """Pieces of the two attention phases of a split-image rank.

    Per 128-query tile: an image held whole -> one piece over all its keys (phase A); an
    image split across GPUs -> the key blocks of this rank's patches (phase A, contiguous)
    and the remote ranges before / after them (phase B).  Pieces longer than the SM-balance
    target are cut further.  A tile with a single piece writes its output directly; the
    others write partials merged by ps_attention_combine."""
    owned = set(int(x) for x in owned)
    tpb = max(1, hw // 128)  # key blocks per patch
    segs = []  # per tile: list of (kb0, nkb, phase)
    for q0, img in zip(q0_host, img_host):
        img = int(img)
        p0, p1 = int(req_off[img]), int(req_off[img + 1])
        nkb = (p1 - p0) * hw // 128
        mine = [p for p in range(p0, p1) if p in owned]
        if len(mine) == p1 - p0:
            segs.append([(0, nkb, 0)])
            continue
        a, b = (mine[0] - p0) * tpb, (mine[-1] + 1 - p0) * tpb
        tile = [(a, b - a, 0)]
        if a > 0:
            tile.append((0, a, 1))
        if b < nkb:
            tile.append((b, nkb - b, 1))
        segs.append(tile)
    total = sum(n for t in segs for _, n, _ in t)
    target = max(SPLITKV_MIN_BLOCKS, -(-total // max(1, 2 * sms)))
    rows = {0: [], 1: []}
    cq0, cs0, cns, cimg = [], [], [], []
    slot = 0
    for (q0, img), tile in zip(zip(q0_host, img_host), segs):
        pieces = []
        for k0, n, ph in tile:
            ns = -(-n // target) if n > target else 1
            q, r = divmod(n, ns)
            k = k0
            for i in range(ns):
                m = q + (1 if i < r else 0)
                pieces.append((k, m, ph))
                k += m
        if len(pieces) == 1:
            k, m, ph = pieces[0]
            rows[ph].append((int(q0), int(img), k, m, -1))
            continue
        cq0.append(int(q0)); cs0.append(slot); cns.append(len(pieces)); cimg.append(int(img))
        for k, m, ph in pieces:
            rows[ph].append((int(q0), int(img), k, m, slot))
            slot += 1
    t = lambda v: torch.as_tensor(np.asarray(v, dtype=np.int32), device=device)

    def launch_list(rs):
        rs = sorted(rs, key=lambda r_: -r_[3])
        if not rs:
            return (None, None, None, None, None, 0)
        c = list(zip(*rs))
        return (t(c[0]), t(c[1]), t(c[2]), t(c[3]), t(c[4]), len(rs))
    comb = (t(cq0), t(cs0), t(cns), t(cimg), len(cq0)) if cq0 else (None, None, None, None, 0)
    return launch_list(rows[0]), launch_list(rows[1]), slot, comb


def skv_q0(plan):
    return plan[9]


def skv_img(plan):
    return plan[10]


def _attn_tiles(ctx: "Ctx", pats: np.ndarray):
    """Attention query tiles (q0, image, n, pairs, q0 host, image host) of these patches,
    longest images first."""
    batch = ctx.b
    sizes = batch.request_offset[1:] - batch.request_offset[:-1]
    pairs = USE_PAIRS and ctx.hw % 256 == 0
    tq = 256 if pairs else 128
    order = sorted(np.asarray(pats).tolist(), key=lambda p: -int(sizes[batch.request_index[p]]))
    n = ctx.hw // tq
    q0 = [p * ctx.hw + tq * j for p in order for j in range(n)]
    img = [int(batch.request_index[p]) for p in order for _ in range(n)]
    # 128-query tiles on the host for the split-KV planner (which runs the single-CTA kernel)
    n1 = ctx.hw // 128
    q0h = np.asarray([p * ctx.hw + 128 * j for p in order for j in range(n1)], np.int64)
    imgh = np.asarray([int(batch.request_index[p]) for p in order for _ in range(n1)], np.int64)
    return (torch.as_tensor(np.asarray(q0, np.int32), device=ctx.device),
            torch.as_tensor(np.asarray(img, np.int32), device=ctx.device), len(q0), pairs, q0h, imgh)


def shard_context(batch: CSPBatch, shard, exch) -> "Ctx":
    """Ctx of one rank of the split-image path (patchshard.py): every stage computes the
    owned patches only; context owned by other ranks arrives through `exch`."""
    ctx = Ctx(batch)
    if batch.n_patches != shard.n_patches:
        raise InputError(f"batch has {batch.n_patches} patches, shard expects {shard.n_patches}")
    if ctx.hw % 128:
        raise InputError(f"split-image path needs patch_size^2 % 128 == 0, got patch {ctx.ps}")
    owned = np.asarray(shard.owned, dtype=np.int64)
    ctx.owned = (torch.as_tensor(owned.astype(np.int32), device=ctx.device), int(owned.size))
    ctx.owned_host = owned
    ctx.exch = exch
    ctx.rows_live = ctx.rows_act = _row_tiles(ctx, owned)
    ctx.attn_live = ctx.attn_act = _attn_tiles(ctx, owned)
    return ctx


def run_block_shard(batch: CSPBatch, x, ops, shard, exch, ctx: "Ctx | None" = None) -> torch.Tensor:
    """run_block for one rank of the split-image path; rows of ghost patches are unspecified."""
    x = _check_data(batch, x, finite=False)  # ghost rows are unspecified by contract
    return _run_ops(ctx or shard_context(batch, shard, exch), x, ops)


def _run_ops(ctx: "Ctx", x: torch.Tensor, ops) -> torch.Tensor:
    for kind, _ in ops:
        if kind not in ("group_norm", "layer_norm", "conv", "attention", "feed_forward", "linear", "residual"):
            raise InputError(f"unknown block stage {kind!r}")
    block_in = _bf16_nchw(x)
    cur = Act("nchw", block_in, x.shape[1])
    frames = None
    fused_residual = False

    def is_context(op):  # stages whose outputs depend on other patches of the image
        k, prm = op
        return k in ("group_norm", "attention") or (k == "conv" and int(np.asarray(prm.weights).shape[2]) == 3)

    for i, (kind, prm) in enumerate(ops):
        nxt = ops[i + 1][0] if i + 1 < len(ops) else None
        # compaction: a stage feeding a later context stage must produce every live-image row
        ctx_after = any(is_context(o) for o in ops[i + 1:])
        ctx.rows = ctx.rows_live if ctx_after else ctx.rows_act
        ctx.attn_tiles = ctx.attn_live if ctx_after else ctx.attn_act
        resid = block_in if (nxt == "residual" and kind in _GEMM_STAGES) else None
        if kind == "group_norm":
            fuse = (nxt == "conv" and int(np.asarray(ops[i + 1][1].weights).shape[2]) == 3)
            a, fr = ctx.group_norm(cur, prm, frames=fuse)
            _launch("group_norm")
            if fuse:
                # the normalised activation only exists as halo frames for the conv
                frames, cur = fr, Act("frames", None, cur.C)
            else:
                cur, frames = a, None
            continue
        if kind == "conv":
            cur = ctx.conv(cur, prm, frames, resid)
        elif kind == "layer_norm":
            cur = ctx.layer_norm(cur, prm)
        elif kind == "attention":
            cur = ctx.attention(cur, prm, resid)
        elif kind == "feed_forward":
            cur = ctx.feed_forward(cur, prm, resid)
        elif kind == "linear":
            cur = ctx.linear(cur, prm, resid)
        elif kind == "residual":
            if not fused_residual:
                if cur.C != block_in.shape[1]:
                    raise InputError(f"residual shape mismatch: {cur.C} vs {block_in.shape[1]} channels")
                cur = Act("nchw", ctx.as_nchw(cur, resid=block_in), cur.C)
        _launch(kind)
        fused_residual = resid is not None
        frames = None
    return ctx.as_nchw(cur)


def _mask_tensor(batch: CSPBatch, mask) -> torch.Tensor:
    if isinstance(mask, torch.Tensor):
        if mask.dtype != torch.bool or tuple(mask.shape) != (batch.n_patches,):
            raise InputError(f"mask must be ({batch.n_patches},) bool, got {tuple(mask.shape)} {mask.dtype}")
        return mask.to(require_cuda()).contiguous()
    m = np.asarray(mask)
    if m.shape != (batch.n_patches,) or m.dtype != np.bool_:
        raise InputError(f"mask must be ({batch.n_patches},) bool, got {m.shape} {m.dtype}")
    return torch.as_tensor(m, device=require_cuda())


def select_patches(mask: torch.Tensor, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """out[p] = a[p] if mask[p] else b[p] (patch arrays of one dtype: bf16, fp32 or fp64)."""
    if a.dtype != b.dtype:
        raise InputError("select_patches: dtype mismatch")
    out = torch.empty_like(b)
    n = b[0].numel() if b.shape[0] else 0
    code = {BF16: _lib.DTYPE_BF16, torch.float32: _lib.DTYPE_F32, torch.float64: _lib.DTYPE_F64}[b.dtype]
    _lib.call("ps_select_patches", stream(), mask.view(torch.uint8).data_ptr(), b.shape[0], n, code,
              a.contiguous().data_ptr(), b.contiguous().data_ptr(), out.data_ptr())
    return out


def masked_block_forward(batch: CSPBatch, x, mask, ops, cached_inputs, cached_outputs) -> torch.Tensor:
    """Run a block reusing cached results for masked patches (patched.py:224-246).

    Masked rows of the result are exact copies of `cached_outputs` at its precision (bf16 on the
    hot path; fp32 / fp64 cached outputs stay exact, as np.where keeps them); the recomputed rows
    are the bf16 block outputs at that precision."""
    x = _check_data(batch, x)
    m = _mask_tensor(batch, mask)
    # the all / none branches (patched.py:237-240) need the count on the host: free for a host
    # (numpy) mask, one read-back for a device mask
    n_masked = int(np.count_nonzero(mask)) if not isinstance(mask, torch.Tensor) else int(m.sum())
    co = _check_data(batch, cached_outputs)
    out_dt = co.dtype if co.dtype in (BF16, torch.float32, torch.float64) else torch.float32
    if n_masked == batch.n_patches:
        return co.to(out_dt).clone()
    if n_masked == 0:
        y = run_block(batch, x, ops)
        return y if out_dt == BF16 else y.to(out_dt)
    ci = _bf16_nchw(_check_data(batch, cached_inputs))
    y = run_block(batch, select_patches(m, ci, _bf16_nchw(x)), ops)
    return select_patches(m, co.to(out_dt).contiguous(), y.to(out_dt))
