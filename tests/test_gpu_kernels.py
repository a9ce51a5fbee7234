"""Kernel-level parity on the B200: tcgen05 GEMM / implicit conv / attention against
plain fp32 torch references (floating point, stated tolerances), copy kernels
bit-exact."""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2501_09253_b200 import _lib  # noqa: E402
from paper_2501_09253_b200._dev import stream  # noqa: E402


def _gemm(a, b, bias=None, epi=0, bn=0, out=None, ldo=None, pair=0):
    M, K = a.shape
    N = b.shape[0]
    if out is None:
        out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    g = _lib.GemmArgs()
    g.a, g.lda, g.M = a.data_ptr(), a.stride(0), M
    g.a_mode = 0
    g.b, g.N, g.K = b.data_ptr(), N, K
    g.bias = None if bias is None else bias.data_ptr()
    g.epi, g.out, g.ldo = epi, out.data_ptr(), ldo or N
    g.bn = bn
    g.cta_pair = pair
    _lib.check(_lib.load().ps_gemm(stream(), C.byref(g)))
    return out


@pytest.mark.parametrize("M,N,K,bn", [(128, 64, 64, 64), (256, 128, 128, 128), (1000, 320, 320, 160),
                                      (384, 160, 192, 160), (512, 256, 640, 256), (200, 1280, 320, 256),
                                      (130, 192, 64, 192), (1000, 320, 1280, 320), (256, 320, 2880, 0)])
def test_gemm_matches_fp32(M, N, K, bn):
    torch.manual_seed(M + N + K)
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda")
    got = _gemm(a, b, bias, bn=bn).float()
    want = a.float() @ b.float().T + bias
    err = (got - want).abs().max().item()
    # bf16 output rounding of O(1..4) values: <= 2^-7 relative
    assert err <= 2e-2 * max(1.0, want.abs().max().item()), err


def test_gemm_gelu_epilogue():
    torch.manual_seed(0)
    a = torch.randn(256, 128, device="cuda").to(torch.bfloat16)
    b = (torch.randn(256, 128, device="cuda") / 11).to(torch.bfloat16)
    bias = torch.randn(256, device="cuda") * 0.1
    got = _gemm(a, b, bias, epi=1).float()
    x = a.float() @ b.float().T + bias
    want = 0.5 * x * (1 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))
    assert (got - want).abs().max().item() <= 2e-2


def test_split_reassemble_bit_exact():
    import paper_2501_09253_b200 as ps
    rng = np.random.default_rng(0)
    lats = [(f"r{i}", torch.tensor(rng.normal(size=(3, d, d)), dtype=torch.float32))
            for i, d in enumerate((64, 96, 64, 128))]
    b = ps.split(lats, patch_size=32)
    back = ps.reassemble(b)
    for rid, lat in lats:
        assert torch.equal(back[rid].cpu(), lat)
    # patch 0 of the first 64-latent is its top-left tile (csp.py:167)
    sl = b.patches_of_request("r0")
    assert torch.equal(b.data[sl.start].cpu(), lats[0][1][:, :32, :32])


# ------------------------------------------------ SDXL-shaped (C=320) stages
# fp32 torch references of the same operators on the stitched images.

def _sdxl_batch(dims=(64, 96, 64), c=320, seed=0):
    import paper_2501_09253_b200 as ps
    g = torch.Generator().manual_seed(seed)
    lats = [(f"r{i}", torch.randn(c, d, d, generator=g).to(torch.bfloat16).float()) for i, d in enumerate(dims)]
    return lats, ps.split(lats, patch_size=32)


def _rel_close(got, want, atol, rtol):
    excess = ((got - want).abs() - (atol + rtol * want.abs())).max().item()
    assert excess <= 0, f"excess {excess:.3e}, max |d| {(got - want).abs().max().item():.3e}"


def test_conv3_sdxl_vs_torch():
    import paper_2501_09253_b200 as ps
    lats, b = _sdxl_batch()
    g = torch.Generator().manual_seed(1)
    w = (torch.randn(320, 320, 3, 3, generator=g) * (0.8 / (9 * 320) ** 0.5)).to(torch.bfloat16).float()
    bias = torch.randn(320, generator=g) * 0.01
    prm = ps.ConvParams(weights=w.double().numpy(), bias=bias.double().numpy())
    got = ps.reassemble(b, ps.patched_conv(b, b.data, prm))
    for rid, lat in lats:
        want = torch.nn.functional.conv2d(lat[None].cuda(), w.cuda(), bias.cuda(), padding=1)[0]
        _rel_close(got[rid].float(), want, 2e-2, 1e-2)


def test_group_norm_sdxl_vs_torch():
    import paper_2501_09253_b200 as ps
    lats, b = _sdxl_batch(seed=2)
    g = torch.Generator().manual_seed(3)
    gamma, beta = 1 + 0.05 * torch.randn(320, generator=g), 0.05 * torch.randn(320, generator=g)
    prm = ps.GroupNormParams(groups=32, gamma=gamma.double().numpy(), beta=beta.double().numpy())
    got = ps.reassemble(b, ps.stitched_group_norm(b, b.data, prm))
    for rid, lat in lats:
        want = torch.nn.functional.group_norm(lat[None].cuda(), 32, gamma.cuda(), beta.cuda(), eps=1e-5)[0]
        _rel_close(got[rid].float(), want, 2e-2, 1e-2)


def test_attention_sdxl_vs_torch():
    import paper_2501_09253_b200 as ps
    lats, b = _sdxl_batch(dims=(64, 96), seed=4)
    g = torch.Generator().manual_seed(5)
    ws = [(torch.randn(320, 320, generator=g) * (0.8 / 320 ** 0.5)).to(torch.bfloat16).float() for _ in range(4)]
    prm = ps.AttentionParams(*(x.double().numpy() for x in ws))
    got = ps.reassemble(b, ps.patched_self_attention(b, b.data, prm))
    for rid, lat in lats:
        t = lat.cuda().reshape(320, -1).T  # (T, C) row-major tokens, kernels.py:270-273
        q, k, v = t @ ws[0].cuda(), t @ ws[1].cuda(), t @ ws[2].cuda()
        s = torch.softmax((q @ k.T) / 320 ** 0.5, dim=1)
        o = (s @ v) @ ws[3].cuda()
        want = o.T.reshape(320, lat.shape[1], lat.shape[2])
        _rel_close(got[rid].float(), want, 5e-2, 2e-2)


def test_feed_forward_residual_sdxl_vs_torch():
    import paper_2501_09253_b200 as ps
    lats, b = _sdxl_batch(dims=(64,), seed=6)
    g = torch.Generator().manual_seed(7)
    w1 = (torch.randn(1280, 320, generator=g) * (0.8 / 320 ** 0.5)).to(torch.bfloat16).float()
    w2 = (torch.randn(320, 1280, generator=g) * (0.8 / 1280 ** 0.5)).to(torch.bfloat16).float()
    b1, b2 = 0.01 * torch.randn(1280, generator=g), 0.01 * torch.randn(320, generator=g)
    prm = ps.FeedForwardParams(w1.double().numpy(), b1.double().numpy(), w2.double().numpy(), b2.double().numpy())
    got = ps.reassemble(b, ps.run_block(b, b.data, [("feed_forward", prm), ("residual", None)]))
    lat = lats[0][1].cuda()
    t = lat.reshape(320, -1).T
    h = t @ w1.cuda().T + b1.cuda()
    h = 0.5 * h * (1 + torch.tanh(0.7978845608028654 * (h + 0.044715 * h ** 3)))
    want = (h @ w2.cuda().T + b2.cuda()).T.reshape(lat.shape) + lat
    _rel_close(got["r0"].float(), want, 5e-2, 2e-2)


@pytest.mark.parametrize("C,ps,mode", [(64, 16, 1), (320, 32, 1), (320, 32, 0), (24, 8, 1), (64, 64, 1)])
def test_frames_cl_register_transpose_matches_smem_kernel(C, ps, mode, monkeypatch):
    """ps_frames_cl / ps_to_cl: the register-transposing streaming kernel (C % 8 == 0,
    ps % 8 == 0) against the shared-memory transposer, bit for bit (same fp32 affine)."""
    import ctypes as Cc
    import paper_2501_09253_b200 as ps_
    from paper_2501_09253_b200 import _lib
    from paper_2501_09253_b200._dev import stream
    torch.manual_seed(0)
    dims = [2 * ps, 3 * ps, ps]
    b = ps_.split([(f"r{i}", torch.randn(C, d, d)) for i, d in enumerate(dims)], patch_size=ps)
    P = b.n_patches
    Cp = (C + 63) // 64 * 64
    x = torch.randn(P, C, ps, ps, device="cuda").to(torch.bfloat16)
    G = 8 if C % 8 == 0 else 4
    stats = torch.rand(b.n_requests, G, 2, device="cuda") + 0.5
    gamma = torch.randn(C, device="cuda")
    beta = torch.randn(C, device="cuda")
    dev = b.device()
    owned = torch.tensor([0, P - 1], dtype=torch.int32, device="cuda")

    def run(smem):
        if smem:
            monkeypatch.setenv("PS_FRAMES_SMEM", "1")
        else:
            monkeypatch.delenv("PS_FRAMES_SMEM", raising=False)
        fr = torch.full((P, ps + 2, ps + 2, Cp), 7.0, device="cuda").to(torch.bfloat16)
        _lib.call("ps_frames_cl", stream(), x.data_ptr(), P, C, ps, Cp, mode, stats.data_ptr(),
                  dev["request_index"].data_ptr(), dev["neighbors"].data_ptr(), G, gamma.data_ptr(),
                  beta.data_ptr(), fr.data_ptr())
        cl = torch.full((P * ps * ps, Cp), 7.0, device="cuda").to(torch.bfloat16)
        _lib.call("ps_to_cl", stream(), x.data_ptr(), P, C, ps, Cp, mode, stats.data_ptr(),
                  dev["request_index"].data_ptr(), G, gamma.data_ptr(), beta.data_ptr(), Cc.c_float(1e-5),
                  cl.data_ptr())
        sub = torch.full((P, ps + 2, ps + 2, Cp), 7.0, device="cuda").to(torch.bfloat16)
        _lib.call("ps_frames_cl_sub", stream(), x.data_ptr(), P, C, ps, Cp, mode, stats.data_ptr(),
                  dev["request_index"].data_ptr(), dev["neighbors"].data_ptr(), G, gamma.data_ptr(),
                  beta.data_ptr(), owned.data_ptr(), 2, sub.data_ptr(), None)
        torch.cuda.synchronize()
        return fr, cl, sub

    a, b2 = run(False), run(True)
    for u, v in zip(a, b2):
        assert torch.equal(u, v)
    # full launches push the frame columns from the neighbours' units, patch lists pull them:
    # every patch listed -> the same frames
    allp = torch.arange(P, dtype=torch.int32, device="cuda")
    pull = torch.full((P, ps + 2, ps + 2, Cp), 7.0, device="cuda").to(torch.bfloat16)
    _lib.call("ps_frames_cl_sub", stream(), x.data_ptr(), P, C, ps, Cp, mode, stats.data_ptr(),
              dev["request_index"].data_ptr(), dev["neighbors"].data_ptr(), G, gamma.data_ptr(),
              beta.data_ptr(), allp.data_ptr(), P, pull.data_ptr(), None)
    torch.cuda.synchronize()
    assert torch.equal(pull, a[0])
    # the interior of each frame is the patch itself (mode 0) / its affine image (mode 1)
    if mode == 0:
        inner = a[0][:, 1:-1, 1:-1, :C].permute(0, 3, 1, 2)
        assert torch.equal(inner, x)


@pytest.mark.parametrize("pairs_kv", [True, False])
@pytest.mark.parametrize("world", [4, 8])
def test_splitkv_attention_matches_single_pass(world, pairs_kv, monkeypatch):
    """Split-KV attention (few query tiles: a rank of a split 2048 px image) against the
    one-pass kernel on the same QKV: the merged partials agree to bf16 rounding.  pairs_kv:
    the persistent CTA-pair kernel's split-KV (ps_attention_pairs_splitkv, the default for
    pair-able tiles) or the single-CTA one."""
    import paper_2501_09253_b200 as ps_
    from paper_2501_09253_b200 import patched
    from paper_2501_09253_b200.patchshard import SplitPlan
    torch.manual_seed(0)
    reqs = [("big", 128), ("s0", 32), ("s1", 64)]
    plan = SplitPlan(reqs, 32, world)
    sh = plan.shard(world - 1)
    b = ps_.split([(rid, torch.randn(64, d, d)) for rid, d in sh.requests], patch_size=32)
    cfg = ps_.ModelConfig(arch="dit_like", channels=64, hidden=128, n_blocks=1, groups=8, seed=2)
    at = ps_.init_weights(cfg)[0][1][1]
    x = torch.randn(b.n_patches, 64, 32, 32, device="cuda").to(torch.bfloat16)
    ctx = patched.Ctx(b)
    owned = np.asarray(sh.owned)
    ctx.attn_tiles = patched._attn_tiles(ctx, owned)
    monkeypatch.setattr(patched, "SPLITKV", False)   # never split
    ref = ctx.as_nchw(ctx.attention(patched.Act("nchw", x, 64), at, None)).float()
    monkeypatch.setattr(patched, "SPLITKV", True)
    monkeypatch.setattr(patched, "SPLITKV_ALL", True)
    patched._SKV_CACHE.clear()
    monkeypatch.setattr(patched, "SPLITKV_MIN_BLOCKS", 1)
    monkeypatch.setattr(patched, "sm_count", lambda: 1000)   # more SMs than tiles: forces splits
    monkeypatch.setattr(patched, "SPLITKV_PAIRS", pairs_kv)
    b._dev.clear()
    ctx2 = patched.Ctx(b)
    ctx2.attn_tiles = patched._attn_tiles(ctx2, owned)
    if pairs_kv:
        assert ctx2.attn_tiles[3], "patch 32: pair tiles"
        plan = ctx2._splitkv_pairs(*ctx2.attn_tiles[4:])
        assert plan is not None and plan[9] > 0 and plan[4] > plan[9] // 2, "expected split pair tiles"
    else:
        plan = ctx2._splitkv(*ctx2.attn_tiles[4:])
        assert plan is not None and plan[3] > plan[8], "expected split tiles"
    got = ctx2.as_nchw(ctx2.attention(patched.Act("nchw", x, 64), at, None)).float()
    torch.cuda.synchronize()
    d = (got[owned] - ref[owned]).abs().max().item()
    assert d <= 2e-2 + 2e-2 * ref[owned].abs().max().item(), d


@pytest.mark.parametrize("M,N,K,bn", [(1000, 320, 320, 160), (512, 256, 640, 256), (640, 320, 1280, 320),
                                      (384, 192, 64, 192), (200, 1280, 320, 256)])
def test_gemm_cta_pair_tiles_bit_identical(M, N, K, bn):
    """tcgen05 cta_group::2 tiles (M = 256 per CTA pair, B halves per CTA, odd tile counts
    leave the pair's second CTA a zero-filled tile) equal the single-CTA tiles bit for bit."""
    torch.manual_seed(M + N)
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda")
    one = _gemm(a, b, bias, bn=bn, pair=1).clone()
    two = _gemm(a, b, bias, bn=bn, pair=2)
    torch.cuda.synchronize()
    assert torch.equal(one, two)


@pytest.mark.parametrize("epi", [2, 3])
def test_gemm_cta_pair_epilogues_bit_identical(epi):
    """The attention's GEMM epilogues on CTA-pair tiles (the default for >= 4 waves of tiles):
    QKV's split epilogue (Q, K channels-last through TMA stores, V^T transposed) and the
    O-projection's bias + residual -> NCHW epilogue equal the single-CTA tiles bit for bit,
    including a ragged last m tile."""
    torch.manual_seed(epi)
    hw, ch = 1024, 320
    M = 9 * hw + 512 if epi == 3 else 9 * hw  # NCHW epilogue: whole patches
    N, K = (960, 320) if epi == 3 else (320, 320)
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda")
    res = torch.randn(M * N, device="cuda").to(torch.bfloat16)
    outs = []
    for pair in (1, 2):
        out = torch.full((M * N + 1024,), float("nan"), dtype=torch.bfloat16, device="cuda")
        out2 = torch.full((N * ((M + 63) // 64 * 64),), float("nan"), dtype=torch.bfloat16, device="cuda")
        g = _lib.GemmArgs()
        g.a, g.lda, g.M, g.a_mode = a.data_ptr(), K, M, 0
        g.b, g.N, g.K, g.bias = b.data_ptr(), N, K, bias.data_ptr()
        g.epi, g.out, g.ldo, g.bn = epi, out.data_ptr(), N, 0
        g.P, g.ps = M // hw, 32
        g.cta_pair = pair
        if epi == 3:
            g.out2, g.ldo2, g.n_split, g.ldo = out2.data_ptr(), (M + 63) // 64 * 64, 2 * N // 3, 2 * N // 3
        else:
            g.resid, g.c_real = res.data_ptr(), ch
        _lib.check(_lib.load().ps_gemm(stream(), C.byref(g)))
        torch.cuda.synchronize()
        outs.append((out.clone(), out2.clone()))
    assert torch.equal(outs[0][0].view(torch.int16), outs[1][0].view(torch.int16))
    assert torch.equal(outs[0][1].view(torch.int16), outs[1][1].view(torch.int16))


def test_attention_pair_kernel_bit_identical_to_single():
    """The default CTA-pair attention (attention2.cu) and the single-CTA kernel agree bit for
    bit on a mixed batch (same MMA accumulation order and softmax arithmetic)."""
    import paper_2501_09253_b200 as ps
    from paper_2501_09253_b200 import patched
    torch.manual_seed(3)
    cfg = ps.ModelConfig(arch="dit_like", channels=128, hidden=256, n_blocks=1, groups=8, seed=4)
    at = ps.init_weights(cfg)[0][1][1]
    b = ps.split([(f"r{i}", torch.randn(128, d, d)) for i, d in enumerate((32, 64, 48, 32))], patch_size=16)
    x = torch.randn(b.n_patches, 128, 16, 16, device="cuda").to(torch.bfloat16)
    outs = []
    for pairs in (False, True):
        patched.USE_PAIRS = pairs
        try:
            outs.append(ps.patched_self_attention(b, x, at).clone())
        finally:
            patched.USE_PAIRS = True
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("C,H,lat,compact", [(320, 1280, (64, 32, 96), False), (320, 1280, (64, 96), True),
                                             (128, 256, (32, 64), False), (192, 384, (64,), False),
                                             (320, 1280, (64, 96, 128) * 4, False)])  # config 2: P = 116
def test_fused_feed_forward_bit_identical_to_two_gemms(C, H, lat, compact, monkeypatch):
    """ps_feed_forward (FF1 + GELU + FF2 + residual with the hidden kept on chip, CTA pairs)
    equals the two-GEMM path bit for bit, with and without a compaction tile map."""
    import paper_2501_09253_b200 as ps
    from paper_2501_09253_b200 import patched
    torch.manual_seed(1)
    cfg = ps.ModelConfig(arch="dit_like", channels=C, hidden=H, n_blocks=1, groups=8, seed=3)
    ff = ps.init_weights(cfg)[0][2][1]
    b = ps.split([(f"r{i}", torch.randn(C, d, d)) for i, d in enumerate(lat)], patch_size=32)
    x = torch.randn(b.n_patches, C, 32, 32, device="cuda").to(torch.bfloat16)
    res = torch.randn(b.n_patches, C, 32, 32, device="cuda").to(torch.bfloat16)
    outs = []
    for fused in (False, True):
        monkeypatch.setattr(patched, "FF_FUSED", fused)
        ctx = patched.Ctx(b)
        if compact:
            act = np.arange(0, b.n_patches, 2)
            ctx.rows = patched._row_tiles(ctx, act)
        y = ctx.feed_forward(patched.Act("nchw", x, C), ff, res)
        outs.append(y.t.clone())
    torch.cuda.synchronize()
    if compact:
        act = np.arange(0, b.n_patches, 2)
        assert torch.equal(outs[0][act], outs[1][act])
    else:
        assert torch.equal(outs[0], outs[1])


def test_persistent_attention_concurrent_streams_and_graph():
    """The persistent pair attention deals tiles from per-stream ticket counters: launches on
    two streams at once, and replays of a graph captured on a third stream, all give the
    single-stream result bit for bit (a shared counter would drop or repeat tiles)."""
    import paper_2501_09253_b200 as ps
    torch.manual_seed(5)
    cfg = ps.ModelConfig(arch="dit_like", channels=128, hidden=256, n_blocks=1, groups=8, seed=6)
    at = ps.init_weights(cfg)[0][1][1]
    b = ps.split([(f"r{i}", torch.randn(128, d, d)) for i, d in enumerate((64, 32, 96, 48, 64))], patch_size=16)
    x = torch.randn(b.n_patches, 128, 16, 16, device="cuda").to(torch.bfloat16)
    want = ps.patched_self_attention(b, x, at).clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    outs = []
    for _ in range(4):
        with torch.cuda.stream(s1):
            outs.append(ps.patched_self_attention(b, x, at))
        with torch.cuda.stream(s2):
            outs.append(ps.patched_self_attention(b, x, at))
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, want)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        got = ps.patched_self_attention(b, x, at)
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(got, want)


def test_persistent_attention_two_graphs_replayed_concurrently():
    """Two graphs captured the default way (torch.cuda.graph's shared capture stream) replayed at
    the same time on two streams: each captured launch owns its tile-ticket pair, so neither
    replay drops or repeats the other's tiles (a per-stream counter would be shared)."""
    import paper_2501_09253_b200 as ps
    torch.manual_seed(7)
    cfg = ps.ModelConfig(arch="dit_like", channels=128, hidden=256, n_blocks=1, groups=8, seed=6)
    at = ps.init_weights(cfg)[0][1][1]
    b = ps.split([(f"r{i}", torch.randn(128, d, d)) for i, d in enumerate((64, 96, 64, 128))], patch_size=16)
    x1 = torch.randn(b.n_patches, 128, 16, 16, device="cuda").to(torch.bfloat16)
    x2 = torch.randn(b.n_patches, 128, 16, 16, device="cuda").to(torch.bfloat16)
    want1 = ps.patched_self_attention(b, x1, at).clone()
    want2 = ps.patched_self_attention(b, x2, at).clone()
    g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1):
        o1 = ps.patched_self_attention(b, x1, at)
    with torch.cuda.graph(g2):
        o2 = ps.patched_self_attention(b, x2, at)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(8):
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            g1.replay()
        with torch.cuda.stream(s2):
            g2.replay()
        torch.cuda.synchronize()
        assert torch.equal(o1, want1)
        assert torch.equal(o2, want2)


@pytest.mark.parametrize("nbytes", [32, 1024, 32 * 777, 76021760])
def test_checksum_xor_fold_bit_exact(nbytes):
    """ps_checksum = XOR of every u32 word of the buffer (the 32-byte-word fold is order-free)."""
    from paper_2501_09253_b200._dev import checksum
    from paper_2501_09253_b200.errors import InputError
    g = torch.Generator(device="cuda").manual_seed(nbytes)
    t = torch.randint(-2 ** 31, 2 ** 31 - 1, (nbytes // 4,), dtype=torch.int32, device="cuda", generator=g)
    want = int(np.bitwise_xor.reduce(t.cpu().numpy().view(np.uint32)))
    assert checksum(t) == want
    t[nbytes // 8] ^= 1 << 7  # one flipped bit changes it
    assert checksum(t) == want ^ (1 << 7)
    if nbytes >= 64:
        with pytest.raises(InputError):
            checksum(t[1:])  # 4 bytes off the 32-byte alignment


def test_copy_segments_var_bit_exact():
    """ps_copy_segments_var: per-segment byte counts, 16-byte aligned segments (vector path) and
    2-byte aligned ones (u16 path) mixed in one launch, against a host copy."""
    rng = np.random.default_rng(5)
    src = torch.randint(0, 255, (1 << 20,), dtype=torch.uint8, device="cuda")
    dst = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    so, do, nb = [], [], []
    pos = 0
    for i in range(300):
        n = int(rng.integers(1, 3000)) * (16 if i % 3 else 2)
        a = int(rng.integers(0, (1 << 20) - n)) & ~(15 if i % 3 else 1)
        so.append(a); do.append(pos); nb.append(n)
        pos += n + (16 if i % 2 else 2)
        if pos >= (1 << 20) - 50000:
            break
    so_d, do_d, nb_d = (torch.as_tensor(np.asarray(v, np.int64), device="cuda") for v in (so, do, nb))
    _lib.check(_lib.load().ps_copy_segments_var(stream(), src.data_ptr(), dst.data_ptr(), len(so), so_d.data_ptr(),
                                                  do_d.data_ptr(), nb_d.data_ptr()))
    torch.cuda.synchronize()
    want = np.zeros(1 << 20, np.uint8)
    s_np = src.cpu().numpy()
    for a, b_, n in zip(so, do, nb):
        want[b_:b_ + n] = s_np[a:a + n]
    assert np.array_equal(dst.cpu().numpy(), want)
