"""Pair attention achieved FLOP rate by image size (all images of one class, ~equal total
work): exposes the per-tile fixed cost (Q load, TMEM setup, O epilogue) against the
per-key-block loop.  python tools/attn_size_check.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2501_09253_b200 as ps

cfg = ps.ModelConfig(arch="unet_like", channels=320, hidden=1280, groups=32, n_blocks=1, seed=0)
w = ps.init_weights(cfg)
at = w[0][2][1]
for d, count in ((64, 64), (96, 14), (128, 4), (192, 1), (128, 8)):
    rng = np.random.default_rng(d)
    reqs = [(f"r{i}", torch.tensor(rng.normal(size=(320, d, d)), dtype=torch.float32)) for i in range(count)]
    b = ps.split(reqs, patch_size=32)
    x = b.data.to(torch.bfloat16)
    for _ in range(2):
        ps.patched_self_attention(b, x, at)
    torch.cuda.synchronize()
    ps.patched.ATTN_TIMER = []
    for _ in range(5):
        ps.patched_self_attention(b, x, at)
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(c) for a, c in ps.patched.ATTN_TIMER]))
    ps.patched.ATTN_TIMER = None
    T = d * d
    flops = count * 4.0 * T * T * 320
    tiles = count * T // 256
    print(f"{count:3d} x {T:6d} tokens: {ms:.3f} ms, {flops / ms / 1e9:.0f} TFLOP/s, {tiles} pair tiles "
          f"({tiles / 74:.2f} waves), {T // 128} key blocks per tile", flush=True)
