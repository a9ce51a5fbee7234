"""Device time of the 2048 px (T = 65,536) attention through the persistent pair kernel and
through the split-KV partials (single-CTA attn_kernel) + combine path.
python tools/attn_splitkv_check.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2501_09253_b200 as ps
import paper_2501_09253_b200.patched as PT

cfg = ps.ModelConfig(arch="unet_like", channels=320, hidden=1280, groups=32, n_blocks=1, seed=2)
at = ps.init_weights(cfg)[0][2][1]
lat = torch.tensor(np.random.default_rng(9).normal(size=(320, 256, 256)), dtype=torch.float32)
b = ps.split([("big", lat)], patch_size=64)
x = b.data.to(torch.bfloat16)
T = 256 * 256
for splitkv in (False, True):
    PT.SPLITKV_ALL = splitkv
    for _ in range(2):
        ps.patched_self_attention(b, x, at)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ps.patched_self_attention(b, x, at)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{'split-KV' if splitkv else 'pairs   '}: {ms:.3f} ms per attention layer (with projections), "
          f"{4.0 * T * T * 320 / ms / 1e9:.0f} TFLOP/s of the core")
PT.SPLITKV_ALL = False
