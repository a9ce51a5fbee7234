"""Stitcher (ps_frames_cl, GroupNorm mode) on the config-2 batch: device time, L2 flushed.
PS_FRAMES_PULL=1 selects the per-pixel frame-column units instead of the push variant."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2501_09253_b200 as ps
from paper_2501_09253_b200 import patched
from paper_2501_09253_b200.params import GroupNormParams

reqs = bench.make_requests(0, 0)
b = ps.split([(r, torch.tensor(x, dtype=torch.float32)) for r, x in reqs], patch_size=32)
x = b.data.to(torch.bfloat16)
rng = np.random.default_rng(0)
prm = GroupNormParams(32, rng.normal(size=320).astype(np.float32), rng.normal(size=320).astype(np.float32))
ctx = patched.Ctx(b)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stats = ctx.gn_stats(x, 320, patched.device_params(prm, 320))
dp = patched.device_params(prm, 320)
nbytes = x.numel() * 2 + b.n_patches * 34 * 34 * 320 * 2
ts = []
for it in range(23):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.gn_stats(x, 320, dp)
    e1.record()
    torch.cuda.synchronize()
    if it >= 3:
        ts.append(e0.elapsed_time(e1) * 1e3)
us = float(np.median(ts))
print(f"gn partials + finalize: {us:.1f} us, {x.numel() * 2 / us / 1e3:.0f} GB/s of x")
for mode in (1, 0):
    ts = []
    for it in range(23):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if mode == 1:
            ctx._frames(x, 320, 320, 1, stats, 32, dp["gamma"], dp["beta"])
        else:
            ctx._frames(x, 320, 320, 0, None, 1, None, None)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    us = float(np.median(ts))
    print(f"frames mode={mode} pull={os.environ.get('PS_FRAMES_PULL', '0')}: {us:.1f} us, "
          f"{nbytes / us / 1e3:.0f} GB/s algorithmic")
