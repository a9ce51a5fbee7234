"""Fused feed-forward (ffused.cu) vs FF1 + FF2 GEMMs on the config-2 block: device time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2501_09253_b200 as ps
from paper_2501_09253_b200 import patched

cfg = ps.ModelConfig(arch="unet_like", channels=320, hidden=1280, groups=32, n_blocks=1, seed=0)
ff = ps.init_weights(cfg)[0][3][1]
reqs = bench.make_requests(0, 0)
b = ps.split([(r, torch.tensor(x, dtype=torch.float32)) for r, x in reqs], patch_size=32)
x = b.data.to(torch.bfloat16)
res = torch.randn_like(x)
for fused in (False, True, False, True):
    patched.FF_FUSED = fused
    ctx = patched.Ctx(b)
    a = patched.Act("cl", ctx.as_cl(patched.Act("nchw", x, 320)), 320)
    for _ in range(3):
        ctx.feed_forward(a, ff, res)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ctx.feed_forward(a, ff, res)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"fused={fused}: {ms * 1e3:.1f} us  ({2 * 2 * b.n_patches * 1024 * 320 * 1280 / ms / 1e9:.0f} TFLOP/s)",
          flush=True)

patched.FF_FUSED = True
from paper_2501_09253_b200 import _lib
dbg = torch.zeros(64 + 40 * 8, dtype=torch.int64, device="cuda")
_lib.load().ps_feed_forward_debug(dbg.data_ptr())
ctx.feed_forward(a, ff, res)
torch.cuda.synchronize()
_lib.load().ps_feed_forward_debug(None)
d = dbg.tolist()
f = lambda x, t: x / t if t else 0
tl = np.array(d[64:64 + 320]).reshape(40, 8)
if tl[0, 4]:
    t0 = tl[1:, :].min()
    print("timeline of CTA 0, chunks 1..15 (cycles from the first stamp): MMA1 issue s/e, MMA2 issue s/e, H ready, "
          "H released, GELU done, Hb handed")
    for gc in range(1, 16):
        print(gc, [int(v - t0) for v in tl[gc]])
print(f"producer: w_empty {f(d[0], d[13]):.2f} x_empty {f(d[1], d[13]):.2f}")
print(f"mma     : w_full {f(d[4], d[8]):.2f} h_empty {f(d[5], d[8]):.2f} hs_full {f(d[6], d[8]):.2f} o_empty {f(d[7], d[8]):.2f}")
print(f"epilogue: h_full {f(d[9], d[12]):.2f} hs_empty {f(d[10], d[12]):.2f} o_full {f(d[11], d[12]):.2f}")
print(f"epilogue phases per chunk (cycles): H load {f(d[16], d[19]):.0f}, load+GELU {f(d[17], d[19]):.0f}, "
      f"Hb store+arrive {f(d[18], d[19]):.0f}; output drain per tile {f(d[20], d[21]):.0f}; "
      f"chunk period {f(d[12], d[19]):.0f} (warp-4 total / chunks); MMA1 issue -> H ready {f(d[22], d[23]):.0f}")

# timing experiment (probe build only): the same launch with the chunk epilogue's GELU skipped
for nogelu in (0, 1):
    dbg.zero_()
    dbg[31] = nogelu
    _lib.load().ps_feed_forward_debug(dbg.data_ptr())
    for _ in range(2):
        ctx.feed_forward(a, ff, res)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ctx.feed_forward(a, ff, res)
    e1.record()
    torch.cuda.synchronize()
    _lib.load().ps_feed_forward_debug(None)
    print(f"probe build, gelu {'off' if nogelu else 'on'}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
