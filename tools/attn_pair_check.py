"""Single-CTA vs CTA-pair attention on the config-2 block: time (CUDA events) and agreement."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_2501_09253_b200 as ps
cfg = ps.ModelConfig(arch="unet_like", channels=320, hidden=1280, groups=32, n_blocks=1, seed=0)
w = ps.init_weights(cfg)
reqs = bench.make_requests(0, 0)
b = ps.split([(r, torch.tensor(x, dtype=torch.float32)) for r, x in reqs], patch_size=32)
x = b.data.to(torch.bfloat16)
at = w[0][2][1]
outs = {}
for pairs in (False, True):
    ps.patched.USE_PAIRS = pairs
    for _ in range(2):
        o = ps.patched_self_attention(b, x, at)
    torch.cuda.synchronize()
    outs[pairs] = o.float()
    ps.patched.ATTN_TIMER = []
    for _ in range(5):
        ps.patched_self_attention(b, x, at)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(c) for a, c in ps.patched.ATTN_TIMER]
    ps.patched.ATTN_TIMER = None
    print("pairs", pairs, "attn ms %.3f" % (sum(ms) / len(ms)), flush=True)
print("max |pairs - single|", (outs[True] - outs[False]).abs().max().item())
