"""Per-role barrier-wait fractions of the attention kernel on the config-2 batch."""
import os, sys
os.environ.setdefault("PS_ATTN_PERSIST", "0")  # the trace / role counters live in the one-tile kernel
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2501_09253_b200 as ps
from paper_2501_09253_b200 import _lib

cfg = ps.ModelConfig(arch="unet_like", channels=bench.C, hidden=bench.HIDDEN, groups=bench.GROUPS, n_blocks=1, seed=0)
w = ps.init_weights(cfg)
reqs = bench.make_requests(0, 0)
b = ps.split([(r, torch.tensor(x, dtype=torch.float32)) for r, x in reqs], patch_size=bench.PATCH)
x = b.data.to(torch.bfloat16)
at = w[0][2][1]
for _ in range(2):
    ps.patched_self_attention(b, x, at)
dbg = torch.zeros(16, dtype=torch.int64, device="cuda")
_lib.load().ps_attention_debug(dbg.data_ptr())
ps.patched_self_attention(b, x, at)
torch.cuda.synchronize()
_lib.load().ps_attention_debug(None)
d = dbg.tolist()
f = lambda a, t: a / t if t else 0
print(f"MMA warp: wait s_free {f(d[0], d[3]):.2f}  wait p_full {f(d[1], d[3]):.2f}  wait K/V {f(d[2], d[3]):.2f}")
print(f"softmax : wait s_full {f(d[4], d[6]):.2f}  wait p_free {f(d[5], d[6]):.2f}")
nb = max(1, d[12])
print(f"softmax per 128-key block (cycles): S load {d[8]/nb:.0f}  exp+sum {d[9]/nb:.0f}  wait PV/rescale {d[10]/nb:.0f}  P store {d[11]/nb:.0f}")
