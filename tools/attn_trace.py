"""Per-key-block timeline of the pair attention kernel's first CTA (ps_attention_trace)."""
import os, sys
os.environ.setdefault("PS_ATTN_PERSIST", "0")  # the trace / role counters live in the one-tile kernel
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
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
tr = torch.zeros(14 * 64, dtype=torch.int64, device="cuda")
_lib.load().ps_attention_trace(tr.data_ptr())
ps.patched_self_attention(b, x, at)
torch.cuda.synchronize()
_lib.load().ps_attention_trace(None)
t = tr.view(14, 64).cpu().numpy().astype(np.int64)
names = ["S_iss0", "S_iss1", "PV_iss0", "PV_iss1", "sm_Srdy", "sm_Sld", "sm_exp", "sm_Pfree", "sm_Pst"]
t0 = t[4, 8]
print("block " + " ".join(f"{n:>8s}" for n in names) + "   (cycles relative to softmax S-ready of block 8)")
for j in range(8, 24):
    print(f"{j:5d} " + " ".join(f"{int(t[e, j] - t0):8d}" for e in range(9)))
per = np.diff(t[4, 8:40])
print("S-ready period: mean %.0f  min %d  max %d cycles" % (per.mean(), per.min(), per.max()))
for a, bb, lab in [(4, 5, "S load (TMEM->regs)"), (5, 6, "exp+max+sum"), (6, 7, "wait P free"), (7, 8, "P store"),
                   (0, 1, "S issue span"), (2, 3, "PV issue span")]:
    d = t[bb, 8:40] - t[a, 8:40]
    print(f"{lab:22s} mean {d.mean():7.0f}  min {d.min():6d}  max {d.max():6d}")
d = t[4, 9:41] - t[1, 8:40]
print(f"{'S(j+1) issued->ready':22s} mean {d.mean():7.0f}")
d = t[4, 9:41] - t[8, 8:40]
print(f"{'P(j) stored->S(j+1) rdy':22s} mean {d.mean():7.0f}")
print("S issuer k_full wait per block: mean %.0f   PV issuer v_full wait per block: mean %.0f" %
      (t[9, 8:40].mean(), t[10, 8:40].mean()))
print("prologue (entry -> first S MMA issued): %d cycles; epilogue (O ready -> stores issued): %d cycles"
      % (t[0, 0] - t[11, 0], t[13, 0] - t[12, 0]))
print("last traced block PV issued -> O ready: see PV_iss1; tile blocks traced: %d" % int((t[4] != 0).sum()))
