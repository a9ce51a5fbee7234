"""Run the config-2 step's HBM-bound kernels back to back for an ncu capture:
split, prompt bias, GN partials, stitcher (GN + halo frames), cache reuse test,
cache substitute / finish, blend, reassemble.  python tools/mem_kernels.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2501_09253_b200 as ps
from paper_2501_09253_b200.engine_step import numeric_step
from paper_2501_09253_b200.model import step_inputs

cfg = ps.ModelConfig(arch="unet_like", channels=bench.C, hidden=bench.HIDDEN, groups=bench.GROUPS,
                     n_blocks=2, seed=0)
w = ps.init_weights(cfg)
reqs = bench.make_requests(0, 0)
prompts = {rid: ps.make_prompt(cfg, rid) for rid, _ in reqs}
lats = [(r, torch.tensor(x, dtype=torch.float32, device="cuda")) for r, x in reqs]
cache = ps.BlockCache(cfg.n_blocks, ps.PredictorConfig(0.1, 3))
for s in range(3):
    b = ps.split(lats, patch_size=bench.PATCH)
    bias, rates = step_inputs(cfg, b, prompts, dict.fromkeys(prompts, s), dict.fromkeys(prompts, 50))
    new, st = numeric_step(b, w, cache, bias, rates)
    out = ps.reassemble(b, new)
    lats = [(r, out[r]) for r, _ in reqs]
torch.cuda.synchronize()
print("ok", st)
