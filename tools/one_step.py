"""Run config-2 denoise steps (for ncu / compute-sanitizer captures): python tools/one_step.py [steps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2501_09253_b200 as ps

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = ps.ModelConfig(arch="unet_like", channels=bench.C, hidden=bench.HIDDEN, groups=bench.GROUPS,
                     n_blocks=bench.BLOCKS, seed=0)
w = ps.init_weights(cfg)
reqs = bench.make_requests(0, 0)
prompts = {r: ps.make_prompt(cfg, r) for r, _ in reqs}
b = ps.split([(r, torch.tensor(x, dtype=torch.float32)) for r, x in reqs], patch_size=bench.PATCH)
for s in range(steps):
    out = ps.denoise_batch(cfg, w, b, prompts, {r: s for r, _ in reqs}, {r: 50 for r, _ in reqs})
torch.cuda.synchronize()
print("ok", float(out.abs().mean()))
