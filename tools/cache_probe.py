"""Config-3 cached step: device busy time (sum of kernel durations, torch.profiler) vs the
CUDA-event step time -- the gap is host work and mask read-back bubbles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
import bench
import paper_2501_09253_b200 as ps
from paper_2501_09253_b200.engine_step import CachedStepGraph, numeric_step
from paper_2501_09253_b200.model import step_inputs

cfg = ps.ModelConfig(arch="unet_like", channels=bench.C, hidden=bench.HIDDEN, groups=bench.GROUPS,
                     n_blocks=bench.BLOCKS, seed=0)
w = ps.init_weights(cfg)
reqs = bench.make_requests(0, 0)
b = ps.split([(r, torch.tensor(x, dtype=torch.float32)) for r, x in reqs], patch_size=bench.PATCH)
prompts = {rid: ps.make_prompt(cfg, rid) for rid, _ in reqs}
cache = ps.BlockCache(cfg.n_blocks, ps.PredictorConfig(0.1, 3))
keys = b.patch_keys()
data = b.data.clone()
GRAPH = "--graph" in sys.argv
PROF_STEP = int(os.environ.get("PROF_STEP", "8"))
step = CachedStepGraph(b, w, cache, keys) if GRAPH else None
for s_ in range(10):
    bias, rates = step_inputs(cfg, b, prompts, dict.fromkeys(prompts, s_), dict.fromkeys(prompts, 50))
    b.data = data
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if s_ == PROF_STEP:
        prof = profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU])
        prof.__enter__()
    e0.record()
    if GRAPH:
        data, st = step.run(data, bias, rates)
    else:
        data, st = numeric_step(b, w, cache, bias, rates, keys=keys)
    e1.record()
    torch.cuda.synchronize()
    if s_ == PROF_STEP:
        prof.__exit__(None, None, None)
    print(s_, f"{e0.elapsed_time(e1):.3f} ms", st)
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
busy = sum(e.device_time for e in ev) / 1e3
print(f"kernels {len(ev)}, device busy {busy:.3f} ms")
agg = {}
for e in ev:
    k = e.name.split("(")[0][:48]
    agg.setdefault(k, [0, 0.0])
    agg[k][0] += 1
    agg[k][1] += e.device_time / 1e3
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{t:8.3f} ms {n:4d}  {k}")
