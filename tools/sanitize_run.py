"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel family of the
path at the benchmark's channel count on a small batch -- one 512 px + one 256 px request (C=320,
ps=32): split+bias, GN partials / finalize, stitcher frames, conv3 / QKV / O-proj GEMMs, the
persistent pair attention and the split-KV attention + combine, the fused FF, blend+reassemble,
the one-kernel reuse test (bf16 and fp64), cache substitute / finish, compaction lists, the
graph-captured cached step.
  compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_09253_b200 as ps  # noqa: E402
import paper_2501_09253_b200.patched as PT  # noqa: E402
from paper_2501_09253_b200.engine_step import CachedStepGraph, numeric_step  # noqa: E402
from paper_2501_09253_b200.model import step_inputs  # noqa: E402
from paper_2501_09253_b200.pipeline import DenoisePipeline  # noqa: E402

cfg = ps.ModelConfig(arch="unet_like", channels=320, hidden=1280, groups=32, n_blocks=1, seed=0)
w = ps.init_weights(cfg)
dims = [64, 32]
reqs = [(f"r{i}", np.random.default_rng(i).normal(size=(320, d, d))) for i, d in enumerate(dims)]
prompts = {r: ps.make_prompt(cfg, r) for r, _ in reqs}
# pipeline step (split+bias, blocks, blend+reassemble)
pipe = DenoisePipeline(cfg, w, dims, 32, use_graph=False)
pipe.set_prompts([prompts[r] for r, _ in reqs])
pipe.prepare()
hin = [torch.tensor(a, dtype=torch.float32).pin_memory() for _, a in reqs]
hout = [torch.empty_like(t).pin_memory() for t in hin]
pipe.run([hin], [[0, 0]], [50, 50], [hout])
# split-KV attention + combine
b = ps.split([(r, torch.tensor(a, dtype=torch.float32)) for r, a in reqs], patch_size=32)
PT.SPLITKV_ALL = True
ps.patched_self_attention(b, b.data.to(torch.bfloat16), w[0][2][1])
PT.SPLITKV_ALL = False
# cache path: eager numeric steps, then the graph-captured cached step
cache = ps.BlockCache(cfg.n_blocks, ps.PredictorConfig(0.1, 3))
for s in range(3):
    bias, rates = step_inputs(cfg, b, prompts, dict.fromkeys(prompts, s), dict.fromkeys(prompts, 50))
    new, st = numeric_step(b, w, cache, bias, rates)
    b.data = new
c2 = ps.BlockCache(cfg.n_blocks, ps.PredictorConfig(0.1, 3))
g = CachedStepGraph(b, w, c2)
data = b.data.clone()
for s in range(3):
    bias, rates = step_inputs(cfg, b, prompts, dict.fromkeys(prompts, s), dict.fromkeys(prompts, 50))
    data, st = g.run(data, bias, rates)
# fp64 reuse test
x = np.random.default_rng(3).normal(size=(4, 320, 8, 8))
c3 = ps.BlockCache(1, dtype=torch.float64)
keys = [("a", i) for i in range(4)]
c3.batched_update(0, keys, np.zeros(4, bool), x, x)
c3.predict_reuse(0, keys, x + 0.01)
torch.cuda.synchronize()
print("sanitize workload ok")
