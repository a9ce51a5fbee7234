"""Config 3: the config-2 batch with the patch cache in the loop, sweeping the
reuse threshold sigma (pkg/scripts/cache_reuse.py:20 uses the same grid).

Per sigma: N denoising steps of the SDXL-shaped model through
engine_step.numeric_step (bit-exact reuse test, compaction of the recomputed
patches), reporting the reuse rate (skipped / all patch-blocks), the share of
patch-blocks whose pixel-wise stages actually ran, and device time per step.
Prints one JSON line per sigma; `--out` also writes them to a file.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2501_09253_b200 as ps  # noqa: E402
from paper_2501_09253_b200.engine_step import CachedStepGraph, numeric_step  # noqa: E402
from paper_2501_09253_b200.model import step_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--sigmas", default="0,0.001,0.01,0.05,0.1,0.5")
    ap.add_argument("--max-streak", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--graph", action="store_true",
                    help="the cached step as one CUDA graph (engine_step.CachedStepGraph, as bench.py config 3)")
    args = ap.parse_args()
    cfg = ps.ModelConfig(arch="unet_like", channels=bench.C, hidden=bench.HIDDEN, groups=bench.GROUPS,
                         n_blocks=bench.BLOCKS, seed=0)
    w = ps.init_weights(cfg)
    reqs = bench.make_requests(0, 0)
    prompts = {rid: ps.make_prompt(cfg, rid) for rid, _ in reqs}
    lines = []
    for sig in [float(x) for x in args.sigmas.split(",")]:
        b = ps.split([(r, torch.tensor(x, dtype=torch.float32)) for r, x in reqs], patch_size=bench.PATCH)
        cache = None if sig == 0 else ps.BlockCache(cfg.n_blocks, ps.PredictorConfig(sig, args.max_streak))
        data = b.data.clone()
        keys = b.patch_keys()
        tot = dict(skipped=0, computed=0, rows_run=0)
        times = []
        gstep = CachedStepGraph(b, w, cache, keys) if (args.graph and cache is not None) else None
        for s in range(args.steps):
            bias, rates = step_inputs(cfg, b, prompts, dict.fromkeys(prompts, s), dict.fromkeys(prompts, 50))
            b.data = data
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if gstep is not None:
                data, st = gstep.run(data, bias, rates)
                data = data.clone()  # the graph's output buffer is overwritten by the next replay
            else:
                data, st = numeric_step(b, w, cache, bias, rates, keys=keys)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            for k in tot:
                tot[k] += getattr(st, k)
        allpb = args.steps * b.n_patches * cfg.n_blocks
        warm = times[2:] or times
        line = {"sigma": sig, "max_streak": args.max_streak, "steps": args.steps, "patches": b.n_patches,
                "reuse_rate": tot["skipped"] / allpb, "rows_run_frac": tot["rows_run"] / allpb,
                "ms_per_step_mean": float(np.mean(warm)), "ms_per_step_first": times[0],
                "patches_per_s": b.n_patches / (float(np.mean(warm)) * 1e-3),
                "cache": cache.stats.as_dict() if cache else None,
                "mode": "graph (CachedStepGraph: reuse decisions on the device)" if gstep is not None else
                        "eager (one mask read-back per block as in engine.py:143-144)",
                "note": "sigma=0: no cache (plain steps); timing with CUDA events per step, steps 2.. averaged"}
        print(json.dumps(line), flush=True)
        lines.append(line)
    if args.out:
        with open(args.out, "w") as f:
            for ln in lines:
                f.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()
