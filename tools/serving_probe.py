"""Where the wall plane's time goes: per composition, the cost of (a) split + one eager cached
step, (b) the CachedStepGraph capture step, (c) a replay, and (d) measure_step_ms (calibration)
-- host wall time and the CUDA-event time the engine charges to the clock.
  python tools/serving_probe.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_09253_b200.cache import BlockCache, PredictorConfig  # noqa: E402
from paper_2501_09253_b200.csp import STANDARD_CLASSES, split  # noqa: E402
from paper_2501_09253_b200.engine_step import CachedStepGraph, numeric_step  # noqa: E402
from paper_2501_09253_b200.model import SDXL_SHAPED, init_weights  # noqa: E402
from paper_2501_09253_b200.serving import measure_step_ms  # noqa: E402

w = init_weights(SDXL_SHAPED)
dev = torch.device("cuda")


def timed(fn):
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    t0.record()
    r = fn()
    t1.record()
    t1.synchronize()
    return r, t0.elapsed_time(t1), (time.perf_counter() - h0) * 1e3


for comp in ({"low": 1}, {"med": 2}, {"low": 4, "med": 4, "high": 4}, {"high": 3, "low": 2}):
    reqs = []
    for cls, k in comp.items():
        for j in range(k):
            d = STANDARD_CLASSES[cls].latent
            reqs.append((f"{cls}{j}", torch.randn((320, d, d), device=dev)))
    row = {"comp": comp}
    b, row["split_ev"], row["split_host"] = timed(lambda: split(reqs, patch_size=32))
    cache = BlockCache(7, PredictorConfig())
    bias = torch.zeros((b.n_requests, 320), device=dev)
    rates = torch.full((b.n_requests,), 0.1, device=dev)
    (_, _), row["eager_cached_ev"], row["eager_cached_host"] = timed(lambda: numeric_step(b, w, cache, bias, rates))
    (_, _), row["eager_cached2_ev"], row["eager_cached2_host"] = timed(lambda: numeric_step(b, w, cache, bias, rates))
    (_, _), row["eager_nocache_ev"], row["eager_nocache_host"] = timed(lambda: numeric_step(b, w, None, bias, rates))
    cache2 = BlockCache(7, PredictorConfig())
    g, row["graph_init_ev"], row["graph_init_host"] = timed(lambda: CachedStepGraph(b, w, cache2))
    _, row["graph_run1_ev"], row["graph_run1_host"] = timed(lambda: g.run(b.data, bias, rates))
    _, row["graph_capture_ev"], row["graph_capture_host"] = timed(lambda: g.run(b.data, bias, rates))
    reps = [timed(lambda: g.run(b.data, bias, rates))[1:] for _ in range(5)]
    row["graph_replay_ev"] = [round(r[0], 3) for r in reps]
    h0 = time.perf_counter()
    ms = measure_step_ms(SDXL_SHAPED, w, [comp], reps=2)
    row["calib_ms"], row["calib_host_s"] = ms[0][1], time.perf_counter() - h0
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in row.items()}), flush=True)
