"""Eager one-step time of a composition (the serving plane's step) with a host profile:
python tools/eager_probe.py [low med high]

Prints the CUDA-event time and host wall time of each rep of measure_step_ms's loop and
the top host functions (cProfile) of one rep -- separates launch/host overhead of the
eager path from device time."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2501_09253_b200 as ps  # noqa: E402
from paper_2501_09253_b200.csp import reassemble, split  # noqa: E402
from paper_2501_09253_b200.engine_step import numeric_step  # noqa: E402
from paper_2501_09253_b200.serving import CLASS_ORDER, STANDARD_CLASSES  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
comp = dict(zip(CLASS_ORDER, map(int, args[:3]))) if len(args) > 2 else {"low": 4, "med": 4, "high": 4}
cfg = ps.ModelConfig(arch="unet_like", channels=bench.C, hidden=bench.HIDDEN, groups=bench.GROUPS,
                     n_blocks=bench.BLOCKS, seed=0)
w = ps.init_weights(cfg)
dev = torch.device("cuda", 0)
reqs = []
for cls in CLASS_ORDER:
    for j in range(comp.get(cls, 0)):
        d = STANDARD_CLASSES[cls].latent
        reqs.append((f"{cls}{j}", torch.as_tensor(np.random.default_rng([0, len(reqs)]).normal(size=(cfg.channels, d, d)),
                                                  dtype=torch.float32, device=dev)))


def once():
    b = split(reqs, patch_size=32)
    bias = torch.zeros((b.n_requests, cfg.channels), dtype=torch.float32, device=dev)
    rates = torch.full((b.n_requests,), 0.1, dtype=torch.float32, device=dev)
    new, _ = numeric_step(b, w, None, bias, rates)
    return reassemble(b, new)


for rep in range(6):
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    t0.record()
    once()
    t1.record()
    h1 = time.perf_counter()
    t1.synchronize()
    print(f"rep {rep}: event {t0.elapsed_time(t1):8.2f} ms  host-enqueue {1e3 * (h1 - h0):8.2f} ms", flush=True)

pr = cProfile.Profile()
torch.cuda.synchronize()
pr.enable()
once()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
pstats.Stats(pr).sort_stats("tottime").print_stats(15)

if "--calib" in sys.argv:
    from paper_2501_09253_b200 import patched
    from paper_2501_09253_b200.serving import CALIBRATION_COMPS, measure_step_ms
    for timer in (None, []):
        patched.ATTN_TIMER = timer
        for rep in range(2):
            s = measure_step_ms(cfg, w, CALIBRATION_COMPS, reps=3)
            print("timer" if timer is not None else "no-timer", rep, [(tuple(c.values()), round(ms, 2)) for c, ms in s], flush=True)
