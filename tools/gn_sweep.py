"""GroupNorm-partials variants (PS_GN_CFG, norm.cu) on the config-2 activation: mean CUDA-event
time per launch with L2 flushed (a 256 MB read) before each, and the HBM fraction.
  for c in 0 1 2 3 4 5 6; do PS_GN_CFG=$c python tools/gn_sweep.py; done"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_09253_b200 import _lib  # noqa: E402
from paper_2501_09253_b200._dev import stream  # noqa: E402

P, C, ps, G = 116, 320, 32, 32
x = torch.randn((P, C, ps, ps), device="cuda").to(torch.bfloat16)
part = torch.empty((P, G, 2), device="cuda")
flush = torch.ones(64 << 20, device="cuda")
sink = torch.zeros(1, device="cuda")
L = _lib.load()
for _ in range(3):
    L.ps_gn_partials(stream(), x.data_ptr(), P, C, ps, G, part.data_ptr())
ts = []
for _ in range(30):
    sink += flush.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.ps_gn_partials(stream(), x.data_ptr(), P, C, ps, G, part.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
us = sum(ts[3:-3]) / len(ts[3:-3])
ref = x.double().view(P, G, -1)
err = float((part[..., 0].double() - ref.mean(-1)).abs().max())
print(json.dumps({"cfg": os.environ.get("PS_GN_CFG", "0"), "us": round(us, 2), "min_us": round(ts[0], 2),
                  "frac": round(x.numel() * 2 / (us * 1e-6) / 1e9 / 6545.0, 3), "mean_err": err}), flush=True)

if os.environ.get("PS_GN_FLOOR"):
    # floors for the same 76 MB: torch's sum (read-only reduction) and clone (read + write)
    x2 = torch.randn((2 * P, C, ps, ps), device="cuda").to(torch.bfloat16)  # 152 MB (the reuse test's reads)
    for name, fn in (("torch_sum", lambda: x.sum(dtype=torch.float32)), ("torch_clone", lambda: x.clone()),
                     ("torch_sum_152MB", lambda: x2.sum(dtype=torch.float32)), ("torch_clone_152MB", lambda: x2.clone())):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(30):
            sink += flush.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        us = sum(ts[3:-3]) / len(ts[3:-3])
        nb = (x2 if "152" in name else x).numel() * 2 * (1 if "sum" in name else 2)
        print(json.dumps({"floor": name, "us": round(us, 2), "frac": round(nb / (us * 1e-6) / 1e9 / 6545.0, 3)}))
