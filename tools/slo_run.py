"""SLO attainment of the B200 path in the wall plane (serving.slo_run) for the SDXL-shaped
config-2 model: one JSON line per (max_active, policy, load) point.  The MLP latency model is
trained once per max_active on >= 200 measured compositions and reused across loads.
  python tools/slo_run.py --loads 0.5 0.9 1.2 1.5 --max-active 12 64 --policies slo_aware fcfs"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2501_09253_b200.model import SDXL_SHAPED, init_weights  # noqa: E402
from paper_2501_09253_b200.serving import calibrate_latency_model, slo_run  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--loads", type=float, nargs="+", default=[0.9])
ap.add_argument("--max-active", type=int, nargs="+", default=[12])
ap.add_argument("--policies", nargs="+", default=["slo_aware"])
ap.add_argument("--n-requests", type=int, default=128)
ap.add_argument("--n-calib", type=int, default=240)
ap.add_argument("--no-cache", action="store_true")
ap.add_argument("--static", action="store_true", help="MLP predictor without the EWMA pace correction")
a = ap.parse_args()
w = init_weights(SDXL_SHAPED)
for ma in a.max_active:
    model, rep = calibrate_latency_model(SDXL_SHAPED, w, n_compositions=a.n_calib, max_batch=ma)
    print(json.dumps({"max_active": ma, "latency_model": rep}), flush=True)
    for policy in a.policies:
        for load in a.loads:
            r = slo_run(SDXL_SHAPED, w, n_requests=a.n_requests, load=load, use_cache=not a.no_cache,
                        policy=policy, adaptive=not a.static, max_active=ma, latency_model=model,
                        calib_report=rep)
            r.pop("latency_model", None)
            print(json.dumps(r), flush=True)
