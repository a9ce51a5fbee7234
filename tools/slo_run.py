"""SLO attainment of the B200 path in the wall plane (serving.slo_run) for the
SDXL-shaped config-2 model; one JSON line per (load, cache) point."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2501_09253_b200.model import SDXL_SHAPED, init_weights  # noqa: E402
from paper_2501_09253_b200.serving import slo_run  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--loads", type=float, nargs="+", default=[0.9])
ap.add_argument("--n-requests", type=int, default=64)
ap.add_argument("--no-cache", action="store_true")
ap.add_argument("--policy", default="slo_aware")
ap.add_argument("--static", action="store_true", help="fitted analytic predictor without the EWMA correction")
a = ap.parse_args()
w = init_weights(SDXL_SHAPED)
for load in a.loads:
    r = slo_run(SDXL_SHAPED, w, n_requests=a.n_requests, load=load, use_cache=not a.no_cache, policy=a.policy,
                adaptive=not a.static)
    print(json.dumps(r), flush=True)
