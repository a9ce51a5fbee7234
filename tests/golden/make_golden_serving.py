"""Record serving-plane golden outputs from the REAL reference.

    python tests/golden/make_golden_serving.py

* traces of `generate_trace` (workload.py:58-77) for several configs;
* cost_only event logs + summaries of `Engine.run` (engine.py:72-250) for
  each scheduler policy (scheduler.py) and 1-3 workers;
* cost-model KATs (latency.py:52-84);
* one small numeric-plane run (unet_like C=4, low-res only, 3 steps, cache on):
  events, summary and final latents (float64) — the GPU numeric plane must give
  the same events and latents within the bf16 tolerance.

Writes serving.json and serving_numeric.npz next to this script.
"""

from __future__ import annotations

import json
import sys
from dataclasses import asdict
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent

COST_RUNS = [
    # (workload kwargs, policy, workers, max_active, steps)
    (dict(seed=0, qps=1.0, n_requests=40), "slo_aware", 1, 12, 50),
    (dict(seed=1, qps=3.0, n_requests=60), "slo_aware", 2, 12, 50),
    (dict(seed=2, qps=0.5, n_requests=30), "fcfs", 1, 12, 50),
    (dict(seed=3, qps=2.0, n_requests=50), "sequential", 3, 12, 20),
    (dict(seed=4, qps=6.0, n_requests=64, slo_scale=2.0), "slo_aware", 1, 64, 50),
    (dict(seed=5, qps=1.5, n_requests=40, class_weights={"low": 1.0, "high": 1.0}), "fcfs", 2, 4, 30),
]
COMPS = [{"low": 1}, {"med": 2}, {"high": 1, "low": 3}, {"low": 4, "med": 4, "high": 4}, {"med": 0, "high": 2}]
NUMERIC = dict(workload=dict(seed=7, qps=20.0, n_requests=3, class_weights={"low": 1.0}, steps=3),
               model=dict(arch="unet_like", channels=4, hidden=8, n_blocks=2, groups=2, seed=0))


def main():
    sys.path.insert(0, REF)
    from mixserve import engine, latency, scheduler, workload
    from mixserve.model import ModelConfig

    out = {"cost": [], "comps": [], "runs": []}
    for comp in COMPS:
        out["comps"].append({"comp": comp, "step_ms": latency.step_latency(comp),
                             "standalone": {c: latency.standalone_latency(c, 50) for c in ("low", "med", "high")}})
    for wl, policy, workers, max_active, steps in COST_RUNS:
        wc = workload.WorkloadConfig(steps=steps, **wl)
        trace = workload.generate_trace(wc)
        ec = engine.EngineConfig(plane="cost_only", n_workers=workers, total_steps=steps,
                                 scheduler=scheduler.SchedulerConfig(policy=policy, max_active=max_active))
        res = engine.Engine(ec).run(trace)
        out["runs"].append({"workload": wl, "policy": policy, "workers": workers, "max_active": max_active,
                            "steps": steps, "trace": [asdict(r) for r in trace], "events": res.events,
                            "completions": res.completions, "summary": res.summary})

    wc = workload.WorkloadConfig(**NUMERIC["workload"])
    trace = workload.generate_trace(wc)
    ec = engine.EngineConfig(plane="numeric", total_steps=wc.steps, model=ModelConfig(**NUMERIC["model"]))
    res = engine.Engine(ec).run(trace)
    out["numeric"] = {"config": NUMERIC, "trace": [asdict(r) for r in trace], "events": res.events,
                      "summary": res.summary}
    np.savez_compressed(HERE / "serving_numeric.npz", **{k: v for k, v in res.latents.items()})
    with open(HERE / "serving.json", "w") as f:
        json.dump(out, f)
    print("wrote", HERE / "serving.json", len(out["runs"]), "runs")


if __name__ == "__main__":
    main()
