"""Serving plane (serving.py) against the reference's own outputs.

Golden file: tests/golden/serving.json, written by make_golden_serving.py from
the real reference (workload.py, latency.py, scheduler.py, engine.py).  The
cost_only plane must reproduce the reference's traces, event logs,
completions and summaries EXACTLY; the GPU numeric plane must reproduce the
event log exactly and the final latents within the north-star tolerance.
"""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2501_09253_b200 import serving as S

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def gold():
    with open(GOLD / "serving.json") as f:
        return json.load(f)


def test_cost_model_kats(gold):
    for c in gold["comps"]:
        assert S.step_latency(c["comp"]) == c["step_ms"]
        for cls, v in c["standalone"].items():
            assert S.standalone_latency(cls, 50) == v


def _run_cost(r):
    wc = S.WorkloadConfig(steps=r["steps"], **r["workload"])
    trace = S.generate_trace(wc)
    ec = S.EngineConfig(plane="cost_only", n_workers=r["workers"], total_steps=r["steps"],
                        scheduler=S.SchedulerConfig(policy=r["policy"], max_active=r["max_active"]))
    return trace, S.Engine(ec).run(trace)


@pytest.mark.parametrize("i", range(6))
def test_cost_only_plane_matches_reference(gold, i):
    r = gold["runs"][i]
    trace, res = _run_cost(r)
    assert [vars(t) for t in trace] == r["trace"]
    assert res.events == r["events"]
    assert res.completions == r["completions"]
    assert res.summary == r["summary"]


def test_trace_roundtrip(tmp_path):
    rows = S.generate_trace(S.WorkloadConfig(seed=3, n_requests=10))
    p = tmp_path / "t.jsonl"
    S.write_trace(rows, p)
    assert S.read_trace(p) == rows
    p.write_text('{"request_id": "a"}\n')
    with pytest.raises(S.InputError):
        S.read_trace(p)


def test_input_errors():
    with pytest.raises(S.InputError):
        S.WorkloadConfig(qps=0)
    with pytest.raises(S.InputError):
        S.SchedulerConfig(policy="lifo")
    with pytest.raises(S.InputError):
        S.EngineConfig(plane="gpu")
    with pytest.raises(S.InputError):
        S.step_latency({})
    with pytest.raises(S.InputError):
        S.Engine().run([])


def test_fit_cost_model_recovers_constants():
    true = S.CostModelParams(c_step_fixed=1.5, c_res_overhead=0.2, c_patch=0.004, c_attn_coeff=3e-8)
    samples = [(c, S.step_latency(c, true)) for c in S.CALIBRATION_COMPS]
    fit = S.fit_cost_model(samples)
    for k in ("c_step_fixed", "c_res_overhead", "c_patch", "c_attn_coeff"):
        assert getattr(fit, k) == pytest.approx(getattr(true, k), rel=1e-6, abs=1e-9)


@pytest.mark.gpu
def test_numeric_plane_matches_reference(gold):
    from paper_2501_09253_b200.model import ModelConfig
    g = gold["numeric"]
    wc = S.WorkloadConfig(**g["config"]["workload"])
    trace = S.generate_trace(wc)
    assert [vars(t) for t in trace] == g["trace"]
    ec = S.EngineConfig(plane="numeric", total_steps=wc.steps, model=ModelConfig(**g["config"]["model"]))
    res = S.Engine(ec).run(trace)
    assert res.events == g["events"]
    want = dict(g["summary"])
    got = {k: v for k, v in res.summary.items() if k in want}
    assert got == want  # includes the cache counters: skip masks are bit-exact
    lat = np.load(GOLD / "serving_numeric.npz")
    for rid in lat.files:
        d = np.abs(res.latents[rid].double().cpu().numpy() - lat[rid]).max()
        assert d <= 1e-2, (rid, d)


@pytest.mark.gpu
def test_wall_plane_runs_on_device():
    from paper_2501_09253_b200.model import ModelConfig
    mc = ModelConfig(arch="unet_like", channels=64, hidden=128, n_blocks=2, groups=8)
    wc = S.WorkloadConfig(seed=1, qps=50.0, n_requests=6, steps=4)
    ec = S.EngineConfig(plane="wall", total_steps=4, model=mc)
    res = S.Engine(ec).run(S.generate_trace(wc))
    s = res.summary
    assert s["n_completed"] + s["n_discarded"] == 6
    assert s["device_step_ms_mean"] > 0
    # the clock advanced by measured device time, not the analytic model (~60 ms a step)
    assert s["makespan_ms"] < 6 * 4 * 60.0


@pytest.mark.gpu
def test_slo_run_two_ranks_pool_completions():
    """slo_run's multi-GPU path (fit shared from rank 0, lowest-load dispatch on the fitted
    model, completions pooled) with two ranks as threads on one GPU."""
    import threading

    import torch

    from paper_2501_09253_b200.model import ModelConfig, init_weights
    mc = ModelConfig(arch="unet_like", channels=64, hidden=128, n_blocks=1, groups=8)
    w = init_weights(mc)
    bar = threading.Barrier(2)
    box: dict = {}

    def share(obj, rank):
        if rank == 0:
            box["fit"] = obj
        bar.wait()
        return box["fit"]

    def gather(obj, rank):
        box[rank] = obj
        bar.wait()
        return [box[0], box[1]]

    res, errs = {}, []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            res[rank] = S.slo_run(mc, w, n_requests=8, load=0.5, steps=3, rank=rank, world=2, n_calib=24,
                                  share=lambda o: share(o, rank), gather=lambda o: gather(o, rank))
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    if errs:
        raise errs[0]
    a, b = res[0], res[1]
    assert a["n_gpus"] == 2 and a["slo_attainment"] == b["slo_attainment"]
    assert a["n_met_slo"] + a["n_discarded"] <= 8
    assert a["latency_model"] == b["latency_model"]


def test_mlp_latency_model_generalises_on_synthetic_steps():
    # the serving plane's predictor (MLP on measured compositions): trained on
    # 200 compositions of a known T^2-attention cost law with 1% noise, held-out error < 5%
    comps = S.random_compositions(260, seed=1)
    assert len({tuple(sorted(c.items())) for c in comps}) == 260
    np.random.default_rng(9).shuffle(comps)
    true = S.CostModelParams(c_step_fixed=0.8, c_res_overhead=0.05, c_patch=0.008, c_attn_coeff=2.2e-9,
                             attn_exponent=2.0)
    y = np.array([S.step_latency(c, true) * (1 + 0.01 * np.random.default_rng(i).normal()) + 0.2 * sum(c.values()) ** 0.5
                  for i, c in enumerate(comps)])
    m = S.MlpLatencyModel()
    m.fit(comps[:200], y[:200])
    err = np.abs(m.predict(comps[200:]) - y[200:]) / y[200:]
    assert err.mean() < 0.05, err.mean()
    pred = S.LearnedPredictor(m)
    assert pred.predict_step_latency({"low": 2}) == m.predict_step_latency({"low": 2})
    pred.observe({"low": 2}, 0.5 * m.predict_step_latency({"low": 2}))
    assert pred.ratio < 1.0


def test_extended_resolution_classes_enter_the_serving_plane():
    # configs 1 (256/384 px) and 5 (2048 px) through the engine
    from paper_2501_09253_b200.csp import STANDARD_CLASSES
    assert {c: STANDARD_CLASSES[c].latent for c in ("tiny", "small", "ultra")} == {"tiny": 32, "small": 48,
                                                                                 "ultra": 256}
    cost = S.CostModelParams(patch_size=16)
    trace = S.generate_trace(S.WorkloadConfig(seed=1, qps=2.0, n_requests=12, steps=4,
                                              class_weights={"tiny": 1, "small": 1, "low": 1}), cost)
    res = S.Engine(S.EngineConfig(plane="cost_only", total_steps=4, patch_size=16, cost=cost,
                                  scheduler=S.SchedulerConfig(cost=cost))).run(trace)
    assert res.summary["n_completed"] + res.summary["n_discarded"] == 12
    cost64 = S.CostModelParams(patch_size=64)
    trace5 = [S.TraceRow("big", 0.0, "ultra", 1e9)] + [S.TraceRow(f"s{i}", 0.0, "low", 1e9) for i in range(8)]
    res5 = S.Engine(S.EngineConfig(plane="cost_only", total_steps=2, patch_size=64, cost=cost64,
                                   scheduler=S.SchedulerConfig(cost=cost64))).run(trace5)
    assert res5.summary["n_completed"] == 9


@pytest.mark.gpu
def test_wall_and_numeric_planes_graph_opt_in_equals_eager():
    """EngineConfig.graph_after_steps > 0 replays a composition's cached step as one CUDA graph
    once it has run that many eager steps: the numeric plane's events and final latents equal
    the all-eager run bit for bit (CachedStepGraph reproduces numeric_step exactly)."""
    import torch

    from paper_2501_09253_b200.model import ModelConfig
    from paper_2501_09253_b200.patched import device_compaction_ok  # noqa: F401 -- the path exercised
    mc = ModelConfig(arch="unet_like", channels=64, hidden=128, n_blocks=2, groups=8, seed=1)
    wc = S.WorkloadConfig(seed=3, qps=5.0, n_requests=5, steps=12)
    trace = S.generate_trace(wc)
    runs = {}
    for k in (0, 2):
        ec = S.EngineConfig(plane="numeric", total_steps=12, model=mc, graph_after_steps=k)
        runs[k] = S.Engine(ec).run(trace)
    assert runs[0].events == runs[2].events
    strip = lambda d: {k: v for k, v in d.items() if k != "device_step_ms_mean"}  # timing differs
    assert strip(runs[0].summary) == strip(runs[2].summary)
    for rid, lat in runs[0].latents.items():
        assert torch.equal(lat, runs[2].latents[rid]), rid
    # the wall plane runs with graphs on as well
    ec = S.EngineConfig(plane="wall", total_steps=12, model=mc, graph_after_steps=2)
    res = S.Engine(ec).run(trace)
    assert res.summary["n_completed"] + res.summary["n_discarded"] == 5
