"""Serving plane around the patch path: cost model, traces, SLO-aware admission
and the event loop — the caller of the hot path.

The reference (latency.py, workload.py, scheduler.py, engine.py) prices every
step with an analytic cost model calibrated to nothing in particular, and its
numeric plane runs the patched model on the CPU while the clock still comes
from that model.  Here the same policy code drives the B200 path, with three
clocks:

* ``cost_only`` — analytic step latency, no compute (the reference's
  cost_only plane; event logs match it exactly, tests/test_serving.py);
* ``numeric``   — analytic clock, every step computed on the GPU through
  engine_step.numeric_step with the patch cache in the loop (the reference's
  numeric plane; same events, latents within the bf16 tolerance);
* ``wall``      — every step computed on the GPU and the clock advanced by the
  step's measured device time (CUDA events around the whole step: split,
  prompt bias, blocks with the cache, blend, reassemble).  SLO attainment in
  this plane is the B200 number the BASELINE metric asks for.

`fit_cost_model` refits the analytic model's constants to measured B200 step
times so admission decisions and SLO budgets (workload.py:74, 3x standalone
latency) are in B200 time.
"""

from __future__ import annotations

import gc
import heapq
import json
import os
import sys
from dataclasses import dataclass, field, replace
from typing import Sequence

import numpy as np

from .csp import STANDARD_CLASSES
from .errors import InputError  # noqa: F401  (re-exported for callers)

CLASS_ORDER = ("low", "med", "high", "tiny", "small", "ultra")

# ------------------------------------------------------------ cost model


@dataclass(frozen=True)
class CostModelParams:
    """latency.py:25-33 (defaults are the reference's)."""

    blocks_per_step: int = 8
    c_step_fixed: float = 60.0
    c_res_overhead: float = 2.0
    c_patch: float = 0.1
    c_attn_coeff: float = 6e-7
    attn_exponent: float = 1.5
    patch_size: int = 32


DEFAULT_COST = CostModelParams()


def _validated(comp: dict) -> dict:
    if not comp:
        raise InputError("empty composition")
    for k, v in comp.items():
        if k not in STANDARD_CLASSES:
            raise InputError(f"unknown resolution class {k!r}")
        if v < 0:
            raise InputError(f"negative count for {k!r}")
    if sum(comp.values()) == 0:
        raise InputError("composition has no requests")
    return comp


def _terms(comp: dict, p: CostModelParams):
    """(distinct resolutions, patches, sum of tokens^exponent) of a composition."""
    n_res, patches, attn = 0, 0, 0.0
    for cls, n in _validated(comp).items():
        if n == 0:
            continue
        lat = STANDARD_CLASSES[cls].latent
        if lat % p.patch_size:
            raise InputError(f"patch size {p.patch_size} does not tile {cls}")
        n_res += 1
        patches += n * (lat // p.patch_size) ** 2
        attn += n * float(lat * lat) ** p.attn_exponent
    return n_res, patches, attn


def step_latency(comp: dict, p: CostModelParams = DEFAULT_COST) -> float:
    """latency.py:52-77: fixed + per-resolution + blocks x (patch term + attention term), ms."""
    n_res, patches, attn = _terms(comp, p)
    return p.c_step_fixed + p.c_res_overhead * n_res + p.blocks_per_step * (p.c_patch * patches
                                                                            + p.c_attn_coeff * attn)


def standalone_latency(cls: str, steps: int, p: CostModelParams = DEFAULT_COST) -> float:
    """latency.py:80-84."""
    if steps < 1:
        raise InputError("steps must be >= 1")
    return steps * step_latency({cls: 1}, p)


class AnalyticPredictor:
    """latency.py:256-263: the scheduler's default predictor."""

    def __init__(self, p: CostModelParams = DEFAULT_COST):
        self.cost_params = p

    def predict_step_latency(self, comp: dict) -> float:
        return step_latency(comp, self.cost_params)


class AdaptivePredictor(AnalyticPredictor):
    """Analytic model x an EWMA of measured / predicted step time (wall plane).

    The analytic model prices a step without the patch cache; once the cache
    is warm most patch-blocks are skipped and steps run several times faster.
    The engine reports every measured step (`observe`), so admission and
    time-out decisions track the pace the GPU actually delivers."""

    def __init__(self, p: CostModelParams = DEFAULT_COST, alpha: float = 0.2):
        super().__init__(p)
        self.alpha, self.ratio = alpha, 1.0

    def predict_step_latency(self, comp: dict) -> float:
        return self.ratio * step_latency(comp, self.cost_params)

    def observe(self, comp: dict, measured_ms: float) -> None:
        r = measured_ms / step_latency(comp, self.cost_params)
        # the fitted model is the uncached cost: only the cache's speed-up is learned; slower
        # steps (cold caches, launch overhead of small batches) must not make admission more
        # conservative than the calibrated model (measured: more discards at low load)
        self.ratio = min(1.0, (1.0 - self.alpha) * self.ratio + self.alpha * r)


def fit_cost_model(samples: Sequence[tuple[dict, float]], base: CostModelParams = DEFAULT_COST) -> CostModelParams:
    """Least-squares fit of (c_step_fixed, c_res_overhead, c_patch, c_attn_coeff) to
    measured (composition, step ms) pairs, keeping the exponent and block count.  The residuals
    are relative (each row divided by its measured time), so 2 ms single-request steps weigh as
    much as 20 ms full batches.  Coefficients are clamped at zero (non-negative least squares by
    elimination)."""
    if len(samples) < 4:
        raise InputError("need at least 4 measured compositions to fit the cost model")
    rows, y = [], []
    for comp, ms in samples:
        n_res, patches, attn = _terms(comp, base)
        rows.append([1.0, n_res, base.blocks_per_step * patches, base.blocks_per_step * attn])
        y.append(float(ms))
    A, y = np.asarray(rows), np.asarray(y)
    A, y = A / y[:, None], np.ones_like(y)
    active = list(range(4))
    while True:
        coef = np.zeros(4)
        sol, *_ = np.linalg.lstsq(A[:, active], y, rcond=None)
        coef[active] = sol
        neg = [i for i in active if coef[i] < 0]
        if not neg:
            break
        active.remove(min(neg, key=lambda i: coef[i]))
    return replace(base, c_step_fixed=float(coef[0]), c_res_overhead=float(coef[1]), c_patch=float(coef[2]),
                   c_attn_coeff=float(coef[3]))


# ------------------------------------------------ learned latency model


def composition_features(comp: dict, patch_size: int = 32) -> np.ndarray:
    """Per-class request counts (CLASS_ORDER) plus the step's cost drivers on B200: distinct
    resolutions, patches (the pixel-wise / conv work), sum of T^2 over images (attention work,
    in units of 2^24) -- the reference's features (latency.py:78-91) plus the attention term."""
    _validated(comp)
    counts = [float(comp.get(c, 0)) for c in CLASS_ORDER]
    lat = [STANDARD_CLASSES[c].latent for c in CLASS_ORDER]
    n_res = float(sum(1 for v in counts if v > 0))
    patches = sum(v * (d // patch_size) ** 2 for v, d in zip(counts, lat))
    attn = sum(v * float(d * d) ** 2 for v, d in zip(counts, lat)) / 2.0 ** 24
    return np.array(counts + [n_res, patches, attn], dtype=np.float64)


class MlpLatencyModel:
    """Step-latency predictor learned from measured B200 steps (the paper's MLP predictor,
    latency.py:140-253, retrained on this hardware).

    A 2 x 32 ReLU network on standardised composition features regresses log(step ms), full-batch
    Adam.  With `residual` (default) the net learns log(measured / analytic) on top of the cost
    model fitted to the same samples (fit_cost_model; exponent 2 = the T^2 attention work), so
    the structure extrapolates and the net absorbs what the analytic form misses.
    `fit` returns the training loss; `predict_step_latency(comp)` is the scheduler's predictor
    interface (scheduler.py:126-128)."""

    def __init__(self, hidden=(32, 32), lr: float = 1e-2, epochs: int = 1500, seed: int = 0, patch_size: int = 32,
                 residual: bool = True):
        self.hidden, self.lr, self.epochs, self.seed, self.patch_size = tuple(hidden), lr, epochs, seed, patch_size
        self.residual = residual
        self.base = None  # fitted CostModelParams (residual mode)
        self.params: list = []
        self.mu = self.sd = None

    def _base_ms(self, comps) -> np.ndarray:
        if self.base is None:
            return np.ones(len(comps))
        return np.array([step_latency(c, self.base) for c in comps])

    def _feats(self, comps) -> np.ndarray:
        return np.stack([composition_features(c, self.patch_size) for c in comps])

    def _net(self, xn):
        acts, h = [xn], xn
        for i in range(0, len(self.params), 2):
            h = h @ self.params[i] + self.params[i + 1]
            if i + 2 < len(self.params):
                h = np.maximum(h, 0.0)
            acts.append(h)
        return acts

    def fit(self, comps, ms) -> float:
        ms = np.asarray(ms, dtype=np.float64)
        if np.any(~(ms > 0)):
            raise InputError("step times must be positive")
        self.base = None
        if self.residual:
            self.base = fit_cost_model(list(zip(comps, ms)), replace(DEFAULT_COST, attn_exponent=2.0,
                                                                       patch_size=self.patch_size))
        x, y = self._feats(comps), np.log(ms / self._base_ms(comps))[:, None]
        self.mu, self.sd = x.mean(0), np.maximum(x.std(0), 1e-8)
        xn = (x - self.mu) / self.sd
        rng = np.random.default_rng(self.seed)
        dims = [x.shape[1], *self.hidden, 1]
        self.params = []
        for a, b in zip(dims, dims[1:]):
            self.params += [rng.normal(size=(a, b)) * np.sqrt(2.0 / a), np.zeros(b)]
        m = [np.zeros_like(p) for p in self.params]
        v = [np.zeros_like(p) for p in self.params]
        loss = np.inf
        for t in range(1, self.epochs + 1):
            acts = self._net(xn)
            err = acts[-1] - y
            loss = float(np.mean(err ** 2))
            g = 2.0 * err / len(xn)
            grads = [None] * len(self.params)
            for li in range(len(self.params) // 2 - 1, -1, -1):
                grads[2 * li] = acts[li].T @ g
                grads[2 * li + 1] = g.sum(0)
                if li:
                    g = (g @ self.params[2 * li].T) * (acts[li] > 0)
            for j, (p, gr) in enumerate(zip(self.params, grads)):
                m[j] = 0.9 * m[j] + 0.1 * gr
                v[j] = 0.999 * v[j] + 0.001 * gr * gr
                p -= self.lr * (m[j] / (1 - 0.9 ** t)) / (np.sqrt(v[j] / (1 - 0.999 ** t)) + 1e-8)
        return loss

    def predict(self, comps) -> np.ndarray:
        if not self.params:
            raise InputError("latency model is not trained")
        return self._base_ms(comps) * np.exp(self._net((self._feats(comps) - self.mu) / self.sd)[-1][:, 0])

    def predict_step_latency(self, comp: dict) -> float:
        return float(self.predict([comp])[0])


class LearnedPredictor:
    """Scheduler predictor on the MLP, optionally following the measured pace: step time =
    MLP(comp) x EWMA(measured / MLP) clamped <= 1 (the cache's speed-up, as AdaptivePredictor)."""

    def __init__(self, model: MlpLatencyModel, alpha: float = 0.2, adaptive: bool = True):
        self.model, self.alpha, self.adaptive, self.ratio = model, alpha, adaptive, 1.0

    def predict_step_latency(self, comp: dict) -> float:
        return self.ratio * self.model.predict_step_latency(comp)

    def observe(self, comp: dict, measured_ms: float) -> None:
        if self.adaptive:
            r = measured_ms / self.model.predict_step_latency(comp)
            self.ratio = min(1.0, (1.0 - self.alpha) * self.ratio + self.alpha * r)


def random_compositions(n: int, seed: int = 0, max_batch: int = 12, classes=("low", "med", "high")) -> list:
    """n distinct compositions of 1..max_batch requests over `classes` (latency.py:102-123)."""
    rng = np.random.default_rng(seed)
    seen, out = set(), []
    while len(out) < n:
        k = int(rng.integers(1, max_batch + 1))
        counts = np.bincount(rng.integers(0, len(classes), size=k), minlength=len(classes))
        key = tuple(int(c) for c in counts)
        if key in seen:
            continue
        seen.add(key)
        out.append({c: v for c, v in zip(classes, key) if v})
    return out


# ------------------------------------------------------------- workload

DEFAULT_WEIGHTS = {"low": 0.4, "med": 0.35, "high": 0.25}


@dataclass(frozen=True)
class WorkloadConfig:
    """workload.py:23-48."""

    seed: int = 0
    qps: float = 1.0
    n_requests: int = 100
    class_weights: dict = field(default_factory=lambda: dict(DEFAULT_WEIGHTS))
    slo_scale: float = 3.0
    steps: int = 50

    def __post_init__(self):
        if self.qps <= 0:
            raise InputError("qps must be positive")
        if self.n_requests < 1:
            raise InputError("n_requests must be >= 1")
        if self.slo_scale <= 0:
            raise InputError("slo_scale must be positive")
        if self.steps < 1:
            raise InputError("steps must be >= 1")
        if any(c not in STANDARD_CLASSES for c in self.class_weights):
            raise InputError(f"unknown resolution class in {sorted(self.class_weights)}")
        if any(w < 0 for w in self.class_weights.values()):
            raise InputError("class weights must be nonnegative")
        if sum(self.class_weights.values()) <= 0:
            raise InputError("class weights must not all be zero")


@dataclass(frozen=True)
class TraceRow:
    request_id: str
    arrival_ms: float
    resolution_class: str
    slo_ms: float


def generate_trace(cfg: WorkloadConfig, cost: CostModelParams = DEFAULT_COST, predictor=None) -> list[TraceRow]:
    """workload.py:58-77: exponential gaps then weighted class picks from one seeded stream.
    SLO budget = slo_scale x the standalone latency of the class: from `cost` (the reference's
    semantics) or, when given, from `predictor`'s one-request step latency x steps."""
    rng = np.random.default_rng(cfg.seed)
    arrivals = np.cumsum(rng.exponential(scale=1000.0 / cfg.qps, size=cfg.n_requests))
    names = sorted(cfg.class_weights)
    w = np.asarray([cfg.class_weights[n] for n in names], dtype=np.float64)
    picks = rng.choice(len(names), size=cfg.n_requests, p=w / w.sum())
    if predictor is not None:
        budget = {n: cfg.slo_scale * cfg.steps * predictor.predict_step_latency({n: 1}) for n in names}
    else:
        budget = {n: cfg.slo_scale * standalone_latency(n, cfg.steps, cost) for n in names}
    return [TraceRow(f"req-{i:05d}", float(arrivals[i]), names[int(k)], budget[names[int(k)]])
            for i, k in enumerate(picks)]


def write_trace(rows: Sequence[TraceRow], path) -> None:
    """JSONL, one object per row (workload.py:80-89)."""
    with open(path, "w") as f:
        for r in rows:
            f.write(json.dumps({"request_id": r.request_id, "arrival_ms": r.arrival_ms,
                                "resolution_class": r.resolution_class, "slo_ms": r.slo_ms}) + "\n")


def read_trace(path) -> list[TraceRow]:
    """workload.py:92-113 (InputError on malformed, empty or unsorted traces)."""
    rows = []
    with open(path) as f:
        for n, line in enumerate(f, 1):
            if not line.strip():
                continue
            try:
                d = json.loads(line)
                rows.append(TraceRow(d["request_id"], float(d["arrival_ms"]), d["resolution_class"],
                                     float(d["slo_ms"])))
            except (KeyError, ValueError) as exc:
                raise InputError(f"{path}:{n}: bad trace row: {exc}") from exc
    if not rows:
        raise InputError(f"{path}: empty trace")
    if any(b.arrival_ms < a.arrival_ms for a, b in zip(rows, rows[1:])):
        raise InputError(f"{path}: arrivals are not sorted")
    return rows


# ------------------------------------------------------------- scheduler

POLICIES = ("slo_aware", "fcfs", "sequential")


@dataclass
class RequestMeta:
    """scheduler.py:25-50."""

    request_id: str
    cls: str
    arrival_ms: float
    slo_ms: float
    total_steps: int
    remaining_steps: int = -1

    def __post_init__(self):
        if self.cls not in STANDARD_CLASSES:
            raise InputError(f"unknown resolution class {self.cls!r}")
        if self.total_steps < 1:
            raise InputError("total_steps must be >= 1")
        if self.remaining_steps < 0:
            self.remaining_steps = self.total_steps

    @property
    def deadline_ms(self) -> float:
        return self.arrival_ms + self.slo_ms

    @property
    def pixels(self) -> int:
        return STANDARD_CLASSES[self.cls].pixel ** 2


@dataclass(frozen=True)
class SchedulerConfig:
    """scheduler.py:53-64."""

    policy: str = "slo_aware"
    max_active: int = 12
    theta_mode: float = 2.0
    cost: CostModelParams = field(default_factory=CostModelParams)

    def __post_init__(self):
        if self.policy not in POLICIES:
            raise InputError(f"policy must be one of {POLICIES}, got {self.policy!r}")
        if self.max_active < 1:
            raise InputError("max_active must be >= 1")


@dataclass
class TickResult:
    admitted: list
    discarded: list


def composition(requests) -> dict:
    comp: dict = {}
    for r in requests:
        comp[r.cls] = comp.get(r.cls, 0) + 1
    return comp


def slack(req: RequestMeta, now_ms: float, predicted_remaining_ms: float,
          cost: CostModelParams = DEFAULT_COST) -> float:
    """scheduler.py:81-90: spare time in units of the request's standalone latency."""
    return (req.deadline_ms - now_ms - predicted_remaining_ms) / standalone_latency(req.cls, req.total_steps, cost)


def time_out(req: RequestMeta, now_ms: float, predicted_remaining_ms: float) -> bool:
    return now_ms + predicted_remaining_ms > req.deadline_ms


class Scheduler:
    """Admission policy (scheduler.py:98-177); owns no queues."""

    def __init__(self, cfg: SchedulerConfig | None = None, predictor=None):
        self.cfg = cfg or SchedulerConfig()
        self.predictor = predictor or AnalyticPredictor(self.cfg.cost)

    def tick(self, now_ms: float, active: list, waiting: list) -> TickResult:
        if self.cfg.policy == "slo_aware":
            return self._slo_aware(now_ms, list(active), list(waiting))
        cap = 1 if self.cfg.policy == "sequential" else self.cfg.max_active
        queue = sorted(waiting, key=lambda r: (r.arrival_ms, r.request_id))
        room = max(0, cap - len(active))
        return TickResult(admitted=queue[:room], discarded=[])

    def _step_ms(self, batch) -> float:
        return self.predictor.predict_step_latency(composition(batch))

    def _slo_aware(self, now: float, active: list, pool: list) -> TickResult:
        cost = self.cfg.cost
        out = TickResult([], [])
        while pool and len(active) < self.cfg.max_active:
            # least slack first, each candidate priced at the pace of the batch it would join
            best = None
            for w in pool:
                rem = self._step_ms(active + [w]) * w.remaining_steps
                key = (slack(w, now, rem, cost), w.arrival_ms, w.request_id)
                if best is None or key < best[0]:
                    best = (key, w, rem)
            (s_min, _, _), cand, rem = best
            if time_out(cand, now, rem):
                out.discarded.append(cand)
                pool.remove(cand)
                continue
            if s_min > self.cfg.theta_mode:
                # nobody urgent: maximise pixel throughput of the grown batch
                px = sum(r.pixels for r in active)
                cand = min(pool, key=lambda w: (-(px + w.pixels) / self._step_ms(active + [w]), w.arrival_ms,
                                                w.request_id))
            if active:
                step = self._step_ms(active + [cand])
                tight = min(active, key=lambda a: (slack(a, now, step * a.remaining_steps, cost), a.arrival_ms,
                                                   a.request_id))
                if time_out(tight, now, step * tight.remaining_steps):
                    break
            active.append(cand)
            pool.remove(cand)
            out.admitted.append(cand)
        return out


# ---------------------------------------------------------------- engine

PLANES = ("cost_only", "numeric", "wall")


@dataclass(frozen=True)
class EngineConfig:
    """engine.py:34-52, plus the `wall` plane."""

    plane: str = "cost_only"
    n_workers: int = 1
    total_steps: int = 50
    patch_size: int = 32
    use_cache: bool = True
    latent_seed: int = 0
    scheduler: SchedulerConfig = field(default_factory=SchedulerConfig)
    cost: CostModelParams = field(default_factory=CostModelParams)
    model: object = None            # model.ModelConfig (None -> the reference default)
    cache: object = None            # cache.PredictorConfig (None -> defaults)
    # GPU planes: capture the cached step of a composition as a CUDA graph once it has run this many
    # eager steps unchanged (0 = never).  A capture costs 10-100 ms of host time on the clock
    # (tools/serving_probe.py) against ~0.5 ms saved per replay, and a Poisson trace changes the
    # composition every few steps, so the default serves eagerly.
    graph_after_steps: int = 0

    def __post_init__(self):
        if self.plane not in PLANES:
            raise InputError(f"plane must be one of {PLANES}, got {self.plane!r}")
        if self.n_workers < 1:
            raise InputError("n_workers must be >= 1")
        if self.total_steps < 1:
            raise InputError("total_steps must be >= 1")


@dataclass
class RunResult:
    events: list
    completions: list
    summary: dict
    latents: dict = field(default_factory=dict)


class _Worker:
    def __init__(self, wid: int):
        self.wid = wid
        self.active: list = []
        self.waiting: list = []
        self.busy = False
        self.steps_run = 0
        self.latents: dict = {}
        self.prompts: dict = {}
        self.cache = None
        self.step_ms: list = []   # measured device time per step (wall plane)
        self.batch = None         # resident CSP batch of the active set (GPU planes)
        self.batch_ids = None
        self.graph = None         # CachedStepGraph of that composition
        self.comp_steps = 0       # steps run since the composition last changed


class Engine:
    """Discrete-event serving loop (engine.py:72-250).

    Events are ordered by (time, insertion sequence); all events sharing a
    timestamp are applied before any worker ticks, then idle touched workers
    tick in worker order.  A step's duration is the analytic step latency
    (cost_only / numeric) or the measured device time of the step (wall).
    """

    def __init__(self, cfg: EngineConfig | None = None, predictor=None, weights=None):
        self.cfg = cfg or EngineConfig()
        self.scheduler = Scheduler(self.cfg.scheduler, predictor)
        self.model_cfg = self.cfg.model
        self.weights = weights
        if self.cfg.plane != "cost_only":
            from .model import ModelConfig, init_weights
            if self.model_cfg is None:
                self.model_cfg = ModelConfig()
            if self.weights is None:
                self.weights = init_weights(self.model_cfg)

    # ------------------------------------------------------------ compute
    def _new_cache(self):
        from .cache import BlockCache, PredictorConfig
        return BlockCache(self.model_cfg.n_blocks, self.cfg.cache or PredictorConfig())

    def _admit_latent(self, w: _Worker, meta: RequestMeta, idx: int) -> None:
        import torch

        from ._dev import require_cuda
        from .model import make_prompt
        d = STANDARD_CLASSES[meta.cls].latent
        lat = np.random.default_rng([self.cfg.latent_seed, idx]).normal(size=(self.model_cfg.channels, d, d))
        w.latents[meta.request_id] = torch.as_tensor(lat, dtype=torch.float32, device=require_cuda())
        w.prompts[meta.request_id] = make_prompt(self.model_cfg, meta.request_id)

    def _materialize(self, w: _Worker) -> None:
        """Resident CSP batch -> per-request latents (on a composition change)."""
        from .csp import reassemble
        if w.batch is not None:
            for rid, lat in reassemble(w.batch, w.batch.data).items():
                w.latents[rid] = lat
        w.batch, w.batch_ids, w.graph = None, None, None
        w.comp_steps = 0

    def _compute_step(self, w: _Worker) -> float:
        """One denoising step of w's active batch on the GPU; returns its device time in ms.

        The batch's fp32 latents stay resident in CSP layout across steps and are re-split only
        when the composition changes (an admission or a completion); while it is unchanged, the
        cached step runs as one CUDA graph (engine_step.CachedStepGraph: the reuse test,
        compaction and every block replay without the host) -- the reference re-splits and
        reassembles every step (engine.py:129,159-160)."""
        import torch

        from ._dev import require_cuda
        from .csp import split
        from .engine_step import CachedStepGraph, numeric_step
        from .model import rate_schedule
        from .patched import device_compaction_ok
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        ids = tuple(r.request_id for r in w.active)
        if w.batch_ids is None or set(w.batch_ids) != set(ids):
            self._materialize(w)
            w.batch = split([(rid, w.latents.pop(rid)) for rid in ids], patch_size=self.cfg.patch_size)
            w.batch_ids = ids
        if (w.graph is None and self.cfg.use_cache and self.cfg.graph_after_steps > 0 and w.cache is not None
                and w.comp_steps >= self.cfg.graph_after_steps and device_compaction_ok(w.batch)):
            w.graph = CachedStepGraph(w.batch, self.weights, w.cache)
        batch = w.batch
        order = [self._meta[e.request_id] for e in batch.requests]
        dev = require_cuda()
        bias = torch.as_tensor(np.stack([w.prompts[m.request_id] for m in order]), dtype=torch.float32, device=dev)
        rates = torch.as_tensor([rate_schedule(m.total_steps - m.remaining_steps, m.total_steps) for m in order],
                                dtype=torch.float32, device=dev)
        if w.graph is not None:
            new, st = w.graph.run(batch.data, bias, rates)
        else:
            cache = w.cache if self.cfg.use_cache else None
            new, st = numeric_step(batch, self.weights, cache, bias, rates)
        batch.data = new
        w.comp_steps += 1
        t1.record()
        t1.synchronize()
        self._skipped += st.skipped
        self._computed += st.computed
        return float(t0.elapsed_time(t1))

    # ------------------------------------------------------------ the loop
    def run(self, trace: Sequence[TraceRow]) -> RunResult:
        if not trace:
            raise InputError("empty trace")
        cfg = self.cfg
        workers = [_Worker(i) for i in range(cfg.n_workers)]
        if cfg.plane != "cost_only":
            for w in workers:
                w.cache = self._new_cache() if cfg.use_cache else None
        events, completions, final = [], [], {}
        self._skipped = self._computed = 0
        self._meta = {}
        heap: list = []
        seq = [0]

        def push(t, kind, payload):
            heapq.heappush(heap, (t, seq[0], kind, payload))
            seq[0] += 1

        def log(t, kind, rid, wid):
            events.append({"t_ms": round(t, 9), "kind": kind, "request_id": rid, "worker": wid})

        index = {}
        for i, row in enumerate(trace):
            m = RequestMeta(row.request_id, row.resolution_class, row.arrival_ms, row.slo_ms, cfg.total_steps)
            self._meta[row.request_id] = m
            index[row.request_id] = i
            push(row.arrival_ms, "arrival", row.request_id)

        unit = {c: step_latency({c: 1}, cfg.cost) for c in sorted({r.resolution_class for r in trace})}

        def backlog(w):  # engine.py:120-124
            return sum(r.remaining_steps * unit[r.cls] for r in w.active + w.waiting)

        def record_done(m, t, wid, discarded):
            completions.append({
                "request_id": m.request_id, "resolution_class": m.cls,
                "arrival_ms": round(m.arrival_ms, 9), "finish_ms": round(t, 9),
                "latency_ms": round(t - m.arrival_ms, 9), "slo_ms": round(m.slo_ms, 9),
                "met_slo": bool(not discarded and t <= m.deadline_ms), "discarded": bool(discarded),
                "worker": wid,
            })

        def begin(w, now):
            w.busy = True
            w.steps_run += 1
            if cfg.plane == "cost_only":
                dt = step_latency(composition(w.active), cfg.cost)
            else:
                dt_dev = self._compute_step(w)
                w.step_ms.append(dt_dev)
                observe = getattr(self.scheduler.predictor, "observe", None)
                if observe is not None and cfg.plane == "wall":
                    observe(composition(w.active), dt_dev)
                dt = dt_dev if cfg.plane == "wall" else step_latency(composition(w.active), cfg.cost)
            push(now + dt, "step_end", w.wid)

        def finish(w, now):
            w.busy = False
            for r in w.active:
                r.remaining_steps -= 1
            done = [r for r in w.active if r.remaining_steps == 0]
            if done and cfg.plane != "cost_only":
                self._materialize(w)
            for r in done:
                w.active.remove(r)
                log(now, "complete", r.request_id, w.wid)
                record_done(r, now, w.wid, False)
                if cfg.plane != "cost_only":
                    final[r.request_id] = w.latents.pop(r.request_id)
                    w.prompts.pop(r.request_id, None)
            if done and w.cache is not None:
                live = [(r.request_id, k) for r in w.active
                        for k in range((STANDARD_CLASSES[r.cls].latent // cfg.patch_size) ** 2)]
                w.cache.evict_expired(live)

        def tick(w, now):
            res = self.scheduler.tick(now, w.active, w.waiting)
            for r in res.discarded:
                w.waiting.remove(r)
                log(now, "discard", r.request_id, w.wid)
                record_done(r, now, w.wid, True)
            for r in res.admitted:
                w.waiting.remove(r)
                w.active.append(r)
                log(now, "admit", r.request_id, w.wid)
            if w.active and not w.busy:
                begin(w, now)

        while heap:
            now = heap[0][0]
            touched = []
            while heap and heap[0][0] == now:
                _, _, kind, payload = heapq.heappop(heap)
                if kind == "arrival":
                    m = self._meta[payload]
                    w = min(workers, key=lambda k: (backlog(k), k.wid))
                    w.waiting.append(m)
                    log(now, "arrival", m.request_id, w.wid)
                    if cfg.plane != "cost_only":
                        self._admit_latent(w, m, index[m.request_id])
                else:
                    w = workers[payload]
                    finish(w, now)
                if w not in touched:
                    touched.append(w)
            for w in sorted(touched, key=lambda k: k.wid):
                if not w.busy:
                    tick(w, now)

        return RunResult(events, completions, self._summary(trace, completions, workers), final)

    def _summary(self, trace, completions, workers) -> dict:
        """engine.py:252-280."""
        met = sum(1 for c in completions if c["met_slo"])
        fin = sorted(c["latency_ms"] for c in completions if not c["discarded"])
        horizon = max([c["finish_ms"] for c in completions] + [r.arrival_ms for r in trace])
        out = {
            "n_requests": len(trace),
            "n_completed": len(fin),
            "n_discarded": len(completions) - len(fin),
            "n_met_slo": met,
            "slo_attainment": met / len(trace),
            "goodput_rps": 1000.0 * met / horizon if horizon > 0 else 0.0,
            "mean_latency_ms": sum(fin) / len(fin) if fin else 0.0,
            "p95_latency_ms": fin[int(0.95 * (len(fin) - 1))] if fin else 0.0,
            "makespan_ms": horizon,
            "steps_run": sum(w.steps_run for w in workers),
            "skipped_patches": self._skipped,
            "computed_patches": self._computed if self.cfg.plane != "cost_only" else 0,
        }
        if self.cfg.plane != "cost_only" and self.cfg.use_cache:
            agg: dict = {}
            for w in workers:
                for k, v in w.cache.stats.as_dict().items():
                    agg[k] = agg.get(k, 0) + v
            out["cache"] = agg
        if self.cfg.plane != "cost_only":
            ms = [x for w in workers for x in w.step_ms]
            out["device_step_ms_mean"] = float(np.mean(ms)) if ms else 0.0
        return out


# --------------------------------------------------------- calibration


def measure_step_ms(model_cfg, weights, comps: Sequence[dict], patch_size: int = 32, reps: int = 3,
                    use_cache: bool = False, seed: int = 0, steps: int = 50) -> list[tuple[dict, float]]:
    """Measured device time (ms) of one steady-state denoising step for each composition, through
    the call the wall plane makes on a resident batch (numeric_step on the CSP latents; the split
    happens once per composition, as in the wall plane).

    Without the cache: median of `reps` steps after one warm-up step (the first step on a new
    batch also builds its plans).  With the cache: the composition is denoised for 12 steps with
    a BlockCache in the loop (outputs fed back as latents); the result is the lifetime-weighted
    mean of a request served for `steps` steps -- the first 4 (cold cache) weighted 4/steps, the
    steady state the rest."""
    import torch

    from ._dev import require_cuda
    from .cache import BlockCache, PredictorConfig
    from .csp import split
    from .engine_step import numeric_step
    dev = require_cuda()
    out = []
    for comp in comps:
        reqs = []
        # seeded N(0,1) latents drawn on the device (a host normal() of 64 x 320 x 128^2 doubles
        # took seconds per composition); the step time does not depend on the values
        gen = torch.Generator(device=dev).manual_seed(seed)
        for cls in CLASS_ORDER:
            for j in range(comp.get(cls, 0)):
                d = STANDARD_CLASSES[cls].latent
                reqs.append((f"{cls}{j}", torch.randn((model_cfg.channels, d, d), generator=gen, device=dev)))
        b = split(reqs, patch_size=patch_size)
        bias = torch.zeros((b.n_requests, model_cfg.channels), dtype=torch.float32, device=dev)
        rates = torch.full((b.n_requests,), 0.1, dtype=torch.float32, device=dev)
        cache = BlockCache(model_cfg.n_blocks, PredictorConfig()) if use_cache else None
        n_runs = 12 if use_cache else reps + 1
        times = []
        # host stalls (a Python GC pass, measured up to ~250 ms once in a long bench process)
        # would land inside the event pair: no collection while a composition is timed
        gc_was = gc.isenabled()
        gc.disable()
        for rep in range(n_runs):
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            new, _ = numeric_step(b, weights, cache, bias, rates)
            t1.record()
            t1.synchronize()
            times.append(t0.elapsed_time(t1))
            if use_cache:
                b.data = new
        if gc_was:
            gc.enable()
        if os.environ.get("PS_CALIB_DEBUG"):
            print("calibration", dict(comp), [round(t, 3) for t in times],
                  f"reserved {torch.cuda.memory_reserved() / 2**30:.1f} GiB",
                  f"allocated {torch.cuda.memory_allocated() / 2**30:.1f} GiB", file=sys.stderr, flush=True)
        if use_cache:
            cold, warm = float(np.mean(times[:4])), float(np.mean(times[4:]))
            k = min(4, steps)
            ms = (k * cold + (steps - k) * warm) / steps
        else:
            ms = float(np.median(times[1:]))
        out.append((dict(comp), ms))
    return out


CALIBRATION_COMPS = ({"low": 1}, {"med": 1}, {"high": 1}, {"low": 4, "med": 4, "high": 4},
                     {"low": 2, "high": 2}, {"med": 3}, {"low": 6}, {"high": 4}, {"low": 1, "med": 1, "high": 1})


def calibrate_latency_model(model_cfg, weights, n_compositions: int = 240, n_train: int = 200,
                            max_batch: int = 12, reps: int = 3, seed: int = 0, classes=("low", "med", "high"),
                            patch_size: int = 32):
    """Measure n_compositions distinct random batch compositions (1..max_batch requests) on the
    GPU (measure_step_ms, uncached), train the MLP latency model on n_train of them (PAPER.md:
    480-484: 200 compositions) and report its mean relative error on the held-out rest.
    Returns (model, report)."""
    comps = random_compositions(n_compositions, seed=seed, max_batch=max_batch, classes=classes)
    np.random.default_rng(seed + 1).shuffle(comps)
    samples = measure_step_ms(model_cfg, weights, comps, patch_size=patch_size, reps=reps)
    ms = np.array([m for _, m in samples])
    model = MlpLatencyModel(patch_size=patch_size)
    loss = model.fit(comps[:n_train], ms[:n_train])
    held = comps[n_train:]
    pred = model.predict(held) if held else np.zeros(0)
    rel = np.abs(pred - ms[n_train:]) / ms[n_train:] if held else np.zeros(0)
    rel_train = np.abs(model.predict(comps[:n_train]) - ms[:n_train]) / ms[:n_train]
    analytic = np.array([step_latency(c, model.base) for c in held]) if held else np.zeros(0)
    return model, {
        "n_measured": len(comps), "n_train": n_train, "n_heldout": len(held), "max_batch": max_batch,
        "train_log_mse": loss, "train_mean_rel_err": float(rel_train.mean()),
        "heldout_mean_rel_err": float(rel.mean()) if held else None,
        "heldout_max_rel_err": float(rel.max()) if held else None,
        "heldout_mean_rel_err_analytic_only": float((np.abs(analytic - ms[n_train:]) / ms[n_train:]).mean())
        if held else None,
        "step_ms_range": [float(ms.min()), float(ms.max())],
        "analytic_base": {k: getattr(model.base, k) for k in ("c_step_fixed", "c_res_overhead", "c_patch",
                                                               "c_attn_coeff", "attn_exponent")},
    }


def slo_run(model_cfg, weights, n_requests: int = 64, load: float = 0.9, steps: int = 50, seed: int = 0,
            use_cache: bool = True, policy: str = "slo_aware", max_active: int = 12, slo_scale: float = 3.0,
            rank: int = 0, world: int = 1, share=None, gather=None, adaptive: bool = True,
            latency_model=None, n_calib: int = 240, calib_report=None) -> dict:
    """SLO attainment of the B200 path in the wall plane.

    1. the step-latency model: an MLP trained on >= 200 measured B200 compositions of up to
       max_active requests (calibrate_latency_model; rank 0's model is shared through `share`;
       pass `latency_model` to reuse one across runs);
    2. a trace whose SLO budgets are slo_scale x the model's standalone latency (workload.py:74)
       at `load` x the capacity of `world` GPUs serving full 12-request mixed batches without
       the cache;
    3. dispatch requests to GPUs lowest-outstanding-work first (engine.py:228) on the model's
       analytic base (a cost_only run with `world` workers, the same on every rank), then each
       rank serves its requests with `policy`, every step run and timed on its device (resident
       CSP latents, one CUDA graph per composition); completions pooled through `gather`.  With
       `adaptive` the scheduler's predictor follows the measured pace (LearnedPredictor)."""
    model, report = latency_model, calib_report
    if model is None:
        model, report = calibrate_latency_model(model_cfg, weights, n_compositions=n_calib,
                                                max_batch=max_active, seed=seed)
    if share is not None:
        model, report = share((model, report))
    fit = model.base
    full = {"low": 4, "med": 4, "high": 4}
    capacity_rps = world * 12 * 1000.0 / (steps * model.predict_step_latency(full))
    qps = load * capacity_rps
    wc = WorkloadConfig(seed=seed, qps=qps, n_requests=n_requests, steps=steps, slo_scale=slo_scale)
    trace = generate_trace(wc, fit, predictor=model)
    sched = SchedulerConfig(policy=policy, max_active=max_active, cost=fit)
    mine = trace
    if world > 1:
        plan = Engine(EngineConfig(plane="cost_only", n_workers=world, total_steps=steps, cost=fit,
                                   scheduler=sched)).run(trace)
        owner = {e["request_id"]: e["worker"] for e in plan.events if e["kind"] == "arrival"}
        mine = [r for r in trace if owner[r.request_id] == rank]
    ec = EngineConfig(plane="wall", total_steps=steps, use_cache=use_cache, cost=fit, model=model_cfg,
                      scheduler=sched)
    pred = LearnedPredictor(model, adaptive=adaptive)
    res = Engine(ec, predictor=pred, weights=weights).run(mine) if mine else None
    local = {"completions": res.completions if res else [], "steps_run": res.summary["steps_run"] if res else 0,
             "skipped": res.summary["skipped_patches"] if res else 0,
             "computed": res.summary["computed_patches"] if res else 0,
             "step_ms": res.summary["device_step_ms_mean"] if res else 0.0}
    parts = gather(local) if gather is not None else [local]
    comp = [c for p in parts for c in p["completions"]]
    met = sum(1 for c in comp if c["met_slo"])
    fin = sorted(c["latency_ms"] for c in comp if not c["discarded"])
    horizon = max([c["finish_ms"] for c in comp] + [r.arrival_ms for r in trace])
    return {
        "slo_attainment": met / len(trace), "goodput_rps": 1000.0 * met / horizon, "qps": qps, "load": load,
        "n_gpus": world, "n_requests": n_requests, "steps": steps, "policy": policy, "max_active": max_active,
        "use_cache": use_cache, "slo_scale": slo_scale, "n_met_slo": met,
        "predictor": "MLP on measured B200 steps" + (" x EWMA(measured/predicted)" if adaptive else ""),
        "n_discarded": sum(1 for c in comp if c["discarded"]),
        "mean_latency_ms": float(np.mean(fin)) if fin else 0.0,
        "p95_latency_ms": fin[int(0.95 * (len(fin) - 1))] if fin else 0.0, "makespan_ms": horizon,
        "steps_run": sum(p["steps_run"] for p in parts),
        "device_step_ms_mean": float(np.mean([p["step_ms"] for p in parts if p["steps_run"]] or [0.0])),
        "skipped_patches": sum(p["skipped"] for p in parts), "computed_patches": sum(p["computed"] for p in parts),
        "latency_model": report,
    }
