"""The cache-in-the-loop step (engine.py:126-160): active-patch compaction is
exact, and the fused device sequence equals the reference's op-by-op sequence
(predict_reuse -> gather -> masked_block_forward -> batched_fill -> batched_update)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2501_09253_b200 as ps  # noqa: E402
from paper_2501_09253_b200 import model as psm  # noqa: E402
from paper_2501_09253_b200.engine_step import numeric_step  # noqa: E402
from paper_2501_09253_b200.model import step_inputs  # noqa: E402
from paper_2501_09253_b200.patched import run_block_active  # noqa: E402


def _setup(seed=0, dims=(32, 64, 48, 32), c=64, ps_=16):
    cfg = ps.ModelConfig(arch="unet_like", channels=c, hidden=2 * c, n_blocks=3, groups=8, seed=seed)
    w = ps.init_weights(cfg)
    rng = np.random.default_rng(seed)
    reqs = [(f"r{i}", torch.tensor(rng.normal(size=(c, d, d)), dtype=torch.float32)) for i, d in enumerate(dims)]
    return cfg, w, reqs, ps.split(reqs, patch_size=ps_)


@pytest.mark.parametrize("seed", [0, 1])
def test_compacted_block_rows_bit_identical(seed):
    cfg, w, reqs, b = _setup(seed)
    rng = np.random.default_rng(100 + seed)
    active = rng.random(b.n_patches) < 0.3
    active[b.patches_of_request("r3")] = False  # one image entirely reused
    x = b.data.to(torch.bfloat16)
    full = ps.run_block(b, x, w[0])
    part = run_block_active(b, x, w[0], active)
    sel = torch.as_tensor(active, device="cuda")
    assert torch.equal(full[sel], part[sel])


def test_fused_cache_step_equals_reference_sequence():
    cfg, w, reqs, b = _setup(2)
    prompts = {rid: ps.make_prompt(cfg, rid) for rid, _ in reqs}
    keys = b.patch_keys()
    fused = ps.BlockCache(cfg.n_blocks, ps.PredictorConfig(mse_threshold=0.05, max_streak=3))
    seq = ps.BlockCache(cfg.n_blocks, ps.PredictorConfig(mse_threshold=0.05, max_streak=3))
    data_f = data_s = b.data.clone()
    total_skipped = 0
    for s in range(6):
        si = dict.fromkeys(prompts, s)
        bias, rates = step_inputs(cfg, b, prompts, si, dict.fromkeys(prompts, 50))
        b.data = data_f
        data_f, st = numeric_step(b, w, fused, bias, rates, keys=keys)
        total_skipped += st.skipped
        # reference op-by-op sequence through the drop-in API
        b.data = data_s
        h = psm.prompt_bias(b, data_s, bias)
        for blk, ops in enumerate(w):
            mask = seq.predict_reuse(blk, keys, h)
            ci, co = seq.gather(blk, keys, mask, h.shape[1:])
            y = ps.masked_block_forward(b, h, mask.cpu().numpy(), ops, ci, co)
            seq.batched_fill(blk, keys, mask)
            seq.batched_update(blk, keys, mask, h, y)
            h = y
        data_s = psm.blend_batch(b, data_s, h, rates)
        assert torch.equal(data_f, data_s), s
        assert fused.stats.as_dict() == seq.stats.as_dict()
    assert total_skipped > 0  # the sweep exercised reuse


def test_compaction_off_matches_on():
    cfg, w, reqs, b = _setup(3)
    prompts = {rid: ps.make_prompt(cfg, rid) for rid, _ in reqs}
    c1 = ps.BlockCache(cfg.n_blocks, ps.PredictorConfig(mse_threshold=0.1, max_streak=2))
    c2 = ps.BlockCache(cfg.n_blocks, ps.PredictorConfig(mse_threshold=0.1, max_streak=2))
    d1 = d2 = b.data.clone()
    for s in range(5):
        bias, rates = step_inputs(cfg, b, prompts, dict.fromkeys(prompts, s), dict.fromkeys(prompts, 50))
        b.data = d1
        d1, s1 = numeric_step(b, w, c1, bias, rates, compact=True)
        b.data = d2
        d2, s2 = numeric_step(b, w, c2, bias, rates, compact=False)
        assert torch.equal(d1, d2)
        assert (s1.skipped, s1.computed) == (s2.skipped, s2.computed)
        assert s1.rows_run <= s2.rows_run


@pytest.mark.parametrize("seed,ps_,frac", [(0, 16, 0.3), (1, 32, 0.5), (2, 16, 0.0), (3, 16, 1.0)])
def test_device_lists_block_bit_identical(seed, ps_, frac):
    """run_block_masked (compaction lists built on the device from the device mask, work
    counts read by the kernels) against run_block_active with the host mask."""
    from paper_2501_09253_b200.patched import run_block_masked
    dims = (32, 64, 96, 32) if ps_ == 32 else (32, 64, 48, 32)
    cfg, w, reqs, b = _setup(seed, dims=dims, ps_=ps_)
    rng = np.random.default_rng(200 + seed)
    active = rng.random(b.n_patches) < frac
    if 0 < frac < 1:
        active[b.patches_of_request("r3")] = False
    x = b.data.to(torch.bfloat16)
    reused = torch.as_tensor(~active, device="cuda")
    got, counts = run_block_masked(b, x, w[0], reused)
    c = counts.cpu().numpy()
    assert c[4] == active.sum()
    live = np.isin(b.request_index, np.unique(b.request_index[active]))
    assert c[5] == live.sum()
    if active.any():
        want = run_block_active(b, x, w[0], active) if not active.all() else ps.run_block(b, x, w[0])
        sel = torch.as_tensor(active, device="cuda")
        assert torch.equal(got[sel], want[sel])


def test_device_compaction_step_equals_host_readback(monkeypatch):
    """numeric_step without any per-block read-back equals the read-back path (outputs,
    StepStats, cache counters) over a run with partial, full and no reuse."""
    from paper_2501_09253_b200 import engine_step
    cfg, w, reqs, b = _setup(4, dims=(32, 64, 96, 32), ps_=32)
    prompts = {rid: ps.make_prompt(cfg, rid) for rid, _ in reqs}
    keys = b.patch_keys()
    caches = [ps.BlockCache(cfg.n_blocks, ps.PredictorConfig(mse_threshold=0.08, max_streak=2)) for _ in range(2)]
    data = [b.data.clone(), b.data.clone()]
    kinds = set()
    for s in range(6):
        bias, rates = step_inputs(cfg, b, prompts, dict.fromkeys(prompts, s), dict.fromkeys(prompts, 50))
        outs = []
        for i, dev in enumerate((True, False)):
            monkeypatch.setattr(engine_step, "DEVICE_COMPACTION", dev)
            b.data = data[i]
            data[i], st = numeric_step(b, w, caches[i], bias, rates, keys=keys)
            outs.append(st)
        assert torch.equal(data[0], data[1]), s
        assert (outs[0].skipped, outs[0].computed) == (outs[1].skipped, outs[1].computed)
        assert caches[0].stats.as_dict() == caches[1].stats.as_dict()
        kinds.add("partial" if 0 < outs[0].skipped < b.n_patches * cfg.n_blocks else str(outs[0].skipped))
    assert len(kinds) > 1


def test_cached_step_graph_equals_eager():
    """CachedStepGraph (the whole cached step as one CUDA graph, decisions on the device)
    reproduces the eager read-back step bit for bit, stats included."""
    from paper_2501_09253_b200.engine_step import CachedStepGraph
    cfg, w, reqs, b = _setup(5, dims=(32, 64, 96, 32), ps_=32)
    prompts = {rid: ps.make_prompt(cfg, rid) for rid, _ in reqs}
    keys = b.patch_keys()
    c_graph = ps.BlockCache(cfg.n_blocks, ps.PredictorConfig(mse_threshold=0.08, max_streak=2))
    c_eager = ps.BlockCache(cfg.n_blocks, ps.PredictorConfig(mse_threshold=0.08, max_streak=2))
    b_graph = ps.split(reqs, patch_size=32)
    g = CachedStepGraph(b_graph, w, c_graph, keys)
    d_graph = d_eager = b.data.clone()
    skipped = []
    for s in range(7):
        bias, rates = step_inputs(cfg, b, prompts, dict.fromkeys(prompts, s), dict.fromkeys(prompts, 50))
        out, st_g = g.run(d_graph, bias, rates)
        d_graph = out.clone()
        b.data = d_eager
        d_eager, st_e = numeric_step(b, w, c_eager, bias, rates, keys=keys)
        assert torch.equal(d_graph, d_eager), s
        assert (st_g.skipped, st_g.computed) == (st_e.skipped, st_e.computed), s
        assert c_graph.stats.as_dict() == c_eager.stats.as_dict()
        skipped.append(st_g.skipped)
    assert g.graph is not None and max(skipped) > 0
