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
