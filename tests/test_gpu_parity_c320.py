"""Parity at the benchmark's shapes (SDXL-shaped unet_like: C=320, hidden 1280, GN 32, ps=32).

The GPU path is checked against the fp64 oracle (oracle/mixref.py, pinned to the reference's
golden vectors) in its BLAS contraction mode (same fp64 arithmetic, summation order of a matrix
product; tests/test_oracle_golden.py::test_blas_mode_matches_reference_goldens) on the box's
host cores.  Inputs are seeded N(0,1) latents (engine.py:233-234) and the reference's
init_weights (model.py:66-94); the oracle keeps the UNROUNDED fp64 weights and fp32 latents,
so the error below is the whole bf16 path's, not only the kernels'.

Tolerances (stated per test):
  * one block (bf16 output):            |d| <= 5e-2 + 2e-2 |ref|
  * latents after one step:             max |d| <= 1e-2                 (north-star budget)
  * latents over 50 steps:              <= 1.25 x the pure-numpy bf16 emulation's drift + 5e-4
                                        (tests/golden/drift_emulation.json; the dynamics amplify
                                        any bf16 rounding to ~0.02 by step 50)
  * attention at T = 65,536 (2048 px): |d| <= 5e-2 + 2e-2 |ref| on sampled query rows
  * cache masks (step-locked):          bit-exact

Set PS_REPORT_DIR to write the measured errors (JSON) there.
"""

import json
import os

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import paper_2501_09253_b200 as ps  # noqa: E402
from oracle import mixref as R  # noqa: E402

C, HID, G = 320, 1280, 32


def _report(name, obj):
    d = os.environ.get("PS_REPORT_DIR")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, f"parity_{name}.json"), "w") as f:
            json.dump(obj, f, indent=1)


def _cfgs(n_blocks, seed=0):
    return (ps.ModelConfig(arch="unet_like", channels=C, hidden=HID, groups=G, n_blocks=n_blocks, seed=seed),
            R.ModelConfig(arch="unet_like", channels=C, hidden=HID, groups=G, n_blocks=n_blocks, seed=seed))


def _latents(dims, seed=0):
    # engine.py:233-234 draws; fp32 master latents on the GPU, the same fp32 values in the oracle
    return [(f"req-{i}", np.random.default_rng([seed, i]).normal(size=(C, d, d)).astype(np.float32).astype(np.float64))
            for i, d in enumerate(dims)]


def _excess(got, want, atol, rtol):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float((np.abs(got - want) - (atol + rtol * np.abs(want))).max()), float(np.abs(got - want).max())


def test_c320_unet_block_p29_mixed_batch():
    """(a) one unet block (GN -> conv3 -> attention -> FF -> residual) on a P=29 mixed batch:
    one 512 / 768 / 1024 px request (latents 64 / 96 / 128, T up to 16,384 per image) --
    inter-patch halos, pooled GroupNorm over 4 / 9 / 16 patches, the pair attention kernel."""
    gcfg, rcfg = _cfgs(1)
    gw, rw = ps.init_weights(gcfg), R.init_weights(rcfg)
    reqs = _latents((64, 96, 128))
    rb = R.split(reqs, patch_size=32)
    x = ps.split([(r, torch.tensor(a, dtype=torch.float32)) for r, a in reqs], patch_size=32)
    xin = x.data.to(torch.bfloat16)  # the block input the GPU path runs on
    got = ps.run_block(x, xin, gw[0]).double().cpu().numpy()
    with R.blas_contractions():
        want = R.run_block(rb, xin.double().cpu().numpy(), rw[0])
    exc, mx = _excess(got, want, 5e-2, 2e-2)
    _report("c320_block_p29", {"max_abs": mx, "excess": exc, "P": rb.n_patches, "ref_max": float(np.abs(want).max())})
    assert exc <= 0, f"max |d| {mx:.3e}"


def test_c320_config2_step_7_blocks():
    """(b) a full SDXL-shaped step (prompt bias -> 7 blocks -> blend) on one 512 px + one
    1024 px request, through the public denoise_batch AND the graph-captured DenoisePipeline
    the bench times, against the oracle's denoise_image with the reference's fp64 weights."""
    from paper_2501_09253_b200.pipeline import DenoisePipeline
    gcfg, rcfg = _cfgs(7)
    gw, rw = ps.init_weights(gcfg), R.init_weights(rcfg)
    reqs = _latents((64, 128), seed=1)
    prompts = {rid: ps.make_prompt(gcfg, rid) for rid, _ in reqs}
    b = ps.split([(r, torch.tensor(a, dtype=torch.float32)) for r, a in reqs], patch_size=32)
    got = ps.reassemble(b, ps.denoise_batch(gcfg, gw, b, prompts, dict.fromkeys(prompts, 3),
                                            dict.fromkeys(prompts, 50)))
    pipe = DenoisePipeline(gcfg, gw, [64, 128], 32)
    pipe.set_prompts([prompts[r] for r, _ in reqs])
    pipe.prepare()
    hin = [torch.tensor(a, dtype=torch.float32).pin_memory() for _, a in reqs]
    hout = [torch.empty_like(t).pin_memory() for t in hin]
    pipe.run([hin], [[3, 3]], [50, 50], [hout])
    torch.cuda.synchronize()
    errs = {}
    with R.blas_contractions():
        for i, (rid, lat) in enumerate(reqs):
            want = R.denoise_image(rcfg, rw, lat, R.make_prompt(rcfg, rid), 3, 50)
            errs[rid] = (float(np.abs(got[rid].double().cpu().numpy() - want).max()),
                         float(np.abs(hout[i].double().numpy() - want).max()))
    _report("c320_step7", {"max_abs_denoise_batch_pipeline": errs})
    for rid, (e_api, e_pipe) in errs.items():
        assert e_api <= 1e-2, (rid, e_api)
        assert e_pipe <= 1e-2, (rid, e_pipe)


def _attention_rows_fp64(tokens, p, rows):
    """kernels.py:257-267 for a subset of query rows (softmax over all keys of the image)."""
    q = tokens[rows] @ p.wq
    k = tokens @ p.wk
    v = tokens @ p.wv
    s = (q @ k.T) / np.sqrt(q.shape[1])
    s -= s.max(axis=1, keepdims=True)
    np.exp(s, out=s)
    s /= s.sum(axis=1, keepdims=True)
    return (s @ v) @ p.wo


@pytest.mark.parametrize("splitkv", [False, True])
def test_attention_2048px_t65536_sampled_rows(splitkv):
    """(c) config 5's 2048 px image (latent 256, ps=64: T = 65,536 tokens in one image) through
    the persistent pair attention and through the split-KV + combine path, against fp64 on 96
    sampled query rows spread over every patch."""
    import paper_2501_09253_b200.patched as PT
    gcfg, rcfg = _cfgs(1, seed=2)
    gw, rw = ps.init_weights(gcfg), R.init_weights(rcfg)
    at_g, at_r = gw[0][2][1], rw[0][2][1]
    lat = np.random.default_rng(9).normal(size=(C, 256, 256))
    lat_bf = torch.tensor(lat, dtype=torch.float32).to(torch.bfloat16)
    b = ps.split([("big", lat_bf.float())], patch_size=64)
    prev = PT.SPLITKV_ALL
    PT.SPLITKV_ALL = splitkv
    try:
        out = ps.patched_self_attention(b, b.data.to(torch.bfloat16), at_g)
    finally:
        PT.SPLITKV_ALL = prev
    img = ps.reassemble(b, out.float())["big"].double().cpu().numpy()  # (C, 256, 256)
    tokens = lat_bf.double().numpy().reshape(C, -1).T.copy()               # (T, C) row-major
    rng = np.random.default_rng(4)
    rows = np.sort(rng.choice(256 * 256, size=96, replace=False))
    want = _attention_rows_fp64(tokens, at_r, rows)                       # (96, C)
    got = img.reshape(C, -1).T[rows]
    exc, mx = _excess(got, want, 5e-2, 2e-2)
    _report(f"attn_t65536_{'splitkv' if splitkv else 'pairs'}", {"max_abs": mx, "excess": exc,
                                                               "ref_max": float(np.abs(want).max())})
    assert exc <= 0, f"max |d| {mx:.3e}"


def test_c320_drift_50_steps_512px():
    """(d) latent drift over the 50-step schedule (rate 0.15 -> 0.05, model.py:56-63) for one
    512 px request with the 7-block SDXL-shaped model: the GPU's fp32 master latents against the
    oracle's fp64 trajectory from the same start, error reported per step.

    Bar.  One step stays within the north-star budget (<= 1e-2; 1.4e-3 measured).  Over 50
    steps the model's dynamics amplify ANY perturbation: pure-numpy emulations of bf16 arithmetic
    (tests/golden/drift_emulation.json, tools/drift_emulation.py) drift to 0.019 with bf16 weights
    alone and to 0.020 with the GPU path's full precision profile.  The GPU trajectory must stay
    within 1.25x the emulated bf16 drift at every step (+5e-4): the kernels add no error of their
    own beyond bf16 arithmetic."""
    gcfg, rcfg = _cfgs(7, seed=3)
    gw, rw = ps.init_weights(gcfg), R.init_weights(rcfg)
    (rid, lat), = _latents((64,), seed=5)
    gp, rp = ps.make_prompt(gcfg, rid), R.make_prompt(rcfg, rid)
    x_g = torch.tensor(lat, dtype=torch.float32)
    x_r = lat.copy()
    curve = []
    with R.blas_contractions():
        for s in range(50):
            b = ps.split([(rid, x_g)], patch_size=32)
            x_g = ps.reassemble(b, ps.denoise_batch(gcfg, gw, b, {rid: gp}, {rid: s}, {rid: 50}))[rid]
            x_r = R.denoise_image(rcfg, rw, x_r, rp, s, 50)
            curve.append(float(np.abs(x_g.double().cpu().numpy() - x_r).max()))
    emu = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "drift_emulation.json")))["curves"]
    bound = [1.25 * max(emu["W+ST+RS"][s], emu["W"][s]) + 5e-4 for s in range(50)]
    _report("drift_50_steps_512px", {"max_abs_per_step": curve, "final": curve[-1], "worst": max(curve),
                                     "bf16_emulation_W+ST+RS": emu["W+ST+RS"], "bound": bound})
    assert curve[0] <= 1e-2, curve[0]
    assert all(c <= b for c, b in zip(curve, bound)), [(s, c, b) for s, (c, b) in enumerate(zip(curve, bound))
                                                        if c > b]


def test_c320_cache_masks_step_locked():
    """(e) config 3 at C=320 / ps=32: the GPU patch cache in the engine's per-block sequence
    (predict_reuse -> gather -> masked_block_forward -> batched_fill -> batched_update,
    engine.py:137-142) over 6 steps of a 512 + 768 px batch, with the oracle's cache driven by
    the SAME block inputs and outputs (step-locked: the GPU's bf16 values, exact in fp64).
    Masks, streaks and stats must be bit-identical (cache.py:107-169)."""
    gcfg, _ = _cfgs(2, seed=4)
    gw = ps.init_weights(gcfg)
    reqs = _latents((64, 96), seed=6)
    prompts = {rid: ps.make_prompt(gcfg, rid) for rid, _ in reqs}
    gcache = ps.BlockCache(2, ps.PredictorConfig(0.1, 3))
    rcache = R.Cache(2, sigma=0.1, max_streak=3)
    lats = {rid: torch.tensor(a, dtype=torch.float32) for rid, a in reqs}
    n_masked = 0
    for s in range(6):
        b = ps.split([(rid, lats[rid]) for rid, _ in reqs], patch_size=32)
        keys = b.patch_keys()
        from paper_2501_09253_b200.model import blend_batch, prompt_bias, step_inputs
        bias, rates = step_inputs(gcfg, b, prompts, dict.fromkeys(prompts, s), dict.fromkeys(prompts, 50))
        h = prompt_bias(b, b.data.float().contiguous(), bias)
        for blk, ops in enumerate(gw):
            mask_g = gcache.predict_reuse(blk, keys, h).cpu().numpy()
            mask_r = rcache.predict_reuse(blk, keys, h.double().cpu().numpy())
            np.testing.assert_array_equal(mask_g, mask_r)
            ci, co = gcache.gather(blk, keys, mask_g, h.shape[1:])
            y = ps.masked_block_forward(b, h, mask_g, ops, ci, co)
            gcache.batched_fill(blk, keys, mask_g)
            gcache.batched_update(blk, keys, mask_g, h, y)
            rcache.batched_fill(blk, keys, mask_r)
            rcache.batched_update(blk, keys, mask_r, h.double().cpu().numpy(), y.double().cpu().numpy())
            n_masked += int(mask_g.sum())
            for k in keys[::7]:
                e_g, e_r = gcache.entry(blk, k), rcache.stores[blk].get(k)
                assert (e_g is None) == (e_r is None)
                if e_g is not None:
                    assert e_g.reuse_streak == e_r.reuse_streak
            h = y
        new = blend_batch(b, b.data.float().contiguous(), h, rates)
        lats = ps.reassemble(b, new)
    st_g, st_r = gcache.stats, rcache.stats
    assert (st_g.predicted_reuse, st_g.fresh_compute, st_g.inserted, st_g.refreshed) == \
        (st_r.predicted_reuse, st_r.fresh_compute, st_r.inserted, st_r.refreshed)
    _report("cache_masks_c320", {"masked_patch_blocks": n_masked, "stats": st_g.as_dict()})
    assert n_masked > 0  # the reuse path was exercised
