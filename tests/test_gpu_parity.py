"""Parity of the CUDA path (through the C ABI / facade) with the CPU oracle.

Bit-exact: CSP metadata and pixel copies, halo frames, skip masks, streaks,
cache snapshots.  Floating point: bf16 activations with fp32 accumulation
against the fp64 oracle on identical (bf16-representable) inputs and weights;
tolerances are stated per test:
  * single stage output (bf16-rounded):  |d| <= 2e-2 + 1e-2 |ref|
  * attention / whole block:              |d| <= 5e-2 + 2e-2 |ref|
  * denoised latents (fp32 master):       max |d| <= 1e-2   (north-star budget)
"""

import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2501_09253_b200 as ps  # noqa: E402
from oracle import mixref as R  # noqa: E402
from tests.golden.cases import bf16_round, cache_trace_inputs, cfg1_requests, mse_inputs, MSE_CASES  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def np_(t):
    return t.detach().double().cpu().numpy()


def close(got, want, atol, rtol):
    got, want = np.asarray(got), np.asarray(want)
    err = np.abs(got - want) - (atol + rtol * np.abs(want))
    assert err.max() <= 0, f"max excess {err.max():.3e}; max |d| {np.abs(got - want).max():.3e}"


def _bf16_params(prm: dict):
    return {k: ({kk: (bf16_round(v) if isinstance(v, np.ndarray) else v) for kk, v in d.items()}) for k, d in prm.items()}


def _small():
    from tests.golden.cases import ops_small_inputs
    reqs, prm, extra = ops_small_inputs()
    prm = _bf16_params(prm)
    rb = R.split(reqs, patch_size=4)
    gb = ps.split([(r, torch.tensor(a, dtype=torch.float32)) for r, a in reqs], patch_size=4)
    P = dict(gn=(ps.GroupNormParams(**prm["gn"]), R.GroupNormParams(**prm["gn"])),
             ln=(ps.LayerNormParams(**prm["ln"]), R.LayerNormParams(**prm["ln"])),
             c3=(ps.ConvParams(**prm["c3"]), R.ConvParams(**prm["c3"])),
             c1=(ps.ConvParams(**prm["c1"]), R.ConvParams(**prm["c1"])),
             at=(ps.AttentionParams(**prm["at"]), R.AttentionParams(**prm["at"])),
             ff=(ps.FeedForwardParams(**prm["ff"]), R.FeedForwardParams(**prm["ff"])))
    return reqs, rb, gb, P, extra


# ------------------------------------------------------------------ CSP


@pytest.mark.parametrize("case", range(11))
def test_csp_metadata_bit_exact(case):
    from tests.golden.cases import CSP_CASES
    with open(os.path.join(GOLD, "csp_kats.json")) as f:
        g = json.load(f)[case]
    dims, psz = CSP_CASES[case]
    reqs = [(f"r{i}", torch.zeros((1, d, d))) for i, d in enumerate(dims)]
    b = ps.split(reqs, patch_size=psz)
    assert b.patch_size == g["patch_size"]
    assert [e.request_id for e in b.requests] == g["order"]
    for k in ("request_offset", "resolution_offset", "request_index", "ordinal", "row", "col", "neighbors"):
        assert getattr(b, k).tolist() == g[k], k
    assert b.resolution_dims == g["resolution_dims"]


def test_split_reassemble_ragged_round_trip():
    rng = np.random.default_rng(5)
    for dims in ([4, 6, 8], [6], [8, 4, 8, 4, 6], [12, 8]):
        reqs = [(f"q{i}", torch.tensor(rng.normal(size=(2, d, d)), dtype=torch.float32)) for i, d in enumerate(dims)]
        b = ps.split(reqs)
        back = ps.reassemble(b)
        for rid, lat in reqs:
            assert torch.equal(back[rid].cpu(), lat)
        rb = R.split([(r, a.double().numpy()) for r, a in reqs])
        np.testing.assert_array_equal(np_(b.data), rb.data)


def test_split_rejects_bad_input():
    with pytest.raises(ps.InputError):
        ps.split([])
    with pytest.raises(ps.InputError):
        ps.split([("a", torch.zeros(2, 8, 8)), ("a", torch.zeros(2, 8, 8))])
    with pytest.raises(ps.InputError):
        ps.split([("a", torch.zeros(2, 8, 6))])
    with pytest.raises(ps.InputError):
        ps.split([("a", torch.zeros(2, 8, 8))], patch_size=3)


# ---------------------------------------------------------------- halos


def test_halo_frames_bit_exact():
    reqs, rb, gb, P, _ = _small()
    np.testing.assert_array_equal(np_(ps.exchange_halos(gb, gb.data)), R.exchange_halos(rb, rb.data))
    x = torch.tensor(bf16_round(rb.data)).to(torch.bfloat16).cuda()
    np.testing.assert_array_equal(np_(ps.exchange_halos(gb, x)), R.exchange_halos(rb, rb.data))


def test_halo_frames_zero_padded_windows_ps16():
    rng = np.random.default_rng(1)
    lat = rng.normal(size=(3, 48, 48))
    gb = ps.split([("a", torch.tensor(lat, dtype=torch.float32))], patch_size=16)
    fr = np_(ps.exchange_halos(gb, gb.data))
    pad = np.zeros((3, 50, 50))
    pad[:, 1:-1, 1:-1] = np.float32(lat)
    for p in range(gb.n_patches):
        r, c = int(gb.row[p]), int(gb.col[p])
        np.testing.assert_array_equal(fr[p], pad[:, r * 16:r * 16 + 18, c * 16:c * 16 + 18])


# ------------------------------------------------------------ operators


def test_group_norm_close():
    reqs, rb, gb, P, _ = _small()
    got = ps.stitched_group_norm(gb, gb.data, P["gn"][0])
    close(np_(got), R.stitched_group_norm(rb, rb.data, P["gn"][1]), 2e-2, 1e-2)
    out, fr = ps.stitched_group_norm(gb, gb.data, P["gn"][0], emit_halos=True)
    np.testing.assert_array_equal(np_(fr), R.exchange_halos(rb, np_(out)))


def test_layer_norm_close():
    reqs, rb, gb, P, _ = _small()
    close(np_(ps.patched_layer_norm(gb, gb.data, P["ln"][0])), R.patched_layer_norm(rb, rb.data, P["ln"][1]),
          2e-2, 1e-2)


@pytest.mark.parametrize("k", ["c3", "c1"])
def test_conv_close(k):
    reqs, rb, gb, P, _ = _small()
    close(np_(ps.patched_conv(gb, gb.data, P[k][0])), R.patched_conv(rb, rb.data, P[k][1]), 2e-2, 1e-2)


def test_conv_with_given_frames():
    reqs, rb, gb, P, _ = _small()
    fr = ps.exchange_halos(gb, gb.data)
    close(np_(ps.patched_conv(gb, gb.data, P["c3"][0], frames=fr)), R.patched_conv(rb, rb.data, P["c3"][1]),
          2e-2, 1e-2)


def test_attention_close():
    reqs, rb, gb, P, _ = _small()
    close(np_(ps.patched_self_attention(gb, gb.data, P["at"][0])),
          R.patched_self_attention(rb, rb.data, P["at"][1]), 5e-2, 2e-2)


def test_feed_forward_close():
    reqs, rb, gb, P, _ = _small()
    from paper_2501_09253_b200.patched import feed_forward
    close(np_(feed_forward(gb, gb.data, P["ff"][0])), R.feed_forward(rb.data, P["ff"][1]), 2e-2, 1e-2)


def _ops(P, arch):
    if arch == "unet":
        names = ("gn", "c3", "at", "ff")
        kinds = ("group_norm", "conv", "attention", "feed_forward")
    else:
        names = ("ln", "at", "ff")
        kinds = ("layer_norm", "attention", "feed_forward")
    g = [(k, P[n][0]) for k, n in zip(kinds, names)] + [("residual", None)]
    r = [(k, P[n][1]) for k, n in zip(kinds, names)] + [("residual", None)]
    return g, r


@pytest.mark.parametrize("arch", ["unet", "dit"])
def test_run_block_close(arch):
    reqs, rb, gb, P, _ = _small()
    g, r = _ops(P, arch)
    close(np_(ps.run_block(gb, gb.data, g)), R.run_block(rb, rb.data, r), 5e-2, 2e-2)


def test_launch_counts_match_reference_semantics():
    reqs, rb, gb, P, _ = _small()
    g, r = _ops(P, "unet")
    ps.reset_launch_counters()
    ps.run_block(gb, gb.data, g)
    R.LAUNCHES.clear()
    R.run_block(rb, rb.data, r)
    assert ps.launch_counters() == R.LAUNCHES
    ps.reset_launch_counters()
    ps.run_block(gb, gb.data, [("conv", P["c3"][0])])
    assert ps.launch_counters() == {"halo_exchange": 1, "conv": 1}


def test_masked_forward_matches_substitution():
    reqs, rb, gb, P, extra = _small()
    g, r = _ops(P, "unet")
    mask = extra["mask"]
    x_prev = rb.data
    x_cur = bf16_round(rb.data + 0.05 * extra["x_cur_noise"])
    y_prev_g = ps.run_block(gb, gb.data, g)
    y_prev = np_(y_prev_g)
    got = ps.masked_block_forward(gb, torch.tensor(x_cur, dtype=torch.float32), mask, g, gb.data, y_prev_g)
    want = R.masked_block_forward(rb, x_cur, mask, r, x_prev, y_prev)
    close(np_(got), want, 5e-2, 2e-2)
    # masked rows are exact copies of the cached outputs (patched.py:246)
    np.testing.assert_array_equal(np_(got)[mask], y_prev[mask])
    ps.reset_launch_counters()
    allm = ps.masked_block_forward(gb, gb.data, np.ones(gb.n_patches, dtype=bool), g, gb.data, y_prev_g)
    assert ps.launch_counters() == {}
    assert torch.equal(allm, y_prev_g)
    with pytest.raises(ps.InputError):
        ps.masked_block_forward(gb, gb.data, np.ones(3, dtype=bool), g, gb.data, y_prev_g)


# ------------------------------------------------------------------ cache


@pytest.mark.parametrize("idx", range(len(MSE_CASES)))
def test_mse_bit_exact(idx):
    shape, seed, kind = MSE_CASES[idx]
    a, b = mse_inputs(shape, seed, kind)
    got = ps.mse(torch.tensor(a, dtype=torch.float32), torch.tensor(b, dtype=torch.float32))
    assert got.hex() == float(np.mean((a - b) ** 2)).hex()


def test_predict_reuse_masks_bit_exact_near_threshold():
    # per-patch MSE straddling sigma within a few ulps: masks must match numpy exactly
    rng = np.random.default_rng(3)
    shape = (320, 16, 16)
    n_p = 24
    snap = bf16_round(rng.normal(size=(n_p,) + shape))
    x = bf16_round(snap + 0.3 * rng.normal(size=snap.shape))
    msev = [float(np.mean((x[i] - snap[i]) ** 2)) for i in range(n_p)]
    keys = [("r", i) for i in range(n_p)]
    for sigma in sorted(msev)[::3] + [np.nextafter(m, 1.0) for m in msev[:6]] + [np.nextafter(m, 0.0) for m in msev[:6]]:
        cache = ps.BlockCache(1, ps.PredictorConfig(mse_threshold=sigma, max_streak=3))
        cache.batched_update(0, keys, np.zeros(n_p, dtype=bool), torch.tensor(snap), torch.tensor(snap))
        got = cache.predict_reuse(0, keys, torch.tensor(x)).cpu().numpy()
        want = np.array([m < sigma for m in msev])
        np.testing.assert_array_equal(got, want)


def test_threshold_is_strict_and_streak_bounded():
    sigma = 0.25
    cache = ps.BlockCache(2, ps.PredictorConfig(mse_threshold=sigma, max_streak=3))
    x = torch.zeros((1, 2, 3, 3))
    cache.batched_update(0, ["a"], np.zeros(1, dtype=bool), x, x)
    assert not cache.predict_reuse(0, ["a"], x + 0.5).any()          # mse == sigma
    assert cache.predict_reuse(0, ["a"], x + 0.49609375).all()       # bf16 below sqrt(sigma)
    assert not cache.predict_reuse(1, ["a"], x).any()                # other block is empty
    hits = 0
    for _ in range(10):
        m = cache.predict_reuse(0, ["a"], x)
        if not bool(m[0]):
            break
        cache.batched_fill(0, ["a"], m)
        hits += 1
    assert hits == 3 and cache.entry(0, "a").reuse_streak == 3
    cache.batched_update(0, ["a"], np.zeros(1, dtype=bool), x, x)
    assert cache.entry(0, "a").reuse_streak == 0


def test_gather_fill_integrity():
    cache = ps.BlockCache(1)
    rng = np.random.default_rng(3)
    x = torch.tensor(bf16_round(rng.normal(size=(1, 2, 3, 3))), dtype=torch.float32)
    y = torch.tensor(bf16_round(rng.normal(size=(1, 2, 3, 3))), dtype=torch.float32)
    cache.batched_update(0, ["a"], np.zeros(1, dtype=bool), x, y)
    ins, outs = cache.gather(0, ["a", "b"], np.array([True, False]), (2, 3, 3))
    assert torch.equal(ins[0].float().cpu(), x[0]) and torch.equal(outs[0].float().cpu(), y[0])
    assert float(ins[1].abs().sum()) == 0.0
    with pytest.raises(ps.IntegrityError):
        cache.gather(0, ["b"], np.array([True]), (2, 3, 3))
    with pytest.raises(ps.IntegrityError):
        cache.batched_fill(0, ["b"], np.array([True]))
    x[:] = 99.0  # snapshots are copies (cache.py:166-167)
    assert float(cache.entry(0, "a").input_snapshot.float().abs().max()) < 99


def test_cache_traces_match_reference():
    with open(os.path.join(GOLD, "cache_traces.json")) as f:
        traces = json.load(f)
    for t in traces:
        c = ps.BlockCache(2, ps.PredictorConfig(0.1, 3))
        o = R.Cache(2, 0.1, 3)
        for (keys, x, live), rec in zip(cache_trace_inputs(t["seed"]), t["steps"]):
            keys = [tuple(k) for k in keys]
            xb = bf16_round(x)  # GPU snapshots are bf16: feed both sides the same values
            xt = torch.tensor(xb, dtype=torch.float32)
            for blk in range(2):
                m = c.predict_reuse(blk, keys, xt)
                mo = o.predict_reuse(blk, keys, xb)
                np.testing.assert_array_equal(m.cpu().numpy(), mo)
                c.batched_fill(blk, keys, m)
                o.batched_fill(blk, keys, mo)
                yb = bf16_round(np.tanh(xb + blk))
                c.batched_update(blk, keys, m, xt, torch.tensor(yb, dtype=torch.float32))
                o.batched_update(blk, keys, mo, xb, yb)
            if live is not None:
                lv = [tuple(k) for k in live]
                assert c.evict_expired(lv) == o.evict_expired(lv)
        for bk in range(2):
            for k, e in o.stores[bk].items():
                ge = c.entry(bk, k)
                assert ge is not None and ge.reuse_streak == e.reuse_streak
                np.testing.assert_array_equal(np_(ge.input_snapshot), e.input_snapshot)
                np.testing.assert_array_equal(np_(ge.output_snapshot), e.output_snapshot)
        assert c.size() == sum(len(s) for s in o.stores)
        assert c.stats.as_dict() == o.stats.__dict__


def test_partition_sets():
    assert ps.partition_sets(["a", "b", "c"], ["b", "d", "a"]) == (["b", "a"], ["d"], ["c"])
    with pytest.raises(ps.InputError):
        ps.partition_sets(["a", "a"], ["b"])


# ------------------------------------------------------------------ model


def test_config1_denoise_within_budget():
    g = np.load(os.path.join(GOLD, "cfg1_steps.npz"))
    cfg = ps.ModelConfig(arch="unet_like", channels=4, hidden=8, n_blocks=2, groups=2, seed=0)
    w = ps.init_weights(cfg)
    reqs = cfg1_requests()
    prompts = {rid: ps.make_prompt(cfg, rid) for rid, _ in reqs}
    b = ps.split([(r, torch.tensor(a, dtype=torch.float32)) for r, a in reqs], patch_size=16)
    data = b.data
    worst = []
    for s in range(4):
        b.data = data
        data = ps.denoise_batch(cfg, w, b, prompts, {r: s for r, _ in reqs}, {r: 4 for r, _ in reqs})
        worst.append(float(np.abs(np_(data) - g[f"step{s}"]).max()))
    assert max(worst) <= 1e-2, worst


def test_dit_denoise_within_budget():
    rng = np.random.default_rng(0)
    cfg = ps.ModelConfig(arch="dit_like", n_blocks=2, seed=3)
    rcfg = R.ModelConfig(arch="dit_like", n_blocks=2, seed=3)
    reqs = [(f"r{i}", rng.normal(size=(4, d, d))) for i, d in enumerate((8, 12, 8))]
    w, rw = ps.init_weights(cfg), R.init_weights(rcfg)
    prompts = {rid: ps.make_prompt(cfg, rid) for rid, _ in reqs}
    si = {"r0": 0, "r1": 3, "r2": 7}
    ts = {"r0": 10, "r1": 10, "r2": 10}
    b = ps.split([(r, torch.tensor(a, dtype=torch.float32)) for r, a in reqs], patch_size=4)
    got = ps.reassemble(b, ps.denoise_batch(cfg, w, b, prompts, si, ts))
    for rid, lat in reqs:
        want = R.denoise_image(rcfg, rw, np.float32(lat).astype(np.float64), prompts[rid], si[rid], ts[rid])
        assert np.abs(np_(got[rid]) - want).max() <= 1e-2


def test_pipeline_graph_matches_denoise_batch():
    """DenoisePipeline (CUDA graph, overlapped copies) reproduces denoise_batch bit for bit."""
    from paper_2501_09253_b200.pipeline import DenoisePipeline
    cfg = ps.ModelConfig(arch="unet_like", channels=64, hidden=128, n_blocks=2, groups=8, seed=5)
    w = ps.init_weights(cfg)
    rng = np.random.default_rng(9)
    dims = [64, 32, 64, 96]
    lats = [rng.normal(size=(64, d, d)).astype(np.float32) for d in dims]
    ids = [f"q{i}" for i in range(len(dims))]
    prompts = [ps.make_prompt(cfg, r) for r in ids]
    pipe = DenoisePipeline(cfg, w, dims, 32)
    pipe.set_prompts(prompts)
    pipe.prepare()
    steps = 3
    host_in = [[torch.tensor(x).pin_memory() for x in lats] for _ in range(steps)]
    host_out = [[torch.empty_like(x).pin_memory() for x in host_in[0]] for _ in range(steps)]
    pipe.run(host_in, [[s, s, s + 1, 0] for s in range(steps)], [5, 5, 5, 5], host_out)
    torch.cuda.synchronize()
    b = ps.split([(r, torch.tensor(x)) for r, x in zip(ids, lats)], patch_size=32)
    for s in range(steps):
        si = dict(zip(ids, [s, s, s + 1, 0]))
        want = ps.reassemble(b, ps.denoise_batch(cfg, w, b, dict(zip(ids, prompts)), si, dict.fromkeys(ids, 5)))
        for r, rid in enumerate(ids):
            assert torch.equal(host_out[s][r], want[rid].cpu()), (s, rid)
