"""Drop-in precision of the cache path and input validation on the device.

* `mse` keeps its operands' precision: numpy float64 inputs (not bf16-representable) give
  numpy's exact fp64 pairwise mean, hex-equal (cache.py:54-55).
* `BlockCache(dtype=torch.float64)` stores fp64 snapshots, so masks on arbitrary fp64
  inputs equal the reference's bit for bit, including thresholds at the MSE's neighbouring
  doubles (cache.py:107-122); the fp32 slab likewise for fp32 inputs.
* Non-finite latents are rejected (kernels.py:20-24): the pipeline's split kernel flags them.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2501_09253_b200 as ps  # noqa: E402


@pytest.mark.parametrize("shape,seed", [((4, 16, 16), 0), ((320, 32, 32), 1), ((7, 5, 3), 2), ((1,), 3),
                                        ((3, 8, 8), 4), ((640, 32, 32), 5)])
def test_mse_fp64_inputs_hex_equal(shape, seed):
    rng = np.random.default_rng(seed)
    a, b = rng.normal(size=shape), rng.normal(size=shape) * 1.7
    assert ps.mse(a, b).hex() == float(np.mean((a - b) ** 2)).hex()
    af, bf = a.astype(np.float32), b.astype(np.float32)
    want32 = float(np.mean((af.astype(np.float64) - bf.astype(np.float64)) ** 2))
    assert ps.mse(torch.tensor(af), torch.tensor(bf)).hex() == want32.hex()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_predict_reuse_fp_slab_masks_exact(dtype):
    rng = np.random.default_rng(11)
    shape, n_p = (64, 8, 8), 20
    np_dt = np.float64 if dtype == torch.float64 else np.float32
    snap = rng.normal(size=(n_p,) + shape).astype(np_dt)
    x = (snap + 0.3 * rng.normal(size=snap.shape)).astype(np_dt)
    msev = [float(np.mean((x[i].astype(np.float64) - snap[i].astype(np.float64)) ** 2)) for i in range(n_p)]
    keys = [("r", i) for i in range(n_p)]
    for sigma in sorted(msev)[::4] + [np.nextafter(m, 1.0) for m in msev[:5]] + [np.nextafter(m, 0.0) for m in msev[:5]]:
        cache = ps.BlockCache(1, ps.PredictorConfig(mse_threshold=sigma, max_streak=3), dtype=dtype)
        cache.batched_update(0, keys, np.zeros(n_p, dtype=bool), snap, snap)
        got = cache.predict_reuse(0, keys, x).cpu().numpy()
        np.testing.assert_array_equal(got, np.array([m < sigma for m in msev]))
        # entries are exact copies at the slab precision
        e = cache.entry(0, keys[3])
        np.testing.assert_array_equal(e.input_snapshot.cpu().numpy(), snap[3])


def test_fp64_cache_gather_fill_round_trip():
    rng = np.random.default_rng(5)
    x, y = rng.normal(size=(6, 4, 4, 4)), rng.normal(size=(6, 4, 4, 4))
    keys = [("a", i) for i in range(6)]
    cache = ps.BlockCache(2, dtype=torch.float64)
    cache.batched_update(1, keys, np.zeros(6, dtype=bool), x, y)
    mask = np.array([1, 0, 1, 0, 0, 1], dtype=bool)
    ins, outs = cache.gather(1, keys, mask, x.shape[1:])
    np.testing.assert_array_equal(ins.cpu().numpy()[mask], x[mask])
    np.testing.assert_array_equal(outs.cpu().numpy()[mask], y[mask])
    np.testing.assert_array_equal(outs.cpu().numpy()[~mask], 0.0)
    out = np.zeros_like(y)
    cache.batched_fill(1, keys, mask, out=out)
    np.testing.assert_array_equal(out[mask], y[mask])
    assert cache.entry(1, keys[0]).reuse_streak == 1


def test_pipeline_rejects_non_finite_latents():
    from paper_2501_09253_b200.pipeline import DenoisePipeline
    cfg = ps.ModelConfig(arch="unet_like", channels=64, hidden=128, groups=8, n_blocks=1, seed=0)
    w = ps.init_weights(cfg)
    pipe = DenoisePipeline(cfg, w, [32, 64], 32, use_graph=True)
    pipe.set_prompts([ps.make_prompt(cfg, f"r{i}") for i in range(2)])
    pipe.prepare()
    ok = [torch.randn((64, d, d)).pin_memory() for d in (32, 64)]
    out = [torch.empty_like(t).pin_memory() for t in ok]
    pipe.run([ok], [[0, 0]], [4, 4], [out])
    bad = [t.clone().pin_memory() for t in ok]
    bad[1][3, 5, 7] = float("nan")
    with pytest.raises(ps.InputError):
        pipe.run([bad], [[0, 0]], [4, 4], [out])
    bad[1][3, 5, 7] = float("inf")
    with pytest.raises(ps.InputError):
        pipe.run([bad], [[0, 0]], [4, 4], [out])
    pipe.run([ok], [[0, 0]], [4, 4], [out])  # the flag is per call


def _bf16_adversarial(shape, seed):
    """bf16 operands whose differences are inexact in fp32 in some 8-element groups: magnitudes
    spread over 2^-60 .. 2^60, exact ties, zeros of both signs, values near the bf16 maximum (the
    fp32 difference overflows) and subnormal bf16."""
    rng = np.random.default_rng(seed)
    n = int(np.prod(shape))
    a = rng.normal(size=n) * np.exp2(rng.integers(-60, 61, size=n))
    b = rng.normal(size=n) * np.exp2(rng.integers(-60, 61, size=n))
    k = rng.choice(n, size=n // 16, replace=False)
    b[k] = a[k]                                   # zero differences
    z = rng.choice(n, size=n // 32, replace=False)
    a[z] = np.where(rng.random(z.size) < 0.5, 0.0, -0.0)
    big = rng.choice(n, size=max(2, n // 512), replace=False)
    a[big], b[big[: big.size // 2]] = 3.3e38, -3.3e38
    sub = rng.choice(n, size=max(2, n // 256), replace=False)
    b[sub] = rng.normal(size=sub.size) * 1e-39    # bf16 subnormals
    ta = torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).reshape(shape)
    tb = torch.tensor(b, dtype=torch.float32).to(torch.bfloat16).reshape(shape)
    return ta, tb


@pytest.mark.parametrize("shape,seed", [((320, 32, 32), 0), ((4, 16, 16), 1), ((64, 8, 8), 2), ((3, 5, 7), 3)])
def test_mse_bf16_mixed_exponents_hex_equal(shape, seed):
    """The bf16 leaf's fp32-difference fast path (exact iff round-down == round-up) and its fp64
    fallback give numpy's fp64 pairwise mean bit for bit, on groups where both paths run."""
    ta, tb = _bf16_adversarial(shape, seed)
    a, b = ta.double().numpy(), tb.double().numpy()
    want = float(np.mean((a - b) ** 2))
    assert ps.mse(ta, tb).hex() == want.hex()
    # the same on moderate values (the all-fast-path case)
    rng = np.random.default_rng(seed + 100)
    ua = torch.tensor(rng.normal(size=shape), dtype=torch.float32).to(torch.bfloat16)
    ub = torch.tensor(rng.normal(size=shape), dtype=torch.float32).to(torch.bfloat16)
    assert ps.mse(ua, ub).hex() == float(np.mean((ua.double().numpy() - ub.double().numpy()) ** 2)).hex()
