"""Seeded input generators shared by the golden-fixture writer and the tests.

Everything here is pure numpy (no reference import), so the GPU box can
regenerate the exact inputs the golden outputs were recorded on.
"""

from __future__ import annotations

import numpy as np

# (dims, patch_size argument) — KATs from pkg/tests/test_csp.py:38-95 plus the
# BASELINE configs 1, 2 and 5 and a few ragged hypothesis-style lists.
CSP_CASES = [
    ([64, 64, 96], None),
    ([96, 64, 96, 64], None),
    ([96], 32),
    ([64, 128, 96, 64], None),
    ([64], None),
    ([32, 48, 64], 16),                       # config 1
    ([64, 96, 128] * 4, 32),                  # config 2
    ([256] + [64] * 8, 64),                   # config 5
    ([4, 6, 8, 6, 4], None),
    ([8, 4, 8], None),
    ([6, 6], None),
]


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bfloat16 (ties to even), returned as float64."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def ops_small_inputs():
    """Small mixed batch (dims 8/12/8, C=4, ps=4) and params in the style of
    pkg/tests/test_patched.py:59-74; values are bf16-representable so the same
    arrays can be fed to the GPU path unchanged."""
    rng = np.random.default_rng(2024)
    c = 4
    reqs = [(f"r{i}", bf16_round(rng.normal(size=(c, d, d)))) for i, d in enumerate((8, 12, 8))]
    prm = {
        "gn": dict(groups=2, gamma=rng.normal(size=c), beta=rng.normal(size=c)),
        "ln": dict(gamma=rng.normal(size=c), beta=rng.normal(size=c)),
        "c3": dict(weights=rng.normal(size=(c, c, 3, 3)) * 0.3, bias=rng.normal(size=c) * 0.1),
        "c1": dict(weights=rng.normal(size=(c, c, 1, 1)) * 0.3, bias=rng.normal(size=c) * 0.1),
        "at": dict(wq=rng.normal(size=(c, c)) * 0.5, wk=rng.normal(size=(c, c)) * 0.5,
                   wv=rng.normal(size=(c, c)) * 0.5, wo=rng.normal(size=(c, c)) * 0.5),
        "ff": dict(w1=rng.normal(size=(2 * c, c)) * 0.3, b1=rng.normal(size=2 * c) * 0.1,
                   w2=rng.normal(size=(c, 2 * c)) * 0.3, b2=rng.normal(size=c) * 0.1),
    }
    n_p = 4 + 9 + 4
    mask = rng.random(n_p) < 0.4
    return reqs, prm, {"mask": mask, "x_cur_noise": rng.normal(size=(n_p, c, 4, 4))}


def cfg1_requests():
    """Config 1: latents 32/48/64 drawn as engine.py:233-234 does (seed 0, idx i)."""
    return [(f"req-{i:05d}", np.random.default_rng([0, i]).normal(size=(4, d, d)))
            for i, d in enumerate((32, 48, 64))]


def cache_trace_inputs(seed: int, n_steps: int = 10):
    """Random trace in the style of pkg/tests/test_cache.py:163-201 (shape (2,3,3))."""
    rng = np.random.default_rng(seed)
    shape = (2, 3, 3)
    pool = [(f"r{i}", j) for i in range(3) for j in range(4)]
    state = {k: rng.normal(size=shape) for k in pool}
    out = []
    for _ in range(n_steps):
        k = int(rng.integers(1, len(pool) + 1))
        keys = [pool[i] for i in rng.choice(len(pool), size=k, replace=False)]
        for key in keys:
            if rng.random() < 0.5:
                state[key] = state[key] + rng.normal(scale=0.2, size=shape)
        x = np.stack([state[key] for key in keys])
        live = [key for key in pool if rng.random() < 0.7] if rng.random() < 0.3 else None
        out.append(([list(kk) for kk in keys], x, None if live is None else [list(kk) for kk in live]))
    return out


# (shape, seed, kind) — kind "rand": two bf16 normal fields; "shift": b = a + const
MSE_CASES = [
    ((4, 16, 16), 1, "rand"), ((4, 32, 32), 2, "rand"), ((320, 32, 32), 3, "rand"),
    ((2, 3, 3), 4, "rand"), ((4, 4, 4), 5, "rand"), ((3, 5, 7), 6, "rand"),
    ((640, 32, 32), 7, "rand"), ((320, 16, 16), 8, "rand"), ((8, 64, 64), 9, "rand"),
    ((320, 32, 32), 10, "near"), ((4, 16, 16), 11, "shift"), ((320, 32, 32), 12, "shift"),
]


def mse_inputs(shape, seed, kind):
    rng = np.random.default_rng(seed)
    a = bf16_round(rng.normal(size=shape))
    if kind == "rand":
        b = bf16_round(rng.normal(size=shape))
    elif kind == "near":
        b = bf16_round(a + 0.3 * rng.normal(size=shape))
    else:
        b = bf16_round(a + np.sqrt(0.1))
    return a, b
