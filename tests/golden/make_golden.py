"""Record golden vectors from the REAL reference (`/root/reference/pkg/src/mixserve`).

Run in the build container (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes small fixtures next to this script.  They pin the oracle restatement
(`oracle/`) — see tests/test_oracle_golden.py — and through it every GPU parity
test.  Inputs are regenerated from seeds where they are large (numpy's
default_rng streams are platform-stable), so only outputs are stored.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
from tests.golden.cases import (  # noqa: E402
    CSP_CASES, MSE_CASES, ops_small_inputs, cfg1_requests, cache_trace_inputs,
)


def main():
    sys.path.insert(0, REF)
    from mixserve import csp, patched, kernels, cache, model  # noqa: F401

    # ---------------------------------------------------------------- CSP KATs
    out = []
    for dims, ps in CSP_CASES:
        rng = np.random.default_rng(0)
        reqs = [(f"r{i}", rng.normal(size=(1, d, d))) for i, d in enumerate(dims)]
        b = csp.split(reqs, patch_size=ps)
        out.append({
            "dims": dims, "ps_arg": ps, "patch_size": b.patch_size,
            "order": [e.request_id for e in b.requests],
            "request_offset": b.request_offset.tolist(),
            "resolution_dims": list(b.resolution_dims),
            "resolution_offset": b.resolution_offset.tolist(),
            "request_index": b.request_index.tolist(),
            "ordinal": b.ordinal.tolist(), "row": b.row.tolist(), "col": b.col.tolist(),
            "neighbors": b.neighbors.tolist(),
        })
    (HERE / "csp_kats.json").write_text(json.dumps(out))

    # ------------------------------------------------------ patched operators
    reqs, prm, extra = ops_small_inputs()
    b = csp.split(reqs, patch_size=4)
    gn = kernels.GroupNormParams(**prm["gn"])
    ln = kernels.LayerNormParams(**prm["ln"])
    c3 = kernels.ConvParams(**prm["c3"])
    c1 = kernels.ConvParams(**prm["c1"])
    at = kernels.AttentionParams(**prm["at"])
    ff = kernels.FeedForwardParams(**prm["ff"])
    unet = [("group_norm", gn), ("conv", c3), ("attention", at), ("feed_forward", ff), ("residual", None)]
    dit = [("layer_norm", ln), ("attention", at), ("feed_forward", ff), ("residual", None)]
    gno, frames_gn = patched.stitched_group_norm(b, b.data, gn, emit_halos=True)
    mask = extra["mask"]
    from tests.golden.cases import bf16_round
    x_cur = bf16_round(b.data + 0.05 * extra["x_cur_noise"])
    y_prev = patched.run_block(b, b.data, unet)
    res = dict(
        data=b.data,
        halos=patched.exchange_halos(b, b.data),
        gn=gno, gn_frames=frames_gn,
        conv3=patched.patched_conv(b, b.data, c3),
        conv1=patched.patched_conv(b, b.data, c1),
        attn=patched.patched_self_attention(b, b.data, at),
        ln=patched.patched_layer_norm(b, b.data, ln),
        ff=kernels.feed_forward(b.data, ff),
        block_unet=y_prev,
        block_dit=patched.run_block(b, b.data, dit),
        x_cur=x_cur, mask=mask,
        masked_unet=patched.masked_block_forward(b, x_cur, mask, unet, b.data, y_prev),
    )
    np.savez_compressed(HERE / "ops_small.npz", **res)

    # -------------------------------------------------- config-1 denoise steps
    cfg = model.ModelConfig(arch="unet_like", channels=4, hidden=8, n_blocks=2, groups=2, seed=0)
    w = model.init_weights(cfg)
    reqs1 = cfg1_requests()
    prompts = {rid: model.make_prompt(cfg, rid) for rid, _ in reqs1}
    b1 = csp.split(reqs1, patch_size=16)
    data = b1.data
    steps = {}
    for s in range(4):
        b1.data = data
        data = model.denoise_batch(cfg, w, b1, prompts, {r: s for r, _ in reqs1}, {r: 4 for r, _ in reqs1})
        steps[f"step{s}"] = data
    wflat = np.concatenate([np.ravel(getattr(p, f)) for ops in w for _, p in ops if p is not None
                            for f in p.__dataclass_fields__ if f not in ("groups", "eps")])
    prom = np.stack([prompts[r] for r, _ in reqs1])
    dense0 = {r: model.denoise_image(cfg, w, lat, prompts[r], 0, 4) for r, lat in reqs1}
    np.savez_compressed(HERE / "cfg1_steps.npz", weights_flat=wflat, prompts=prom,
                        **steps, **{f"dense0_{r}": v for r, v in dense0.items()})

    # ------------------------------------------------------- cache traces
    traces = []
    for seed in range(6):
        steps_in = cache_trace_inputs(seed)
        c = cache.BlockCache(2, cache.PredictorConfig(mse_threshold=0.1, max_streak=3))
        rec = []
        for keys, x, live in steps_in:
            keys = [tuple(k) for k in keys]
            step_rec = {"masks": [], "evicted": None}
            for blk in range(2):
                m = c.predict_reuse(blk, keys, x)
                outb = np.zeros_like(x)
                c.batched_fill(blk, keys, m, outb)
                c.batched_update(blk, keys, m, x, np.tanh(x + blk))
                step_rec["masks"].append(m.astype(int).tolist())
            if live is not None:
                step_rec["evicted"] = c.evict_expired([tuple(k) for k in live])
            rec.append(step_rec)
        final = [sorted([[list(k), c.entry(bk, k).reuse_streak] for k in c._stores[bk]]) for bk in range(2)]
        traces.append({"seed": seed, "steps": rec, "final": final, "stats": c.stats.as_dict()})
    (HERE / "cache_traces.json").write_text(json.dumps(traces))

    # ------------------------------------------------------------ MSE bits
    mse_out = []
    for shape, seed, kind in MSE_CASES:
        from tests.golden.cases import mse_inputs
        a, bb = mse_inputs(shape, seed, kind)
        mse_out.append({"shape": list(shape), "seed": seed, "kind": kind,
                        "mse_hex": float(cache.mse(a, bb)).hex()})
    (HERE / "mse_bits.json").write_text(json.dumps(mse_out))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
