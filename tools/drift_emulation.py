"""Where does the 50-step latent drift of the bf16 path come from?  Pure-numpy emulation (oracle,
BLAS mode): the fp64 trajectory of one 512 px request (the SDXL-shaped 7-block model of
tests/test_gpu_parity_c320.py::test_c320_drift_50_steps_512px) against the same trajectory with
  W  : weights rounded to bf16 (what the GPU's tensor cores multiply),
  RS : the residual stream (every block output) rounded to bf16,
  W+RS both,
  W+ST: weights and every intra-block stage output (GN / frames, conv, attention, FF) in bf16,
        residual stream (block outputs) exact -- an fp32 residual stream on the GPU,
  W+ST+RS: the bf16 GPU path as built in round 1.
Prints / writes the per-step max |d| of each variant.
  python tools/drift_emulation.py [steps] [out.json] [variant,...]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import mixref as R  # noqa: E402
from tests.golden.cases import bf16_round  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
out = sys.argv[2] if len(sys.argv) > 2 else None
cfg = R.ModelConfig(arch="unet_like", channels=320, hidden=1280, groups=32, n_blocks=7, seed=3)
w = R.init_weights(cfg)


def rounded(ops_list):
    res = []
    for ops in ops_list:
        new = []
        for kind, p in ops:
            if p is None or kind == "residual":
                new.append((kind, p))
                continue
            kw = {f: (bf16_round(getattr(p, f)) if isinstance(getattr(p, f), np.ndarray) else getattr(p, f))
                  for f in p.__dataclass_fields__}
            new.append((kind, type(p)(**kw)))
        res.append(new)
    return res


wb = rounded(w)
rid = "req-0"
lat = np.random.default_rng([5, 0]).normal(size=(320, 64, 64)).astype(np.float32).astype(np.float64)
prompt = R.make_prompt(cfg, rid)
all_variants = {"exact": (w, None, False), "W": (wb, None, False), "RS": (w, bf16_round, False),
                "W+RS": (wb, bf16_round, False), "W+ST": (wb, None, True), "W+ST+RS": (wb, bf16_round, True)}
pick = sys.argv[3].split(",") if len(sys.argv) > 3 else ["W", "RS", "W+RS"]
variants = {k: all_variants[k] for k in ["exact"] + pick}
xs = {k: lat.copy() for k in variants}
curves = {k: [] for k in variants if k != "exact"}
with R.blas_contractions():
    for s in range(steps):
        for k, (ww, rf, st) in variants.items():
            b = R.split([(rid, xs[k])], patch_size=32)
            R.STAGE_ROUND = bf16_round if st else None
            d = R.denoise_batch(cfg, ww, b, {rid: prompt}, {rid: s}, {rid: 50}, round_fn=rf)
            R.STAGE_ROUND = None
            xs[k] = R.reassemble(b, d)[rid]
        for k in curves:
            curves[k].append(float(np.abs(xs[k] - xs["exact"]).max()))
        print(s, {k: round(v[-1], 5) for k, v in curves.items()}, flush=True)
if out:
    with open(out, "w") as f:
        json.dump(curves, f, indent=1)
