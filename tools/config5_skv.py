"""Config-5 batch on one GPU (bench.measure_config5) with and without the pair split-KV:
  PS_SPLITKV_SINGLE_MIN_BLOCKS=1000000 python tools/config5_skv.py   # one-pass pair kernel
  python tools/config5_skv.py                                       # default rule
prints the bench's config5 line plus whether a split plan was used."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_09253_b200 as ps  # noqa: E402
from paper_2501_09253_b200 import patched  # noqa: E402

cfg = ps.ModelConfig(arch="unet_like", channels=bench.C, hidden=bench.HIDDEN, groups=bench.GROUPS,
                     n_blocks=bench.BLOCKS, seed=0)
w = ps.init_weights(cfg)
line = bench.measure_config5(cfg, w)
plans = [k for k, v in patched._SKV_CACHE.items() if k[0] == "pairs"]
line["pair_splitkv_plans"] = [(v is not None) and {"pair_tiles": v[4], "split_halves": v[9], "slots": v[12]}
                              for k, v in patched._SKV_CACHE.items() if k[0] == "pairs"]
line["single_min_blocks"] = patched.SPLITKV_SINGLE_MIN_BLOCKS
print(json.dumps(line))
