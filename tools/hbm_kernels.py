"""The config-2 HBM kernel table (bench.measure_hbm_kernels) on its own, for an ncu capture:
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv python tools/hbm_kernels.py
prints the CUDA-event table as JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_09253_b200 as ps  # noqa: E402
from paper_2501_09253_b200.pipeline import DenoisePipeline  # noqa: E402

cfg = ps.ModelConfig(arch="unet_like", channels=bench.C, hidden=bench.HIDDEN, groups=bench.GROUPS,
                     n_blocks=int(os.environ.get("HBM_BLOCKS", 2)), seed=0)
w = ps.init_weights(cfg)
reqs = bench.make_requests(0, 0)
pipe = DenoisePipeline(cfg, w, bench.DIMS, bench.PATCH, use_graph=False)
pipe.set_prompts([ps.make_prompt(cfg, rid) for rid, _ in reqs])
import torch  # noqa: E402
for k in range(pipe.n_sets):
    for r, (_, lat) in enumerate(reqs):
        pipe.lat_in[k][r].copy_(torch.as_tensor(lat, dtype=torch.float32))
    pipe.rates[k].fill_(0.1)
pipe.prepare()
print(json.dumps(bench.measure_hbm_kernels(pipe, bench._peaks().get("hbm_gbs", 6548.5)), indent=1))
