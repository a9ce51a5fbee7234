"""Config 5 (1x 2048 px + 8x 512 px, patch 64, SDXL-shaped model) on the split-image
path, projected to W GPUs from one B200.

For each rank of SplitPlan(W), the rank's full denoising step (its local CSP batch,
owned patches only, pack/unpack kernels included) runs on this GPU with the
collectives replaced by no-ops (NullComm); its device time is measured with CUDA
events.  The projected W-GPU step = max over ranks of (device time + bytes the
rank exchanges / NVLink bandwidth), with the exchange NOT overlapped (upper bound).
Bandwidth: 770 GB/s per direction (measured peer copy, B200_PROFILING.md).
SPLIT_WORLDS=8 SPLIT_RANKS=0 SPLIT_GRAPH=0 times one rank of one world (for an ncu launch list).
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2501_09253_b200 as ps
from paper_2501_09253_b200.model import denoise_batch_shard, step_inputs
from paper_2501_09253_b200.patched import shard_context
from paper_2501_09253_b200.patchshard import ShardExchange, SplitPlan

NVLINK_GBS = 770.0
GRAPH = os.environ.get("SPLIT_GRAPH", "1") == "1"
MODE = os.environ.get("SPLIT_MODE", "balanced")
C, H, G, NB, PS = 320, 1280, 32, 7, 64
REQS = [("big", 256)] + [(f"s{i}", 64) for i in range(8)]


class NullComm:
    def __init__(self, world):
        self.world = world

    def all_gather(self, rank, t):
        return torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)

    def exchange(self, rank, sends, recv_like):
        return {s: torch.empty(shape, dtype=dt, device=dev) for s, (shape, dt, dev) in recv_like.items()}


def time_rank(cfg, w, plan, r, reps=3):
    sh = plan.shard(r)
    lats = {rid: torch.randn(C, d, d, device="cuda") for rid, d in sh.requests}
    b = ps.split([(rid, lats[rid]) for rid, _ in sh.requests], patch_size=PS)
    prompts = {rid: ps.make_prompt(cfg, rid) for rid, _ in sh.requests}
    si = {rid: 3 for rid, _ in sh.requests}
    ts = {rid: 50 for rid, _ in sh.requests}
    ex = ShardExchange(sh, NullComm(plan.world))
    denoise_batch_shard(cfg, w, b, sh, ex, prompts, si, ts)  # warm-up (plans, tables, allocations)
    torch.cuda.synchronize()
    ex.bytes_moved = 0
    denoise_batch_shard(cfg, w, b, sh, ex, prompts, si, ts)
    sent = ex.bytes_moved
    torch.cuda.synchronize()
    inputs = step_inputs(cfg, b, prompts, si, ts)
    ctx = shard_context(b, sh, ex)
    step = lambda: denoise_batch_shard(cfg, w, b, sh, ex, prompts, si, ts, inputs=inputs, ctx=ctx)
    if GRAPH:
        # the whole rank step as one CUDA graph: device time without host launch gaps
        # (with NCCL the collectives are captured too)
        g = torch.cuda.CUDAGraph()
        s_ = torch.cuda.Stream()
        s_.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_):
            step()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s_):
                step()
        torch.cuda.current_stream().wait_stream(s_)
        step = g.replay
    ts_ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        ts_ms.append(e0.elapsed_time(e1))
    # received: every all-gather delivers (world-1) peer buffers of the same size; halos ~ sent
    return float(np.median(ts_ms)), sent, len(sh.owned)


def main():
    cfg = ps.ModelConfig(arch="unet_like", channels=C, hidden=H, groups=G, n_blocks=NB, seed=0)
    w = ps.init_weights(cfg)
    out = []
    worlds = [int(x) for x in os.environ.get("SPLIT_WORLDS", "1,2,4,8").split(",")]
    only = os.environ.get("SPLIT_RANKS")  # e.g. "0": time only these ranks (ncu launch lists)
    for world in worlds:
        plan = SplitPlan(REQS, PS, world, mode=MODE)
        ranks = []
        for r in range(world):
            if only is not None and str(r) not in only.split(","):
                continue
            ms, sent, owned = time_rank(cfg, w, plan, r)
            comm_ms = sent * (world - 1) / (NVLINK_GBS * 1e9) * 1e3 if world > 1 else 0.0
            ranks.append({"rank": r, "owned_patches": owned, "device_ms": ms, "sent_MB": sent / 1e6,
                          "comm_ms_est": comm_ms, "total_ms": ms + comm_ms})
        step = max(x["total_ms"] for x in ranks)
        line = {"world": world, "graph": GRAPH, "mode": plan.mode,
                "owned": [len(plan.owned_by(r)) for r in range(world)], "split_images": len(plan.split_requests()),
                "step_ms_projected": step, "patches_per_s": 24 / (step * 1e-3), "ranks": ranks}
        out.append(line)
        print(json.dumps(line), flush=True)
    if only is not None or worlds[0] != 1:
        return
    base = out[0]["patches_per_s"]
    for l in out:
        print(f"W={l['world']}: {l['step_ms_projected']:.2f} ms/step projected, {l['patches_per_s']:.0f} patches/s, "
              f"scaling efficiency {l['patches_per_s'] / (base * l['world']):.2f}", flush=True)


if __name__ == "__main__":
    main()
