"""Request-to-GPU ownership for the multi-GPU path (one process per GPU).

The patch path never mixes requests: halo neighbours are intra-image
(csp.py:171-174), GroupNorm statistics are per request (patched.py:132-140)
and attention is per image (patched.py:164-176).  Whole-request ownership
therefore shards the work with no data-path collective.  Ownership follows
the reference's lowest-outstanding-work dispatch (engine.py:120-124, 228:
argmin over (outstanding work, worker id)), computed identically on every rank
from the same request list, so ranks agree without communicating.

Work per request is the algorithmic FLOP count of one denoising step of the
configured model (attention 4 T^2 D + 8 T D^2, conv3 18 C^2 T, FF 4 C H T per
block), which is what a B200 step time is proportional to.
"""

from __future__ import annotations

from typing import Sequence


def step_flops(latent: int, channels: int, hidden: int, n_blocks: int, arch: str = "unet_like") -> float:
    t = latent * latent
    per_block = 4.0 * t * t * channels + 8.0 * t * channels * channels + 4.0 * channels * hidden * t
    if arch == "unet_like":
        per_block += 18.0 * channels * channels * t
    return n_blocks * per_block


def assign(requests: Sequence[tuple], world: int, cost) -> list[int]:
    """Owner rank of each request, in input order.

    `requests` items are (request_id, latent_dim, ...); `cost(latent_dim)`
    gives the per-step work.  Greedy lowest-load with ties to the lowest rank,
    in arrival order (engine.py:228).
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    load = [0.0] * world
    owner = []
    for req in requests:
        r = min(range(world), key=lambda k: (load[k], k))
        owner.append(r)
        load[r] += cost(req[1])
    return owner


def local_requests(requests: Sequence[tuple], rank: int, world: int, cost) -> list:
    owners = assign(requests, world, cost)
    return [req for req, o in zip(requests, owners) if o == rank]
