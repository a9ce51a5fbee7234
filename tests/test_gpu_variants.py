"""Default kernels against their A/B baselines: a faster variant that keeps the arithmetic order
of the kernel it replaced must produce identical bytes; one that reorders a reduction is held to
the fp64 statistics.  The baseline runs in a subprocess with the variant's off switch set (the
switches are read once per process).

  * GroupNorm partials: the warp-per-slice kernel (shifted single-pass moments) and the
    one-CTA-per-(patch, group) two-pass kernel (PS_GN_WARP_OFF=1) against fp64 statistics, over
    the whole batch and over a device patch list with a device count.
"""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

GN_SCRIPT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2501_09253_b200 import _lib
from paper_2501_09253_b200._dev import stream
P, C, ps, G = 116, 320, 32, 32
g = torch.Generator(device="cuda").manual_seed(5)
x = (torch.randn((P, C, ps, ps), device="cuda", generator=g) * 2 + 0.5).to(torch.bfloat16)
full = torch.full((P, G, 2), float("nan"), device="cuda")
_lib.check(_lib.load().ps_gn_partials(stream(), x.data_ptr(), P, C, ps, G, full.data_ptr()))
lst = torch.arange(3, P, 2, dtype=torch.int32, device="cuda")
n_dev = torch.tensor([lst.numel() - 4], dtype=torch.int32, device="cuda")
sub = torch.full((P, G, 2), float("nan"), device="cuda")
_lib.check(_lib.load().ps_gn_partials_sub(stream(), x.data_ptr(), P, C, ps, G, lst.data_ptr(), lst.numel(),
                                          sub.data_ptr(), n_dev.data_ptr()))
torch.cuda.synchronize()
torch.save({"x": x.cpu(), "full": full.cpu(), "sub": sub.cpu(), "lst": lst.cpu()}, sys.argv[2])
"""


def _run(tmp_path, name, env_extra):
    out = tmp_path / f"{name}.pt"
    env = dict(os.environ, **env_extra)
    subprocess.run([sys.executable, "-c", GN_SCRIPT, ROOT, str(out)], check=True, env=env, timeout=300)
    return torch.load(out)


def test_gn_partials_warp_kernel(tmp_path):
    """The warp-per-slice shifted-moment kernel against the one-CTA-per-slice two-pass kernel and
    fp64 statistics (tolerance: both are fp32 reductions in different orders)."""
    new = _run(tmp_path, "warp", {})
    base = _run(tmp_path, "base", {"PS_GN_WARP_OFF": "1"})
    assert torch.equal(new["x"], base["x"])
    x = new["x"].double().numpy().reshape(116, 32, -1)
    mean = x.mean(-1)
    m2 = ((x - mean[..., None]) ** 2).sum(-1)
    for r in (new, base):
        np.testing.assert_allclose(r["full"][..., 0].double().numpy(), mean, rtol=0, atol=2e-5)
        np.testing.assert_allclose(r["full"][..., 1].double().numpy(), m2, rtol=2e-5)
        # the sub-list launch writes exactly the first n_dev listed patches and nothing else
        written = r["lst"][: r["lst"].numel() - 4].long()
        mask = torch.zeros(116, dtype=torch.bool)
        mask[written] = True
        assert not r["sub"][mask].isnan().any() and r["sub"][~mask].isnan().all()
        assert torch.equal(r["sub"][mask], r["full"][mask])


@pytest.mark.parametrize("P,ps_", [(29, 32), (6, 64)])
def test_gn_partials_offset_and_outlier_shift(P, ps_):
    """Shifted single-pass moments stay accurate when the shift (the slice's first element) is an
    outlier and the data sit on a large offset: mean 50, std 1, first element of every slice at
    50 + 8 (M2 is then a difference of two sums ~65x larger than itself).  ps = 64: 80 KB slices,
    four warps per slice whose sums share the shift."""
    from paper_2501_09253_b200 import _lib
    from paper_2501_09253_b200._dev import stream
    C, G = 320, 32
    g = torch.Generator(device="cuda").manual_seed(11)
    x = (50.0 + torch.randn((P, C, ps_, ps_), device="cuda", generator=g))
    xv = x.view(P, G, -1)
    xv[:, :, 0] = 58.0
    x = x.to(torch.bfloat16)
    part = torch.empty((P, G, 2), device="cuda")
    _lib.check(_lib.load().ps_gn_partials(stream(), x.data_ptr(), P, C, ps_, G, part.data_ptr()))
    torch.cuda.synchronize()
    ref = x.double().view(P, G, -1)
    mean = ref.mean(-1)
    m2 = ((ref - mean[..., None]) ** 2).sum(-1)
    assert float((part[..., 0].double() - mean).abs().max()) <= 2e-4  # fp32 mean of ~50 (ulp 4e-6)
    assert float(((part[..., 1].double() - m2).abs() / m2).max()) <= 1e-4


CONV_SCRIPT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2501_09253_b200 as ps
cfg = ps.ModelConfig(arch="unet_like", channels=320, hidden=1280, n_blocks=1, groups=32, seed=2)
conv = ps.init_weights(cfg)[0][1][1]
g = torch.Generator().manual_seed(3)
reqs = [(f"r{i}", torch.randn((320, d, d), generator=g)) for i, d in enumerate([64, 96, 128] * 4)]
b = ps.split(reqs, patch_size=32)  # P = 116: 464 CTA-pair tiles on 74 pairs -> a 20-tile tail wave
x = b.data.to(torch.bfloat16).cuda()
y = ps.patched_conv(b, x, conv)
torch.cuda.synchronize()
torch.save(y.cpu(), sys.argv[2])
"""


def test_conv3_tail_split_bit_identical(tmp_path):
    """conv3 (CTA-pair tiles, BN = 320) with the last partial wave split into column-half work
    items equals the unsplit schedule bit for bit (every column keeps its k order)."""
    outs = {}
    for name, env in (("split", {}), ("whole", {"PS_GEMM_TAIL_SPLIT": "0"})):
        out = tmp_path / f"{name}.pt"
        subprocess.run([sys.executable, "-c", CONV_SCRIPT, ROOT, str(out)], check=True, timeout=300,
                       env=dict(os.environ, **env))
        outs[name] = torch.load(out)
    assert torch.equal(outs["split"], outs["whole"])
