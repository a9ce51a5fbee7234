"""Restatement of numpy's float64 pairwise summation — TEST INFRASTRUCTURE ONLY.

The reference decides cache reuse with `mse(a, b) = float(np.mean((a - b) ** 2))`
(`/root/reference/pkg/src/mixserve/cache.py:54-55`, used by `_mse_predictor`,
`cache.py:87-88`).  The bits of that mean come from numpy's add-reduce, a
third-party dependency that is not vendored in `/root/reference`:

* dependency: numpy (unpinned in `pkg/pyproject.toml:10`; restated from and
  verified against numpy 2.3.5, the version in this image);
* algorithm: `pairwise_sum` in `numpy/_core/src/umath/loops_utils.h.src`
  (PW_BLOCKSIZE = 128), entered once over the whole C-contiguous array because
  the reduce iterator coalesces the axes; the add identity 0.0 is added in front
  and `np.mean` then divides by the element count.

`tests/test_oracle_pairwise.py` checks `np_mean_sq_diff` bitwise against
`np.mean` on the patch shapes the GPU kernel (`csrc/cache.cu`) has to match.
`leaf_plan` is the same tree expressed as leaves + combine order, which is what
the CUDA kernel's plan builder (`csrc/capi.cpp: ps_pairwise_plan`) produces.
"""

from __future__ import annotations

import numpy as np

PW_BLOCKSIZE = 128


def pairwise_sum(a: np.ndarray, lo: int = 0, n: int | None = None) -> float:
    """Sum a[lo:lo+n] (float64, 1-D) with numpy's pairwise tree."""
    if n is None:
        n = a.shape[0] - lo
    if n < 8:
        res = -0.0
        for i in range(n):
            res += float(a[lo + i])
        return res
    if n <= PW_BLOCKSIZE:
        r = [float(a[lo + j]) for j in range(8)]
        i = 8
        stop = n - (n % 8)
        while i < stop:
            for j in range(8):
                r[j] += float(a[lo + i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += float(a[lo + i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a, lo, n2) + pairwise_sum(a, lo + n2, n - n2)


def np_mean_sq_diff(a, b) -> float:
    """Restated `float(np.mean((a - b) ** 2))` for C-contiguous float64 inputs."""
    d = (np.ascontiguousarray(a, dtype=np.float64) - np.ascontiguousarray(b, dtype=np.float64)).ravel()
    sq = d * d
    total = 0.0 + pairwise_sum(sq)
    return total / sq.shape[0]


def leaf_plan(n: int):
    """Leaves (start, length) in order and the binary combine tree of pairwise_sum(n).

    Returns (leaves, nodes) where nodes is a post-order list of
    ("leaf", idx) / ("add", left_node, right_node); the last node is the root.
    """
    leaves: list[tuple[int, int]] = []
    nodes: list[tuple] = []

    def rec(lo: int, m: int) -> int:
        if m <= PW_BLOCKSIZE:
            leaves.append((lo, m))
            nodes.append(("leaf", len(leaves) - 1))
            return len(nodes) - 1
        m2 = m // 2
        m2 -= m2 % 8
        left = rec(lo, m2)
        right = rec(lo + m2, m - m2)
        nodes.append(("add", left, right))
        return len(nodes) - 1

    rec(0, n)
    return leaves, nodes
