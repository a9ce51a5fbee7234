"""CPU oracle for the PatchedServe patch-execution path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy float64, the algorithm of the reference
`mixserve` package (`/root/reference/pkg/src/mixserve/*.py`) for the hot path
named by BASELINE.json's north star: CSP split/merge + halos, per-image
GroupNorm, per-image attention, the pixel-wise ops, the block interpreter and
the patch-cache reuse test.  Every function cites the reference file:line it
follows.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
reference-arm legs may import this package, and only as the checker (or the
timed CPU reference).  The product (`paper_2501_09253_b200`) never imports it:
its path is the CUDA library and it fails loudly when that is missing.

Parity pinning: `tests/golden/make_golden.py` imports the real reference in the
build container and records golden input/output vectors under `tests/golden/`;
`tests/test_oracle_golden.py` checks this restatement against them (integer and
copy results bit-exact, float results to 1e-12 or bit-exact where the reference
itself is order-deterministic).  The numpy pairwise-summation dependency that
makes cache masks bit-exact is restated in `pairwise.py` and checked bitwise
against `np.mean` (numpy 2.3.5).
"""
