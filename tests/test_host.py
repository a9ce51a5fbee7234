"""CPU-only checks: the C-ABI library loads and exports every declared symbol, the
host-side plan builders (CSP metadata, numpy pairwise-summation tree) match the
oracle / golden vectors, error mapping, and the multi-rank ownership logic
(gloo, world size 2)."""

import ctypes as C
import json
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "patchserve.h")
GOLD = os.path.join(ROOT, "tests", "golden")


def _lib():
    from paper_2501_09253_b200 import _lib as L
    if not os.path.exists(L.LIB_PATH):
        subprocess.run(["make", "-j8", "-C", os.path.join(ROOT, "paper_2501_09253_b200", "csrc")], check=True)
    return L


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib()
    lib = L.load()
    decl = declared_symbols()
    assert len(decl) >= 25
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(L.EXPORTED) == decl
    assert lib.ps_abi_version() == L.ABI_VERSION
    hdr = open(HEADER).read()
    assert re.search(rf"#define PS_ABI_VERSION {L.ABI_VERSION}\b", hdr)
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    for name in decl:
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a():
    L = _lib()
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", L.LIB_PATH], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):  # tcgen05.mma, TMA, tcgen05.ld
        assert mnem in sass, mnem


def _csp_plan(dims, ps):
    L = _lib()
    lib = L.load()
    n = len(dims)
    d = (C.c_int32 * n)(*dims)
    P, nres = C.c_int32(), C.c_int32()
    L.check(lib.ps_csp_count(n, d, ps, C.byref(P), C.byref(nres)))
    P, nres = P.value, nres.value
    arrs = [np.zeros(k, np.int32) for k in (n, n + 1, nres, nres + 1, P, P, P, P, 8 * P)]
    L.check(lib.ps_csp_build(n, d, ps, *[a.ctypes.data_as(C.c_void_p) for a in arrs]))
    return arrs


def test_csp_plan_matches_golden():
    from math import gcd
    from tests.golden.cases import CSP_CASES
    gold = json.load(open(os.path.join(GOLD, "csp_kats.json")))
    for (dims, ps), g in zip(CSP_CASES, gold):
        ps = ps or gcd(*dims)
        order, ro, rd, so, ri, od, rw, cl, nb = _csp_plan(dims, ps)
        assert [f"r{i}" for i in order] == g["order"]
        assert ro.tolist() == g["request_offset"] and so.tolist() == g["resolution_offset"]
        assert rd.tolist() == g["resolution_dims"]
        assert ri.tolist() == g["request_index"] and od.tolist() == g["ordinal"]
        assert rw.tolist() == g["row"] and cl.tolist() == g["col"]
        assert nb.reshape(-1, 8).tolist() == g["neighbors"]


def test_csp_plan_rejects_bad_input():
    from paper_2501_09253_b200.errors import InputError
    with pytest.raises(InputError):
        _csp_plan([64, 48], 32)
    with pytest.raises(InputError):
        _csp_plan([64, 0], 32)


def _pairwise_plan(n):
    L = _lib()
    lib = L.load()
    nl, ni, nh = C.c_int32(), C.c_int32(), C.c_int32()
    L.check(lib.ps_pairwise_plan(n, C.byref(nl), C.byref(ni), C.byref(nh), None, None, None))
    leaves = np.zeros(2 * nl.value, np.int32)
    nodes = np.zeros(max(1, 2 * ni.value), np.int32)
    lvl = np.zeros(nh.value + 1, np.int32)
    L.check(lib.ps_pairwise_plan(n, C.byref(nl), C.byref(ni), C.byref(nh), leaves.ctypes.data_as(C.c_void_p),
                                 nodes.ctypes.data_as(C.c_void_p), lvl.ctypes.data_as(C.c_void_p)))
    return leaves.reshape(-1, 2), nodes[:2 * ni.value].reshape(-1, 2), lvl


@pytest.mark.parametrize("shape", [(2, 3, 3), (4, 4, 4), (4, 16, 16), (3, 5, 7), (320, 32, 32), (320, 16, 16),
                                   (8, 64, 64), (1, 1, 5), (4, 32, 32)])
def test_pairwise_plan_reproduces_numpy_mean(shape):
    """Evaluate the GPU kernel's plan on the CPU, level by level, and compare with np.mean bitwise."""
    from oracle.pairwise import leaf_plan, pairwise_sum
    n = int(np.prod(shape))
    leaves, nodes, lvl = _pairwise_plan(n)
    ref_leaves, _ = leaf_plan(n)
    assert [tuple(x) for x in leaves.tolist()] == ref_leaves
    rng = np.random.default_rng(n)
    a = rng.normal(size=shape)
    b = rng.normal(size=shape) * 1.1
    sq = ((a - b) ** 2).ravel()
    L = len(leaves)
    vals = np.zeros(L + len(nodes))
    for k, (s, ln) in enumerate(leaves.tolist()):
        vals[k] = pairwise_sum(sq, s, ln)
    for h in range(len(lvl) - 1):
        for i in range(lvl[h], lvl[h + 1]):
            vals[L + i] = vals[nodes[i, 0]] + vals[nodes[i, 1]]
    root = vals[L + len(nodes) - 1] if len(nodes) else vals[0]
    assert ((0.0 + root) / n) == float(np.mean((a - b) ** 2))


def test_pairwise_restatement_matches_numpy_and_differs_from_naive():
    from oracle.pairwise import np_mean_sq_diff
    rng = np.random.default_rng(11)
    naive_diff = 0
    for shape in [(320, 32, 32), (4, 16, 16), (7, 11, 13), (640, 16, 16)]:
        for _ in range(3):
            a, b = rng.normal(size=shape), rng.normal(size=shape)
            assert np_mean_sq_diff(a, b) == float(np.mean((a - b) ** 2))
            d = ((a - b) ** 2).ravel()
            s = 0.0
            for v in d.tolist():
                s += v
            naive_diff += (s / d.size) != float(np.mean((a - b) ** 2))
    assert naive_diff > 0  # the tree matters: sequential summation gives other bits



def test_integration_ctypes_stub_matches_header():
    """INTEGRATION.md's ctypes stub for ps_cache_predict declares as many arguments as the C
    prototype in include/patchserve.h and the facade's signature table."""
    import re

    from paper_2501_09253_b200 import _lib
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    stub = re.search(r"lib\.ps_cache_predict\.argtypes = \[(.*?)\]", doc, re.S).group(1)
    n_stub = len([a for a in stub.split(",") if a.strip()])
    hdr = open(os.path.join(ROOT, "include", "patchserve.h")).read()
    proto = re.search(r"int ps_cache_predict\((.*?)\);", hdr, re.S).group(1)
    n_hdr = len(proto.split(","))
    assert n_stub == n_hdr == len(_lib._SIGS["ps_cache_predict"][0])
