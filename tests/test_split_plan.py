"""Split-image multi-GPU plan, host side, CPU only.

The exchange tables of patchshard.py are checked by simulating every device
mover in numpy (halo strip pack/unpack, segment copies) and every collective in
Python, then comparing what each rank's owned patches would read with the
single-GPU arrays: halo frames (exchange_halos, patched.py:57-89), GroupNorm
partial rows (patched.py:132-140) and attention K / V^T (patched.py:164-176).
The gloo test runs the torch.distributed adapter at world size 2.
"""

import itertools
import os

import numpy as np
import pytest

from paper_2501_09253_b200.patchshard import SplitPlan, kv_plan, linear_partition, patch_cost


def _brute(w, parts):
    n = len(w)
    best = None
    for cuts in itertools.combinations_with_replacement(range(n + 1), parts - 1):
        c = [0, *cuts, n]
        m = max(sum(w[c[i]:c[i + 1]]) for i in range(parts))
        best = m if best is None else min(best, m)
    return best


@pytest.mark.parametrize("seed", range(6))
def test_linear_partition_optimal(seed):
    rng = np.random.default_rng(seed)
    w = rng.integers(1, 20, size=int(rng.integers(3, 9))).astype(float).tolist()
    for parts in (1, 2, 3):
        cuts = linear_partition(w, parts)
        assert cuts[0] == 0 and cuts[-1] == len(w) and len(cuts) == parts + 1
        assert all(a <= b for a, b in zip(cuts, cuts[1:]))
        got = max(sum(w[cuts[i]:cuts[i + 1]]) for i in range(parts))
        assert got == pytest.approx(_brute(w, parts))
        if len(w) >= parts:
            assert all(cuts[i + 1] > cuts[i] for i in range(parts))


def test_config5_plan():
    """Config 5: 1x2048 px + 8x512 px, patch 64, 8 GPUs."""
    reqs = [("big", 256)] + [(f"s{i}", 64) for i in range(8)]
    plan = SplitPlan(reqs, 64, 8, mode="contiguous")
    assert plan.n_patches == 24
    assert plan.split_requests() == [8]  # the 2048 px image, last in CSP order
    per_patch = patch_cost(256, 64)
    assert max(plan.load) <= 3 * per_patch  # bottleneck <= 3 big patches
    assert all(plan.cuts[k + 1] > plan.cuts[k] for k in range(8))
    for r in range(8):
        sh = plan.shard(r)
        assert len(sh.owned) == plan.cuts[r + 1] - plan.cuts[r]
    # balanced: every GPU gets 2 patches of the 2048 px image and one whole 512 px image
    bal = SplitPlan(reqs, 64, 8)
    assert bal.split_requests() == [8]
    for r in range(8):
        own = bal.owned_by(r)
        assert len(own) == 3
        assert sum(1 for g in own if bal.req_of(g) == 8) == 2
    assert max(bal.load) / min(bal.load) < 1.01


def test_balanced_keeps_small_requests_whole():
    reqs = [(f"r{i}", d) for i, d in enumerate([64, 96, 128] * 4)]
    plan = SplitPlan(reqs, 32, 8)
    split = set(plan.split_requests())
    for k, rq in enumerate(plan.reqs):
        owners = {plan.owner(g) for g in range(rq.g0, rq.g0 + rq.count)}
        assert (len(owners) > 1) == (k in split)
    assert SplitPlan(reqs, 32, 1).split_requests() == []


def _cases():
    for mode in ("balanced", "contiguous"):
        yield [("a", 64), ("b", 16), ("c", 32), ("d", 16)], 16, 2, mode
        yield [("a", 64), ("b", 16), ("c", 32), ("d", 16)], 16, 3, mode
        yield [("big", 128), ("x", 32), ("y", 64)], 32, 4, mode
        yield [("big", 96), ("x", 48), ("y", 48)], 16, 5, mode
        yield [("only", 64)], 16, 4, mode
        yield [("big", 256)] + [(f"s{i}", 64) for i in range(8)], 64, 8, mode


def _neighbour_frames(arr, plan, sh, g):
    """(C, ps+2, ps+2) frame of global patch g read from a local array (zero outside the image)."""
    ps = plan.ps
    C = arr.shape[1]
    f = np.zeros((C, ps + 2, ps + 2))
    f[:, 1:-1, 1:-1] = arr[sh.local(g)]
    sl = {0: (slice(0, 1), slice(1, -1), slice(ps - 1, ps), slice(None)),
          1: (slice(0, 1), slice(-1, None), slice(ps - 1, ps), slice(0, 1)),
          2: (slice(1, -1), slice(-1, None), slice(None), slice(0, 1)),
          3: (slice(-1, None), slice(-1, None), slice(0, 1), slice(0, 1)),
          4: (slice(-1, None), slice(1, -1), slice(0, 1), slice(None)),
          5: (slice(-1, None), slice(0, 1), slice(0, 1), slice(ps - 1, ps)),
          6: (slice(1, -1), slice(0, 1), slice(None), slice(ps - 1, ps)),
          7: (slice(0, 1), slice(0, 1), slice(ps - 1, ps), slice(ps - 1, ps))}
    for d in range(8):
        q = plan.neighbour(g, d)
        if q < 0:
            continue
        fy, fx, sy, sx = sl[d]
        f[:, fy, fx] = arr[sh.local(q)][:, sy, sx]
    return f


def _strip_io(arr, q, code, ps, buf=None):
    if buf is None:
        return (arr[q][:, code, :] if code < ps else arr[q][:, :, code - ps]).copy()
    if code < ps:
        arr[q][:, code, :] = buf
    else:
        arr[q][:, :, code - ps] = buf


@pytest.mark.parametrize("case", list(_cases()))
def test_halo_exchange_simulated(case):
    reqs, ps, world, mode = case
    plan = SplitPlan(reqs, ps, world, mode=mode)
    C = 3
    rng = np.random.default_rng(1)
    full = rng.normal(size=(plan.n_patches, C, ps, ps))
    shards = [plan.shard(r) for r in range(world)]
    local = []
    for sh in shards:
        a = np.full((sh.n_patches, C, ps, ps), np.nan)
        for g in plan.owned_by(sh.rank):
            a[sh.local(g)] = full[g]
        local.append(a)
    # pack on every sender, then unpack on every receiver
    msgs = {}
    for sh in shards:
        for d, strips in sh.halo_send.items():
            msgs[(sh.rank, d)] = np.stack([_strip_io(local[sh.rank], q, c, ps) for q, c in strips])
    for sh in shards:
        for s, strips in sh.halo_recv.items():
            buf = msgs.pop((s, sh.rank))
            assert buf.shape == (len(strips), C, ps)
            for (q, c), b in zip(strips, buf):
                _strip_io(local[sh.rank], q, c, ps, b)
    assert not msgs
    # every owned patch's frame equals the single-GPU frame (no NaN ghost read)
    for sh in shards:
        for g in plan.owned_by(sh.rank):
            got = _neighbour_frames(local[sh.rank], plan, sh, g)
            ref = _frames_full(full, plan, g)
            assert not np.isnan(got).any()
            np.testing.assert_array_equal(got, ref)


def _frames_full(full, plan, g):
    class _Id:
        @staticmethod
        def local(x):
            return x
    return _neighbour_frames(full, plan, _Id, g)


def _copy_segments(src: np.ndarray, dst: np.ndarray, so, do, nbytes):
    for a, b in zip(so, do):
        dst[b:b + nbytes] = src[a:a + nbytes]


@pytest.mark.parametrize("case", list(_cases()))
def test_gn_partials_exchange_simulated(case):
    reqs, ps, world, mode = case
    plan = SplitPlan(reqs, ps, world, mode=mode)
    G = 4
    rng = np.random.default_rng(2)
    full = rng.normal(size=(plan.n_patches, G, 2)).astype(np.float32)
    shards = [plan.shard(r) for r in range(world)]
    loc = []
    for sh in shards:
        a = np.full((sh.n_patches, G, 2), np.nan, np.float32)
        for g in plan.owned_by(sh.rank):
            a[sh.local(g)] = full[g]
        loc.append(a)
    if shards[0].gn_max == 0:
        assert not plan.split_requests()
        return
    sends = []
    for sh in shards:
        ps_, pd, us, ud, row = sh.gn_offsets(G)
        buf = np.zeros(sh.gn_max * G * 2, np.float32)
        _copy_segments(loc[sh.rank].view(np.uint8).reshape(-1), buf.view(np.uint8), ps_, pd, row)
        sends.append(buf)
    got = np.stack(sends)
    for sh in shards:
        ps_, pd, us, ud, row = sh.gn_offsets(G)
        _copy_segments(got.view(np.uint8).reshape(-1), loc[sh.rank].view(np.uint8).reshape(-1), us, ud, row)
        for k in sh.slots:
            rq = plan.reqs[k]
            if k in plan.split_requests():
                for g in range(rq.g0, rq.g0 + rq.count):
                    np.testing.assert_array_equal(loc[sh.rank][sh.local(g)], full[g])


@pytest.mark.parametrize("case", list(_cases()))
def test_kv_exchange_simulated(case):
    reqs, ps, world, mode = case
    plan = SplitPlan(reqs, ps, world, mode=mode)
    hw = ps * ps
    dpp = 64
    rng = np.random.default_rng(3)
    # global token-major K and V (bf16 stand-ins as uint16)
    Kf = rng.integers(0, 65535, size=(plan.n_patches * hw, dpp), dtype=np.uint16)
    Vf = rng.integers(0, 65535, size=(plan.n_patches * hw, dpp), dtype=np.uint16)
    shards = [plan.shard(r) for r in range(world)]
    if shards[0].kv_max_tokens == 0:
        return
    st = []
    for sh in shards:
        T = sh.n_patches * hw
        ldv = (T + 63) // 64 * 64
        qk = np.zeros((T, 2 * dpp), np.uint16)
        vt = np.zeros((dpp, ldv), np.uint16)
        for g in plan.owned_by(sh.rank):
            t = sh.local(g) * hw
            qk[t:t + hw, dpp:] = Kf[g * hw:(g + 1) * hw]
            vt[:, t:t + hw] = Vf[g * hw:(g + 1) * hw].T
        pl = kv_plan(sh, dpp, ldv)
        send = np.zeros(pl["buf_bytes"], np.uint8)
        ks, kd, kb = pl["k_pack"]
        _copy_segments(qk.view(np.uint8).reshape(-1), send, ks, kd, kb)
        vs, vd, vn = pl["v_pack_var"]  # the merged variable-length list the GPU path launches
        for a, b_, n in zip(vs, vd, vn):
            _copy_segments(vt.view(np.uint8).reshape(-1), send, [a], [b_], n)
        st.append((sh, qk, vt, pl, send))
    got = np.stack([s[4] for s in st]).reshape(-1)
    split = set(plan.split_requests())
    for sh, qk, vt, pl, _ in st:
        ks, kd, kb = pl["k_unpack"]
        _copy_segments(got, qk.view(np.uint8).reshape(-1), ks, kd, kb)
        vs, vd, vn = pl["v_unpack_var"]
        for a, b_, n in zip(vs, vd, vn):
            _copy_segments(got, vt.view(np.uint8).reshape(-1), [a], [b_], n)
        for k in sh.slots:
            if k not in split:
                continue
            rq = plan.reqs[k]
            for g in range(rq.g0, rq.g0 + rq.count):
                t = sh.local(g) * hw
                np.testing.assert_array_equal(qk[t:t + hw, dpp:], Kf[g * hw:(g + 1) * hw])
                np.testing.assert_array_equal(vt[:, t:t + hw], Vf[g * hw:(g + 1) * hw].T)


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2501_09253_b200.patchshard import DistComm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = DistComm()
        g = comm.all_gather(rank, torch.full((3,), float(rank)))
        sends = {(rank + 1) % world: torch.arange(4, dtype=torch.float32) + 10 * rank}
        src = (rank - 1) % world
        got = comm.exchange(rank, sends, {src: ((4,), torch.float32, torch.device("cpu"))})
        q.put((rank, g.tolist(), got[src].tolist()))
    finally:
        dist.destroy_process_group()


def test_dist_comm_gloo_ws2():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (g, x)) for r, g, x in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for r in range(2):
        g, x = res[r]
        assert g == [[0.0] * 3, [1.0] * 3]
        assert x == [10.0 * ((r - 1) % 2) + i for i in range(4)]


@pytest.mark.parametrize("sms,min_base", [(148, 0), (600, 0), (148, 10 ** 6)])
def test_splitkv_plan_pairs_layout(sms, min_base):
    """Pair split-KV plan (ps_attention_pairs_splitkv + ps_attention_combine): every pair tile's
    key blocks are covered exactly once by its pieces; a split tile's two 128-row halves own
    contiguous slot ranges [s0, s0 + ns) / [s0 + ns, s0 + 2 ns) listed in the combine tables;
    unsplit tiles write directly (slots -1); pieces are dealt longest first; a makespan under
    min_base gives no plan."""
    from paper_2501_09253_b200.patched import splitkv_plan_pairs
    hw = 64 * 64
    sizes = [16, 1, 1, 1, 1, 1, 1, 1, 1]  # config 5: one 2048 px image (16 patches) + 8x 512 px
    tok0 = np.concatenate([[0], np.cumsum(sizes)]) * hw
    pq0, pimg = [], []
    for r, n in enumerate(sizes):
        for q in range(int(tok0[r]), int(tok0[r + 1]), 256):
            pq0.append(q)
            pimg.append(r)
    plan = splitkv_plan_pairs(np.asarray(pq0), np.asarray(pimg), tok0, sms, "cpu", min_base)
    if min_base:
        assert plan is None
        return
    assert plan is not None
    kb0, nkb, s0, s1, n_rows, cq0, cs0, cns, cimg, n_q, rq0, rimg, n_slots = plan
    kb0, nkb, s0, s1 = (t.numpy() for t in (kb0, nkb, s0, s1))
    rq0, rimg = rq0.numpy(), rimg.numpy()
    assert len(kb0) == n_rows and list(nkb) == sorted(nkb, reverse=True)
    cover = {}
    for q, img, k0, n, a, b in zip(rq0, rimg, kb0, nkb, s0, s1):
        cover.setdefault(int(q), []).append((int(k0), int(n), int(a), int(b), int(img)))
    comb = {int(q): (int(s), int(n)) for q, s, n in zip(cq0.numpy(), cs0.numpy(), cns.numpy())}
    assert len(comb) == n_q
    used = []
    for q, img in zip(pq0, pimg):
        pieces = sorted(cover[q])
        total = (int(tok0[img + 1] - tok0[img]) + 127) // 128
        pos = 0
        for k0, n, a, b, im in pieces:
            assert k0 == pos and im == img
            pos += n
        assert pos == total
        if len(pieces) == 1:
            assert pieces[0][2] == pieces[0][3] == -1 and q not in comb
            continue
        ns = len(pieces)
        base, n0 = comb[q]
        assert n0 == ns and comb[q + 128] == (base + ns, ns)
        assert sorted(p[2] for p in pieces) == list(range(base, base + ns))
        assert sorted(p[3] for p in pieces) == list(range(base + ns, base + 2 * ns))
        used += list(range(base, base + 2 * ns))
    assert sorted(used) == list(range(n_slots))
