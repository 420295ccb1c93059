"""Multi-rank host logic on CPU: gloo world_size 2, partitions, rank-ordered sums,
and the slab property the multi-GPU build relies on (checked with the oracle)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2604_13433_b200 import dist as D
from paper_2604_13433_b200 import stencil


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = D.Comm()
        # rank-ordered local sums
        loc = torch.arange(8, dtype=torch.float64) + 100 * rank
        glob = torch.zeros(world * 8, dtype=torch.float64)
        comm.all_gather_into(glob, loc)
        # in-place slab all-gather of a direction vector
        n = 6
        full = torch.zeros(world * n, dtype=torch.float32)
        full[rank * n:(rank + 1) * n] = rank + 1.0
        comm.all_gather_vec(full, full[rank * n:(rank + 1) * n])
        kmax = comm.allreduce_max(10 + rank)
        q.put((rank, glob.numpy().copy(), full.numpy().copy(), kmax))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_collectives():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for rank, glob, full, kmax in res:
        want = np.concatenate([np.arange(8) + 100 * r for r in range(world)])
        assert np.array_equal(glob, want)
        assert np.array_equal(full, np.repeat([1.0, 2.0], 6))
        assert kmax == 11
        assert D.rank_order_sum(glob.reshape(world, 8)[:, 3]) == 3.0 + 103.0


def test_partitions():
    sl = D.equal_row_slabs(16 * 256, 4, 256)
    assert sl == [(0, 1024), (1024, 2048), (2048, 3072), (3072, 4096)]
    D.check_equal(sl)
    with pytest.raises(ValueError):
        D.check_equal(D.equal_row_slabs(1000, 3, 256))
    w = np.ones(4096, dtype=np.int64)
    w[:256] = 100  # first block heavy
    ws = D.word_balanced_slabs(w, 2, 256)
    assert ws[0][0] == 0 and ws[-1][1] == 4096 and all(a % 256 == 0 for a, _ in ws)
    assert ws[0][1] - ws[0][0] < ws[1][1] - ws[1][0]


@pytest.mark.parametrize("preset,world", [("fp16", 2), ("e8m14", 3), ("fp16", 4)])
def test_slab_packs_concatenate_to_global(preset, world):
    """Per-rank slab builds with the global k_left == the single build (oracle)."""
    A = stencil.stencil27(10)
    f = O.preset(preset)
    G = O.build(A.row_ptr, A.col_idx, A.values, A.n_cols, 32, 256, f, "implicit")
    packs, perms, offs = [], [], [0]
    for a, b in D.equal_row_slabs(A.n_rows, world, 256):
        S = stencil.stencil_rows("stencil27", 10, a, b)
        M = O.build(S.row_ptr, S.col_idx, S.values, S.n_cols, 32, 256, f, "implicit", k_left=G.k_left, row0=a)
        packs.append(M.pack)
        perms.append(M.perm)
        offs.extend((M.offset[1:] + offs[-1]).tolist())
        x = np.random.default_rng(a).uniform(-1, 1, A.n_cols).astype(np.float32)
        assert np.array_equal(O.spmv(M, x), O.spmv(G, x)[a:b])
    assert np.array_equal(np.concatenate(packs), G.pack)
    assert np.array_equal(np.concatenate(perms), G.perm)
    assert np.array_equal(np.array(offs), G.offset)


def test_stencil_rows_match_full():
    A = stencil.poisson3d(7)
    S = stencil.stencil_rows("poisson3d", 7, 50, 200)
    assert np.array_equal(S.col_idx, A.col_idx[A.row_ptr[50]:A.row_ptr[200]])
    assert np.array_equal(S.row_ptr, A.row_ptr[50:201] - A.row_ptr[50])


def _halo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = D.Comm()
        nx = 8
        n = nx ** 3
        slabs = D.equal_row_slabs(n, world, 32)
        r0, r1 = slabs[rank]
        A = stencil.poisson3d(nx)
        cols = A.col_idx[A.row_ptr[r0]:A.row_ptr[r1]]
        h = D.Halo(comm, r0, r1, cols)
        # the exchange on host tensors (the device path runs K7 pack/unpack around the same p2p)
        full_ref = torch.arange(n, dtype=torch.float64) * 0.5 + 1.0
        full = torch.zeros(n, dtype=torch.float64)
        full[r0:r1] = full_ref[r0:r1]
        send = full[r0:r1][torch.as_tensor(h.send_idx)]
        recv = torch.zeros(h.volume, dtype=torch.float64)
        h.p2p(send, recv)
        full[torch.as_tensor(h.recv_idx)] = recv
        need = np.unique(cols.astype(np.int64))
        ok = bool(torch.equal(full[torch.as_tensor(need)], full_ref[torch.as_tensor(need)]))
        # an irregular operator (every row reads everything) falls back to the all-gather
        g = D.Halo(comm, r0, r1, np.arange(n))
        q.put((rank, ok, h.volume, h.use_allgather, g.use_allgather, list(h.recv_counts), list(h.send_counts)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_halo_exchange():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for rank, ok, vol, h_ag, g_ag, rc, sc in res:
        assert ok
        assert vol == 8 * 8  # one boundary plane of the 7-point stencil from the neighbour slab
        assert not h_ag and g_ag
    # what rank 0 receives from rank 1 is what rank 1 sends to rank 0, and vice versa
    assert res[0][5][1] == res[1][6][0] and res[1][5][0] == res[0][6][1]


def _push_worker(rank, world, port, slabs, use_halo, q):
    """Simulate the peer transport's pushes: every rank contributes its push lists; the
    entries pushed to rank s are applied to rank s's full vector; the columns rank s's
    rows read must then hold their owners' values (equal or unequal slabs)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = D.Comm()
        nx = 8
        n = nx ** 3
        r0, r1 = slabs[rank]
        A = stencil.poisson3d(nx)
        cols = A.col_idx[A.row_ptr[r0]:A.row_ptr[r1]]
        h = D.Halo(comm, r0, r1, cols, n_cols=n) if use_halo else None
        dst, loc = D.push_lists(h, rank, world, r1 - r0)
        vals = (r0 + loc.astype(np.int64)) * 0.25 + 3.0   # the owner's p at those global rows
        pushed = [None] * world
        dist.all_gather_object(pushed, (dst, r0 + loc.astype(np.int64), vals))
        full = np.zeros(n)
        full[r0:r1] = np.arange(r0, r1) * 0.25 + 3.0
        for d_, g_, v_ in pushed:
            sel = d_ == rank
            full[g_[sel]] = v_[sel]
        need = np.unique(cols)
        ok = bool(np.array_equal(full[need], need * 0.25 + 3.0))
        # the same pushes as contiguous ranges (the direction kernel's fused halo push)
        rg = D.push_ranges(dst, loc)
        ok_rg = None
        if rg is not None:
            pushed = [None] * world
            dist.all_gather_object(pushed, rg)
            full_r = np.zeros(n)
            full_r[r0:r1] = np.arange(r0, r1) * 0.25 + 3.0
            for src, rgs in enumerate(pushed):
                for lo, hi, d_ in rgs:
                    if d_ == rank:
                        g = slabs[src][0] + np.arange(lo, hi)
                        full_r[g] = g * 0.25 + 3.0
            ok_rg = bool(np.array_equal(full_r[need], need * 0.25 + 3.0))
        else:
            dist.all_gather_object([None] * world, None)
        q.put((rank, ok and ok_rg is not False, int(len(dst)), None if h is None else h.volume, rg))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,slabs,use_halo", [
    (2, [(0, 256), (256, 512)], True),
    (3, [(0, 96), (96, 352), (352, 512)], True),     # unequal slabs: addressed by global index
    (3, [(0, 96), (96, 352), (352, 512)], False),    # all-gather fallback over peer memory
])
def test_peer_push_lists_cover_every_read_column(world, slabs, use_halo):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_push_worker, args=(r, world, port, slabs, use_halo, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _, _ in res), res
    if not use_halo:
        assert [k for _, _, k, _, _ in res] == [(b - a) * (world - 1) for a, b in slabs]
    # stencil slabs: every rank's pushes are <= 2 contiguous ranges (boundary planes, or the
    # whole slab to each of the other two ranks), so the direction kernel can push them
    assert all(rg is not None and len(rg) <= 2 for _, _, _, _, rg in res), res


def test_push_ranges():
    assert D.push_ranges(np.array([1, 1, 1], np.int32), np.array([4, 5, 6], np.int32)) == [(4, 7, 1)]
    assert D.push_ranges(np.array([2, 0, 2, 0], np.int32), np.array([9, 0, 8, 1], np.int32)) == [(0, 2, 0), (8, 10, 2)]
    assert D.push_ranges(np.array([1, 1], np.int32), np.array([4, 6], np.int32)) is None        # gap
    assert D.push_ranges(np.array([1, 1], np.int32), np.array([4, 4], np.int32)) is None        # duplicate
    assert D.push_ranges(np.array([0, 1, 2], np.int32), np.array([0, 0, 0], np.int32)) is None  # 3 destinations
    assert D.push_ranges(np.zeros(0, np.int32), np.zeros(0, np.int32)) == []


def _slab_check_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_13433_b200 import solvers as S
        comm = D.Comm()
        out = []
        # equal, rank-ordered slabs pass the all-gather check
        S._check_slabs(comm, rank * 512, 512, None, None)
        out.append("equal ok")
        # unequal slabs: refused for the all-gather transport ...
        r0, n = (0, 256) if rank == 0 else (256, 768)
        try:
            S._check_slabs(comm, r0, n, None, None)
            out.append("unequal accepted")
        except ValueError:
            out.append("unequal refused")
        # ... accepted with the peer transport (global indices)
        S._check_slabs(comm, r0, n, None, object())
        out.append("peer ok")
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_allgather_transport_refuses_unequal_slabs():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_slab_check_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for _, out in res:
        assert out == ["equal ok", "unequal refused", "peer ok"], out


def test_peer_capable():
    """The peer transport is used only when every rank's GPU is on this node and reachable."""
    from paper_2604_13433_b200.dist import peer_capable
    local = ["GPU-a", "GPU-b", "GPU-c"]
    allp = lambda i, j: True  # noqa: E731
    assert peer_capable(0, ["GPU-a", "GPU-b", "GPU-c"], local, allp)
    assert peer_capable(1, ["GPU-b", "GPU-b"], local, lambda i, j: False)  # ranks sharing one GPU
    assert not peer_capable(0, ["GPU-a", "GPU-z"], local, allp)  # a rank on another node
    assert not peer_capable(0, ["GPU-a", "GPU-c"], local, lambda i, j: (i, j) != (0, 2))  # no P2P path
