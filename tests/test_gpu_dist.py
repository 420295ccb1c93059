"""Distributed PCG path with real ranks on one GPU (gloo transport through host memory;
the NCCL run differs only in the transport).  Rank slabs + halo exchange (or the
all-gather) must reproduce the single-GPU solve: same convergence, outer
iterations within 1, x within 1e-6 relative (only the association of the FP64 dot
sums differs); halo and all-gather solves are bitwise identical."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, nx, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_13433_b200 as P
        from paper_2604_13433_b200 import dist as D
        from paper_2604_13433_b200 import solvers as S
        torch.cuda.set_device(0)
        comm = D.Comm()
        n = nx ** 3
        (r0, r1) = D.equal_row_slabs(n, world, 256)[rank]
        A = P.stencil_device("poisson3d", nx, scale="sym", row_begin=r0, row_end=r1)
        b, _ = S.make_rhs_and_x0(n, 42)
        cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=20, a_backend="packsell-e8m14", max_outer=200)
        rep = S.iocg(A, b[r0:r1], cfg, comm=comm)
        pc = S.pcg(P.stencil_device("poisson3d", nx, scale="sym", row_begin=r0, row_end=r1), b[r0:r1],
                   S.SolveConfig(tol=1e-9, max_outer=2000), comm=comm)
        halo = S._halo_for(comm, A)
        # the same solve with the full all-gather: the SpMVs read identical values -> identical x
        os.environ["PSELL_HALO"] = "0"
        A2 = P.stencil_device("poisson3d", nx, scale="sym", row_begin=r0, row_end=r1)
        rep_ag = S.iocg(A2, b[r0:r1], cfg, comm=comm)
        q.put((rank, r0, r1, rep.converged, rep.outer_iters, rep.total_inner_iters, rep.final_true_relres,
               rep.x, pc.converged, pc.outer_iters, pc.x,
               None if halo is None else (halo.volume, halo.use_allgather), rep_ag.x))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_distributed_iocg_matches_single_gpu(world):
    import torch.multiprocessing as mp
    import paper_2604_13433_b200 as P
    from paper_2604_13433_b200 import solvers as S
    nx = 16
    n = nx ** 3
    A = P.sym_diag_scale(P.poisson3d(nx))
    b, _ = S.make_rhs_and_x0(n, 42)
    cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=20, a_backend="packsell-e8m14", max_outer=200)
    ref = S.iocg(A, b, cfg)
    refp = S.pcg(A, b, S.SolveConfig(tol=1e-9, max_outer=2000))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank, args=(r, world, port, nx, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=120)
    assert all(len(r) > 2 for r in res), res
    x = np.zeros(n)
    xp = np.zeros(n)
    for (rank, r0, r1, conv, outer, inner, relres, xs, pconv, pouter, pxs, halo, xs_ag) in res:
        assert halo is not None and halo == (nx * nx, False)  # one boundary plane, point-to-point
        assert np.array_equal(xs, xs_ag)
        assert conv and abs(outer - ref.outer_iters) <= 1
        assert inner == cfg.m_in * outer
        assert relres < 1e-9
        x[r0:r1] = xs
        assert pconv and abs(pouter - refp.outer_iters) <= 1
        xp[r0:r1] = pxs
    assert np.abs(x - ref.x).max() / np.abs(ref.x).max() < 1e-6
    assert np.abs(xp - refp.x).max() / np.abs(refp.x).max() < 1e-9


def _rank_peer(rank, world, port, nx, slabs, q):
    """Same solves over the peer-memory transport (K8: CUDA IPC arenas, one exchange
    kernel, graph-captured inner loop) next to the gloo-staged collectives."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["PSELL_PEER_TIMEOUT_S"] = "120"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_13433_b200 as P
        from paper_2604_13433_b200 import dist as D
        from paper_2604_13433_b200 import solvers as S
        from paper_2604_13433_b200.packed import lower_bandwidth
        torch.cuda.set_device(0)
        comm = D.Comm()
        n = nx ** 3
        r0, r1 = slabs[rank]
        b, _ = S.make_rhs_and_x0(n, 42)
        cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=20, a_backend="packsell-e8m14", max_outer=200)
        out = {}
        # "nccl" = the torch.distributed collectives (gloo here); "peer0" = the peer transport
        # with separate exchange kernels; "peer" = the fused dot all-reduces (default)
        # "peer1" = fused dot all-reduces with the halo still pushed by its own K8 kernel
        for xport in ("nccl", "peer0", "peer1", "peer"):
            os.environ["PSELL_XPORT"] = "nccl" if xport == "nccl" else "peer"
            os.environ["PSELL_PEER_FUSED"] = "0" if xport == "peer0" else "1"
            os.environ["PSELL_PEER_HALO_FUSED"] = "0" if xport == "peer1" else "1"
            A = P.stencil_device("poisson3d", nx, scale="sym", row_begin=r0, row_end=r1)
            kl = comm.allreduce_max(lower_bandwidth(A))
            be = S.make_backend(A, "packsell-e8m14", k_left=kl)
            rep = S.iocg(A, b[r0:r1], cfg, backend=be, comm=comm)
            inner = next(iter(be._inner_cache.values()))
            rep2 = S.iocg(A, b[r0:r1], cfg, backend=be, comm=comm)  # graph replay
            pc = S.pcg(P.stencil_device("poisson3d", nx, scale="sym", row_begin=r0, row_end=r1), b[r0:r1],
                       S.SolveConfig(tol=1e-9, max_outer=2000), comm=comm)
            out[xport] = (rep.converged, rep.outer_iters, rep.total_inner_iters, rep.final_true_relres, rep.x,
                          rep2.x, pc.converged, pc.outer_iters, pc.x, inner.use_graph, inner.peer is not None,
                          inner.peer is not None and inner.peer.ranges(inner.halo, inner.n) is not None)
        comm.close()
        q.put((rank, r0, r1, out))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("split", ["equal", "unequal", "three"])
def test_peer_transport_matches_collectives_and_single_gpu(split):
    """2 ranks on one GPU: the peer-memory path with separate exchange kernels gives the
    same x bit for bit as the collective path, on equal and unequal slabs; the fused path
    (dot sums all-reduced over the arenas by the SpMV's and the update's last CTAs, the
    halo pushed by the direction kernel: 3 launches per inner iteration) the same solve up
    to the association of the local dot sums (its last-CTA tree), deterministic across
    graph replays, and bitwise the same with the halo pushed by a separate K8 kernel."""
    import torch.multiprocessing as mp
    import paper_2604_13433_b200 as P
    from paper_2604_13433_b200 import solvers as S
    nx = 16
    n = nx ** 3
    world = 3 if split == "three" else 2   # three ranks: the middle one pushes two halo ranges
    slabs = {"equal": [(0, n // 2), (n // 2, n)], "unequal": [(0, 1280), (1280, n)],
             "three": [(0, 1280), (1280, 2560), (2560, n)]}[split]
    A = P.sym_diag_scale(P.poisson3d(nx))
    b, _ = S.make_rhs_and_x0(n, 42)
    ref = S.iocg(A, b, S.SolveConfig(solver="iocg", tol=1e-9, m_in=20, a_backend="packsell-e8m14", max_outer=200))
    refp = S.pcg(A, b, S.SolveConfig(tol=1e-9, max_outer=2000))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank_peer, args=(r, world, port, nx, slabs, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=900) for _ in ps]
    for p in ps:
        p.join(timeout=120)
    assert all(len(r) == 4 for r in res), res
    x, xp = np.zeros(n), np.zeros(n)
    for rank, r0, r1, out in res:
        cg = out["nccl"]
        pe = out["peer0"]
        fu = out["peer"]
        assert pe[9] and pe[10] and fu[9] and fu[10], "peer transport + CUDA graph not used"
        assert not cg[10]
        assert pe[0] and pe[1] == cg[1] and pe[2] == cg[2] and pe[3] < 1e-9
        assert np.array_equal(pe[4], cg[4]) and np.array_equal(pe[5], pe[4])
        assert pe[6] and pe[7] == cg[7] and np.array_equal(pe[8], cg[8])
        assert abs(pe[1] - ref.outer_iters) <= 1
        assert fu[0] and abs(fu[1] - pe[1]) <= 1 and fu[3] < 1e-9 and np.array_equal(fu[5], fu[4])
        # the halo pushed by the direction kernel itself: the same values as its K8 push
        f1 = out["peer1"]
        assert fu[11], "the halo push list did not reduce to contiguous ranges"
        assert (f1[1], f1[2]) == (fu[1], fu[2]) and np.array_equal(f1[4], fu[4])
        assert np.abs(fu[4] - pe[4]).max() <= 1e-6 * np.abs(pe[4]).max()
        x[r0:r1] = fu[4]
        xp[r0:r1] = pe[8]
    assert np.abs(x - ref.x).max() / np.abs(ref.x).max() < 1e-6
    assert np.abs(xp - refp.x).max() / np.abs(refp.x).max() < 1e-9
