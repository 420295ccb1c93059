"""Multi-GPU plumbing: row-slab partitions and the two collectives the path needs.

The reference is single-process; the only parallelism SURVEY.md §2.1/§8e
allows is row-slice data parallelism.  A rank owns a contiguous,
sigma-aligned slab of rows (so the implicit permutation stays rank-local and
the concatenation of slab packs equals the single-GPU pack).  Standalone SpMV
needs no collective (x replicated).  The PCG needs exactly two, over NCCL
(NVLink / NVSwitch) through torch.distributed:

* all-gather of the direction vector before every SpMV (in place: each rank's
  slab is its chunk of the global vector), and
* all-gather of the per-rank FP64 local dot sums, summed in rank order on the
  device (deterministic regardless of the collective's reduction tree).

`Comm` wraps a process group (NCCL on GPUs, gloo in the CPU tests).  `Halo`
 replaces the direction all-gather by a neighbour exchange
of just the columns a rank's rows read: for banded operators (the stencils)
that is two thin boundary layers instead of the whole vector.
"""

from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


class Comm:
    """torch.distributed process-group wrapper used by the solvers and the bench."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        # NCCL moves device buffers directly over NVLink; gloo (CPU tests, or
        # several ranks sharing one GPU) stages through host memory
        self.nccl = dist.get_backend(group) == "nccl"

    def _gather(self, out_flat, local):
        if self.nccl or not out_flat.is_cuda:
            self.dist.all_gather_into_tensor(out_flat, local.contiguous(), group=self.group)
            return
        h_out = out_flat.cpu()
        self.dist.all_gather_into_tensor(h_out, local.contiguous().cpu(), group=self.group)
        out_flat.copy_(h_out)

    def all_gather_into(self, out_flat, local):
        """out_flat[r * len(local):(r+1) * len(local)] <- local of rank r (rank order)."""
        self._gather(out_flat, local)

    def all_gather_vec(self, full, local):
        """In-place all-gather of equal slabs: `local` is this rank's chunk of `full`."""
        if self.nccl or not full.is_cuda:
            self.dist.all_gather_into_tensor(full, local, group=self.group)
        else:
            self._gather(full, local.clone())

    def padded_len(self, n_glob: int) -> int:
        return n_glob

    def allreduce_max(self, v: int) -> int:
        import torch
        dev = "cuda" if torch.cuda.is_available() and self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([int(v)], dtype=torch.int64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def barrier(self):
        self.dist.barrier(group=self.group)

    def slabs(self, row0: int, n: int) -> List[Tuple[int, int]]:
        """Every rank's (row0, row1), in rank order (host all-gather, setup only)."""
        out = [None] * self.world
        self.dist.all_gather_object(out, (int(row0), int(row0) + int(n)), group=self.group)
        return [tuple(map(int, s)) for s in out]

    def peer(self, n_cols: int):
        """The peer-memory transport for vectors of n_cols entries, or None.

        Used when the ranks share a node and CUDA IPC works: by default on NCCL
        process groups, and on any group with PSELL_XPORT=peer (several ranks
        sharing one GPU over gloo, the tests); PSELL_XPORT=nccl keeps the NCCL
        collectives (A/B)."""
        import os
        mode = os.environ.get("PSELL_XPORT", "auto")
        if mode == "nccl" or (mode == "auto" and not self.nccl):
            return None
        if mode == "auto" and not self._peer_capable():
            return None  # another node, or no P2P path between two ranks' GPUs: NCCL
        cache = self.__dict__.setdefault("_peers", {})
        if n_cols not in cache:
            cache[n_cols] = PeerTransport(self, n_cols)
        return cache[n_cols]

    def _peer_capable(self) -> bool:
        """Every rank can map every other rank's arena (collective, cached): all GPUs are
        visible on this node and each pair has a P2P path (NVLink / NVSwitch), so no rank
        fails in cudaIpcOpenMemHandle while the others wait in the exchange kernel."""
        if "_p2p" not in self.__dict__:
            import torch
            mine = str(torch.cuda.get_device_properties(torch.cuda.current_device()).uuid)
            uuids = [None] * self.world
            self.dist.all_gather_object(uuids, mine, group=self.group)
            local = [str(torch.cuda.get_device_properties(i).uuid) for i in range(torch.cuda.device_count())]
            ok = peer_capable(torch.cuda.current_device(), uuids, local, torch.cuda.can_device_access_peer)
            votes = [None] * self.world
            self.dist.all_gather_object(votes, bool(ok), group=self.group)
            self._p2p = all(votes)
        return self._p2p

    def close(self):
        """Release the peer arenas (collective)."""
        for t in self.__dict__.pop("_peers", {}).values():
            t.close()


def peer_capable(my_dev: int, rank_uuids: Sequence[str], local_uuids: Sequence[str], can_access) -> bool:
    """This rank can map every rank's device memory: each rank's GPU (by UUID) is one of this
    node's devices, and the same GPU or one `can_access(my_dev, dev)` reaches."""
    for u in rank_uuids:
        if u not in local_uuids:
            return False
        d = list(local_uuids).index(u)
        if d != my_dev and not can_access(my_dev, d):
            return False
    return True


class _CudaView:
    """__cuda_array_interface__ over raw device memory (arena views as torch tensors)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class PeerTransport:
    """One-kernel collectives over NVLink peer memory (csrc/peer.cu, K8).

    Each rank allocates an arena holding the exchange flags, the FP64 dot
    slots and the full-length f32 / f64 vectors, exports it through a CUDA IPC
    handle and maps every peer's.  `exchange` then pushes this rank's halo
    entries straight into the peers' full vectors and its local dot sums into
    their dot slots, signals, waits, and leaves the rank-ordered dot sums in
    `out` — one stream-ordered kernel, so the distributed inner PCG iteration
    is a kernel chain captured in one CUDA graph (no NCCL call, no host wait).
    """

    def __init__(self, comm: "Comm", n_cols: int):
        import ctypes
        import os

        import torch
        from . import _lib
        self.comm, self.n_cols = comm, int(n_cols)
        self.lib = lib = _lib.lib()
        self.G, self.rank = comm.world, comm.rank
        self.timeout_ns = int(float(os.environ.get("PSELL_PEER_TIMEOUT_S", "60")) * 1e9)
        nbytes = lib.psell_peer_arena_bytes(self.n_cols)
        ptr = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        if lib.psell_peer_alloc(nbytes, ctypes.byref(ptr), handle):
            raise _lib.LibpsellError("psell_peer_alloc failed (cudaMalloc / cudaIpcGetMemHandle)")
        self.arena = int(ptr.value)
        handles = [None] * self.G
        comm.dist.all_gather_object(handles, bytes(handle), group=comm.group)
        bases, self._opened = [], []
        for r, h in enumerate(handles):
            if r == self.rank:
                bases.append(self.arena)
                continue
            p = ctypes.c_void_p()
            hb = (ctypes.c_char * 64).from_buffer_copy(h)
            if lib.psell_peer_open(hb, ctypes.byref(p)):
                raise _lib.LibpsellError(f"psell_peer_open of rank {r}'s arena failed (CUDA IPC)")
            bases.append(int(p.value))
            self._opened.append(int(p.value))
        self.d_peers = torch.tensor(bases, dtype=torch.int64, device="cuda")
        off32 = lib.psell_peer_vec_offset(self.n_cols, 4)
        off64 = lib.psell_peer_vec_offset(self.n_cols, 8)
        self.vec_off = {4: off32, 8: off64}
        self.full32 = torch.as_tensor(_CudaView(self.arena + off32, self.n_cols, "<f4"), device="cuda")
        self.full64 = torch.as_tensor(_CudaView(self.arena + off64, self.n_cols, "<f8"), device="cuda")
        self._plans = {}
        torch.cuda.synchronize()
        comm.barrier()

    def full(self, dtype):
        """The arena's full-length vector of `dtype` (f32 inner / f64 outer)."""
        import torch
        return self.full32 if dtype == torch.float32 else self.full64

    def plan(self, halo: "Halo", row0: int, n_local: int):
        """Device (dst rank, local index) lists of the entries this rank pushes: the halo
        plan's send lists, or its whole slab to every peer when the plan falls back to
        the all-gather (irregular matrices)."""
        key = None if halo is None else id(halo)
        if key not in self._plans:
            import torch
            dst, loc = push_lists(halo, self.rank, self.G, n_local)
            self._plans[key] = (torch.as_tensor(dst).cuda(), torch.as_tensor(loc).cuda(), int(row0), len(dst))
        return self._plans[key]

    def ranges(self, halo: "Halo", n_local: int):
        """The push list as at most 2 contiguous local row ranges, each owed to one peer
        ((lo, hi, dst) host tuples; stencil slabs: the first / last boundary planes), or
        None when it does not decompose so (irregular halos, all-gather fallback): the
        direction kernel can then push it itself (psell_ipcg_direction_x_push)."""
        key = ("ranges", None if halo is None else id(halo))
        if key not in self._plans:
            self._plans[key] = push_ranges(*push_lists(halo, self.rank, self.G, n_local))
        return self._plans[key]

    def exchange(self, local=None, plan=None, loc=None, n_loc: int = 0, out=None):
        """Push `local`'s planned entries and loc[:n_loc], wait for all ranks, out <- dot sums."""
        from . import _lib
        if plan is not None:
            dst, li, row0, n_send = plan
            es = local.element_size()
            rc = self.lib.psell_peer_exchange(self.G, self.rank, self.d_peers.data_ptr(), n_send, dst.data_ptr(),
                                              li.data_ptr(), row0, local.data_ptr(), es, self.vec_off[es],
                                              None if loc is None else loc.data_ptr(), n_loc,
                                              None if out is None else out.data_ptr(), self.timeout_ns,
                                              _lib.stream_handle())
        else:
            rc = self.lib.psell_peer_exchange(self.G, self.rank, self.d_peers.data_ptr(), 0, None, None, 0, None,
                                              8, 0, loc.data_ptr(), n_loc, out.data_ptr(), self.timeout_ns,
                                              _lib.stream_handle())
        if rc:
            raise _lib.LibpsellError(f"psell_peer_exchange failed ({rc})")

    def check(self):
        """Raise if any exchange of this rank timed out waiting for a peer."""
        import ctypes
        from . import _lib
        v = ctypes.c_int32(0)
        if self.lib.psell_peer_error(self.arena, ctypes.byref(v)) or v.value:
            raise _lib.LibpsellError("peer exchange timed out waiting for a rank (PSELL_PEER_TIMEOUT_S)")

    def close(self):
        import torch
        torch.cuda.synchronize()
        self.comm.barrier()
        for p in self._opened:
            self.lib.psell_peer_close(p)
        self._opened = []
        self.comm.barrier()
        if self.arena:
            self.lib.psell_peer_free(self.arena)
            self.arena = 0


class Halo:
    """Point-to-point halo plan of one row-partitioned operator (built once, collectively).

    `needed` are the sorted unique global columns this rank's rows read
    (the CSR slab's col_idx).  Columns outside the own slab [row0, row1) are
    requested from their owners; `exchange(full, local)` then packs what each
    peer needs from `local` (K7 pack), moves it with NCCL send/recv over
    NVLink, and scatters the received entries into `full` (K7 unpack) — the
    entries of `full` the SpMV reads are then exactly those of the all-gathered
    vector.  When the halo covers more than `max_frac` of the remote part of
    the vector (irregular matrices) the plan sets `use_allgather` and the
    solvers keep the all-gather.
    """

    def __init__(self, comm: "Comm", row0: int, row1: int, needed, max_frac: float = 0.5, n_cols: int = None):
        self.comm = comm
        self.row0, self.row1 = int(row0), int(row1)
        needed = np.unique(np.asarray(needed, dtype=np.int64))
        slabs = [None] * comm.world
        comm.dist.all_gather_object(slabs, (self.row0, self.row1), group=comm.group)
        self.slabs = [tuple(map(int, s)) for s in slabs]
        ends = np.array([b for _, b in self.slabs], dtype=np.int64)
        remote = needed[(needed < self.row0) | (needed >= self.row1)]
        owner = np.searchsorted(ends, remote, side="right")
        self.recv_lists = [remote[owner == s] for s in range(comm.world)]
        wanted = [None] * comm.world  # wanted[s][r]: columns rank s needs from rank r
        comm.dist.all_gather_object(wanted, self.recv_lists, group=comm.group)
        self.send_lists = [np.asarray(wanted[s][comm.rank], dtype=np.int64) for s in range(comm.world)]
        self.recv_counts = [len(v) for v in self.recv_lists]
        self.send_counts = [len(v) for v in self.send_lists]
        n_glob = max(b for _, b in self.slabs)
        n_remote = n_glob - (self.row1 - self.row0)
        tot = [0] * comm.world
        comm.dist.all_gather_object(tot, int(sum(self.recv_counts)), group=comm.group)
        self.use_allgather = max(tot) > max_frac * max(n_remote, 1)
        self.send_idx = np.concatenate(self.send_lists + [np.zeros(0, np.int64)]) - self.row0
        self.recv_idx = np.concatenate(self.recv_lists + [np.zeros(0, np.int64)])
        # every index lands inside the full-length vector and the own slab
        n_full = n_glob if n_cols is None else int(n_cols)
        if self.recv_idx.size and (self.recv_idx.min() < 0 or self.recv_idx.max() >= n_full):
            raise ValueError(f"halo column outside [0, {n_full}): the slabs do not cover the columns read")
        if self.send_idx.size and (self.send_idx.min() < 0 or self.send_idx.max() >= self.row1 - self.row0):
            raise ValueError("a peer requested a column outside this rank's slab")
        self._dev = None

    @property
    def volume(self) -> int:
        """Entries this rank receives per exchange (the all-gather would deliver n_glob - n_own)."""
        return int(sum(self.recv_counts))

    def _device_plan(self):
        if self._dev is None:
            import torch
            self._dev = (torch.as_tensor(self.send_idx.astype(np.int32)).cuda(),
                         torch.as_tensor(self.recv_idx).cuda(), {})
        return self._dev

    def p2p(self, send, recv):
        """Move send[slice for peer s] to peer s and fill recv[slice from peer s] (stream-ordered on NCCL)."""
        dist, grp = self.comm.dist, self.comm.group
        staged = send.is_cuda and not self.comm.nccl  # gloo moves host tensors
        s_buf = send.cpu() if staged else send
        r_buf = recv.cpu() if staged else recv
        ops, so, ro = [], 0, 0
        for peer in range(self.comm.world):
            ns, nr = self.send_counts[peer], self.recv_counts[peer]
            if nr:
                ops.append(dist.P2POp(dist.irecv, r_buf[ro:ro + nr], peer, grp))
            if ns:
                ops.append(dist.P2POp(dist.isend, s_buf[so:so + ns], peer, grp))
            so += ns
            ro += nr
        if ops:
            if self.comm.nccl:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            else:
                reqs = [op.op(op.tensor, op.peer, op.group) for op in ops]
                for req in reqs:
                    req.wait()
        if staged:
            recv.copy_(r_buf)

    def exchange(self, full, local):
        """full[recv_idx] <- the owners' entries; `local` is this rank's slab (any 4/8-byte dtype)."""
        import torch
        from . import _lib
        lib = _lib.lib()
        send_idx, recv_idx, bufs = self._device_plan()
        key = full.dtype
        if key not in bufs:
            bufs[key] = (torch.empty(len(self.send_idx), dtype=full.dtype, device=full.device),
                         torch.empty(len(self.recv_idx), dtype=full.dtype, device=full.device))
        send, recv = bufs[key]
        st = _lib.stream_handle()
        es = full.element_size()
        if lib.psell_halo_pack(len(self.send_idx), local.data_ptr(), send_idx.data_ptr(), send.data_ptr(), es, st):
            raise _lib.LibpsellError("psell_halo_pack failed")
        self.p2p(send, recv)
        if lib.psell_halo_unpack(len(self.recv_idx), recv.data_ptr(), recv_idx.data_ptr(), full.data_ptr(), es, st):
            raise _lib.LibpsellError("psell_halo_unpack failed")
        return full


def push_lists(halo, rank: int, world: int, n_local: int):
    """(destination rank, local row) of every entry this rank pushes per exchange over peer
    memory: the halo plan's send lists (each peer gets the columns its slab reads from this
    rank), or the whole slab to every other rank when the plan falls back to the
    all-gather (halo None or use_allgather).  Host side of PeerTransport.plan."""
    if halo is not None and not halo.use_allgather:
        dst = np.concatenate([np.full(len(v), s, np.int32) for s, v in enumerate(halo.send_lists)]
                             + [np.zeros(0, np.int32)])
        return dst, halo.send_idx.astype(np.int32)
    peers = [s for s in range(world) if s != rank]
    return (np.repeat(np.asarray(peers, np.int32), n_local),
            np.tile(np.arange(n_local, dtype=np.int32), len(peers)))


def push_ranges(dst, loc, max_ranges: int = 2):
    """A push list (destination rank, local row) as contiguous local row ranges, one per
    destination: [(lo, hi, dst), ...] sorted by destination, or None when some destination's
    rows are not one contiguous duplicate-free range or there are more than `max_ranges`
    destinations (the fused halo push of psell_ipcg_direction_x_push then does not apply)."""
    dst = np.asarray(dst)
    loc = np.asarray(loc, dtype=np.int64)
    out = []
    for q in np.unique(dst):
        li = np.sort(loc[dst == q])
        if len(li) == 0:
            continue
        if li[-1] - li[0] + 1 != len(li) or np.any(np.diff(li) == 0):
            return None
        out.append((int(li[0]), int(li[-1]) + 1, int(q)))
    return out if len(out) <= max_ranges else None


def equal_row_slabs(n: int, world: int, sigma: int) -> List[Tuple[int, int]]:
    """sigma-aligned contiguous row slabs, as equal as the sigma granularity allows.

    The PCG requires exactly equal slabs (in-place all-gather of equal chunks),
    i.e. n % (world * sigma) == 0; `check_equal` enforces it.
    """
    nb = -(-n // sigma)
    out = []
    for r in range(world):
        a = min(n, (nb * r // world) * sigma)
        b = min(n, (nb * (r + 1) // world) * sigma)
        out.append((a, b))
    return out


def check_equal(slabs: Sequence[Tuple[int, int]]):
    sizes = {b - a for a, b in slabs}
    if len(sizes) != 1:
        raise ValueError(f"the distributed PCG needs equal row slabs, got sizes {sorted(sizes)}; "
                         "choose n divisible by world * sigma")


def word_balanced_slabs(row_words: np.ndarray, world: int, sigma: int) -> List[Tuple[int, int]]:
    """sigma-aligned slabs balancing stored words (power-law matrices).

    `row_words` are the per-row stored word counts (len + dummies, or the
    padded slice widths spread over rows); cuts are placed at sigma-block
    boundaries nearest to equal prefix sums.
    """
    n = len(row_words)
    nb = -(-n // sigma)
    blk = np.add.reduceat(np.asarray(row_words, dtype=np.int64), np.arange(0, n, sigma)) if n else np.zeros(0)
    pref = np.concatenate([[0], np.cumsum(blk)])
    total = pref[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        j = int(np.searchsorted(pref, target))
        j = min(max(j, cuts[-1]), nb)
        cuts.append(j)
    cuts.append(nb)
    return [(min(n, cuts[r] * sigma), min(n, cuts[r + 1] * sigma)) for r in range(world)]


def rank_order_sum(parts: np.ndarray) -> float:
    """Host mirror of psell_sum_strided: sequential sum in rank order."""
    s = 0.0
    for v in np.asarray(parts, dtype=np.float64):
        s += float(v)
    return s


__all__ = ["Comm", "PeerTransport", "push_lists", "Halo", "equal_row_slabs", "check_equal", "word_balanced_slabs", "rank_order_sum"]
