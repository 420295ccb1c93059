"""CG drivers over pluggable SpMV backends — drop-in for reference `packsell.solvers`.

Same names, signatures, config validation and report fields as the reference
(solvers.py:31-333).  Vectors live in HBM; every vector operation and every
reduction runs in libpsell (K3 kernels, deterministic fixed-grid FP64
reductions), every operator application in K2 (PackSELL) or K4 (CSR).

* `_InnerPCG` is the hot loop of the mixed-precision solver
  (_inner_pcg, solvers.py:278-308): m_in f32 PCG steps with the curvature dot
  fused into the PackSELL SpMV epilogue, alpha / beta / the breakdown flag kept
  on the device, and — on one GPU — the whole m_in-step loop captured once as
  a CUDA graph and replayed every outer iteration (no host round trip inside).
* `fcg` / `pcg` are the f64 outer / comparator loops; they read back one
  small status block per iteration (the reference's residual history needs it).

Multi-GPU (`comm=` a paper_2604_13433_b200.dist.Comm): every rank passes its
sigma-aligned row slab (DeviceCsrMatrix with row0, n_cols global) and the
matching slab of b.  The direction vectors are all-gathered over NCCL before
each SpMV and every dot's per-rank FP64 sum is all-gathered and summed in rank
order on the device, so the iteration is identical for any rank count up to
the dot association.
"""

from __future__ import annotations

import logging
import os
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import codec
from .matrix import CsrMatrix, DeviceCsrMatrix, csr_spmv
from .packed import PackSellMatrix, build_packsell, packsell_spmv

log = logging.getLogger(__name__)

BACKEND_NAMES = ("csr64", "sell64", "sell32", "sell16", "packsell-fp16")

_PRECISIONS = {"real32": np.dtype(np.float32), "real64": np.dtype(np.float64)}


@dataclass
class SolveConfig:
    solver: str = "pcg"
    tol: float = 1e-9
    max_outer: int = 1000
    m_in: int = 50
    inner_precision: str = "real32"
    a_backend: str = "csr64"
    preconditioner: str = "identity"

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.m_in < 1:
            raise ValueError("m_in must be >= 1")
        if self.inner_precision not in _PRECISIONS:
            raise ValueError(f"inner_precision must be one of {sorted(_PRECISIONS)}")
        if self.preconditioner not in ("identity", "jacobi"):
            raise ValueError("preconditioner must be 'identity' or 'jacobi'")


@dataclass
class SolveReport:
    converged: bool
    outer_iters: int
    total_inner_iters: int
    residual_history: list
    final_true_relres: float
    elapsed: float
    reason: Optional[str] = None
    x: np.ndarray = field(repr=False, compare=False, default=None)

    def to_dict(self) -> dict:
        return {
            "converged": self.converged,
            "outer_iters": self.outer_iters,
            "total_inner_iters": self.total_inner_iters,
            "residual_history": self.residual_history,
            "final_true_relres": self.final_true_relres,
            "elapsed": self.elapsed,
            "reason": self.reason,
        }


def make_rhs_and_x0(n: int, seed: int):
    """b ~ U[0,1) from PCG64(seed), x0 = 0 (solvers.py:81-84) — identical stream to the reference."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.random(n), np.zeros(n)


# ----------------------------------------------------------------------------
# backends
# ----------------------------------------------------------------------------

class SpmvBackend:
    """A device-resident operator plus its unquantised f64 CSR source (solvers.py:96-111).

    `apply(x)` takes numpy (returns numpy, the reference call) or a CUDA tensor
    (returns a CUDA tensor); it runs in x's precision.  For a rank slab, x is
    the global vector and the result has the slab's rows.
    """

    def __init__(self, name: str, matrix, kernel: Callable, source, kernel_into: Callable = None):
        self.name = name
        self.matrix = matrix
        self._kernel = kernel
        self._into = kernel_into
        self.source = source

    def apply(self, x):
        return self._kernel(x)

    def apply_into(self, x, out):
        """out <- A x for device tensors (no temporary when the backend writes in place)."""
        if self._into is not None:
            return self._into(x, out)
        out.copy_(self._kernel(x))
        return out

    @property
    def is_packsell(self) -> bool:
        return isinstance(self.matrix, PackSellMatrix)


def make_backend(A, name: str, c: int = 32, sigma: int = 256, mode: str = "implicit", *,
                 k_left: Optional[int] = None) -> SpmvBackend:
    """Named backend from an f64 CSR matrix (solvers.py:114-131).

    `k_left` passes the global lower bandwidth when A is one rank's slab.
    """
    if name == "csr64":
        return SpmvBackend(name, A, lambda x: csr_spmv(A, x, _dtype_of(x)), A,
                           lambda x, out: csr_spmv(A, x, _dtype_of(x), out=out))
    if name in ("sell64", "sell32", "sell16"):
        from .sellfmt import build_sell, sell_spmv
        dt = {"sell64": np.float64, "sell32": np.float32, "sell16": np.float16}[name]
        S = build_sell(A, c, sigma, mode, value_dtype=dt)
        return SpmvBackend(name, S, lambda x: sell_spmv(S, x), A, lambda x, out: sell_spmv(S, x, out=out))
    if name.startswith("packsell-"):
        fmt = codec.parse_format(name[len("packsell-"):])
        M = build_packsell(A, c, sigma, fmt, mode, _k_left_override=k_left)
        return SpmvBackend(name, M, lambda x: packsell_spmv(M, x), A, lambda x, out: packsell_spmv(M, x, out=out))
    raise ValueError(f"unknown backend {name!r}")


def _dtype_of(x):
    import torch
    if isinstance(x, torch.Tensor):
        from . import _dev
        return _dev.T2NP[x.dtype]
    return np.asarray(x).dtype


def _as_backend(A) -> SpmvBackend:
    if isinstance(A, SpmvBackend):
        return A
    if isinstance(A, (CsrMatrix, DeviceCsrMatrix)):
        return make_backend(A, "csr64")
    raise TypeError("expected an SpmvBackend or CsrMatrix")


# ----------------------------------------------------------------------------
# device reduction / scalar plumbing
# ----------------------------------------------------------------------------

class _Dev:
    """Per-solve device scratch: partials, local sums, gathered sums, global scalars, flags.

    loc[8]   this rank's sums (written by the fused reduction kernels)
    glob[G,8] all ranks' loc (rank order) after `gather`
    scal[32] global scalars (rank-ordered sums and the coefficients)
    """

    def __init__(self, n_partials: int, comm=None):
        import torch
        from . import _lib
        self.torch = torch
        self.lib = _lib.lib()
        self.L = _lib
        self.comm = comm
        self.G = 1 if comm is None else comm.world
        self.peer = None  # dist.PeerTransport: gathers become one peer-memory kernel
        np_ = max(int(n_partials), 2 * _lib.RED_BLOCKS)
        self.partials = torch.zeros(np_ + -(-np_ // 32) + 8, dtype=torch.float64, device="cuda")
        self.loc = torch.zeros(8, dtype=torch.float64, device="cuda")
        self.glob = torch.zeros(self.G * 8, dtype=torch.float64, device="cuda")
        self.scal = torch.zeros(32, dtype=torch.float64, device="cuda")
        self.flags = torch.zeros(4, dtype=torch.int32, device="cuda")
        # last-CTA tickets of the fused epilogues: [0, T) SpMV + alpha, [T, 2T) update + beta
        self.tstride = 1 + -(-np_ // 32)  # groups of >= 32 CTAs
        self.ticket = torch.zeros(2 * self.tstride, dtype=torch.int32, device="cuda")

    def st(self):
        return self.L.stream_handle()

    def p(self, t, off: int = 0):
        return t.data_ptr() + off * t.element_size()

    def gather(self):
        """(pointer base, stride) of every rank's loc[] in rank order."""
        if self.G == 1:
            return self.loc, 8
        if self.peer is not None:
            self.peer.exchange(loc=self.loc, n_loc=8, out=self.glob)
        else:
            self.comm.all_gather_into(self.glob, self.loc)
        return self.glob, 8

    def reduce(self, k0: int, n_out: int, dst: int):
        """scal[dst:dst+n_out] <- rank-ordered global sums of loc[k0:k0+n_out]."""
        g, stride = self.gather()
        self.lib.psell_sum_strided(self.p(g, k0), self.G, stride, n_out, self.p(self.scal, dst), self.st())

    def status(self, i: int, j: int):
        """(flags[0], scal[i], scal[j]) on the host: two small D2H copies into page-locked
        buffers and one stream sync (no gather kernels on the per-iteration path)."""
        torch = self.torch
        if not hasattr(self, "_h_scal"):
            self._h_scal = torch.zeros(32, dtype=torch.float64, pin_memory=True)
            self._h_flags = torch.zeros(4, dtype=torch.int32, pin_memory=True)
        self._h_scal.copy_(self.scal, non_blocking=True)
        self._h_flags.copy_(self.flags, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        hs = self._h_scal.numpy()
        return int(self._h_flags[0]), float(hs[i]), float(hs[j])

    def norm(self, a, slot: int = 15) -> float:
        """sqrt of the global a.a (solvers.py:92-93)."""
        self.lib.psell_dot(a.data_ptr(), a.data_ptr(), 2 if a.dtype == self.torch.float64 else 1, a.numel(),
                           self.p(self.partials), self.p(self.loc, 7), self.st())
        self.reduce(7, 1, slot)
        return float(np.sqrt(float(self.scal[slot].item())))


def _gather_full(comm, local, full, halo=None, peer=None, row0: int = 0):
    """Entries of `full` the slab's rows read <- their owners' values.

    With the peer transport, `full` is its arena vector and every rank pushes the
    entries its peers read straight into theirs (one kernel, K8).  Otherwise, with
    a halo plan (dist.Halo): NCCL point-to-point exchange of the
    boundary columns only; else the in-place all-gather of equal slabs."""
    if comm is None or comm.world == 1:
        return local
    if peer is not None:
        peer.exchange(local, peer.plan(halo, row0, local.numel()))
        return full
    if halo is not None and not halo.use_allgather:
        return halo.exchange(full, local)
    comm.all_gather_vec(full, local)
    return full


def _halo_for(comm, src):
    """The operator's halo plan (cached on its CSR slab); None on one GPU or with PSELL_HALO=0."""
    import os
    if comm is None or comm.world == 1 or os.environ.get("PSELL_HALO", "1") == "0":
        return None
    D = src.to_device()
    cache = D.__dict__.setdefault("_halo", {})
    if id(comm) not in cache:
        import torch
        from .dist import Halo
        needed = torch.unique(D.col_idx).cpu().numpy() if D.nnz else np.zeros(0, np.int64)
        cache[id(comm)] = Halo(comm, D.row0, D.row0 + D.n_rows, needed, n_cols=D.n_cols)
    return cache[id(comm)]


def _check_slabs(comm, row0: int, n: int, halo, peer):
    """The NCCL all-gather path places rank r's chunk at r * n: it needs equal, rank-ordered
    slabs.  The halo exchanges and the peer transport address entries by
    global index and take any sigma-aligned partition."""
    if comm is None or comm.world == 1 or peer is not None or (halo is not None and not halo.use_allgather):
        return
    slabs = comm.slabs(row0, n)
    if any(s != (r * n, (r + 1) * n) for r, s in enumerate(slabs)):
        raise ValueError(f"the all-gather transport needs equal rank-ordered row slabs, got {slabs}; use the "
                         "halo exchange or the peer transport for other partitions")


# ----------------------------------------------------------------------------
# inner mixed-precision PCG (solvers.py:278-308)
# ----------------------------------------------------------------------------

class _InnerPCG:
    """f32 fixed-count PCG on the PackSELL operator; CUDA-graph captured on one GPU."""

    def __init__(self, backend: SpmvBackend, m_in: int, inv_diag=None, comm=None, use_graph: bool = True):
        import torch
        from . import _lib
        self.torch = torch
        self.backend = backend
        self.m_in = int(m_in)
        self.comm = comm
        M = backend.matrix
        if not isinstance(M, PackSellMatrix):
            raise TypeError("_InnerPCG drives a PackSELL backend")
        self.halo = _halo_for(comm, backend.source)
        self.M = M
        self.n = M.n_rows
        self.row0 = M.row0
        self.peer = None if comm is None or comm.world == 1 else comm.peer(M.n_cols)
        _check_slabs(comm, self.row0, self.n, self.halo, self.peer)
        self.inv = inv_diag
        f32 = torch.float32
        self.x = torch.zeros(self.n, dtype=f32, device="cuda")
        self.r = torch.zeros(self.n, dtype=f32, device="cuda")
        self.q = torch.zeros(self.n, dtype=f32, device="cuda")
        self.z = torch.zeros(self.n, dtype=f32, device="cuda") if inv_diag is not None else self.r
        G = 1 if comm is None else comm.world
        if G == 1:
            self.p_full = torch.zeros(self.n, dtype=f32, device="cuda")
            self.p = self.p_full
        else:
            self.p_full = self.peer.full32 if self.peer is not None else \
                torch.zeros(M.n_cols, dtype=f32, device="cuda")
            self.p = self.p_full[self.row0:self.row0 + self.n]
        lib = _lib.lib()
        self.desc = M.desc()
        self.npart = lib.psell_spmv_dot_partials(self.desc, M.spmv_flags())
        self.d = _Dev(max(self.npart, _lib.RED_BLOCKS), comm)
        self.d.peer = self.peer
        self.graph = None
        self.graph_in = None
        # one GPU, or ranks joined by the peer transport: the inner loop is kernels only
        self.use_graph = use_graph and (G == 1 or self.peer is not None)
        self._io = None
        # outer-loop gate (fcg look-ahead): nonzero turns the whole inner solve into a no-op
        self.gate = torch.zeros(2, dtype=torch.int32, device="cuda")

    def buffers(self):
        """Persistent f64 (r, z) the outer loop can hand to solve(): the captured graph
        is bound to them, so repeated solves replay without re-capture."""
        if self._io is None:
            f64 = self.torch.float64
            self._io = (self.torch.zeros(self.n, dtype=f64, device="cuda"),
                        self.torch.zeros(self.n, dtype=f64, device="cuda"))
        return self._io

    def _sequence(self, r64, z64):
        d, L, lib = self.d, self.d.L, self.d.lib
        st = d.st()
        inv = None if self.inv is None else self.inv.data_ptr()
        M = self.M
        err = L.PsellError()
        lib.psell_ipcg_begin(self.n, r64.data_ptr(), self.x.data_ptr(), self.r.data_ptr(), self.z.data_ptr(),
                             self.p.data_ptr(), inv, d.p(d.partials), d.p(d.loc, 0), st)
        g, stride = d.gather()
        lib.psell_ipcg_set_rz_gated(d.p(g, 0), d.G, stride, d.p(d.scal), d.p(d.flags), self.gate.data_ptr(), st)
        if d.G == 1:
            # one GPU: 3 launches per iteration -- SpMV + p.q + alpha, r/z update + r.z + beta,
            # x += alpha p with p = z + beta p
            # (the scalar steps run in the last CTA of the preceding kernel, fixed-order sums)
            for _ in range(self.m_in):
                rc = lib.psell_spmv_dot_alpha(self.desc, L.ptr(M.d_pack), L.ptr(M.d_offset), L.ptr(M.d_perm),
                                              self.p_full.data_ptr(), self.q.data_ptr(), self.p.data_ptr(),
                                              d.p(d.partials), d.p(d.scal), d.p(d.flags), d.p(d.ticket, 0),
                                              M.spmv_flags(), st, err)
                L.check(rc, err, M.fmt)
                lib.psell_ipcg_update_beta(self.n, None, self.r.data_ptr(), self.z.data_ptr(),
                                           self.p.data_ptr(), self.q.data_ptr(), inv, d.p(d.scal), d.p(d.flags),
                                           d.p(d.partials), d.p(d.ticket, d.tstride), st)
                lib.psell_ipcg_direction_x(self.n, self.p.data_ptr(), self.z.data_ptr(), self.x.data_ptr(),
                                           d.p(d.scal), d.p(d.flags), st)
            lib.psell_ipcg_end(self.n, self.x.data_ptr(), z64.data_ptr(), st)
            return
        if self.peer is not None and os.environ.get("PSELL_PEER_FUSED", "1") != "0":
            # G ranks over the peer arenas: the halo push (K8) and the single-GPU iteration's
            # three kernels, the SpMV's and the update's last CTAs all-reducing their dot
            # sums over the arenas before the alpha / beta steps -- 4 launches per iteration
            pe = self.peer
            peers = pe.d_peers.data_ptr()
            # the halo of p: pushed by K8 before the first SpMV, then by each iteration's direction
            # kernel itself when the push list is <= 2 contiguous ranges (stencil slabs)
            rg = pe.ranges(self.halo, self.n) if os.environ.get("PSELL_PEER_HALO_FUSED", "1") != "0" else None
            if rg is not None:
                import ctypes
                k = len(rg)
                lo = (ctypes.c_int64 * 2)(*[r[0] for r in rg], *([0] * (2 - k)))
                hi = (ctypes.c_int64 * 2)(*[r[1] for r in rg], *([0] * (2 - k)))
                dst = (ctypes.c_int32 * 2)(*[r[2] for r in rg], *([0] * (2 - k)))
                _gather_full(self.comm, self.p, self.p_full, self.halo, self.peer, self.row0)
            for it in range(self.m_in):
                if rg is None:
                    _gather_full(self.comm, self.p, self.p_full, self.halo, self.peer, self.row0)
                rc = lib.psell_spmv_dot_alpha_peer(self.desc, L.ptr(M.d_pack), L.ptr(M.d_offset), L.ptr(M.d_perm),
                                                   self.p_full.data_ptr(), self.q.data_ptr(), self.p.data_ptr(),
                                                   d.p(d.partials), d.p(d.scal), d.p(d.flags), d.p(d.ticket, 0),
                                                   M.spmv_flags(), pe.G, pe.rank, peers, pe.timeout_ns, st, err)
                L.check(rc, err, M.fmt)
                rc = lib.psell_ipcg_update_beta_peer(self.n, None, self.r.data_ptr(), self.z.data_ptr(),
                                                     self.p.data_ptr(), self.q.data_ptr(), inv, d.p(d.scal),
                                                     d.p(d.flags), d.p(d.partials), d.p(d.ticket, d.tstride), pe.G,
                                                     pe.rank, peers, pe.timeout_ns, st)
                if rc:
                    raise L.LibpsellError(f"psell_ipcg_update_beta_peer failed ({rc})")
                if rg is not None and it + 1 < self.m_in:
                    rc = lib.psell_ipcg_direction_x_push(self.n, self.p.data_ptr(), self.z.data_ptr(),
                                                         self.x.data_ptr(), d.p(d.scal), d.p(d.flags), pe.G, pe.rank,
                                                         peers, self.row0, pe.vec_off[4], k, lo, hi, dst,
                                                         pe.timeout_ns, st)
                    if rc:
                        raise L.LibpsellError(f"psell_ipcg_direction_x_push failed ({rc})")
                else:
                    lib.psell_ipcg_direction_x(self.n, self.p.data_ptr(), self.z.data_ptr(), self.x.data_ptr(),
                                               d.p(d.scal), d.p(d.flags), st)
            lib.psell_ipcg_end(self.n, self.x.data_ptr(), z64.data_ptr(), st)
            return
        for _ in range(self.m_in):
            _gather_full(self.comm, self.p, self.p_full, self.halo, self.peer, self.row0)
            rc = lib.psell_spmv_dot(self.desc, L.ptr(M.d_pack), L.ptr(M.d_offset), L.ptr(M.d_perm),
                                    self.p_full.data_ptr(), self.q.data_ptr(), self.p.data_ptr(),
                                    d.p(d.partials), d.p(d.flags), M.spmv_flags(), st, err)
            L.check(rc, err, M.fmt)
            lib.psell_sum_partials(d.p(d.partials), self.npart, 1, d.p(d.loc, 1), d.p(d.flags), st)
            g, stride = d.gather()
            lib.psell_ipcg_alpha(d.p(g, 1), d.G, stride, d.p(d.scal), d.p(d.flags), st)
            lib.psell_ipcg_update(self.n, self.x.data_ptr(), self.r.data_ptr(), self.z.data_ptr(),
                                  self.p.data_ptr(), self.q.data_ptr(), inv, d.p(d.scal), d.p(d.flags),
                                  d.p(d.partials), d.p(d.loc, 2), st)
            g, stride = d.gather()
            lib.psell_ipcg_beta(d.p(g, 2), d.G, stride, d.p(d.scal), d.p(d.flags), st)
            lib.psell_ipcg_direction(self.n, self.p.data_ptr(), self.z.data_ptr(), d.p(d.scal), d.p(d.flags), st)
        lib.psell_ipcg_end(self.n, self.x.data_ptr(), z64.data_ptr(), st)

    def solve(self, r64, z64) -> int:
        """z64 <- m_in f32 PCG steps on A z = r64 from zero; returns completed iterations."""
        self.launch(r64, z64)
        return _inner_done(self.d)

    def launch(self, r64, z64):
        """Queue the inner solve (no host synchronisation); d.flags[:2] = {breakdown, done}."""
        torch = self.torch
        if self.use_graph:
            if self.graph is None or self.graph_in is None or \
                    self.graph_in[0] is not r64 or self.graph_in[1] is not z64:
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    self._sequence(r64, z64)  # warm-up outside capture
                torch.cuda.current_stream().wait_stream(s)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._sequence(r64, z64)
                self.graph = g
                self.graph_in = (r64, z64)
            self.graph.replay()
        else:
            self._sequence(r64, z64)


def _inner_done(d, flags=None) -> int:
    """Completed inner iterations from an inner solver's {breakdown, done} flags (logs a breakdown)."""
    if flags is None:
        flags = d.flags[:2].cpu().numpy()
    if int(flags[0]):
        log.warning("inner PCG breakdown at iteration %d (p'Ap=%r); returning current iterate",
                    int(flags[1]), float(d.scal[1].item()))
    return int(flags[1])


class _GenericInner:
    """Inner PCG (solvers.py:278-308) on any device backend: the SELL-C-sigma / CSR
    comparators in f32 (the FP32 IO-CG of config 5) and every backend in f64
    (inner_precision="real64").  One GPU.  The same K3 scalar kernels as _InnerPCG
    (breakdown flags, alpha / beta on the device).  f32: the _InnerPCG launch
    structure (fused r/z update + beta, fused x / direction) captured in one CUDA
    graph per backend, with the operator's SpMV and a fixed-grid FP64 p.q in place
    of the fused PackSELL SpMV + p.q + alpha; f64: eager, the outer loop's f64
    kernels."""

    def __init__(self, backend, m_in, dtype, inv, use_graph: bool = True):
        import torch
        from . import _dev, _lib
        self.torch = torch
        self.use_graph = use_graph
        self.graph, self.graph_in, self._io = None, None, None
        self.gate = torch.zeros(2, dtype=torch.int32, device="cuda")  # see _InnerPCG.gate
        self.backend = backend
        self.m_in = int(m_in)
        self.tdt = _dev.torch_dtype(dtype)
        self.f32 = self.tdt == torch.float32
        self.dt_code = _dev.T_DT_CODE[self.tdt]
        self.inv = inv
        # f32 SELL-C-sigma (C = 32) comparator: SpMV + p.q + alpha as one launch, like the PackSELL
        # inner loop (psell_sell_spmv_dot_alpha; PSELL_SELL_FUSED=0 restores the three launches)
        M = backend.matrix
        self.sell_fused = (self.f32 and backend.name == "sell32" and getattr(M, "c", 0) == 32
                           and os.environ.get("PSELL_SELL_FUSED", "1") != "0")
        n_part = _lib.RED_BLOCKS
        if self.sell_fused:
            n_part = max(n_part, int(_lib.lib().psell_sell_spmv_dot_partials(M.desc())))
        self.d = _Dev(n_part)
        self.n = None

    def _alloc(self, n):
        if self.n != n:
            t = self.torch
            self.n = n
            self.x, self.r, self.p, self.q = (t.zeros(n, dtype=self.tdt, device="cuda") for _ in range(4))
            self.z = t.zeros(n, dtype=self.tdt, device="cuda") if self.inv is not None else self.r
            self.graph = None

    def buffers(self):
        """Persistent f64 (r, z) for the outer loop (the f32 graph is bound to them)."""
        if getattr(self, "_io", None) is None:
            n = self.backend.source.n_rows
            f64 = self.torch.float64
            self._io = (self.torch.zeros(n, dtype=f64, device="cuda"), self.torch.zeros(n, dtype=f64, device="cuda"))
        return self._io

    def _sequence_f32(self, r64, z64):
        """The f32 inner loop in the _InnerPCG launch structure (SpMV; p.q + alpha;
        r/z update + r.z + beta in one launch; x += alpha p with p = z + beta p)."""
        d, lib = self.d, self.d.lib
        n = self.n
        st = d.st()
        inv = None if self.inv is None else self.inv.data_ptr()
        x, r, z, p, q = self.x, self.r, self.z, self.p, self.q
        lib.psell_ipcg_begin(n, r64.data_ptr(), x.data_ptr(), r.data_ptr(), z.data_ptr(), p.data_ptr(), inv,
                             d.p(d.partials), d.p(d.loc, 0), st)
        lib.psell_ipcg_set_rz_gated(d.p(d.loc, 0), 1, 8, d.p(d.scal), d.p(d.flags), self.gate.data_ptr(), st)
        M, L = self.backend.matrix, d.L
        if self.sell_fused:
            from . import _dev
            sdesc, err = M.desc(), L.PsellError()
        for _ in range(self.m_in):
            if self.sell_fused:
                rc = lib.psell_sell_spmv_dot_alpha(sdesc, L.ptr(M.d_val), _dev.DT_CODE[M.value_dtype], L.ptr(M.d_col),
                                                   L.ptr(M.d_offset), L.ptr(M.d_perm), p.data_ptr(), q.data_ptr(),
                                                   p.data_ptr(), d.p(d.partials), d.p(d.scal), d.p(d.flags),
                                                   d.p(d.ticket, 0), st, err)
                L.check(rc, err)
            else:
                self.backend.apply_into(p, q)
                lib.psell_dot(p.data_ptr(), q.data_ptr(), self.dt_code, n, d.p(d.partials), d.p(d.loc, 1), st)
                lib.psell_ipcg_alpha(d.p(d.loc, 1), 1, 8, d.p(d.scal), d.p(d.flags), st)
            lib.psell_ipcg_update_beta(n, None, r.data_ptr(), z.data_ptr(), p.data_ptr(), q.data_ptr(), inv,
                                       d.p(d.scal), d.p(d.flags), d.p(d.partials), d.p(d.ticket, d.tstride), st)
            lib.psell_ipcg_direction_x(n, p.data_ptr(), z.data_ptr(), x.data_ptr(), d.p(d.scal), d.p(d.flags), st)
        lib.psell_ipcg_end(n, x.data_ptr(), z64.data_ptr(), st)

    def _eager(self, r64, z64):
        """The loop launched op by op (f64 vectors, or use_graph=False)."""
        d, lib = self.d, self.d.lib
        n = self.n
        st = d.st()
        inv = None if self.inv is None else self.inv.data_ptr()
        x, r, z, p = self.x, self.r, self.z, self.p
        if self.f32:
            self._sequence_f32(r64, z64)
            return
        x.zero_()
        r.copy_(r64)
        lib.psell_precond_dot(n, z.data_ptr(), r.data_ptr(), inv, d.p(d.partials), d.p(d.loc, 0), st)
        lib.psell_xpby(n, p.data_ptr(), z.data_ptr(), None, st)
        lib.psell_ipcg_set_rz_gated(d.p(d.loc, 0), 1, 8, d.p(d.scal), d.p(d.flags), self.gate.data_ptr(), st)
        for _ in range(self.m_in):
            q = self.backend.apply(p)
            lib.psell_dot(p.data_ptr(), q.data_ptr(), self.dt_code, n, d.p(d.partials), d.p(d.loc, 1), st)
            lib.psell_ipcg_alpha(d.p(d.loc, 1), 1, 8, d.p(d.scal), d.p(d.flags), st)
            lib.psell_axpy2(n, x.data_ptr(), r.data_ptr(), p.data_ptr(), q.data_ptr(), d.p(d.scal, 2),
                            d.p(d.flags), d.p(d.partials), d.p(d.loc, 3), st)
            lib.psell_precond_dot(n, z.data_ptr(), r.data_ptr(), inv, d.p(d.partials), d.p(d.loc, 2), st)
            lib.psell_ipcg_beta(d.p(d.loc, 2), 1, 8, d.p(d.scal), d.p(d.flags), st)
            lib.psell_xpby_checked(n, p.data_ptr(), z.data_ptr(), d.p(d.scal, 3), d.p(d.flags), st)
        z64.copy_(x)

    def solve(self, r64, z64) -> int:
        self.launch(r64, z64)
        return _inner_done(self.d)

    def launch(self, r64, z64):
        """Queue the inner solve (no host synchronisation); d.flags[:2] = {breakdown, done}."""
        self._alloc(int(r64.numel()))
        if self.f32 and self.use_graph:
            torch = self.torch
            if self.graph is None or self.graph_in[0] is not r64 or self.graph_in[1] is not z64:
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    self._sequence_f32(r64, z64)  # warm-up outside capture
                torch.cuda.current_stream().wait_stream(s)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._sequence_f32(r64, z64)
                self.graph, self.graph_in = g, (r64, z64)
            self.graph.replay()
        else:
            self._eager(r64, z64)


# ----------------------------------------------------------------------------
# f64 drivers
# ----------------------------------------------------------------------------

def _diag_of(src) -> np.ndarray:
    """Stored diagonal of a (slab) CSR in global column numbering."""
    if isinstance(src, DeviceCsrMatrix):
        H = src.to_host()
        rows = np.repeat(np.arange(H.n_rows, dtype=np.int64), H.row_lengths()) + src.row0
        dg = np.zeros(H.n_rows)
        on = rows == H.col_idx
        dg[rows[on] - src.row0] = H.values[on]
        return dg
    return src.diagonal()


def _jacobi_inv(backend: SpmvBackend, dtype):
    """1/diag of the f64 source, rounded to dtype (solvers.py:145-149)."""
    from . import _dev
    diag = _diag_of(backend.source)
    if np.any(diag == 0.0):
        raise ValueError("jacobi preconditioner requires a fully nonzero diagonal")
    return _dev.upload((1.0 / diag).astype(dtype))


class _Outer:
    """f64 vectors + operator of a (possibly distributed) outer loop."""

    def __init__(self, backend: SpmvBackend, b, comm):
        import torch
        from . import _lib
        self.torch = torch
        self.backend = backend
        self.comm = comm
        self.G = 1 if comm is None else comm.world
        src = backend.matrix if not backend.is_packsell else backend.source
        self.row0 = getattr(src, "row0", 0)
        self.halo = _halo_for(comm, src)
        b = np.asarray(b, dtype=np.float64)
        self.n = len(b)
        from . import _dev
        self.b = _dev.upload(b)
        self.d = _Dev(_lib.RED_BLOCKS, comm)
        self.lib = self.d.lib
        f64 = torch.float64
        self.n_glob = src.n_cols
        self.peer = comm.peer(self.n_glob) if self.G > 1 else None
        self.d.peer = self.peer
        _check_slabs(comm, self.row0, self.n, self.halo, self.peer)
        if self.G == 1:
            self.full = None
        else:
            self.full = self.peer.full64 if self.peer is not None else \
                torch.zeros(self.n_glob, dtype=f64, device="cuda")

    def vec(self):
        return self.torch.zeros(self.n, dtype=self.torch.float64, device="cuda")

    def slab_of_full(self):
        return self.full[self.row0:self.row0 + self.n]

    def apply(self, v, out):
        """out <- A v (v local slab; all-gathered to the global vector first)."""
        if self.G == 1:
            return self.backend.apply_into(v, out)
        self.slab_of_full().copy_(v)
        _gather_full(self.comm, self.slab_of_full(), self.full, self.halo, self.peer, self.row0)
        return self.backend.apply_into(self.full, out)

    def apply_pq(self, p, q, slot: int) -> bool:
        """q <- A p and loc[slot] <- this rank's p.q in one fused K4 launch when the
        operator is the f64 CSR (FP64 PCG); False (nothing done) otherwise."""
        if self.backend.name != "csr64" or p.dtype != self.torch.float64:
            return False
        D = self.backend.source.to_device()
        x = p
        if self.G > 1:
            self.slab_of_full().copy_(p)
            x = _gather_full(self.comm, self.slab_of_full(), self.full, self.halo, self.peer, self.row0)
        L, d = self.d.L, self.d
        err = L.PsellError()
        rc = self.lib.psell_csr_spmv_dot(D.n_rows, L.ptr(D.row_ptr), L.ptr(D.col_idx), L.ptr(D.values),
                                         x.data_ptr(), q.data_ptr(), p.data_ptr(), d.p(d.partials),
                                         d.p(d.loc, slot), d.st(), err)
        L.check(rc, err)
        return True

    def audit(self, report: SolveReport, x, bnorm, tol) -> SolveReport:
        """True residual in f64 on the device, demote drifted runs (solvers.py:152-168)."""
        d = self.d
        if bnorm == 0.0:
            report.final_true_relres = 0.0
            return report
        ax = self.vec()
        src = self.backend.source
        if self.G == 1:
            csr_spmv(src, x, np.float64, out=ax)
        else:
            self.slab_of_full().copy_(x)
            _gather_full(self.comm, self.slab_of_full(), self.full, self.halo, self.peer, self.row0)
            csr_spmv(src, self.full, np.float64, out=ax)
        self.lib.psell_resid(self.n, self.b.data_ptr(), ax.data_ptr(), d.p(d.partials), d.p(d.loc, 6), d.st())
        d.reduce(6, 1, 14)
        report.final_true_relres = float(np.sqrt(float(d.scal[14].item()))) / bnorm
        if self.peer is not None:
            self.peer.check()
        if report.converged and not report.final_true_relres < 10.0 * tol:
            report.converged = False
            msg = f"true residual {report.final_true_relres:.3e} exceeds 10x tolerance"
            report.reason = f"{report.reason}; {msg}" if report.reason else msg
        return report


class _HostMirror:
    """The per-iteration status block read back on a side stream: the few-byte D2H copy
    waits for its producer kernel there, so the next kernel of the iteration does not
    queue behind a PCIe round trip on the solver's stream."""

    def __init__(self):
        import torch
        self.torch = torch
        self.side = torch.cuda.Stream()

    def copy(self, dst, src):
        """dst (pinned host) <- src once the work queued so far on the current stream is
        done; returns the event that marks the copy complete."""
        torch = self.torch
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream())
        self.side.wait_event(ready)
        with torch.cuda.stream(self.side):
            dst.copy_(src, non_blocking=True)
        done = torch.cuda.Event()
        done.record(self.side)
        return done


def _dev_mod():
    from . import _dev
    return _dev


def pcg(A, b, cfg: SolveConfig = None, x0=None, *, comm=None) -> SolveReport:
    """f64 PCG stopping on the recurred residual (solvers.py:171-217), on the GPU."""
    import torch
    cfg = cfg or SolveConfig()
    backend = _as_backend(A)
    t0 = time.perf_counter()
    o = _Outer(backend, b, comm)
    d, lib, n = o.d, o.lib, o.n
    st = d.st()
    x = o.vec() if x0 is None else torch.as_tensor(np.asarray(x0, dtype=np.float64)).cuda()
    inv = _jacobi_inv(backend, np.float64) if cfg.preconditioner == "jacobi" else None
    bnorm = d.norm(o.b)
    if bnorm == 0.0:
        return SolveReport(True, 0, 0, [], 0.0, time.perf_counter() - t0, x=x.cpu().numpy())
    r = o.b.clone()
    if x0 is not None and np.any(np.asarray(x0)):
        ax = o.vec()
        o.apply(x, ax)
        r.copy_(ax)
        neg1 = torch.tensor([-1.0], dtype=torch.float64, device="cuda")
        lib.psell_xpby(n, r.data_ptr(), o.b.data_ptr(), neg1.data_ptr(), st)   # r = b - Ax
    history = [d.norm(r) / bnorm]
    z = o.vec() if inv is not None else r
    invp = None if inv is None else inv.data_ptr()
    lib.psell_precond_dot(n, z.data_ptr(), r.data_ptr(), invp, d.p(d.partials), d.p(d.loc, 0), st)
    d.reduce(0, 1, 4)                                                      # scal4 = rz
    p = z.clone()
    q = o.vec()
    # The host reads iteration k's status while iteration k+1 is already queued:
    # psell_pcg_status closes a device gate (flags[2]) on convergence, and a
    # breakdown closes it through scalar_div's curvature check, so the iteration
    # queued past the stop leaves x and r untouched -- no idle GPU between
    # iterations, and the same iterates, history and stopping point as the loop
    # of solvers.py:183-207 evaluated one iteration at a time.
    gate = d.flags[2:4]
    gate.zero_()
    gp = gate.data_ptr()
    h_stat = torch.zeros(6, dtype=torch.float64, pin_memory=True)
    mirror = _HostMirror()
    events = [None, None]  # per status slot: the event of its last read-back

    def body(k):
        st = d.st()
        if not o.apply_pq(p, q, 0):
            o.apply(p, q)
            lib.psell_pq_pr(n, p.data_ptr(), q.data_ptr(), None, d.p(d.partials), d.p(d.loc, 0), st)
        d.reduce(0, 1, 10)                                                 # scal10 = pq
        lib.psell_scalar_div(d.p(d.scal, 4), d.p(d.scal, 10), 1, 1, d.p(d.scal, 0), gp, 1, st)  # alpha
        lib.psell_axpy2(n, x.data_ptr(), r.data_ptr(), p.data_ptr(), q.data_ptr(), d.p(d.scal, 0),
                        gp, d.p(d.partials), d.p(d.loc, 2), st)
        d.reduce(2, 1, 12)                                                 # scal12 = rr
        slot = 16 + 3 * (k % 2)
        lib.psell_pcg_status(d.p(d.scal, 10), d.p(d.scal, 12), gp, bnorm, cfg.tol, d.p(d.scal, slot), st)
        events[k % 2] = mirror.copy(h_stat[3 * (k % 2):3 * (k % 2) + 3], d.scal[slot:slot + 3])
        if invp is None:
            # identity: z = r, and r.z is the r.r just reduced -- the same kernel
            # grid, per-thread order and tree as psell_precond_dot, so the same bits
            rz_slot = 12
        else:
            lib.psell_precond_dot(n, z.data_ptr(), r.data_ptr(), invp, d.p(d.partials), d.p(d.loc, 3), st)
            d.reduce(3, 1, 5)                                              # scal5 = rz_new
            rz_slot = 5
        lib.psell_scalar_div(d.p(d.scal, rz_slot), d.p(d.scal, 4), 1, 1, d.p(d.scal, 2), None, 0, st)  # beta
        lib.psell_sum_strided(d.p(d.scal, rz_slot), 1, 1, 1, d.p(d.scal, 4), st)                   # rz = rz_new
        lib.psell_xpby(n, p.data_ptr(), z.data_ptr(), d.p(d.scal, 2), st)

    # one GPU, f64 CSR operator, identity preconditioner (the FP64 comparator of config 5):
    # three launches per iteration -- SpMV + p.q + alpha, update + r.r + status + beta,
    # direction -- with the scalar steps in the last CTA of the first two (fixed order)
    fused = (o.G == 1 and backend.name == "csr64" and invp is None
             and os.environ.get("PSELL_PCG_FUSED", "1") != "0")
    if fused:
        D = backend.source.to_device()
        L = d.L

    def body_fused(k):
        st = d.st()
        slot = 16 + 3 * (k % 2)
        err = L.PsellError()
        rc = lib.psell_csr_spmv_dot_alpha(D.n_rows, L.ptr(D.row_ptr), L.ptr(D.col_idx), L.ptr(D.values),
                                          p.data_ptr(), q.data_ptr(), p.data_ptr(), d.p(d.partials), d.p(d.scal),
                                          gp, d.p(d.ticket, 0), st, err)
        L.check(rc, err)
        lib.psell_pcg_update_status(n, x.data_ptr(), r.data_ptr(), p.data_ptr(), q.data_ptr(), d.p(d.scal), gp,
                                    bnorm, cfg.tol, d.p(d.scal, slot), d.p(d.partials), d.p(d.ticket, d.tstride), st)
        events[k % 2] = mirror.copy(h_stat[3 * (k % 2):3 * (k % 2) + 3], d.scal[slot:slot + 3])
        lib.psell_xpby_checked(n, p.data_ptr(), r.data_ptr(), d.p(d.scal, 2), gp, st)

    def enqueue(k):
        if events[k % 2] is not None:  # slot k % 2 is rewritten only after its last read-back
            torch.cuda.current_stream().wait_event(events[k % 2])
        (body_fused if fused else body)(k)

    converged, reason, it = False, None, 0
    if cfg.max_outer <= 0:
        reason = f"maximum iterations ({cfg.max_outer}) reached"
    elif history[-1] < cfg.tol:
        converged = True
    else:
        enqueue(0)
        k = 0
        while True:
            if k + 1 < cfg.max_outer:
                enqueue(k + 1)
            events[k % 2].synchronize()
            brk, pq, rel = (float(v) for v in h_stat[3 * (k % 2):3 * (k % 2) + 3].numpy())
            if brk == 1.0:
                reason = f"breakdown: non-positive curvature p'Ap = {pq!r} at iteration {it}"
                break
            it = k + 1
            history.append(rel)
            if rel < cfg.tol:
                converged = True
                break
            k += 1
            if k >= cfg.max_outer:
                reason = f"maximum iterations ({cfg.max_outer}) reached"
                break
    if not converged and history[-1] < cfg.tol:
        converged = True
        reason = None
    torch.cuda.synchronize()
    report = SolveReport(converged, it, 0, history, 0.0, time.perf_counter() - t0, reason)
    report = o.audit(report, x, bnorm, cfg.tol)
    report.x = _dev_mod().download(x, np.float64)
    return report


def fcg(A, b, cfg: SolveConfig = None, inner_preconditioner: Callable = None, *, _inner=None,
        comm=None) -> SolveReport:
    """Truncated flexible CG in f64 (solvers.py:220-275), on the GPU.

    `inner_preconditioner` may be a Python callable on numpy vectors (the
    reference contract; runs through host copies); iocg passes a device inner
    solver via `_inner`.
    """
    import torch
    cfg = cfg or SolveConfig()
    backend = _as_backend(A)
    t0 = time.perf_counter()
    o = _Outer(backend, b, comm)
    d, lib, n = o.d, o.lib, o.n
    st = d.st()
    x = o.vec()
    bnorm = d.norm(o.b)
    if bnorm == 0.0:
        return SolveReport(True, 0, 0, [], 0.0, time.perf_counter() - t0, x=x.cpu().numpy())
    inv = None
    if _inner is None and inner_preconditioner is None and cfg.preconditioner == "jacobi":
        inv = _jacobi_inv(backend, np.float64)
    if _inner is not None and hasattr(_inner, "buffers"):
        r, z = _inner.buffers()  # the inner solver's graph is bound to these
        r.copy_(o.b)
    else:
        r, z = o.b.clone(), o.vec()
    history = [d.norm(r) / bnorm]
    p, q, r_prev = o.vec(), o.vec(), o.vec()
    converged, reason, it = False, None, 0
    inner_total = 0
    # Look-ahead as in pcg: iteration k+1 (inner solve included) is queued before
    # iteration k's status is read.  The gate closed by psell_pcg_status (or by a
    # curvature breakdown in scalar_div) gates the outer x / r update and, through
    # psell_ipcg_set_rz_gated, turns the queued inner solve into a no-op.  A host
    # callable preconditioner needs r on the host every iteration: no look-ahead.
    ahead = inner_preconditioner is None
    gate = _inner.gate if (_inner is not None and hasattr(_inner, "gate")) else d.flags[2:4]
    if _inner is not None and not hasattr(_inner, "launch"):
        ahead = False
    gate.zero_()
    gp = gate.data_ptr()
    h_stat = torch.zeros(6, dtype=torch.float64, pin_memory=True)
    h_in = torch.zeros(4, dtype=torch.int32, pin_memory=True)
    mirror = _HostMirror()
    events = [None, None]  # per slot: the read-back of the iteration's status (after its h_in)
    in_done = [None]       # the read-back of the inner flags (rewritten by the next inner solve)

    def enqueue(k):
        slot = k % 2
        main = torch.cuda.current_stream()
        for ev in (events[slot], in_done[0]):
            if ev is not None:
                main.wait_event(ev)
        if _inner is not None:
            if ahead:
                _inner.launch(r, z)
                in_done[0] = mirror.copy(h_in[2 * slot:2 * slot + 2], _inner.d.flags[:2])
            else:
                h_in[2 * slot + 1] = _inner.solve(r, z)
        elif inner_preconditioner is not None:
            z.copy_(torch.as_tensor(np.asarray(inner_preconditioner(r.cpu().numpy()), dtype=np.float64)))
        elif inv is not None:
            lib.psell_precond_dot(n, z.data_ptr(), r.data_ptr(), inv.data_ptr(), d.p(d.partials), d.p(d.loc, 7), st)
        else:
            z.copy_(r)
        lib.psell_fcg_zr(n, z.data_ptr(), r.data_ptr(), None if k == 0 else r_prev.data_ptr(),
                         d.p(d.partials), d.p(d.loc, 0), st)
        d.reduce(0, 2, 8)                                  # scal8 = z.(r - r_prev), scal9 = z.r
        if k == 0:
            lib.psell_xpby(n, p.data_ptr(), z.data_ptr(), None, st)
        else:
            lib.psell_scalar_div(d.p(d.scal, 8), d.p(d.scal, 6), 1, 1, d.p(d.scal, 2), None, 0, st)  # beta
            lib.psell_xpby(n, p.data_ptr(), z.data_ptr(), d.p(d.scal, 2), st)
        lib.psell_sum_strided(d.p(d.scal, 9), 1, 1, 1, d.p(d.scal, 6), st)                        # zr_prev
        r_prev.copy_(r)
        o.apply(p, q)
        lib.psell_pq_pr(n, p.data_ptr(), q.data_ptr(), r.data_ptr(), d.p(d.partials), d.p(d.loc, 2), st)
        d.reduce(2, 2, 10)                                 # scal10 = p.q, scal11 = p.r
        lib.psell_scalar_div(d.p(d.scal, 11), d.p(d.scal, 10), 1, 1, d.p(d.scal, 0), gp, 1, st)     # alpha
        lib.psell_axpy2(n, x.data_ptr(), r.data_ptr(), p.data_ptr(), q.data_ptr(), d.p(d.scal, 0),
                        gp, d.p(d.partials), d.p(d.loc, 4), st)
        d.reduce(4, 1, 12)                                 # scal12 = r.r
        sl = 16 + 3 * slot
        lib.psell_pcg_status(d.p(d.scal, 10), d.p(d.scal, 12), gp, bnorm, cfg.tol, d.p(d.scal, sl), st)
        events[slot] = mirror.copy(h_stat[3 * slot:3 * slot + 3], d.scal[sl:sl + 3])

    if cfg.max_outer <= 0:
        reason = f"maximum iterations ({cfg.max_outer}) reached"
    elif history[-1] < cfg.tol:
        converged = True
    else:
        enqueue(0)
        k = 0
        while True:
            if ahead and k + 1 < cfg.max_outer:
                enqueue(k + 1)
            events[k % 2].synchronize()
            if _inner is not None:
                if ahead:
                    inner_total += _inner_done(_inner.d, h_in[2 * (k % 2):2 * (k % 2) + 2].numpy())
                else:
                    inner_total += int(h_in[2 * (k % 2) + 1])
            brk, pq, rel = (float(v) for v in h_stat[3 * (k % 2):3 * (k % 2) + 3].numpy())
            if brk == 1.0:
                reason = f"breakdown: non-positive curvature p'Ap = {pq!r} at iteration {it}"
                break
            it = k + 1
            history.append(rel)
            if rel < cfg.tol:
                converged = True
                break
            k += 1
            if k >= cfg.max_outer:
                reason = f"maximum iterations ({cfg.max_outer}) reached"
                break
            if not ahead:
                enqueue(k)
    gate.zero_()  # leave the inner solver ungated for direct use
    if not converged and history[-1] < cfg.tol:
        converged = True
        reason = None
    torch.cuda.synchronize()
    report = SolveReport(converged, it, inner_total, history, 0.0, time.perf_counter() - t0, reason)
    report = o.audit(report, x, bnorm, cfg.tol)
    report.x = _dev_mod().download(x, np.float64)
    return report


def iocg(A, b, cfg: SolveConfig = None, *, backend: SpmvBackend = None, comm=None,
         use_graph: bool = True) -> SolveReport:
    """Inner-outer CG (solvers.py:311-333): m_in f32 PackSELL PCG steps precondition f64 FCG.

    `backend` passes a prebuilt inner backend (e.g. to keep the build out of a
    timing); by default it is built from cfg.a_backend like the reference.
    With `comm`, A and b are this rank's slabs.
    """
    cfg = cfg or SolveConfig(solver="iocg")
    if not isinstance(A, (CsrMatrix, DeviceCsrMatrix)):
        raise TypeError("iocg drives the outer iteration with the float64 CSR matrix")
    if backend is None:
        kl = None
        if comm is not None and comm.world > 1:
            from .packed import lower_bandwidth
            kl = comm.allreduce_max(lower_bandwidth(A))
        backend = make_backend(A, cfg.a_backend, k_left=kl)
    dtype = _PRECISIONS[cfg.inner_precision]
    inv = _jacobi_inv(backend, dtype) if cfg.preconditioner == "jacobi" else None
    if dtype == np.float32 and backend.is_packsell:
        # one inner solver (vectors + captured CUDA graph) per operator and setting,
        # reused by every solve on this backend
        key = (cfg.m_in, cfg.preconditioner, id(comm), use_graph)
        cache = backend.__dict__.setdefault("_inner_cache", {})
        inner = cache.get(key)
        if inner is None:
            inner = cache[key] = _InnerPCG(backend, cfg.m_in, inv, comm=comm, use_graph=use_graph)
    else:
        if comm is not None and comm.world > 1:
            raise NotImplementedError("distributed iocg needs a PackSELL inner backend in real32")
        key = ("generic", cfg.m_in, cfg.preconditioner, np.dtype(dtype).name, use_graph)
        cache = backend.__dict__.setdefault("_inner_cache", {})
        inner = cache.get(key)
        if inner is None:
            inner = cache[key] = _GenericInner(backend, cfg.m_in, dtype, inv, use_graph=use_graph)
    outer = make_backend(A, "csr64")
    return fcg(outer, b, cfg, _inner=inner, comm=comm)
