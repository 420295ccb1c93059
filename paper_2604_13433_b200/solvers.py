"""CG drivers over pluggable SpMV backends — drop-in for reference `packsell.solvers`.

Same names, signatures, config validation and report fields as the reference
(solvers.py:31-333).  Vectors live in HBM; every vector operation and every
reduction runs in libpsell (K3 kernels, deterministic fixed-grid FP64
reductions), every operator application in K2 (PackSELL) or K4 (CSR).

* `_InnerPCG` is the hot loop of the mixed-precision solver
  (_inner_pcg, solvers.py:278-308): m_in f32 PCG steps with the curvature dot
  fused into the PackSELL SpMV epilogue, alpha / beta / the breakdown flag kept
  on the device, and — on one GPU — the whole m_in-step loop captured once as
  a CUDA graph and replayed per outer iteration (no host round trip inside).
* `fcg` / `pcg` are the f64 outer / comparator loops; they read back one
  small status block per iteration (the reference's residual history needs it).

Multi-GPU: when a `Comm` is given (paper_2604_13433_b200.dist), each rank
owns a sigma-aligned row slab; the direction vector is all-gathered (NCCL over
NVLink) before every SpMV and every dot's local FP64 sum is all-gathered and
summed in rank order, so results do not depend on the reduction tree of the
collective.
"""

from __future__ import annotations

import logging
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
    (returns a CUDA tensor); it runs in x's precision.
    """

    def __init__(self, name: str, matrix, kernel: Callable, source):
        self.name = name
        self.matrix = matrix
        self._kernel = kernel
        self.source = source

    def apply(self, x):
        return self._kernel(x)

    @property
    def is_packsell(self) -> bool:
        return isinstance(self.matrix, PackSellMatrix)


def make_backend(A, name: str, c: int = 32, sigma: int = 256, mode: str = "implicit") -> SpmvBackend:
    """Named backend from an f64 CSR matrix (solvers.py:114-131)."""
    if name == "csr64":
        return SpmvBackend(name, A, lambda x: csr_spmv(A, x, _dtype_of(x)), A)
    if name in ("sell64", "sell32", "sell16"):
        from .sellfmt import build_sell, sell_spmv
        dt = {"sell64": np.float64, "sell32": np.float32, "sell16": np.float16}[name]
        S = build_sell(A, c, sigma, mode, value_dtype=dt)
        return SpmvBackend(name, S, lambda x: sell_spmv(S, x), A)
    if name.startswith("packsell-"):
        fmt = codec.parse_format(name[len("packsell-"):])
        M = build_packsell(A, c, sigma, fmt, mode)
        return SpmvBackend(name, M, lambda x: packsell_spmv(M, x), A)
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
    """Per-solve device scratch: partials, local sums, gathered sums, scalars, flags."""

    def __init__(self, n_partials: int, comm=None):
        import torch
        from . import _lib
        self.torch = torch
        self.lib = _lib.lib()
        self.L = _lib
        self.comm = comm
        self.G = 1 if comm is None else comm.world
        self.partials = torch.zeros(max(int(n_partials), 2 * _lib.RED_BLOCKS), dtype=torch.float64, device="cuda")
        self.loc = torch.zeros(8, dtype=torch.float64, device="cuda")
        self.glob = torch.zeros(self.G, 8, dtype=torch.float64, device="cuda")
        self.scal = torch.zeros(16, dtype=torch.float64, device="cuda")
        self.flags = torch.zeros(4, dtype=torch.int32, device="cuda")

    def st(self):
        return self.L.stream_handle()

    def p(self, t, off: int = 0):
        return t.data_ptr() + off * t.element_size()

    def gather(self):
        """All ranks' local sums -> glob[G][8] (rank order); G == 1: a view."""
        if self.G == 1:
            return self.loc, 8
        self.comm.all_gather_into(self.glob.view(-1), self.loc)
        return self.glob, 8


# ----------------------------------------------------------------------------
# inner mixed-precision PCG (solvers.py:278-308)
# ----------------------------------------------------------------------------

class _InnerPCG:
    """f32 fixed-count PCG on the PackSELL operator; CUDA-graph captured on one GPU."""

    def __init__(self, backend: SpmvBackend, m_in: int, inv_diag=None, comm=None, use_graph: bool = True):
        import torch
        self.torch = torch
        self.backend = backend
        self.m_in = int(m_in)
        self.comm = comm
        M = backend.matrix
        self.M = M if isinstance(M, PackSellMatrix) else None
        self.n = M.n_rows
        self.row0 = getattr(M, "row0", 0)
        self.n_glob = M.n_cols
        self.inv = inv_diag
        f32 = torch.float32
        self.x = torch.zeros(self.n, dtype=f32, device="cuda")
        self.r = torch.zeros(self.n, dtype=f32, device="cuda")
        self.q = torch.zeros(self.n, dtype=f32, device="cuda")
        self.z = torch.zeros(self.n, dtype=f32, device="cuda") if inv_diag is not None else self.r
        if comm is None or comm.world == 1:
            self.p_full = torch.zeros(self.n, dtype=f32, device="cuda")
            self.p = self.p_full
        else:
            self.p_full = torch.zeros(comm.padded_len(self.n_glob), dtype=f32, device="cuda")
            self.p = self.p_full[self.row0:self.row0 + self.n]
        from . import _lib
        lib = _lib.lib()
        npart = lib.psell_spmv_dot_partials(self.M.desc()) if self.M is not None else 1
        self.d = _Dev(max(npart, _lib.RED_BLOCKS), comm)
        self.graph = None
        self.graph_in = None
        self.use_graph = use_graph and (comm is None or comm.world == 1) and self.M is not None

    # one launch sequence; r64 / z64 are f64 device vectors of the local slab
    def _sequence(self, r64, z64):
        d, L, lib = self.d, self.d.L, self.d.lib
        st = d.st()
        inv = None if self.inv is None else self.inv.data_ptr()
        lib.psell_ipcg_begin(self.n, r64.data_ptr(), self.x.data_ptr(), self.r.data_ptr(), self.z.data_ptr(),
                             self.p.data_ptr(), inv, d.p(d.partials), d.p(d.loc, 0), st)
        g, stride = d.gather()
        lib.psell_ipcg_set_rz(d.p(g, 0), d.G, stride, d.p(d.scal), d.p(d.flags), st)
        desc = self.M.desc() if self.M is not None else None
        err = L.PsellError()
        for _ in range(self.m_in):
            if d.G > 1:
                self.comm.all_gather_vec(self.p_full, self.p)
            if self.M is not None:
                rc = lib.psell_spmv_dot(desc, L.ptr(self.M.d_pack), L.ptr(self.M.d_offset), L.ptr(self.M.d_perm),
                                        self.p_full.data_ptr(), self.q.data_ptr(), self.p.data_ptr(),
                                        d.p(d.partials), d.p(d.flags), st, err)
                L.check(rc, err, self.M.fmt)
                lib.psell_sum_partials(d.p(d.partials), lib.psell_spmv_dot_partials(desc), 1, d.p(d.loc, 1),
                                       d.p(d.flags), st)
            else:
                self.q.copy_(self.backend.apply(self.p_full))
                lib.psell_dot(self.p.data_ptr(), self.q.data_ptr(), 1, self.n, d.p(d.partials), d.p(d.loc, 1), st)
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
        torch = self.torch
        if self.use_graph:
            if self.graph is None or self.graph_in is not (r64, z64):
                self._r_static, self._z_static = r64, z64
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
        done = int(self.d.flags[1].item())
        if int(self.d.flags[0].item()):
            log.warning("inner PCG breakdown at iteration %d (p'Ap=%r); returning current iterate",
                        done, float(self.d.scal[1].item()))
        return done


# ----------------------------------------------------------------------------
# f64 drivers
# ----------------------------------------------------------------------------

class _Op64:
    """f64 operator on device vectors (local slab rows, global x)."""

    def __init__(self, backend: SpmvBackend, comm=None):
        self.backend = backend
        self.comm = comm
        src = backend.matrix
        self.n = src.n_rows
        self.n_glob = src.n_cols
        self.row0 = getattr(src, "row0", 0)

    def __call__(self, p_full, out):
        out.copy_(self.backend.apply(p_full))
        return out


def _prep(b, comm):
    import torch
    from . import _dev
    b = np.asarray(b, dtype=np.float64)
    return b, _dev.upload(b)


def _vec_norm(d: _Dev, a) -> float:
    d.lib.psell_dot(a.data_ptr(), a.data_ptr(), 2, a.numel(), d.p(d.partials), d.p(d.loc, 0), d.st())
    g, _ = d.gather()
    if d.G == 1:
        return float(np.sqrt(float(d.loc[0].item())))
    return float(np.sqrt(float(d.glob[:, 0].cpu().numpy().sum())))


def _audit(report: SolveReport, src, b_dev, bnorm, tol, d: _Dev, x_full) -> SolveReport:
    """True residual in f64 on the device, demote drifted runs (solvers.py:152-168)."""
    import torch
    if bnorm == 0.0:
        report.final_true_relres = 0.0
        return report
    ax = csr_spmv(src, x_full, np.float64)
    d.lib.psell_resid(b_dev.numel(), b_dev.data_ptr(), ax.data_ptr(), d.p(d.partials), d.p(d.loc, 0), d.st())
    d.gather()
    rr = float(d.loc[0].item()) if d.G == 1 else float(d.glob[:, 0].cpu().numpy().sum())
    report.final_true_relres = float(np.sqrt(rr)) / bnorm
    if report.converged and not report.final_true_relres < 10.0 * tol:
        report.converged = False
        msg = f"true residual {report.final_true_relres:.3e} exceeds 10x tolerance"
        report.reason = f"{report.reason}; {msg}" if report.reason else msg
    return report


def _jacobi_inv(backend: SpmvBackend, dtype):
    """1/diag of the f64 source, rounded to dtype (solvers.py:145-149)."""
    from . import _dev
    src = backend.source
    if isinstance(src, DeviceCsrMatrix):
        src = src.to_host()
    diag = src.diagonal()
    if np.any(diag == 0.0):
        raise ValueError("jacobi preconditioner requires a fully nonzero diagonal")
    return _dev.upload((1.0 / diag).astype(dtype))


def pcg(A, b, cfg: SolveConfig = None, x0=None) -> SolveReport:
    """f64 PCG stopping on the recurred residual (solvers.py:171-217), on the GPU."""
    import torch
    from . import _lib
    cfg = cfg or SolveConfig()
    backend = _as_backend(A)
    b, bd = _prep(b, None)
    t0 = time.perf_counter()
    n = len(b)
    d = _Dev(_lib.RED_BLOCKS)
    lib = d.lib
    st = d.st()
    f64 = torch.float64
    x = torch.zeros(n, dtype=f64, device="cuda") if x0 is None else \
        torch.as_tensor(np.asarray(x0, dtype=np.float64)).cuda()
    inv = _jacobi_inv(backend, np.float64) if cfg.preconditioner == "jacobi" else None
    bnorm = _vec_norm(d, bd)
    if bnorm == 0.0:
        return SolveReport(True, 0, 0, [], 0.0, time.perf_counter() - t0, x=x.cpu().numpy())
    r = bd.clone()
    if x0 is not None and np.any(np.asarray(x0)):
        ax = backend.apply(x)
        r.copy_(ax)
        neg1 = torch.tensor([-1.0], dtype=f64, device="cuda")
        lib.psell_xpby(n, r.data_ptr(), bd.data_ptr(), neg1.data_ptr(), st)   # r = b - Ax
    history = [_vec_norm(d, r) / bnorm]
    z = torch.empty_like(r) if inv is not None else r
    lib.psell_precond_dot(n, z.data_ptr(), r.data_ptr(), None if inv is None else inv.data_ptr(),
                          d.p(d.partials), d.p(d.scal, 4), st)               # scal[4] = rz
    p = z.clone()
    q = torch.empty_like(r)
    converged, reason, it = False, None, 0
    while it < cfg.max_outer:
        if history[-1] < cfg.tol:
            converged = True
            break
        q.copy_(backend.apply(p))
        lib.psell_pq_pr(n, p.data_ptr(), q.data_ptr(), None, d.p(d.partials), d.p(d.loc, 0), st)
        d.flags.zero_()
        # alpha = rz / pq with the curvature test -> scal[0], scal[1] = pq
        lib.psell_scalar_div(d.p(d.scal, 4), d.p(d.loc, 0), 1, 1, d.p(d.scal, 0), d.p(d.flags), 1, st)
        lib.psell_axpy2(n, x.data_ptr(), r.data_ptr(), p.data_ptr(), q.data_ptr(), d.p(d.scal, 0),
                        d.p(d.flags), d.p(d.partials), d.p(d.loc, 2), st)
        status = torch.stack([d.flags[0].to(f64), d.loc[0], d.loc[2]]).cpu().numpy()
        if status[0]:
            reason = f"breakdown: non-positive curvature p'Ap = {float(status[1])!r} at iteration {it}"
            break
        it += 1
        history.append(float(np.sqrt(status[2])) / bnorm)
        lib.psell_precond_dot(n, z.data_ptr(), r.data_ptr(), None if inv is None else inv.data_ptr(),
                              d.p(d.partials), d.p(d.loc, 3), st)            # rz_new
        lib.psell_scalar_div(d.p(d.loc, 3), d.p(d.scal, 4), 1, 1, d.p(d.scal, 2), None, 0, st)  # beta
        d.scal[4].copy_(d.loc[3])
        lib.psell_xpby(n, p.data_ptr(), z.data_ptr(), d.p(d.scal, 2), st)
    else:
        reason = f"maximum iterations ({cfg.max_outer}) reached"
    if not converged and history[-1] < cfg.tol:
        converged = True
        reason = None
    torch.cuda.synchronize()
    report = SolveReport(converged, it, 0, history, 0.0, time.perf_counter() - t0, reason)
    report = _audit(report, backend.source, bd, bnorm, cfg.tol, d, x)
    report.x = x.cpu().numpy()
    return report


def fcg(A, b, cfg: SolveConfig = None, inner_preconditioner: Callable = None, *, _inner=None) -> SolveReport:
    """Truncated flexible CG in f64 (solvers.py:220-275), on the GPU.

    `inner_preconditioner` may be a Python callable on numpy vectors (the
    reference contract; runs through host copies) — the iocg path passes a
    device `_InnerPCG` via `_inner` instead.
    """
    import torch
    from . import _lib
    cfg = cfg or SolveConfig()
    backend = _as_backend(A)
    b, bd = _prep(b, None)
    t0 = time.perf_counter()
    n = len(b)
    d = _Dev(_lib.RED_BLOCKS)
    lib = d.lib
    st = d.st()
    f64 = torch.float64
    x = torch.zeros(n, dtype=f64, device="cuda")
    bnorm = _vec_norm(d, bd)
    if bnorm == 0.0:
        return SolveReport(True, 0, 0, [], 0.0, time.perf_counter() - t0, x=x.cpu().numpy())
    inv = None
    if _inner is None and inner_preconditioner is None and cfg.preconditioner == "jacobi":
        inv = _jacobi_inv(backend, np.float64)
    r = bd.clone()
    history = [_vec_norm(d, r) / bnorm]
    z = torch.empty_like(r)
    p = torch.empty_like(r)
    q = torch.empty_like(r)
    r_prev = torch.empty_like(r)
    converged, reason, it, first = False, None, 0, True
    inner_total = 0
    while it < cfg.max_outer:
        if history[-1] < cfg.tol:
            converged = True
            break
        if _inner is not None:
            inner_total += _inner.solve(r, z)
        elif inner_preconditioner is not None:
            z.copy_(torch.as_tensor(np.asarray(inner_preconditioner(r.cpu().numpy()), dtype=np.float64)))
        else:
            lib.psell_precond_dot(n, z.data_ptr(), r.data_ptr(), None if inv is None else inv.data_ptr(),
                                  d.p(d.partials), d.p(d.loc, 7), st)
            if inv is None:
                z.copy_(r)
        lib.psell_fcg_zr(n, z.data_ptr(), r.data_ptr(), None if first else r_prev.data_ptr(),
                         d.p(d.partials), d.p(d.loc, 0), st)                 # loc0 = z.(r - r_prev), loc1 = z.r
        if first:
            lib.psell_xpby(n, p.data_ptr(), z.data_ptr(), None, st)
            first = False
        else:
            lib.psell_scalar_div(d.p(d.loc, 0), d.p(d.scal, 6), 1, 1, d.p(d.scal, 2), None, 0, st)  # beta
            lib.psell_xpby(n, p.data_ptr(), z.data_ptr(), d.p(d.scal, 2), st)
        d.scal[6].copy_(d.loc[1])                                            # zr_prev
        r_prev.copy_(r)
        q.copy_(backend.apply(p))
        lib.psell_pq_pr(n, p.data_ptr(), q.data_ptr(), r.data_ptr(), d.p(d.partials), d.p(d.loc, 2), st)
        d.flags.zero_()
        lib.psell_scalar_div(d.p(d.loc, 3), d.p(d.loc, 2), 1, 1, d.p(d.scal, 0), d.p(d.flags), 1, st)  # alpha
        lib.psell_axpy2(n, x.data_ptr(), r.data_ptr(), p.data_ptr(), q.data_ptr(), d.p(d.scal, 0),
                        d.p(d.flags), d.p(d.partials), d.p(d.loc, 4), st)
        status = torch.stack([d.flags[0].to(f64), d.loc[2], d.loc[4]]).cpu().numpy()
        if status[0]:
            reason = f"breakdown: non-positive curvature p'Ap = {float(status[1])!r} at iteration {it}"
            break
        it += 1
        history.append(float(np.sqrt(status[2])) / bnorm)
    else:
        reason = f"maximum iterations ({cfg.max_outer}) reached"
    if not converged and history[-1] < cfg.tol:
        converged = True
        reason = None
    torch.cuda.synchronize()
    report = SolveReport(converged, it, inner_total, history, 0.0, time.perf_counter() - t0, reason)
    report = _audit(report, backend.source, bd, bnorm, cfg.tol, d, x)
    report.x = x.cpu().numpy()
    return report


def iocg(A: CsrMatrix, b, cfg: SolveConfig = None, *, backend: SpmvBackend = None) -> SolveReport:
    """Inner-outer CG (solvers.py:311-333): m_in f32 PackSELL PCG steps precondition f64 FCG.

    `backend` may pass a prebuilt inner backend (e.g. to exclude the build
    from a timing); by default it is built from cfg.a_backend like the reference.
    """
    cfg = cfg or SolveConfig(solver="iocg")
    if not isinstance(A, (CsrMatrix, DeviceCsrMatrix)):
        raise TypeError("iocg drives the outer iteration with the float64 CSR matrix")
    inner_backend = backend or make_backend(A, cfg.a_backend)
    dtype = _PRECISIONS[cfg.inner_precision]
    inv = _jacobi_inv(inner_backend, dtype) if cfg.preconditioner == "jacobi" else None
    if dtype == np.float32 and inner_backend.is_packsell:
        inner = _InnerPCG(inner_backend, cfg.m_in, inv)
        return fcg(A, b, cfg, _inner=inner)
    # generic inner backend / precision: reference-shaped inner loop through the device backend
    inner = _GenericInner(inner_backend, cfg.m_in, dtype, inv)
    return fcg(A, b, cfg, _inner=inner)


class _GenericInner:
    """Inner PCG for non-PackSELL backends or f64 inner precision (device vectors, host scalars)."""

    def __init__(self, backend, m_in, dtype, inv):
        import torch
        from . import _dev, _lib
        self.torch = torch
        self.backend = backend
        self.m_in = m_in
        self.tdt = _dev.torch_dtype(dtype)
        self.dt_code = _dev.T_DT_CODE[self.tdt]
        self.inv = inv
        self.d = _Dev(_lib.RED_BLOCKS)

    def _dot(self, a, b) -> float:
        d = self.d
        d.lib.psell_dot(a.data_ptr(), b.data_ptr(), self.dt_code, a.numel(), d.p(d.partials), d.p(d.loc, 0), d.st())
        return float(d.loc[0].item())

    def solve(self, r64, z64) -> int:
        torch = self.torch
        rhs = r64.to(self.tdt)
        x = torch.zeros_like(rhs)
        r = rhs.clone()
        P = (lambda v: v) if self.inv is None else (lambda v: v * self.inv)
        z = P(r)
        p = z.clone()
        rz = self._dot(r, z)
        done = 0
        for _ in range(self.m_in):
            q = self.backend.apply(p)
            pq = self._dot(p, q)
            if pq <= 0.0 or not np.isfinite(pq) or rz == 0.0:
                log.warning("inner PCG breakdown at iteration %d (p'Ap=%r); returning current iterate", done, pq)
                break
            a = torch.tensor(rz / pq, dtype=self.tdt, device="cuda")
            x.add_(a * p)
            r.sub_(a * q)
            done += 1
            z = P(r)
            rzn = self._dot(r, z)
            beta = torch.tensor(rzn / rz, dtype=self.tdt, device="cuda")
            rz = rzn
            p = z + beta * p
        z64.copy_(x.to(torch.float64))
        return done
