"""GPU solver parity: pcg / fcg / iocg on the device vs the reference fixtures.

Tolerance: same convergence flag, |outer - ref| <= 1,
total inner = m_in * outer, true relres < tol, ||x - x_ref||_inf / ||x_ref||_inf <= 1e-6.
Residual histories differ from the reference only through the FP64 reduction
order (device tree vs numpy pairwise), so they are compared to 1e-6 relative.
"""

import numpy as np
import pytest

import paper_2604_13433_b200 as P
from paper_2604_13433_b200 import solvers as S

pytestmark = pytest.mark.gpu


def _problem(nx=10, seed=42):
    A = P.sym_diag_scale(P.poisson3d(nx))
    b, _ = S.make_rhs_and_x0(A.n_rows, seed)
    return A, b


def _close(x, xr, tol=1e-6):
    return np.abs(x - xr).max() / np.abs(xr).max() <= tol


@pytest.mark.parametrize("backend", ["packsell-e8m14", "packsell-fp16"])
def test_iocg_matches_reference(golden_solver, backend):
    z, meta = golden_solver
    A, b = _problem()
    assert np.array_equal(b, z["b"])
    m = meta[f"iocg_{backend}"]
    cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=m["m_in"], a_backend=backend, max_outer=200)
    r = S.iocg(A, b, cfg)
    assert r.converged == m["converged"]
    assert abs(r.outer_iters - m["outer"]) <= 1
    assert r.total_inner_iters == m["m_in"] * r.outer_iters
    assert r.final_true_relres < 1e-9
    assert _close(r.x, z[f"iocg_{backend}_x"])
    # the inner SpMV is FP32-FMA (the reference rounds product and sum separately), so the
    # preconditioner differs at ~1e-7 and CG amplifies it: compare histories in log space
    h = np.array(r.residual_history)
    hr = z[f"iocg_{backend}_hist"]
    n = min(len(h), len(hr))
    assert h[0] == hr[0]
    assert np.all(np.abs(np.log10(h[1:n] / hr[1:n])) < 0.5)


def test_pcg_f64_matches_reference(golden_solver):
    z, meta = golden_solver
    A, b = _problem()
    r = S.pcg(A, b, S.SolveConfig(tol=1e-9, max_outer=1000))
    assert r.converged and abs(r.outer_iters - meta["pcg"]["outer"]) <= 1
    assert _close(r.x, z["pcg_x"], 1e-9)
    n = min(len(r.residual_history), len(z["pcg_hist"]))
    assert np.allclose(r.residual_history[:n], z["pcg_hist"][:n], rtol=1e-9)


def test_iocg_csr64_inner_generic(golden_solver):
    z, meta = golden_solver
    A, b = _problem()
    m = meta["iocg_csr64"]
    r = S.iocg(A, b, S.SolveConfig(solver="iocg", tol=1e-9, m_in=m["m_in"], a_backend="csr64", max_outer=200))
    assert r.converged and abs(r.outer_iters - m["outer"]) <= 1
    assert _close(r.x, z["iocg_csr64_x"])


def test_iocg_deterministic():
    A, b = _problem(12, 7)
    cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=20, a_backend="packsell-e8m14", max_outer=200)
    r1 = S.iocg(A, b, cfg)
    r2 = S.iocg(A, b, cfg)
    assert r1.residual_history == r2.residual_history
    assert np.array_equal(r1.x, r2.x)
    assert r1.converged


def test_inner_graph_equals_eager():
    A, b = _problem(12, 3)
    be = S.make_backend(A, "packsell-e8m14")
    import torch
    r = torch.as_tensor(b).cuda()
    za = torch.empty_like(r)
    zb = torch.empty_like(r)
    ia = S._InnerPCG(be, 15, use_graph=True)
    ib = S._InnerPCG(be, 15, use_graph=False)
    assert ia.solve(r, za) == ib.solve(r, zb) == 15
    assert torch.equal(za, zb)
    assert ia.solve(r, za) == 15  # graph replay
    assert torch.equal(za, zb)


def test_inner_pcg_vs_oracle_f32():
    """The fused inner loop follows the reference recurrence (f32 vectors, f64 dots)."""
    import oracle as O
    import torch
    A, b = _problem(10, 5)
    be = S.make_backend(A, "packsell-e8m14")
    OM = O.build(A.row_ptr, A.col_idx, A.values, A.n_cols, 32, 256, O.preset("e8m14"), "implicit")
    zr, done = O.inner_pcg(lambda v: O.spmv(OM, v), b, 20, np.float32)
    inner = S._InnerPCG(be, 20)
    z = torch.empty(A.n_rows, dtype=torch.float64, device="cuda")
    k = inner.solve(torch.as_tensor(b).cuda(), z)
    assert k == done == 20
    zz = z.cpu().numpy()
    assert np.abs(zz - zr).max() / np.abs(zr).max() < 1e-4


def test_breakdown_and_zero_rhs():
    A = P.to_csr(P.CooMatrix(3, 3, [0, 1, 2], [0, 1, 2], [1.0, -1.0, 1.0]))
    r = S.pcg(A, np.array([1.0, 1.0, 1.0]), S.SolveConfig(tol=1e-12, max_outer=10))
    assert not r.converged and r.reason.startswith("breakdown")
    r0 = S.pcg(A, np.zeros(3))
    assert r0.converged and r0.outer_iters == 0


def test_jacobi_preconditioner():
    A = P.poisson3d(8)
    b, _ = S.make_rhs_and_x0(A.n_rows, 1)
    r = S.pcg(A, b, S.SolveConfig(tol=1e-10, preconditioner="jacobi"))
    assert r.converged and r.final_true_relres < 1e-9
    ri = S.iocg(A, b, S.SolveConfig(solver="iocg", tol=1e-9, m_in=20, a_backend="packsell-e8m14",
                                    preconditioner="jacobi"))
    assert ri.converged


def test_iocg_sell32_inner_matches_reference(golden_solver):
    """The FP32 IO-CG comparator (SELL-C-sigma f32 inner) on the device kernels."""
    z, meta = golden_solver
    A, b = _problem()
    m = meta["iocg_sell32"]
    r = S.iocg(A, b, S.SolveConfig(solver="iocg", tol=1e-9, m_in=m["m_in"], a_backend="sell32", max_outer=200))
    assert r.converged == m["converged"] and abs(r.outer_iters - m["outer"]) <= 1
    assert r.total_inner_iters == m["m_in"] * r.outer_iters
    assert _close(r.x, z["iocg_sell32_x"])


@pytest.mark.parametrize("backend", ["packsell-e8m14", "sell64", "csr64"])
def test_iocg_real64_inner_vs_oracle(backend):
    """inner_precision="real64": f64 inner PCG kernels vs the oracle's f64 IO-CG."""
    import oracle as O
    A, b = _problem(8, 3)
    cfg = S.SolveConfig(solver="iocg", tol=1e-10, m_in=10, a_backend=backend, inner_precision="real64",
                        max_outer=200)
    r = S.iocg(A, b, cfg)
    if backend.startswith("packsell"):
        OM = O.build(A.row_ptr, A.col_idx, A.values, A.n_cols, 32, 256, O.preset("e8m14"), "implicit")
        inner_apply = lambda v: O.spmv(OM, v)  # noqa: E731
    else:
        inner_apply = lambda v: O.csr_spmv(A.row_ptr, A.col_idx, A.values, v, np.float64)  # noqa: E731
    ro = O.iocg(lambda v: O.csr_spmv(A.row_ptr, A.col_idx, A.values, v, np.float64), inner_apply, b,
                1e-10, 200, 10, np.float64)
    assert r.converged and ro["converged"]
    assert abs(r.outer_iters - ro["outer_iters"]) <= 1
    assert r.total_inner_iters == 10 * r.outer_iters
    assert _close(r.x, ro["x"], 1e-8)


def test_iocg_and_pcg_64cubed_vs_reference():
    """Config-5 protocol at 64^3 (e8m14 inner, m_in 50) against the real reference's solve."""
    import json
    import os
    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, "solver64_golden.npz"))
    with open(os.path.join(GOLDEN, "solver64_golden.json")) as f:
        meta = json.load(f)
    A = P.sym_diag_scale(P.poisson3d(64))
    b, _ = S.make_rhs_and_x0(A.n_rows, 42)
    r = S.iocg(A, b, S.SolveConfig(solver="iocg", tol=1e-9, m_in=50, a_backend="packsell-e8m14", max_outer=400))
    m = meta["iocg"]
    assert r.converged == m["converged"] and abs(r.outer_iters - m["outer"]) <= 1
    assert r.total_inner_iters == 50 * r.outer_iters and r.final_true_relres < 1e-9
    assert _close(r.x, z["iocg_x"])
    p = S.pcg(A, b, S.SolveConfig(tol=1e-9, max_outer=2000))
    assert p.converged and abs(p.outer_iters - meta["pcg"]["outer"]) <= 1
    assert _close(p.x, z["pcg_x"], 1e-9)


def test_pcg_stopping_rules_vs_oracle():
    """The look-ahead PCG loop stops exactly where the one-at-a-time loop does:
    iteration caps 0 / 1 / 2 / 7, convergence on the last allowed iteration, the
    initial-residual check, and a breakdown a few iterations in (indefinite A)."""
    import oracle as O
    A = P.sym_diag_scale(P.poisson3d(6))
    b, _ = S.make_rhs_and_x0(A.n_rows, 3)
    a64 = lambda v: O.csr_spmv(A.row_ptr, A.col_idx, A.values, v, np.float64)  # noqa: E731
    full = O.pcg(a64, b, 1e-8, 1000)
    cases = [(0, 1e-8), (1, 1e-8), (2, 1e-8), (7, 1e-8), (full["outer_iters"], 1e-8),
             (full["outer_iters"] - 1, 1e-8), (50, 10.0)]
    for max_outer, tol in cases:
        r = S.pcg(A, b, S.SolveConfig(tol=tol, max_outer=max_outer))
        ro = O.pcg(a64, b, tol, max_outer)
        assert (r.converged, r.outer_iters) == (ro["converged"], ro["outer_iters"]), (max_outer, tol)
        assert len(r.residual_history) == len(ro["history"])
        assert np.allclose(r.residual_history, ro["history"], rtol=1e-10, atol=0), (max_outer, tol)
        assert np.abs(r.x - ro["x"]).max() <= 1e-10 * max(1.0, np.abs(ro["x"]).max())
    # indefinite: diagonal with mixed signs breaks down after a few steps
    n = 40
    d = np.concatenate([np.linspace(1, 2, n - 3), [-1.0, -2.0, -3.0]])
    Ai = P.to_csr(P.CooMatrix(n, n, np.arange(n), np.arange(n), d))
    bi = np.ones(n)
    ri = S.pcg(Ai, bi, S.SolveConfig(tol=1e-14, max_outer=100))
    ro = O.pcg(lambda v: d * v, bi, 1e-14, 100)
    assert ro["reason"] == "breakdown" and ri.reason.startswith("breakdown")
    assert ri.outer_iters == ro["outer_iters"] and len(ri.residual_history) == len(ro["history"])


def test_iocg_stopping_rules_vs_oracle():
    """IO-CG with the outer look-ahead stops where the reference loop does: caps 1 / 2 /
    exact / one short, convergence, and counts only the inner iterations of outer
    iterations that ran (the queued, gated one adds none); a direct inner solve after
    an IO-CG solve is not gated."""
    import oracle as O
    import torch
    A = P.sym_diag_scale(P.poisson3d(8))
    b, _ = S.make_rhs_and_x0(A.n_rows, 4)
    a64 = lambda v: O.csr_spmv(A.row_ptr, A.col_idx, A.values, v, np.float64)  # noqa: E731
    OM = O.build(A.row_ptr, A.col_idx, A.values, A.n_cols, 32, 256, O.preset("e8m14"), "implicit")
    inner = lambda v: O.spmv(OM, v)  # noqa: E731
    full = O.iocg(a64, inner, b, 1e-9, 200, 10)
    be = S.make_backend(A, "packsell-e8m14")
    for max_outer in (1, 2, full["outer_iters"] - 1, full["outer_iters"], 200):
        cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=10, a_backend="packsell-e8m14", max_outer=max_outer)
        r = S.iocg(A, b, cfg, backend=be)
        ro = O.iocg(a64, inner, b, 1e-9, max_outer, 10)
        assert (r.converged, r.outer_iters, r.total_inner_iters) == \
            (ro["converged"], ro["outer_iters"], ro["total_inner_iters"]), max_outer
        assert len(r.residual_history) == len(ro["history"])
        assert np.abs(r.x - ro["x"]).max() <= 1e-6 * np.abs(ro["x"]).max()
    inner_solver = next(iter(be._inner_cache.values()))
    z = torch.empty(A.n_rows, dtype=torch.float64, device="cuda")
    assert inner_solver.solve(torch.as_tensor(b).cuda(), z) == 10


@pytest.mark.parametrize("nx,tol,max_outer", [(24, 1e-9, 2000), (6, 1e-8, 7), (6, 10.0, 50)])
def test_pcg_fused_iteration_matches_unfused(monkeypatch, nx, tol, max_outer):
    """The fused FP64 PCG iteration (SpMV + p.q + alpha, update + r.r + status + beta,
    direction: 3 launches) against the 11-launch sequence: same stopping point and
    iterates up to the association of the two dot reductions."""
    A, b = _problem(nx, 5)
    cfg = S.SolveConfig(tol=tol, max_outer=max_outer)
    monkeypatch.setenv("PSELL_PCG_FUSED", "1")
    rf = S.pcg(A, b, cfg)
    monkeypatch.setenv("PSELL_PCG_FUSED", "0")
    ru = S.pcg(A, b, cfg)
    assert (rf.converged, rf.outer_iters, rf.reason) == (ru.converged, ru.outer_iters, ru.reason)
    assert len(rf.residual_history) == len(ru.residual_history)
    assert np.allclose(rf.residual_history, ru.residual_history, rtol=1e-9, atol=0)
    assert np.abs(rf.x - ru.x).max() <= 1e-10 * max(1.0, np.abs(ru.x).max())
    assert abs(rf.final_true_relres - ru.final_true_relres) <= 1e-6 * ru.final_true_relres + 1e-300
