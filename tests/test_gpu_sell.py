"""SELL-C-sigma comparator on the GPU vs the reference (sell.py:114-204) and the
acceptance c08 relation: e8m14 IO-CG needs <= 1.25x the FP32-SELL inner iterations."""

import json
import os

import numpy as np
import pytest

import paper_2604_13433_b200 as P
from paper_2604_13433_b200 import solvers as S
from conftest import GOLDEN, golden_x

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def test_sell_layout_and_spmv_bitwise():
    z = np.load(os.path.join(GOLDEN, "sell_golden.npz"))
    with open(os.path.join(GOLDEN, "sell_golden.json")) as f:
        meta = json.load(f)
    for i, m in enumerate(meta):
        p = f"s{i}_"
        A = P.CsrMatrix(m["n_rows"], m["n_cols"], z[p + "row_ptr"], z[p + "col_idx"], z[p + "values"])
        M = P.build_sell(A, m["c"], m["sigma"], m["mode"], np.dtype(m["vdt"]))
        assert np.array_equal(_bits(M.val), _bits(z[p + "val"])), i
        assert np.array_equal(M.col, z[p + "col"]), i
        assert np.array_equal(M.offset, z[p + "offset"]), i
        assert M.n_padding == m["n_padding"], i
        if m["has_perm"]:
            assert np.array_equal(M.perm, z[p + "perm"]), i
        else:
            assert M.perm is None
        for dt in (np.float16, np.float32, np.float64):
            y = P.sell_spmv(M, golden_x(5000 + i, m["n_cols"], dt))
            want = z[p + f"y_{np.dtype(dt).name}"]
            assert y.dtype == want.dtype and np.array_equal(_bits(y), _bits(want)), (i, dt)


def test_iocg_sell32_and_acceptance_ordering(golden_solver):
    z, meta = golden_solver
    A = P.sym_diag_scale(P.poisson3d(10))
    b = z["b"]
    cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=20, a_backend="sell32", max_outer=200)
    r = S.iocg(A, b, cfg)
    ref = meta["iocg_sell32"]
    assert r.converged and abs(r.outer_iters - ref["outer"]) <= 1
    assert np.abs(r.x - z["iocg_sell32_x"]).max() / np.abs(z["iocg_sell32_x"]).max() < 1e-6
    r14 = S.iocg(A, b, S.SolveConfig(solver="iocg", tol=1e-9, m_in=20, a_backend="packsell-e8m14", max_outer=200))
    assert r14.converged and r14.total_inner_iters <= 1.25 * r.total_inner_iters


def test_make_backend_all_names():
    A = P.sym_diag_scale(P.poisson3d(6))
    x = np.random.default_rng(0).uniform(-1, 1, A.n_cols)
    want = P.csr_spmv(A, x, np.float64)
    for name in ("csr64", "sell64", "sell32", "sell16", "packsell-fp16", "packsell-e8m14", "packsell-fp32embed"):
        be = S.make_backend(A, name)
        y = be.apply(x)
        assert y.dtype == np.float64 and np.abs(y - want).max() < 1e-2, name


def test_sell32_c32_kernel_large_vs_row_sequential():
    """The C = 32 chunked SELL kernel at a multi-wave size, ragged and empty rows,
    sigma sorting: y equals the row-sequential CSR sum in f32 (padding adds +0 * x,
    which leaves a non-zero finite sum unchanged)."""
    import oracle as O
    rng = np.random.default_rng(12)
    n = 300_000
    lens = rng.integers(0, 20, n)
    lens[rng.integers(0, n, 100)] = 200
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.sort(rng.integers(0, n, int(rp[-1])).astype(np.int32))
    A = P.CsrMatrix(n, n, rp, ci, rng.standard_normal(int(rp[-1])))
    x = rng.standard_normal(n).astype(np.float32)
    want = O.csr_spmv(rp, ci, A.values, x, np.float32)
    for mode, sigma in (("implicit", 256), ("explicit", 4096), ("none", 1)):
        M = P.build_sell(A, 32, sigma, mode, np.dtype(np.float32))
        y = P.sell_spmv(M, x)
        w = want[O.sort_order(lens, sigma)] if mode == "explicit" else want  # explicit: storage order
        nz = w != 0
        assert np.array_equal(_bits(y[nz]), _bits(w[nz])), mode
        assert np.all(y[~nz] == 0), mode


@pytest.mark.parametrize("mode,sigma", [("implicit", 256), ("implicit", 4096), ("explicit", 1024), ("none", 1)])
def test_sell_spmv_dot_alpha_fused(mode, sigma):
    """psell_sell_spmv_dot_alpha (the FP32 IO-CG comparator's inner operator): y bitwise equal
    to psell_sell_spmv, p.y equal to the FP64 sum of the f32 products (exact in f64) up to
    summation order, alpha = rz / pq in scal[2], the tickets re-armed for the next launch."""
    import torch
    from paper_2604_13433_b200 import _lib, _dev
    rng = np.random.default_rng(21)
    n = 200_003
    lens = rng.integers(0, 14, n)
    lens[rng.integers(0, n, 50)] = 150
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.sort(rng.integers(0, n, int(rp[-1])).astype(np.int32))
    A = P.CsrMatrix(n, n, rp, ci, rng.standard_normal(int(rp[-1])))
    M = P.build_sell(A, 32, sigma, mode, np.dtype(np.float32))
    lib = _lib.lib()
    p = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).cuda()
    want = P.sell_spmv(M, p)
    n_part = int(lib.psell_sell_spmv_dot_partials(M.desc()))
    parts = torch.zeros(n_part + n_part // 32 + 8, dtype=torch.float64, device="cuda")
    ticket = torch.zeros(2 + n_part // 32, dtype=torch.int32, device="cuda")
    y = torch.empty_like(p)
    for rep in range(3):
        scal = torch.zeros(32, dtype=torch.float64, device="cuda")
        scal[0] = 3.0 + rep
        flags = torch.zeros(4, dtype=torch.int32, device="cuda")
        err = _lib.PsellError()
        rc = lib.psell_sell_spmv_dot_alpha(M.desc(), _lib.ptr(M.d_val), _dev.DT_CODE[M.value_dtype],
                                           _lib.ptr(M.d_col), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                                           p.data_ptr(), y.data_ptr(), p.data_ptr(), parts.data_ptr(),
                                           scal.data_ptr(), flags.data_ptr(), ticket.data_ptr(),
                                           _lib.stream_handle(), err)
        _lib.check(rc, err)
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int32), want.view(torch.int32)), (mode, rep)
        pq = float((p.double() * y.double()).sum())
        assert abs(float(scal[1]) - pq) <= 1e-12 * float((p.double() * y.double()).abs().sum())
        assert int(flags[0]) == (1 if pq <= 0 else 0)
        if pq > 0:
            assert float(scal[2]) == (3.0 + rep) / float(scal[1])
        assert int(ticket.abs().sum()) == 0


def test_iocg_sell32_fused_matches_unfused(monkeypatch):
    """The fused comparator inner loop and the three-launch one agree to summation order."""
    A = P.sym_diag_scale(P.poisson3d(24))
    b, _ = S.make_rhs_and_x0(A.n_rows, 9)
    cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=30, a_backend="sell32", max_outer=200)
    r1 = S.iocg(A, b, cfg)
    monkeypatch.setenv("PSELL_SELL_FUSED", "0")
    r0 = S.iocg(A, b, cfg)
    assert r1.converged and r0.converged and abs(r1.outer_iters - r0.outer_iters) <= 1
    assert np.abs(r1.x - r0.x).max() <= 1e-7 * np.abs(r0.x).max()


def test_iocg_sell32_fused_stopping_rules_vs_oracle():
    """The fused FP32 SELL comparator inside IO-CG (outer look-ahead, gated inner graph)
    stops where the oracle's IO-CG with an f32 row-sequential SELL inner operator does."""
    import oracle as O
    A = P.sym_diag_scale(P.poisson3d(8))
    b, _ = S.make_rhs_and_x0(A.n_rows, 4)
    a64 = lambda v: O.csr_spmv(A.row_ptr, A.col_idx, A.values, v, np.float64)  # noqa: E731
    v32 = A.values.astype(np.float32).astype(np.float64)
    inner = lambda v: O.csr_spmv(A.row_ptr, A.col_idx, v32, v, np.float32)  # noqa: E731
    full = O.iocg(a64, inner, b, 1e-9, 200, 10)
    be = S.make_backend(A, "sell32")
    for max_outer in (1, 2, full["outer_iters"] - 1, full["outer_iters"], 200):
        cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=10, a_backend="sell32", max_outer=max_outer)
        r = S.iocg(A, b, cfg, backend=be)
        ro = O.iocg(a64, inner, b, 1e-9, max_outer, 10)
        assert (r.converged, r.outer_iters, r.total_inner_iters) == \
            (ro["converged"], ro["outer_iters"], ro["total_inner_iters"]), max_outer
        assert np.abs(r.x - ro["x"]).max() <= 1e-6 * np.abs(ro["x"]).max()
    assert next(iter(be._inner_cache.values())).sell_fused
