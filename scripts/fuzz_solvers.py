"""Randomised solver parity (one-off): IO-CG / PCG on random sparse SPD matrices vs the oracle.
usage: fuzz_solvers.py [n_cases] [seed]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import solvers as S  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
fails = 0
for it in range(n_cases):
    n = int(rng.integers(50, 4000))
    k = int(n * rng.uniform(2, 12))
    r, c = rng.integers(0, n, k), rng.integers(0, n, k)
    off = r != c
    r, c = r[off], c[off]
    v = -rng.uniform(0.05, 1.0, len(r))
    rows = np.concatenate([r, c, np.arange(n)])
    cols = np.concatenate([c, r, np.arange(n)])
    dsum = np.zeros(n)
    np.add.at(dsum, r, -v)
    np.add.at(dsum, c, -v)
    vals = np.concatenate([v, v, dsum * rng.uniform(1.0, 1.5) + 1e-3])
    A = P.sym_diag_scale(P.to_csr(P.CooMatrix(n, n, rows, cols, vals)))
    b = S.make_rhs_and_x0(n, it)[0]
    backend = ["packsell-e8m14", "packsell-fp16", "packsell-e8m10", "sell32", "csr64"][it % 5]
    m_in = int(rng.choice([5, 10, 20]))
    try:
        rep = S.iocg(A, b, S.SolveConfig(solver="iocg", tol=1e-9, m_in=m_in, a_backend=backend, max_outer=300))
        a64 = lambda v_: O.csr_spmv(A.row_ptr, A.col_idx, A.values, v_, np.float64)  # noqa: E731
        if backend.startswith("packsell"):
            OM = O.build(A.row_ptr, A.col_idx, A.values, n, 32, 256, O.preset(backend[9:]), "implicit")
            inner = lambda v_: O.spmv(OM, v_)  # noqa: E731
        else:
            inner = lambda v_: O.csr_spmv(A.row_ptr, A.col_idx, A.values, v_, np.float32)  # noqa: E731
        ref = O.iocg(a64, inner, b, 1e-9, 300, m_in)
        assert rep.converged == ref["converged"], "converged"
        assert abs(rep.outer_iters - ref["outer_iters"]) <= 1, f"outer {rep.outer_iters} vs {ref['outer_iters']}"
        assert rep.total_inner_iters == m_in * rep.outer_iters or not rep.converged, "inner count"
        assert np.abs(rep.x - ref["x"]).max() <= 1e-6 * np.abs(ref["x"]).max(), "x"
        p = S.pcg(A, b, S.SolveConfig(tol=1e-9, max_outer=3000))
        pr = O.pcg(a64, b, 1e-9, 3000)
        assert p.converged == pr["converged"] and abs(p.outer_iters - pr["outer_iters"]) <= 1, "pcg"
        assert np.abs(p.x - pr["x"]).max() <= 1e-9 * np.abs(pr["x"]).max(), "pcg x"
    except AssertionError as e:
        fails += 1
        print(f"case {it}: n={n} nnz={A.nnz} {backend} m_in={m_in}: FAIL {e}", flush=True)
print(f"{n_cases} cases, {fails} failures")
sys.exit(1 if fails else 0)
