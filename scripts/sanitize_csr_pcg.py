"""Small runs of the bulk-staged K4 CSR kernel (ragged rows: empty rows, unaligned spans,
blocks longer than one stage, a partial last block) and of the fused FP64 PCG iteration,
for compute-sanitizer; each checked against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import solvers as S  # noqa: E402

rng = np.random.default_rng(11)
for n in (1, 3, 255, 257, 5000):
    lens = rng.integers(0, 12, n)
    lens[rng.integers(0, n, max(1, n // 500))] = rng.integers(0, 2500, max(1, n // 500))
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = rng.integers(0, n, int(rp[-1])).astype(np.int32)
    v = rng.standard_normal(int(rp[-1]))
    A = P.CsrMatrix(n, n, rp, ci, v)
    for dt in (np.float16, np.float32, np.float64):
        x = rng.standard_normal(n).astype(dt)
        y = P.csr_spmv(A, x, dt)
        assert np.array_equal(y.view(np.uint8), O.csr_spmv(rp, ci, v, x, dt).view(np.uint8)), (n, dt)
B = P.sym_diag_scale(P.poisson3d(10))
b, _ = S.make_rhs_and_x0(B.n_rows, 5)
r = S.pcg(B, b, S.SolveConfig(tol=1e-9, max_outer=500))
ro = O.pcg(lambda u: O.csr_spmv(B.row_ptr, B.col_idx, B.values, u, np.float64), b, 1e-9, 500)
assert r.converged and r.outer_iters == ro["outer_iters"]
assert np.abs(r.x - ro["x"]).max() <= 1e-9 * np.abs(ro["x"]).max()
print("sanitize_csr_pcg ok")
