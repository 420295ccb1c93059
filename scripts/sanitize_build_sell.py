"""Small runs of the builder's folded k_left pass, the 8-bit-digit sorts (sigma 256 in shared
memory, sigma 4096 and 65536 in global scratch) and the
fused FP32 SELL comparator kernel, for compute-sanitizer (sigma 1024: the 1024-thread kernel with keys in shared memory, 4-bit digits); each checked against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import solvers as S  # noqa: E402

rng = np.random.default_rng(5)
n = 70_000
lens = rng.integers(0, 30, n)
lens[rng.integers(0, n, 40)] = rng.integers(65, 3000, 40)  # long rows (warp-per-row kernels)
rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
ci = np.concatenate([np.sort(rng.choice(n, int(k), replace=False)) for k in lens]).astype(np.int32)
A = P.CsrMatrix(n, n, rp, ci, rng.standard_normal(int(rp[-1])))
for sigma in (256, 1024, 4096, 65536):
    for name in ("fp16", "e8m10"):
        M = P.build_packsell(A, 32, sigma, P.parse_format(name), "implicit")
        OM = O.build(rp, ci, A.values, n, 32, sigma, O.preset(name), "implicit")
        assert np.array_equal(M.pack, OM.pack) and np.array_equal(M.offset, OM.offset), (sigma, name)
        assert np.array_equal(M.perm, OM.perm) and M.k_left == OM.k_left, (sigma, name)
B = P.sym_diag_scale(P.poisson3d(12))
b, _ = S.make_rhs_and_x0(B.n_rows, 2)
r = S.iocg(B, b, S.SolveConfig(solver="iocg", tol=1e-8, m_in=10, a_backend="sell32", max_outer=100))
assert r.converged
print("sanitize_build_sell ok")
