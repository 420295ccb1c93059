"""Small runs of the narrow kernels (register and cp.async.bulk-staged) for compute-sanitizer:
plain SpMV and the fused SpMV + p.q on a 7-point matrix and a ragged narrow one (tail
steps, odd slice count), each checked against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle as O  # noqa: E402
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import _lib  # noqa: E402
from paper_2604_13433_b200 import solvers as S  # noqa: E402

lib = _lib.lib()
rng = np.random.default_rng(5)
lens = rng.integers(3, 11, 20_011)
rows = np.repeat(np.arange(lens.size), lens)
cols = np.clip(rows + rng.integers(-100, 101, rows.size), 0, lens.size - 1)
order = np.lexsort((cols, rows))
r, c = rows[order], cols[order]
keep = np.ones(r.size, bool)
keep[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
r, c = r[keep], c[keep]
v = rng.uniform(0.01, 1, r.size)
rp = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=lens.size))]).astype(np.int64)
for A in (P.sym_diag_scale(P.poisson3d(21)), P.CsrMatrix(lens.size, lens.size, rp, c.astype(np.int32), v)):
    M = P.build_packsell(A, 32, 256, P.parse_format("e8m14"), "implicit")
    OM = O.build(A.row_ptr, A.col_idx, A.values, A.n_cols, 32, 256, O.preset("e8m14"), "implicit")
    x = rng.uniform(-1, 1, A.n_cols).astype(np.float32)
    ref = O.spmv(OM, x)
    for tma in ("0", "1"):
        os.environ["PSELL_NARROW_TMA"] = tma
        lib.psell_reload_env()
        y = P.packsell_spmv(M, x)
        assert np.abs(y - ref).max() < 1e-4, tma
    # fused p.q through the IO-CG inner loop (graph-captured)
    b = np.random.default_rng(1).random(A.n_rows)
    rep = S.iocg(A, b, S.SolveConfig(solver="iocg", tol=1e-6, m_in=10, a_backend="packsell-e8m14", max_outer=3))
    assert rep.outer_iters >= 1
print("sanitize_narrow ok")
