"""Small runs of this round's new kernels for compute-sanitizer: the TMA slot kernel (A/B),
the SM-affine dual kernel (A/B), the far-column generator, psell_max_column and the
segmented path, each checked against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import _lib  # noqa: E402
from paper_2604_13433_b200.stencil import powerlaw_device, powerlaw_far_rows  # noqa: E402

lib = _lib.lib()
A = P.sym_diag_scale(P.poisson3d(24))
M = P.build_packsell(A, 32, 256, P.parse_format("e8m14"), "implicit")
OM = O.build(A.row_ptr, A.col_idx, A.values, A.n_cols, 32, 256, O.preset("e8m14"), "implicit")
x = np.random.default_rng(0).uniform(-1, 1, A.n_cols).astype(np.float32)
ref = O.spmv(OM, x)
for slot in ("0", "1"):
    os.environ["PSELL_SLOT"] = slot
    lib.psell_reload_env()
    y = P.packsell_spmv(M, x)
    assert np.abs(y - ref).max() < 1e-5, slot
F = powerlaw_far_rows(1 << 15, 3)
D = powerlaw_device(1 << 15, 3, far=True).to_host()
assert np.array_equal(D.col_idx, F.col_idx)
MF = P.build_packsell(F, 32, 4096, P.parse_format("fp16"), "implicit")
OF = O.build(F.row_ptr, F.col_idx, F.values, F.n_cols, 32, 4096, O.preset("fp16"), "implicit")
xf = np.random.default_rng(1).uniform(-1, 1, F.n_cols).astype(np.float16)
for aff in ("0", "1"):
    os.environ["PSELL_AFF"] = aff
    lib.psell_reload_env()
    yf = P.packsell_spmv(MF, xf).astype(np.float64)
    assert np.abs(yf - O.spmv(OF, xf.astype(np.float32))).max() < 0.05, aff
import io  # noqa: E402
buf = io.BytesIO()
P.write_psell(MF, buf)
buf.seek(0)
P.read_psell(buf)  # psell_max_column pass
print("sanitize_r02 ok")
