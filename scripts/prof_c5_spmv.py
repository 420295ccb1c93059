"""Launch the config-5 inner SpMV (7-pt 256^3 e8m14, f32 x) a few times for ncu.
DOT=1: the fused SpMV + p.q (psell_spmv_dot) instead of the plain SpMV."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import _lib  # noqa: E402

S = P.stencil_device("poisson3d", 256, scale="sym")
M = P.build_packsell(S, 32, 256, P.parse_format("e8m14"), "implicit")
del S
x = torch.rand(M.n_cols, device="cuda")
y = torch.empty(M.n_rows, device="cuda")
if os.environ.get("DOT"):
    lib = _lib.lib()
    npart = lib.psell_spmv_dot_partials(M.desc(), M.spmv_flags())
    part = torch.zeros(npart, dtype=torch.float64, device="cuda")
    err = _lib.PsellError()
    for _ in range(6):
        rc = lib.psell_spmv_dot(M.desc(), _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                                x.data_ptr(), y.data_ptr(), x.data_ptr(), part.data_ptr(), None, M.spmv_flags(),
                                _lib.stream_handle(), err)
        _lib.check(rc, err)
else:
    for _ in range(6):
        P.packsell_spmv(M, x, out=y)
torch.cuda.synchronize()
print("ok", M.n_stored, M.counts)
