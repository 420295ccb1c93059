"""Launch the config-5 inner SpMV (7-pt 256^3 e8m14, f32 x) a few times for ncu."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402

S = P.stencil_device("poisson3d", 256, scale="sym")
M = P.build_packsell(S, 32, 256, P.parse_format("e8m14"), "implicit")
del S
x = torch.rand(M.n_cols, device="cuda")
y = torch.empty(M.n_rows, device="cuda")
for _ in range(6):
    P.packsell_spmv(M, x, out=y)
torch.cuda.synchronize()
print("ok", M.n_stored, M.counts)
