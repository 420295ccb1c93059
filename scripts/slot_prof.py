"""One SpMV of each narrow kernel (pair, slot) on the 7-point 256^3 e8m14 operator, for ncu."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import _lib  # noqa: E402

S = P.stencil_device("poisson3d", 256, scale="sym")
M = P.build_packsell(S, 32, 256, P.parse_format("e8m14"), "implicit")
del S
x = torch.rand(M.n_cols, device="cuda") * 2 - 1
y = torch.empty_like(x)
for slot in ("0", "1"):
    os.environ["PSELL_SLOT"] = slot
    _lib.lib().psell_reload_env()
    for _ in range(3):
        P.packsell_spmv(M, x, out=y)
torch.cuda.synchronize()
