"""Launch the SpMV of one config a few times (for ncu A/B of kernel variants via env vars).
usage: prof_spmv_ab.py c2|c3|c5"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402

cfg = {"c2": ("stencil27", None, "fp16", torch.float16), "c3": ("stencil27", "rowsum", "e8m10", torch.float32),
       "c5": ("poisson3d", "sym", "e8m14", torch.float32)}[sys.argv[1]]
S = P.stencil_device(cfg[0], 256, scale=cfg[1])
M = P.build_packsell(S, 32, 256, P.parse_format(cfg[2]), "implicit")
del S
x = (torch.rand(M.n_cols, device="cuda") * 2 - 1).to(cfg[3])
y = torch.empty(M.n_rows, dtype=cfg[3], device="cuda")
for _ in range(4):
    P.packsell_spmv(M, x, out=y)
torch.cuda.synchronize()
