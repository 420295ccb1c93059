"""A/B threads-per-CTA (PSELL_NT) of the one-warp-per-slice SpMV (PSELL_DUAL=0) on configs 2/3/5."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from pair_sweep import timed as bench  # noqa: E402

for name, kind, scale, pre, dt in [("c2 27pt fp16 f16x", "stencil27", None, "fp16", torch.float16),
                                   ("c3 27pt e8m10 f32x", "stencil27", "rowsum", "e8m10", torch.float32),
                                   ("c5 7pt e8m14 f32x", "poisson3d", "sym", "e8m14", torch.float32)]:
    S = P.stencil_device(kind, 256, scale=scale)
    M = P.build_packsell(S, 32, 256, P.parse_format(pre), "implicit")
    del S
    torch.cuda.empty_cache()
    x = (torch.rand(M.n_cols, device="cuda") * 2 - 1).to(dt)
    y = torch.empty(M.n_rows, dtype=dt, device="cuda")
    nb = M.spmv_bytes(x.element_size())
    os.environ["PSELL_DUAL"] = "0"
    for nt in (256, 128, 64):
        os.environ["PSELL_NT"] = str(nt)
        ms = bench(lambda: P.packsell_spmv(M, x, out=y))
        print(f"{name:22s} NT={nt:3d} {ms * 1e3:8.1f} us {nb / ms / 1e6:8.1f} GB/s", flush=True)
    os.environ.pop("PSELL_NT")
    os.environ.pop("PSELL_DUAL")
    del M
    torch.cuda.empty_cache()
