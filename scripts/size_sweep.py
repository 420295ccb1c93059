"""SpMV throughput vs grid size (27-point fp16 / f16 x; 7-point e8m14 / f32 x), production kernels.
Small grids are L2-resident (126 MB), so their GB/s exceeds HBM; large ones are HBM-bound."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import _lib  # noqa: E402
from pair_sweep import timed  # noqa: E402

lib = _lib.lib()
print(f"{'matrix':28s} {'n':>10s} {'nnz':>11s} {'MB':>8s} {'us':>8s} {'GB/s':>8s} {'GFLOP/s':>8s}  kernel")
for kind, pre, dt, sizes in [("stencil27", "fp16", torch.float16, (64, 96, 128, 192, 256, 320)),
                             ("poisson3d", "e8m14", torch.float32, (64, 128, 192, 256, 320, 400))]:
    for nx in sizes:
        S = P.stencil_device(kind, nx, scale="sym" if kind == "poisson3d" else None)
        nnz = S.nnz
        M = P.build_packsell(S, 32, 256, P.parse_format(pre), "implicit")
        del S
        torch.cuda.empty_cache()
        x = (torch.rand(M.n_cols, device="cuda") * 2 - 1).to(dt)
        y = torch.empty(M.n_rows, dtype=dt, device="cuda")
        nb = M.spmv_bytes(x.element_size())
        ms = timed(lambda: P.packsell_spmv(M, x, out=y), reps=30)
        kn = lib.psell_spmv_kernel_name(M.desc(), 0 if dt == torch.float16 else 1, M.spmv_flags()).decode()
        print(f"{kind + ' ' + pre:28s} {M.n_rows:10d} {nnz:11d} {nb / 1e6:8.1f} {ms * 1e3:8.1f} "
              f"{nb / ms / 1e6:8.1f} {2 * nnz / ms / 1e6:8.1f}  {kn}", flush=True)
        del M, x, y
        torch.cuda.empty_cache()
