"""Warm FP64 PCG solve on config 5 (7-point 256^3, tol 1e-9): wall time + per-kernel table."""
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import solvers as S  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = P.stencil_device("poisson3d", nx, scale="sym")
b = S.make_rhs_and_x0(nx ** 3, 42)[0]
be = S.make_backend(A, "csr64")
cfg = S.SolveConfig(tol=1e-9, max_outer=3000)
S.pcg(be, b, cfg)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = S.pcg(be, b, cfg)
    torch.cuda.synchronize()
    print(f"warm pcg {time.perf_counter() - t0:.3f} s, iters {r.outer_iters}")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    S.pcg(be, b, cfg)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14, max_name_column_width=50))
