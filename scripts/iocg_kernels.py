"""Kernel-time table of one warm config-5 IO-CG solve (torch.profiler / CUPTI), plus host gaps."""
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import solvers as S  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n = nx ** 3
A = P.stencil_device("poisson3d", nx, scale="sym")
b = S.make_rhs_and_x0(n, 42)[0]
be = S.make_backend(A, "packsell-e8m14")
cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=50, a_backend="packsell-e8m14", max_outer=400)
S.iocg(A, b, cfg, backend=be)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    r = S.iocg(A, b, cfg, backend=be)
    torch.cuda.synchronize()
    tt = time.perf_counter() - t0
print(f"warm iocg {tt:.3f} s, outer {r.outer_iters}")
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
