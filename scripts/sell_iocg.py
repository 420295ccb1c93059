"""FP32 SELL-C-sigma IO-CG comparator on config 5 (7-point 256^3): warm solve time + SELL SpMV time."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import solvers as S  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = P.stencil_device("poisson3d", nx, scale="sym")
b = S.make_rhs_and_x0(nx ** 3, 42)[0]
be = S.make_backend(A, "sell32")
cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=50, a_backend="sell32", max_outer=400)
S.iocg(A, b, cfg, backend=be)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = S.iocg(A, b, cfg, backend=be)
    torch.cuda.synchronize()
    print(f"warm sell32 iocg {time.perf_counter() - t0:.3f} s, outer {r.outer_iters} inner {r.total_inner_iters} "
          f"relres {r.final_true_relres:.3e}")
x = torch.rand(nx ** 3, device="cuda")
y = torch.empty_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
be.apply_into(x, y)
torch.cuda.synchronize()
e0.record()
for _ in range(50):
    be.apply_into(x, y)
e1.record()
torch.cuda.synchronize()
print(f"sell32 SpMV {e0.elapsed_time(e1) / 50 * 1e3:.1f} us  checksum {float(y.double().sum()):.10e}")
