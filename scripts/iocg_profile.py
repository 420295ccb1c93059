"""Where does the config-5 IO-CG time go?  Times inner solves (graph replays) vs the outer loop."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import solvers as S  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n = nx ** 3
A = P.stencil_device("poisson3d", nx, scale="sym")
b = S.make_rhs_and_x0(n, 42)[0]
be = S.make_backend(A, "packsell-e8m14")
cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=50, a_backend="packsell-e8m14", max_outer=400)
orig = S._InnerPCG.solve
acc = {"t": 0.0, "n": 0, "first": None}


def timed_solve(self, r64, z64):
    torch.cuda.synchronize()
    t = time.perf_counter()
    k = orig(self, r64, z64)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    if acc["first"] is None:
        acc["first"] = dt
    acc["t"] += dt
    acc["n"] += 1
    return k


S._InnerPCG.solve = timed_solve
for rep in range(2):
    acc.update(t=0.0, n=0, first=None)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = S.iocg(A, b, cfg, backend=be)
    torch.cuda.synchronize()
    tt = time.perf_counter() - t0
    print(f"iocg total {tt:.3f} s  outer {r.outer_iters}  inner calls {acc['n']}  inner time {acc['t']:.3f} s "
          f"(first call incl. capture {acc['first']:.3f} s)  rest {tt - acc['t']:.3f} s")
