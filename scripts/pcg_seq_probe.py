"""The bench's config-5 sequence (IO-CG warm-up, IO-CG, FP64 PCG, FP32 SELL IO-CG) repeated,
to see the run-to-run spread of each solve in the order bench.py runs them."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import solvers as S  # noqa: E402
from paper_2604_13433_b200.packed import lower_bandwidth  # noqa: E402

A = P.stencil_device("poisson3d", 256, scale="sym")
b = S.make_rhs_and_x0(256 ** 3, 42)[0]
be = S.make_backend(A, "packsell-e8m14", k_left=lower_bandwidth(A))
cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=50, a_backend="packsell-e8m14", max_outer=400)


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t


import gc  # noqa: E402
pads = []
for a in sys.argv[1:]:
    if a.startswith("pad="):  # shift the solver vectors' placement by a dummy allocation (MB)
        pads.append(torch.empty(int(float(a[4:]) * 2 ** 20), dtype=torch.uint8, device="cuda"))
heap = None
if "heap" in sys.argv[1:]:  # a bench-sized live heap: many small objects the cyclic GC must walk
    heap = [{"i": i, "s": str(i)} for i in range(3_000_000)]
if "nogc" in sys.argv[1:]:
    gc.disable()
for rep in range(4):
    S.iocg(A, b, S.SolveConfig(solver="iocg", tol=1e-9, m_in=50, a_backend="packsell-e8m14", max_outer=1), backend=be)
    r1, t1 = timed(lambda: S.iocg(A, b, cfg, backend=be))
    r2, t2 = timed(lambda: S.pcg(A, b, S.SolveConfig(tol=1e-9, max_outer=5000)))
    print(f"rep {rep}: iocg {t1:.4f} s ({r1.outer_iters}/{r1.total_inner_iters})  fp64 pcg {t2:.4f} s ({r2.outer_iters})",
          flush=True)
