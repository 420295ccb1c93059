"""Run-to-run spread of the config-5 solves (6 warm FP64 PCG and IO-CG solves each),
with Python's cyclic GC on or off (argument "nogc"), to find where the slow repeats come from."""
import gc
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import solvers as S  # noqa: E402

nogc = "nogc" in sys.argv[1:]
nx = 256
A = P.stencil_device("poisson3d", nx, scale="sym")
b = S.make_rhs_and_x0(nx ** 3, 42)[0]
be = S.make_backend(A, "packsell-e8m14")
cio = S.SolveConfig(solver="iocg", tol=1e-9, m_in=50, a_backend="packsell-e8m14", max_outer=400)
c64 = S.SolveConfig(tol=1e-9, max_outer=3000)
S.iocg(A, b, cio, backend=be)
S.pcg(A, b, c64)
if nogc:
    gc.collect()
    gc.disable()
for name, fn in (("fp64_pcg", lambda: S.pcg(A, b, c64)), ("iocg", lambda: S.iocg(A, b, cio, backend=be))):
    ts = []
    for _ in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{'nogc' if nogc else 'gc'} {name:9s} " + " ".join(f"{t:.4f}" for t in ts), flush=True)
