"""FP32 SELL-C-sigma IO-CG comparator (config 5, sell32 inner), warm solves: run once per
setting of an environment A/B knob (e.g. PSELL_SELL_DOT_MINB, PSELL_SELL_FUSED)."""
import os
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
ts = []
for _ in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = S.iocg(A, b, cfg, backend=be)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
knobs = {k: v for k, v in os.environ.items() if k.startswith("PSELL_")}
print(f"{knobs} sell32 iocg outer {r.outer_iters} inner {r.total_inner_iters} "
      + " ".join(f"{t:.4f}" for t in ts), flush=True)
