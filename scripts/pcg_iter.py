"""Per-inner-iteration time of the config-5 inner PCG (CUDA graph, 50 iterations), current env knobs."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import solvers as S  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = P.stencil_device("poisson3d", nx, scale="sym")
be = S.make_backend(A, "packsell-e8m14")
r64 = torch.rand(A.n_rows, dtype=torch.float64, device="cuda")
z64 = torch.empty_like(r64)
g = S._InnerPCG(be, 50)
g.solve(r64, z64)
ref = z64.clone()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    g.solve(r64, z64)
torch.cuda.synchronize()
knobs = {k: v for k, v in os.environ.items() if k.startswith("PSELL_")}
print(f"{str(knobs):40s} graph inner iteration {(time.perf_counter() - t) / 250 * 1e6:7.1f} us  "
      f"deterministic={torch.equal(ref, z64)}  z[0]={float(z64[0]):.17g}")
