"""Config-5 IO-CG, one warm solve under torch.profiler: device time per kernel / memcpy kind
against the wall time of the call (what is outside the inner iterations)."""
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
be = S.make_backend(A, "packsell-e8m14")
cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=50, a_backend="packsell-e8m14", max_outer=400)
S.iocg(A, b, cfg, backend=be)
torch.cuda.synchronize()
t0 = time.perf_counter()
S.iocg(A, b, cfg, backend=be)
torch.cuda.synchronize()
wall_plain = time.perf_counter() - t0
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    r = S.iocg(A, b, cfg, backend=be)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
tot = 0.0
rows = []
for e in prof.key_averages():
    dt = e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    if dt > 0 and e.key not in ("cudaDeviceSynchronize",):
        rows.append((dt, e.count, e.key))
rows.sort(reverse=True)
print(f"wall {wall_plain * 1e3:.1f} ms (unprofiled), {wall * 1e3:.1f} ms profiled; outer {r.outer_iters} inner {r.total_inner_iters}")
for dt, cnt, k in rows[:22]:
    print(f"  {dt / 1e3:9.2f} ms  {cnt:6d}  {dt / cnt:9.1f} us  {k[:90]}")
print(f"  device total {sum(d for d, _, k in rows if not k.startswith('cuda')) / 1e3:.1f} ms")
