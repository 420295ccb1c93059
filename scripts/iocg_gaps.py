"""Idle gaps between consecutive GPU kernels of one warm config-5 IO-CG solve (kineto trace)."""
import json
import sys
import tempfile

import numpy as np
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
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    S.iocg(A, b, cfg, backend=be)
    torch.cuda.synchronize()
f = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(f)
ev = [e for e in json.load(open(f))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
ts = np.array([e["ts"] for e in ev])
te = ts + np.array([e["dur"] for e in ev])
gaps = ts[1:] - te[:-1]
names = [e["name"][:40] for e in ev]
span = te[-1] - ts[0]
busy = sum(e["dur"] for e in ev)
print(f"events {len(ev)}  span {span / 1e3:.1f} ms  busy {busy / 1e3:.1f} ms  idle {(span - busy) / 1e3:.1f} ms")
by = {}
for i, g in enumerate(gaps):
    k = (names[i][:28], names[i + 1][:28])
    by.setdefault(k, []).append(g)
for k, v in sorted(by.items(), key=lambda t: -sum(t[1]))[:10]:
    print(f"{sum(v) / 1e3:7.2f} ms  n={len(v):5d}  median {np.median(v):6.2f} us   {k[0]} -> {k[1]}")
