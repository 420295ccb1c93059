"""A/B of two library builds on one config SpMV (run once per PSELL_LIB): prints the time
and a checksum of y, so two runs can be compared bitwise.

    python scripts/lib_ab.py c2 [reps]     (configs as in bench.py)
"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_13433_b200 as P  # noqa: E402

C5 = dict(kind="poisson3d", nx=256, preset="e8m14", xdt="float32", scale="sym", c=32, sigma=256, mode="implicit")
cfg = dict(C5) if sys.argv[1] == "c5" else dict(bench.CONFIGS[sys.argv[1]])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
S = bench.make_slab(cfg, 0, bench.cfg_rows(cfg))
M = P.build_packsell(S, cfg["c"], cfg["sigma"], P.parse_format(cfg["preset"]), cfg["mode"])
del S
torch.cuda.empty_cache()
xt = getattr(torch, cfg["xdt"])
g = torch.Generator(device="cuda")
g.manual_seed(1234)
x = (torch.rand(M.n_cols, generator=g, device="cuda") * 2 - 1).to(xt)
y = torch.empty(M.n_rows, dtype=xt, device="cuda")
for _ in range(20):
    P.packsell_spmv(M, x, out=y)
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        P.packsell_spmv(M, x, out=y)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / reps)
nb = M.spmv_bytes(x.element_size())
h = hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"{os.environ.get('PSELL_LIB', 'libpsell.so'):20s} {sys.argv[1]:5s} {best * 1e3:8.1f} us "
      f"{nb / best / 1e6:8.1f} GB/s  y sha {h}", flush=True)
