"""Config 4 per-kernel time split (torch.profiler / CUPTI) and slice-width histogram."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200.packed import SEG_LEN, _seg_schedule  # noqa: E402
from paper_2604_13433_b200.stencil import powerlaw_device  # noqa: E402

n = 2 ** 23
A = powerlaw_device(n, 2604)
sigma = int(os.environ.get("SIGMA", "65536"))
M = P.build_packsell(A, 32, sigma, P.parse_format("fp16"), "implicit")
w = np.diff(M.offset) // 32
print("nnz", A.nnz, "n_stored", M.n_stored, "counts", tuple(M.counts), "SEG_LEN", SEG_LEN)
for lo, hi in ((0, 4), (4, 8), (8, 16), (16, 32), (32, 64), (64, 256), (256, 10 ** 9)):
    m = (w >= lo) & (w < hi)
    print(f"width [{lo},{hi}): slices {m.sum():7d}  words {32 * w[m].sum():11d} ({32 * w[m].sum() / M.n_stored:.3f})")
s = _seg_schedule(M)
print("n_seg", s["n_seg"], "n_long", s["n_long"])
x = (torch.rand(n, device="cuda") * 2 - 1).half()
y = torch.empty(n, dtype=torch.float16, device="cuda")
for _ in range(5):
    P.packsell_spmv(M, x, out=y)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(20):
        P.packsell_spmv(M, x, out=y)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=8))
