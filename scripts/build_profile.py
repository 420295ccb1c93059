"""Where the PackSELL build time goes (warm): config 4 power-law (default) or config 2 27-point."""
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c4"
if which == "c4":
    from paper_2604_13433_b200 import stencil
    A = stencil.powerlaw_device(1 << 23)
    args = (32, 65536, P.parse_format("fp16"), "implicit")
else:
    A = P.stencil_device("stencil27", 256)
    args = (32, 256, P.parse_format("fp16"), "implicit")
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    M = P.build_packsell(A, *args)
    torch.cuda.synchronize()
    print(f"{which} build {1e3 * (time.perf_counter() - t0):.2f} ms, nnz {A.nnz}, stored {M.n_stored}")
    del M
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    M = P.build_packsell(A, *args)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=45))
