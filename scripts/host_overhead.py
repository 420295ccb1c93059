"""Host cost of one packsell_spmv call on a small (config-1, 5-point 512^2) matrix: wall time per
call over 2000 back-to-back calls vs the kernel time (CUDA events over a CUDA-graph replay)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402

S = P.stencil_device("poisson2d", 512)
M = P.build_packsell(S, 32, 256, P.parse_format("fp16"), "implicit")
x = torch.rand(M.n_cols, device="cuda").half()
y = torch.empty(M.n_rows, dtype=torch.float16, device="cuda")
for _ in range(50):
    P.packsell_spmv(M, x, out=y)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000):
    P.packsell_spmv(M, x, out=y)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e6 * (t1 - t0) / 2000:.2f} us/call, wall incl. drain {1e6 * (t2 - t0) / 2000:.2f} us/call")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    P.packsell_spmv(M, x, out=y)
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(g):
    for _ in range(100):
        P.packsell_spmv(M, x, out=y)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"kernel (graph replay) {e0.elapsed_time(e1) / 1000 * 1e3:.2f} us/call")
