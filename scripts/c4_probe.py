"""Config 4 probe: power-law (n = 2^23) build + SpMV time per sigma / codec."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200.stencil import powerlaw_device  # noqa: E402

n = 2 ** 23
t = time.perf_counter()
A = powerlaw_device(n, 2604)
torch.cuda.synchronize()
print(f"gen {time.perf_counter() - t:.3f}s nnz {A.nnz}", flush=True)
for sigma in (256, 4096, 65536):
    for pre, dt in (("fp16", torch.float16), ("e8m14", torch.float32)):
        torch.cuda.synchronize()
        t = time.perf_counter()
        M = P.build_packsell(A, 32, sigma, P.parse_format(pre), "implicit")
        torch.cuda.synchronize()
        tb = time.perf_counter() - t
        x = (torch.rand(n, device="cuda") * 2 - 1).to(dt)
        y = torch.empty(n, dtype=dt, device="cuda")
        for _ in range(3):
            P.packsell_spmv(M, x, out=y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            P.packsell_spmv(M, x, out=y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        nb = M.spmv_bytes(x.element_size())
        w = (M.offset[1:] - M.offset[:-1]) // 32
        print(f"sigma={sigma:6d} {pre:6s} build {tb * 1e3:7.1f} ms  n_stored {M.n_stored:11d} "
              f"(stored/nnz {M.n_stored / A.nnz:.2f}) max width {w.max():5d}  spmv {ms * 1e3:8.1f} us "
              f"{nb / ms / 1e6:8.1f} GB/s  {2 * A.nnz / ms / 1e6:8.1f} GFLOP/s", flush=True)
        del M
        torch.cuda.empty_cache()
