"""K4 CSR SpMV timing (7-point 256^3, f64 x): CUDA events over 50 launches."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = P.stencil_device("poisson3d", nx, scale="sym")
torch.manual_seed(0)
x = torch.rand(nx ** 3, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
P.csr_spmv(A, x, out=y)
ref = y.clone()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(50):
    P.csr_spmv(A, x, out=y)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 50 * 1e3
nnz = int(A.nnz)
n = nx ** 3
by = 8 * (n + 1) + 12 * nnz + 8 * n + 8 * n
print(f"csr f64 {us:.1f} us  {by / us / 1e3:.0f} GB/s (algorithmic {by / 1e6:.0f} MB)  checksum {float(ref.sum()):.17g}")
