"""K4 CSR SpMV timing (default 7-point 256^3, f64 x): CUDA events over 50 launches, and a
digest of y so the PSELL_CSR variants (bulk default / pipe / tiled) can be checked bitwise.
usage: csr_ab.py [nx] [kind] [dtype]"""
import hashlib
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
kind = sys.argv[2] if len(sys.argv) > 2 else "poisson3d"
dt = getattr(torch, sys.argv[3]) if len(sys.argv) > 3 else torch.float64
A = P.stencil_device(kind, nx, scale="sym" if kind == "poisson3d" else None)
n = A.n_rows
torch.manual_seed(0)
x = torch.rand(n, dtype=torch.float64, device="cuda").to(dt)
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
es = x.element_size()
by = 8 * (n + 1) + 12 * nnz + es * n + es * n
h = hashlib.sha256(ref.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"csr {kind} {nx} {str(dt)[6:]} {us:.1f} us  {by / us / 1e3:.0f} GB/s (algorithmic {by / 1e6:.0f} MB)  y {h}")
