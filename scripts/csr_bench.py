"""Time the K4 CSR SpMV (f64, the outer FCG / FP64 PCG operator) on the config-5 matrix."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402

A = P.stencil_device("poisson3d", 256, scale="sym")
x = torch.rand(A.n_cols, dtype=torch.float64, device="cuda")
for _ in range(3):
    y = P.csr_spmv(A, x, np.float64)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    y = P.csr_spmv(A, x, np.float64)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
nb = 8 * (A.n_rows + 1) + 12 * A.nnz + 8 * A.n_cols + 8 * A.n_rows
print(f"csr_spmv f64 7pt 256^3: {ms * 1e3:.1f} us  {nb / ms / 1e6:.1f} GB/s")
