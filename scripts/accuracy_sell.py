"""Config 3's accuracy claim and the SELL comparison on the 27-point 256^3 matrix:
backward errors ||y - A x||_inf / (||A||_inf ||x||_inf) (K6, against the unquantised f64 A) of
PackSELL e8m10 / e8m11 / fp16 and of FP32 / FP16 CSR; SpMV time of PackSELL vs our SELL-C-sigma kernels."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from pair_sweep import timed  # noqa: E402

S = P.stencil_device("stencil27", 256, scale="rowsum")
g = torch.Generator(device="cuda")
g.manual_seed(3)
x32 = torch.rand(S.n_cols, generator=g, device="cuda") * 2 - 1
print(f"{'operator':36s} {'backward error':>15s} {'SpMV us':>9s}")
for pre, dt in (("e8m11", torch.float32), ("e8m10", torch.float32), ("e8m7", torch.float32),
                ("fp16", torch.float16)):
    M = P.build_packsell(S, 32, 256, P.parse_format(pre), "implicit")
    x = x32.to(dt)
    y = P.packsell_spmv(M, x)
    us = timed(lambda: P.packsell_spmv(M, x, out=y), reps=20) * 1e3
    print(f"{'PackSELL ' + pre + ' / ' + str(dt).split('.')[1] + ' x':36s} {P.backward_error(S, x, y):15.3e} {us:9.1f}")
    del M
    torch.cuda.empty_cache()
for dt, name in ((torch.float32, "csr32"), (torch.float16, "csr16")):
    x = x32.to(dt)
    y = P.csr_spmv(S, x, np.dtype(str(dt).split(".")[1]))
    print(f"{'CSR ' + name + ' (values and ops in ' + str(dt).split('.')[1] + ')':36s} {P.backward_error(S, x, y):15.3e}")
for vdt, dt in ((np.float32, torch.float32), (np.float16, torch.float16)):
    Sm = P.build_sell(S, 32, 256, "implicit", vdt)
    x = x32.to(dt)
    y = P.sell_spmv(Sm, x)
    us = timed(lambda: P.sell_spmv(Sm, x, out=y), reps=20) * 1e3
    print(f"{'SELL-C-sigma ' + np.dtype(vdt).name:36s} {P.backward_error(S, x, y):15.3e} {us:9.1f}")
    del Sm
    torch.cuda.empty_cache()
