"""Vendor baseline: cuSPARSE CSR SpMV (through torch.sparse_csr_tensor @ x) vs PackSELL on configs 2/3/5.
CSR values in the same precision as PackSELL's x (f16 for config 2, f32 otherwise)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from pair_sweep import timed  # noqa: E402

print(f"{'config':34s} {'PackSELL us':>12s} {'cuSPARSE CSR us':>16s} {'speedup':>8s}")
for name, kind, scale, pre, dt in [("c2 27pt fp16 / f16 x", "stencil27", None, "fp16", torch.float16),
                                   ("c3 27pt e8m10 / f32 x", "stencil27", "rowsum", "e8m10", torch.float32),
                                   ("c5 7pt e8m14 / f32 x", "poisson3d", "sym", "e8m14", torch.float32)]:
    S = P.stencil_device(kind, 256, scale=scale)
    M = P.build_packsell(S, 32, 256, P.parse_format(pre), "implicit")
    x = (torch.rand(S.n_cols, device="cuda") * 2 - 1).to(dt)
    y = torch.empty(S.n_rows, dtype=dt, device="cuda")
    t_ps = timed(lambda: P.packsell_spmv(M, x, out=y), reps=30)
    A = torch.sparse_csr_tensor(S.row_ptr.to(torch.int32), S.col_idx, S.values.to(dt), (S.n_rows, S.n_cols))
    del S
    torch.cuda.empty_cache()
    xv = x.unsqueeze(1)
    try:
        yc = A @ xv
        t_cs = timed(lambda: A @ xv, reps=30)
        err = float((yc.squeeze(1).float() - y.float()).abs().max())
        print(f"{name:34s} {t_ps * 1e3:12.1f} {t_cs * 1e3:16.1f} {t_cs / t_ps:8.2f}   (max |y_csr - y_psell| {err:.2e})",
              flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{name:34s} {t_ps * 1e3:12.1f}   cuSPARSE failed: {e}", flush=True)
    del A, M, x, y
    torch.cuda.empty_cache()
