"""A/B the dual-slice SpMV kernel (PSELL_DUAL) chunk size (PSELL_DUAL_U = 8 | 12) on configs 2/3/5."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402


def bench(M, x, y, reps=50):
    for _ in range(5):
        P.packsell_spmv(M, x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        P.packsell_spmv(M, x, out=y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, kind, scale, pre, dt in [("c2 27pt fp16 f16x", "stencil27", None, "fp16", torch.float16),
                                   ("c3 27pt e8m10 f32x", "stencil27", "rowsum", "e8m10", torch.float32),
                                   ("c5 7pt e8m14 f32x", "poisson3d", "sym", "e8m14", torch.float32)]:
    S = P.stencil_device(kind, 256, scale=scale)
    M = P.build_packsell(S, 32, 256, P.parse_format(pre), "implicit")
    del S
    torch.cuda.empty_cache()
    x = (torch.rand(M.n_cols, device="cuda") * 2 - 1).to(dt)
    y = torch.empty(M.n_rows, dtype=dt, device="cuda")
    nb = M.spmv_bytes(x.element_size())
    ref = P.packsell_spmv(M, x).float()
    for env in ({"PSELL_NT": "128"}, {"PSELL_DUAL": "1", "PSELL_DUAL_U": "8"}, {"PSELL_DUAL": "1", "PSELL_DUAL_U": "12"}):
        os.environ.update(env)
        ms = bench(M, x, y)
        ok = torch.allclose(y.float(), ref, rtol=1e-3, atol=1e-3)
        print(f"{name:22s} {str(env):44s} {ms * 1e3:8.1f} us {nb / ms / 1e6:8.1f} GB/s {'ok' if ok else 'BAD'}",
              flush=True)
        for k in env:
            os.environ.pop(k)
    del M
    torch.cuda.empty_cache()
