"""SpMV kernel time (CUDA events, 50 launches) for c2 / c3 / c5 matrices: default path and the TMA stream variant.
usage: spmv_time.py c5 [c2 ...]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402

CFG = {"c2": ("stencil27", None, "fp16", torch.float16), "c3": ("stencil27", "rowsum", "e8m10", torch.float32),
       "c5": ("poisson3d", "sym", "e8m14", torch.float32)}
for name in sys.argv[1:] or ["c5"]:
    c = CFG[name]
    S = P.stencil_device(c[0], 256, scale=c[1])
    M = P.build_packsell(S, 32, 256, P.parse_format(c[2]), "implicit")
    del S
    torch.manual_seed(0)
    x = (torch.rand(M.n_cols, device="cuda") * 2 - 1).to(c[3])
    out = {}
    ys = {}
    for pipe in (0, 1):
        y = torch.empty(M.n_rows, dtype=c[3], device="cuda")
        for _ in range(3):
            P.packsell_spmv(M, x, out=y, _pipe=pipe)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(50):
            P.packsell_spmv(M, x, out=y, _pipe=pipe)
        e1.record()
        torch.cuda.synchronize()
        out[pipe] = e0.elapsed_time(e1) / 50 * 1e3
        ys[pipe] = y
    same = torch.equal(ys[0].view(torch.int16 if c[3] == torch.float16 else torch.int32),
                       ys[1].view(torch.int16 if c[3] == torch.float16 else torch.int32))
    iv = ys[0].view(torch.int16 if c[3] == torch.float16 else torch.int32).to(torch.int64)
    ck = int((iv * torch.arange(1, len(iv) + 1, device=iv.device, dtype=torch.int64)).sum())
    print(f"{name}: default {out[0]:.1f} us   stream {out[1]:.1f} us   bitwise-equal {same}  checksum {ck}", flush=True)
    del M
