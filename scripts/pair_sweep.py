"""A/B: exact-tail pair kernel (PSELL_PAIR=1, default) vs the chunk-rounded dual kernel (PSELL_PAIR=0).

Both accumulate the same FMAs in the same order, so y must be bitwise equal.
Also times the fused SpMV + p.q (psell_spmv_dot) used by the inner PCG."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import _lib  # noqa: E402


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


if __name__ == "__main__":
    cases = [("c2 27pt fp16 f16x", "stencil27", None, "fp16", torch.float16),
             ("c3 27pt e8m10 f32x", "stencil27", "rowsum", "e8m10", torch.float32),
             ("c5 7pt e8m14 f32x", "poisson3d", "sym", "e8m14", torch.float32),
             ("c5 7pt fp16 f32x", "poisson3d", "sym", "fp16", torch.float32)]
    lib = _lib.lib()
    for name, kind, scale, pre, dt in cases:
        S = P.stencil_device(kind, 256, scale=scale)
        M = P.build_packsell(S, 32, 256, P.parse_format(pre), "implicit")
        del S
        torch.cuda.empty_cache()
        x = (torch.rand(M.n_cols, device="cuda") * 2 - 1).to(dt)
        y = torch.empty(M.n_rows, dtype=dt, device="cuda")
        nb = M.spmv_bytes(x.element_size())
        outs = {}
        for pair in ("0", "1"):
            os.environ["PSELL_PAIR"] = pair
            kname = lib.psell_spmv_kernel_name(M.desc(), 0 if dt == torch.float16 else 1, M.spmv_flags()).decode()
            ms = timed(lambda: P.packsell_spmv(M, x, out=y))
            outs[pair] = y.clone()
            line = f"{name:20s} PAIR={pair} {kname:24s} {ms * 1e3:8.1f} us {nb / ms / 1e6:8.1f} GB/s"
            if dt == torch.float32:
                npart = lib.psell_spmv_dot_partials(M.desc(), M.spmv_flags())
                part = torch.zeros(max(npart, 1), dtype=torch.float64, device="cuda")
                err = _lib.PsellError()
                st = _lib.stream_handle()
                q = torch.empty_like(x)
                f = lambda: lib.psell_spmv_dot(M.desc(), _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                                               x.data_ptr(), q.data_ptr(), x.data_ptr(), part.data_ptr(), None,
                                               M.spmv_flags(), st, err)
                ms2 = timed(f)
                line += f" | spmv_dot {ms2 * 1e3:8.1f} us"
            print(line, flush=True)
        os.environ.pop("PSELL_PAIR")
        print(f"{name:20s} bitwise equal: {torch.equal(outs['0'], outs['1'])}", flush=True)
        del M
        torch.cuda.empty_cache()
