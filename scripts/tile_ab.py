"""A/B: tile-TMA producer/consumer kernel (PSELL_TILE=1) vs the persistent pair kernel on narrow slices.
Same FMA order per row, so y must be bitwise equal; also the fused SpMV + p.q."""
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


lib = _lib.lib()
for name, kind, scale, pre, dt, nx in [("c5 7pt e8m14 f32x", "poisson3d", "sym", "e8m14", torch.float32, 256),
                                       ("c5 7pt fp16 f32x", "poisson3d", "sym", "fp16", torch.float32, 256),
                                       ("7pt fp16 f16x 64^3", "poisson3d", "sym", "fp16", torch.float16, 64)]:
    S = P.stencil_device(kind, nx, scale=scale)
    M = P.build_packsell(S, 32, 256, P.parse_format(pre), "implicit")
    del S
    x = (torch.rand(M.n_cols, device="cuda") * 2 - 1).to(dt)
    y = torch.empty(M.n_rows, dtype=dt, device="cuda")
    nb = M.spmv_bytes(x.element_size())
    outs = {}
    for tile in ("0", "1"):
        os.environ["PSELL_TILE"] = tile
        kname = lib.psell_spmv_kernel_name(M.desc(), 0 if dt == torch.float16 else 1, M.spmv_flags()).decode()
        ms = timed(lambda: P.packsell_spmv(M, x, out=y))
        outs[tile] = y.clone()
        line = f"{name:20s} TILE={tile} {kname:36s} {ms * 1e3:8.1f} us {nb / ms / 1e6:8.1f} GB/s"
        if dt == torch.float32:
            npart = lib.psell_spmv_dot_partials(M.desc(), M.spmv_flags())
            part = torch.zeros(max(npart, 1), dtype=torch.float64, device="cuda")
            err = _lib.PsellError()
            q = torch.empty_like(x)
            f = lambda: lib.psell_spmv_dot(M.desc(), _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                                           x.data_ptr(), q.data_ptr(), x.data_ptr(), part.data_ptr(), None,
                                           M.spmv_flags(), _lib.stream_handle(), err)
            line += f" | spmv_dot {timed(f) * 1e3:8.1f} us  dot={float(part.sum()):.10e}"
        print(line, flush=True)
    os.environ.pop("PSELL_TILE")
    print(f"{name:20s} bitwise equal: {torch.equal(outs['0'], outs['1'])}", flush=True)
