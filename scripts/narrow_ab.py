"""A/B: narrow kernel (PSELL_NARROW=1, resident CTAs per SM PSELL_NARROW_MINB = 4 | 5 | 6)
vs the persistent pair kernel (PSELL_NARROW=0) on 7-point slices (config-5 inner
operator): SpMV and the fused SpMV + p.q (psell_spmv_dot).  y must be bitwise equal
(same FMAs in the same order); the dot partials differ in grouping only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import _lib  # noqa: E402
from pair_sweep import timed  # noqa: E402

lib = _lib.lib()
nx = int(os.environ.get("NX", "256"))
variants = os.environ.get("VARIANTS", "PSELL_NARROW=0;PSELL_NARROW=1").split(";")
cases = [("e8m14", torch.float32), ("fp16", torch.float32), ("fp16", torch.float16)]
if os.environ.get("QUICK"):
    cases = cases[:1]
for pre, dt in cases:
    S = P.stencil_device("poisson3d", nx, scale="sym")
    M = P.build_packsell(S, 32, 256, P.parse_format(pre), "implicit")
    del S
    torch.cuda.empty_cache()
    x = (torch.rand(M.n_cols, device="cuda") * 2 - 1).to(dt)
    y = torch.empty(M.n_rows, dtype=dt, device="cuda")
    nb = M.spmv_bytes(x.element_size())
    outs, dots = {}, {}
    knobs = sorted({kv.split("=")[0] for v in variants for kv in v.split(",")})
    for var in variants:
        for k in knobs:
            os.environ.pop(k, None)
        for kv in var.split(","):
            k, v = kv.split("=")
            os.environ[k] = v
        lib.psell_reload_env()
        kname = lib.psell_spmv_kernel_name(M.desc(), 0 if dt == torch.float16 else 1, M.spmv_flags()).decode()
        ms = min(timed(lambda: P.packsell_spmv(M, x, out=y), reps=100) for _ in range(3))
        key = var
        outs[key] = y.clone()
        line = f"7pt {nx}^3 {pre:6s} {str(dt)[6:]:8s} {var:36s} {kname[:20]:20s} {ms * 1e3:8.1f} us {nb / ms / 1e6:8.1f} GB/s"
        if dt == torch.float32:
            npart = lib.psell_spmv_dot_partials(M.desc(), M.spmv_flags())
            part = torch.zeros(max(npart, 1), dtype=torch.float64, device="cuda")
            err = _lib.PsellError()
            st = _lib.stream_handle()
            q = torch.empty_like(x)
            f = lambda: lib.psell_spmv_dot(M.desc(), _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                                           x.data_ptr(), q.data_ptr(), x.data_ptr(), part.data_ptr(), None,
                                           M.spmv_flags(), st, err)
            ms2 = min(timed(f, reps=100) for _ in range(3))
            dots[key] = (q.clone(), float(part[:npart].sum().item()))
            line += f" | spmv_dot {ms2 * 1e3:8.1f} us"
        print(line, flush=True)
    for k in knobs:
        os.environ.pop(k, None)
    lib.psell_reload_env()
    k0 = next(iter(outs))
    ref = outs[k0]
    eq = all(torch.equal(ref, o) for o in outs.values())
    msg = f"   y bitwise equal across variants: {eq}"
    if dots:
        eq2 = all(torch.equal(dots[k0][0], d[0]) for d in dots.values())
        rel = max(abs(d[1] - dots[k0][1]) / abs(dots[k0][1]) for d in dots.values())
        msg += f"; dot q bitwise {eq2}; p.q rel diff {rel:.2e}"
    print(msg, flush=True)
    del M
    torch.cuda.empty_cache()
