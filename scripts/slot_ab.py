"""A/B: TMA-slot narrow kernel (PSELL_SLOT=1, default) vs the persistent pair kernel
(PSELL_SLOT=0) on 7-point slices (config-5 inner operator): SpMV and the fused SpMV + p.q
(psell_spmv_dot); outputs must be bitwise equal (same FMAs, same order)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import _lib  # noqa: E402
from pair_sweep import timed  # noqa: E402

lib = _lib.lib()
nx = int(os.environ.get("NX", "256"))
for pre, dt in (("e8m14", torch.float32), ("fp16", torch.float32), ("fp16", torch.float16)):
    S = P.stencil_device("poisson3d", nx, scale="sym")
    M = P.build_packsell(S, 32, 256, P.parse_format(pre), "implicit")
    del S
    torch.cuda.empty_cache()
    x = (torch.rand(M.n_cols, device="cuda") * 2 - 1).to(dt)
    y = torch.empty(M.n_rows, dtype=dt, device="cuda")
    nb = M.spmv_bytes(x.element_size())
    outs, dots = {}, {}
    for slot in ("0", "1"):
        os.environ["PSELL_SLOT"] = slot
        lib.psell_reload_env()
        kname = lib.psell_spmv_kernel_name(M.desc(), 0 if dt == torch.float16 else 1, M.spmv_flags()).decode()
        ms = timed(lambda: P.packsell_spmv(M, x, out=y), reps=100)
        outs[slot] = y.clone()
        line = f"7pt {nx}^3 {pre:6s} {str(dt)[6:]:8s} SLOT={slot} {kname:48s} {ms * 1e3:8.1f} us {nb / ms / 1e6:8.1f} GB/s"
        if dt == torch.float32:
            npart = lib.psell_spmv_dot_partials(M.desc(), M.spmv_flags())
            part = torch.zeros(max(npart, 1), dtype=torch.float64, device="cuda")
            err = _lib.PsellError()
            st = _lib.stream_handle()
            q = torch.empty_like(x)
            f = lambda: lib.psell_spmv_dot(M.desc(), _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                                           x.data_ptr(), q.data_ptr(), x.data_ptr(), part.data_ptr(), None,
                                           M.spmv_flags(), st, err)
            ms2 = timed(f, reps=100)
            dots[slot] = (q.clone(), part.clone())
            line += f" | spmv_dot {ms2 * 1e3:8.1f} us"
        print(line, flush=True)
    os.environ.pop("PSELL_SLOT")
    lib.psell_reload_env()
    eq = torch.equal(outs["0"], outs["1"])
    if dots:
        eq = eq and torch.equal(dots["0"][0], dots["1"][0]) and torch.equal(dots["0"][1], dots["1"][1])
    print(f"   bitwise equal: {eq}", flush=True)
    del M
    torch.cuda.empty_cache()
