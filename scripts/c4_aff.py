"""Config 4 A/B: SM-affine persistent short-slice kernel (PSELL_AFF=1, default) vs the
block-linear dual kernel (PSELL_AFF=0), per sigma; outputs must be bitwise equal
(same FMAs per row in the same order, only the warp that runs a slice differs)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import _lib  # noqa: E402
from paper_2604_13433_b200.stencil import powerlaw_device  # noqa: E402


def timed(fn, reps=30):
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


n = 2 ** 23
A = powerlaw_device(n, 2604)
sigmas = [int(s) for s in os.environ.get("SIGMAS", "256,4096,65536").split(",")]
for sigma in sigmas:
    M = P.build_packsell(A, 32, sigma, P.parse_format("fp16"), "implicit")
    x = (torch.rand(n, device="cuda") * 2 - 1).half()
    ys = {}
    for aff in ("0", "1"):
        for ctas in (["6"] if aff == "0" else os.environ.get("CTAS", "6").split(",")):
            os.environ["PSELL_AFF"] = aff
            os.environ["PSELL_AFF_CTAS"] = ctas
            _lib.lib().psell_reload_env()
            y = torch.empty(n, dtype=torch.float16, device="cuda")
            ms = timed(lambda: P.packsell_spmv(M, x, out=y))
            P.packsell_spmv(M, x, out=y)
            ys[(aff, ctas)] = y.clone()
            nb = M.spmv_bytes(2)
            print(f"sigma={sigma:6d} aff={aff} ctas/SM={ctas} stored/nnz {M.n_stored / A.nnz:.2f} "
                  f"spmv {ms * 1e3:7.1f} us {nb / ms / 1e6:7.1f} GB/s {2 * A.nnz / ms / 1e6:7.1f} GFLOP/s",
                  flush=True)
    base = ys[("0", "6")]
    print("  bitwise equal to the block-linear kernel:",
          all(torch.equal(v.view(torch.int16), base.view(torch.int16)) for v in ys.values()), flush=True)
    del M
    torch.cuda.empty_cache()
