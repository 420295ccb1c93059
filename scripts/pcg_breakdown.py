"""Per-kernel CUDA-event breakdown of one inner PCG iteration (config 5, 256^3)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import solvers as S  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = P.stencil_device("poisson3d", nx, scale="sym")
be = S.make_backend(A, "packsell-e8m14")
inner = S._InnerPCG(be, 1, use_graph=False)
d, L, lib = inner.d, inner.d.L, inner.d.lib
n = inner.n
r64 = torch.rand(n, dtype=torch.float64, device="cuda")
z64 = torch.empty_like(r64)
inner.solve(r64, z64)
M = inner.M
st = d.st()
err = L.PsellError()
steps = {
    "spmv_dot": lambda: lib.psell_spmv_dot(inner.desc, L.ptr(M.d_pack), L.ptr(M.d_offset), L.ptr(M.d_perm),
                                           inner.p_full.data_ptr(), inner.q.data_ptr(), inner.p.data_ptr(),
                                           d.p(d.partials), d.p(d.flags), M.spmv_flags(), st, err),
    "sum_partials(spmv)": lambda: lib.psell_sum_partials(d.p(d.partials), inner.npart, 1, d.p(d.loc, 1),
                                                         d.p(d.flags), st),
    "alpha": lambda: lib.psell_ipcg_alpha(d.p(d.loc, 1), 1, 8, d.p(d.scal), d.p(d.flags), st),
    "update+sum": lambda: lib.psell_ipcg_update(n, inner.x.data_ptr(), inner.r.data_ptr(), inner.z.data_ptr(),
                                                inner.p.data_ptr(), inner.q.data_ptr(), None, d.p(d.scal),
                                                d.p(d.flags), d.p(d.partials), d.p(d.loc, 2), st),
    "beta": lambda: lib.psell_ipcg_beta(d.p(d.loc, 2), 1, 8, d.p(d.scal), d.p(d.flags), st),
    "direction": lambda: lib.psell_ipcg_direction(n, inner.p.data_ptr(), inner.z.data_ptr(), d.p(d.scal),
                                                  d.p(d.flags), st),
}
res = {}
for name, fn in steps.items():
    for _ in range(3):
        d.flags.zero_()
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d.flags.zero_()
    e0.record()
    for _ in range(50):
        fn()
    e1.record()
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / 50
for k, v in res.items():
    print(f"{k:22s} {v * 1e3:9.1f} us")
print(f"{'sum':22s} {sum(res.values()) * 1e3:9.1f} us")
bytes_spmv = M.spmv_bytes(4, 4)
print("spmv GB/s", bytes_spmv / (res["spmv_dot"] * 1e-3) / 1e9, "update GB/s", 24 * n / (res["update+sum"] * 1e-3) / 1e9,
      "direction GB/s", 12 * n / (res["direction"] * 1e-3) / 1e9)
# full inner solve with graph: per-iteration time
g = S._InnerPCG(be, 50)
g.solve(r64, z64)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    g.solve(r64, z64)
torch.cuda.synchronize()
print("graph inner iteration", (time.perf_counter() - t) / 250 * 1e6, "us")
e = S._InnerPCG(be, 50, use_graph=False)
e.solve(r64, z64)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    e.solve(r64, z64)
torch.cuda.synchronize()
print("eager inner iteration", (time.perf_counter() - t) / 250 * 1e6, "us")
