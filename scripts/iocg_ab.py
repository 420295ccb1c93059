"""Mixed-precision IO-CG on config 5 (7-point 256^3, e8m14 inner, m_in 50, tol 1e-9): warm solve time per variant
(env switches given as NAME=VALUE[,NAME=VALUE] arguments, each run in a fresh process) and
the solution's digest, so variants can be checked bitwise against each other."""
import hashlib
import os
import subprocess
import sys
import time

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import numpy as np
    import torch
    sys.path.insert(0, ".")
    import paper_2604_13433_b200 as P  # noqa: E402
    from paper_2604_13433_b200 import solvers as S  # noqa: E402
    nx = int(os.environ.get("NX", "256"))
    A = P.stencil_device("poisson3d", nx, scale="sym")
    b = S.make_rhs_and_x0(nx ** 3, 42)[0]
    be = S.make_backend(A, "packsell-e8m14")
    cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=50, a_backend="packsell-e8m14", max_outer=400)
    S.iocg(A, b, cfg, backend=be)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = S.iocg(A, b, cfg, backend=be)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    h = hashlib.sha256(np.ascontiguousarray(r.x).view(np.uint8)).hexdigest()[:16]
    print(f"  iters {r.outer_iters} solve_s {' '.join(f'{t:.4f}' for t in ts)} "
          f"inner {r.total_inner_iters} us/inner {1e6 * min(ts) / r.total_inner_iters:.1f} relres {r.final_true_relres:.3e} x {h}", flush=True)
    sys.exit(0)

for variant in sys.argv[1:] or ["PSELL_PCG_GRAPH=0", "PSELL_PCG_GRAPH=1"]:
    env = dict(os.environ)
    for kv in variant.split(","):
        if kv:
            k, v = kv.split("=", 1)
            env[k] = v
    print(f"== {variant}", flush=True)
    subprocess.run([sys.executable, __file__, "--child"], env=env, check=False)
