"""Config 3 (§VI-B, Fig. 6): the D sweep on the row-sum-scaled 27-point 256^3
matrix with f32 x / y — PackSELL e8m(22-D) for D = 1..12 (e8m21 ... e8m10): SpMV time,
algorithmic GB/s and % of measured HBM peak, GFLOP/s, backward error against the
unquantised f64 A (K6), dummies; and the FP32 comparators on the same matrix: our
SELL-C-sigma f32 kernel, cuSPARSE SELL f32 (cuSELL, explicitly sigma-reordered rows),
cuSPARSE CSR f32.  Config 2's fp16 point vs cuSELL f16 closes the table.

    python scripts/c3_dsweep.py [--nx 256] [--reps 100] [--out gpurun_out/c3_dsweep.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import _lib  # noqa: E402


def timed(fn, reps):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=256)
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--out", default="gpurun_out/c3_dsweep.json")
    ap.add_argument("--d", default="1-12")
    a = ap.parse_args()
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6545.9
    lo, hi = (int(t) for t in a.d.split("-"))
    S = P.stencil_device("stencil27", a.nx, scale="rowsum")
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    x = torch.rand(S.n_cols, generator=g, device="cuda") * 2 - 1
    y = torch.empty(S.n_rows, dtype=torch.float32, device="cuda")
    rows = []
    print(f"{'codec':8s} {'D':>3s} {'dummies':>11s} {'us':>8s} {'GB/s':>7s} {'%peak':>6s} {'GFLOP/s':>8s} "
          f"{'bwd err':>9s}", flush=True)
    for d in range(lo, hi + 1):
        pre = f"e8m{22 - d}"
        M = P.build_packsell(S, 32, 256, P.parse_format(pre), "implicit")
        ms = timed(lambda: P.packsell_spmv(M, x, out=y), a.reps)
        P.packsell_spmv(M, x, out=y)
        be = P.backward_error(S, x, y)
        nb = M.spmv_bytes(4, 4, with_perm=True)
        r = {"codec": pre, "d": d, "n_stored": M.n_stored, "n_dummy": M.counts.n_dummy,
             "n_padding": M.counts.n_padding, "us": ms * 1e3, "bytes": nb, "gbs": nb / ms / 1e6,
             "frac_peak": nb / ms / 1e6 / peak, "gflops": 2 * S.nnz / ms / 1e6, "backward_error": be,
             "kernel": _lib.lib().psell_spmv_kernel_name(M.desc(), 1, M.spmv_flags()).decode()}
        rows.append(r)
        print(f"{pre:8s} {d:3d} {r['n_dummy']:11d} {r['us']:8.1f} {r['gbs']:7.0f} {100 * r['frac_peak']:6.1f} "
              f"{r['gflops']:8.1f} {be:9.2e}  {r['kernel']}", flush=True)
        del M
        torch.cuda.empty_cache()
    comp = {}
    # FP32 CSR accuracy (reference-order arithmetic) and the FP32 comparators' speed
    yc = P.csr_spmv(S, x, np.float32)
    comp["csr32_backward_error"] = P.backward_error(S, x, yc)
    Sm = P.build_sell(S, 32, 256, "implicit", np.float32)
    ys = torch.empty_like(y)
    ms = timed(lambda: P.sell_spmv(Sm, x, out=ys), a.reps)
    comp["sell32_ours"] = {"us": ms * 1e3, "backward_error": P.backward_error(S, x, P.sell_spmv(Sm, x))}
    del Sm
    torch.cuda.empty_cache()
    from paper_2604_13433_b200.vendor import CuSell
    for dt, key in ((np.float32, "cusell32"), (np.float16, "cusell16")):
        try:
            V = CuSell(S, 32, 256, dt)
            V.x.copy_(x.to(V.x.dtype))
            ms = timed(V.spmv, a.reps)
            V.spmv()
            yv = V.to_original()
            comp[key] = {"us": ms * 1e3, "backward_error": P.backward_error(S, V.x, yv),
                         "bytes": V.bytes, "gbs": V.bytes / ms / 1e6}
            V.close()
            del V
        except Exception as e:  # noqa: BLE001
            comp[key] = {"unavailable": repr(e)[:300]}
        torch.cuda.empty_cache()
    try:
        A = torch.sparse_csr_tensor(S.row_ptr.to(torch.int32), S.col_idx, S.values.float(), (S.n_rows, S.n_cols))
        xv = x.unsqueeze(1)
        ms = timed(lambda: A @ xv, max(10, a.reps // 5))
        comp["cucsr32"] = {"us": ms * 1e3}
        del A
    except Exception as e:  # noqa: BLE001
        comp["cucsr32"] = {"unavailable": repr(e)[:300]}
    torch.cuda.empty_cache()
    # config 2's point: PackSELL fp16 (f16 x/y) vs cuSELL f16 on the unscaled matrix
    S2 = P.stencil_device("stencil27", a.nx)
    M2 = P.build_packsell(S2, 32, 256, P.parse_format("fp16"), "implicit")
    x16 = x.half()
    y16 = torch.empty(S2.n_rows, dtype=torch.float16, device="cuda")
    comp["c2_packsell_fp16_us"] = timed(lambda: P.packsell_spmv(M2, x16, out=y16), a.reps) * 1e3
    del M2
    torch.cuda.empty_cache()
    try:
        V = CuSell(S2, 32, 256, np.float16)
        V.x.copy_(x16)
        comp["c2_cusell16_us"] = timed(V.spmv, a.reps) * 1e3
        V.close()
    except Exception as e:  # noqa: BLE001
        comp["c2_cusell16_us"] = repr(e)[:300]
    for k, v in comp.items():
        print(k, v, flush=True)
    for r in rows:
        for k in ("sell32_ours", "cusell32"):
            if "us" in comp.get(k, {}):
                r["speedup_vs_" + k] = comp[k]["us"] / r["us"]
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump({"matrix": f"27-point {a.nx}^3 row-sum scaled, f32 x/y", "peak_gbs": peak, "rows": rows,
                   "comparators": comp}, f, indent=1)


if __name__ == "__main__":
    main()
