#!/usr/bin/env python
"""PackSELL SpMV benchmark on B200 (BASELINE config 2 by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c1] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step is one PackSELL SpMV over the configured matrix.  The matrix is generated
and packed directly in HBM (rows row-partitioned in sigma-aligned slabs across
ranks, x replicated, no collective on the data path).  Rank 0 prints one JSON
line.  `value` = aggregate algorithmic GB/s (SURVEY.md §8d bytes: packed words +
int64 slice offsets + perm + x once + y) over the max-over-ranks CUDA-event time
of the K timed SpMVs with everything resident in HBM; `e2e` is the same metric
through the public API `packsell_spmv(M, x_cpu_pinned, out=y_cpu_pinned)`, i.e.
with the x H2D and y D2H copies inside the timed region.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port of packsell.packsell_spmv, oracle/) on the box's host cores,
one worker process per core, each on its own sigma-aligned slab sample of the
same matrix, and prints the same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PackSELL SpMV GB/s (% HBM peak), GFLOP/s at 1-8 B200; mixed-prec PCG solve s"

CONFIGS = {
    "c2": dict(kind="stencil27", nx=256, preset="fp16", xdt="float16", scale=None, c=32, sigma=256,
               mode="implicit",
               workload="config 2: 27-point stencil 256^3 (HPCG_8_8_8), PackSELL fp16 (W=32, D=15), "
                        "C=32, sigma=256, implicit perm; x, y f16; FP32 FMA accumulation"),
    "c3": dict(kind="stencil27", nx=256, preset="e8m21", xdt="float32", scale="rowsum", c=32, sigma=256,
               mode="implicit",
               workload="config 3: 27-point stencil 256^3 row-sum scaled, PackSELL e8m21 (30-bit float, D=1: "
                        "the FP32-accurate point of the D sweep, backward error 2.9e-7 = FP32 CSR's), C=32, "
                        "sigma=256, implicit; x, y f32"),
    "c3-e8m10": dict(kind="stencil27", nx=256, preset="e8m10", xdt="float32", scale="rowsum", c=32, sigma=256,
                     mode="implicit",
                     workload="config 3 (BASELINE's example codec): 27-point stencil 256^3 row-sum scaled, PackSELL "
                              "e8m10 (20-bit float, D=12), C=32, sigma=256, implicit; x, y f32"),
    "c1": dict(kind="poisson2d", nx=512, preset="fp16", xdt="float16", scale=None, c=32, sigma=256,
               mode="implicit",
               workload="config 1: 5-point Laplacian 512^2, PackSELL fp16, C=32, sigma=256, implicit; x, y f16"),
    "c4": dict(kind="powerlaw", n=2 ** 23, seed=2604, nx=0, preset="fp16", xdt="float16", scale=None, c=32,
               sigma=65536, mode="implicit",
               workload="config 4: power-law rows (Pareto alpha 1.5, n=2^23, ~95M nnz, csrc/gen.cu), PackSELL fp16, "
                        "C=32, sigma=65536 (--sigma), implicit; x, y f16; long slices segmented"),
    "c4b": dict(kind="powerlaw_far", n=2 ** 23, seed=2604, nx=0, preset="fp16", xdt="float16", scale=None, c=32,
                sigma=65536, mode="implicit",
                workload="config 4b: power-law rows with ~20% of entries uniform over [0, n) (SURVEY 8d's "
                         "generator: k_left ~ n, every d_i = 0, dummy-heavy), n=2^23, PackSELL fp16, C=32, "
                         "sigma=65536, implicit; x, y f16; long slices segmented"),
}


def dtype_label(cfg, impl: str) -> str:
    """The arithmetic the path computes in: x / y storage type and accumulator.  Ours
    accumulates with FP32 FMA (FP64 for f64 x); the reference (packed.py:268) rounds
    every product and sum in x's dtype."""
    x = {"float16": "f16", "float32": "f32", "float64": "f64"}[cfg["xdt"]]
    if impl == "reference":
        return f"{x} x/y, {x} accumulate"
    return f"{x} x/y, {'f64' if x == 'f64' else 'f32'} FMA accumulate"


def stencil_k_left(kind: str, nx: int) -> int:
    """Lower bandwidth of the generated matrices (checked against the device in tests)."""
    if kind == "stencil27":
        return nx * nx + nx + 1
    if kind == "poisson3d":
        return nx * nx
    if kind == "powerlaw":
        return 4096  # every row starts at max(0, i - 4096) (csrc/gen.cu)
    if kind == "powerlaw_far":
        from paper_2604_13433_b200.stencil import powerlaw_far_k_left
        return _cached("k_left_far", lambda: powerlaw_far_k_left(2 ** 23, 2604))
    return nx


_CACHE = {}


def _cached(key, fn):
    if key not in _CACHE:
        _CACHE[key] = fn()
    return _CACHE[key]


def cfg_rows(cfg) -> int:
    if cfg["kind"] in ("powerlaw", "powerlaw_far"):
        return cfg["n"]
    return cfg["nx"] ** (2 if cfg["kind"] == "poisson2d" else 3)


def partition(cfg, world):
    """sigma-aligned row slabs: equal for stencils, nnz-balanced for the power-law matrix."""
    from paper_2604_13433_b200 import dist as D
    n = cfg_rows(cfg)
    if not cfg["kind"].startswith("powerlaw") or world == 1:
        return D.equal_row_slabs(n, world, cfg["sigma"])
    from paper_2604_13433_b200.stencil import powerlaw_row_lengths
    return D.word_balanced_slabs(powerlaw_row_lengths(n, cfg["seed"], far=cfg["kind"] == "powerlaw_far"), world,
                                 cfg["sigma"])


def make_slab(cfg, r0, r1):
    import paper_2604_13433_b200 as P
    if cfg["kind"].startswith("powerlaw"):
        from paper_2604_13433_b200.stencil import powerlaw_device
        return powerlaw_device(cfg["n"], cfg["seed"], row_begin=r0, row_end=r1, far=cfg["kind"] == "powerlaw_far")
    return P.stencil_device(cfg["kind"], cfg["nx"], scale=cfg["scale"], row_begin=r0, row_end=r1)


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def ncu_traffic(config: str):
    """(dram bytes per launch of the SpMV kernel, where from) out of the committed ncu --set
    full summary; the summary is stamped with the commit its captures ran at."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(config, {})
        meta = d.get("_meta", {})
        src = (f"profiles/ncu_summary.json['{config}']: ncu --set full of {e.get('kernel', '?')}, captured at "
               f"commit {meta.get('commit', '?')} ({meta.get('when', '?')})")
        return e.get("dram_bytes_per_launch"), src
    except Exception:  # noqa: BLE001
        return None, None


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu_id}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        for ln in getattr(self, "lines", []):
            f = [t.strip() for t in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"),
                                 f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU side
def _digest(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


def reference_pkg():
    """The reference package itself (`packsell` 0.1.0, pure Python/numpy), pip-installed from
    /root/reference into baseline/_ref (git-ignored; it travels to the GPU box with the
    snapshot; __graft_entry__.build() installs it).  None when absent: the CPU legs then
    time the oracle port instead (kind "port")."""
    p = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(p, "packsell")):
        return None
    if p not in sys.path:
        sys.path.append(p)
    try:
        import packsell
        return packsell
    except Exception:  # noqa: BLE001
        return None


class CpuPath:
    """One CPU implementation of the path on a row slab [r0, r1) of a config matrix:
    the reference's own build_packsell / packsell_spmv (kind "reference") or the oracle
    port (kind "port").  The reference has no row origin, so its slab is a CsrMatrix of
    r1 rows whose first r0 rows are empty: same base offsets (global rows, global k_left),
    hence the same words as the production matrix's slices over [r0, r1), at the cost of
    r0 empty rows (no words)."""

    def __init__(self, cfg, A, vals, r0, k_left, prefer_reference=True):
        self.ref = reference_pkg() if prefer_reference else None
        self.kind = "reference" if self.ref is not None else "port"
        self.r0, self.n = r0, A.n_rows
        c, sg = cfg["c"], cfg["sigma"]
        if self.ref is not None:
            R = self.ref
            rp = np.concatenate([np.zeros(r0, np.int64), A.row_ptr])
            Af = R.CsrMatrix(r0 + A.n_rows, A.n_cols, rp, A.col_idx, vals)
            self.M = R.build_packsell(Af, c, sg, R.parse_format(cfg["preset"]), cfg["mode"], _k_left_override=k_left)
            s0 = r0 // c
            off = self.M.offset
            self.pack = self.M.pack
            self.offset = off[s0:] - off[s0]
            self.perm = self.M.perm[r0:] if self.M.perm is not None else None
            self.k_left = self.M.k_left
            self.counts = tuple(self.M.counts)
        else:
            import oracle as O
            self.M = O.build(A.row_ptr, A.col_idx, vals, A.n_cols, c, sg, O.preset(cfg["preset"]), cfg["mode"],
                             k_left=k_left, row0=r0)
            self.pack, self.offset, self.perm = self.M.pack, self.M.offset, self.M.perm
            self.k_left, self.counts = self.M.k_left, tuple(self.M.counts)

    def spmv(self, x):
        """y over the slab's rows (the reference call: packed.py:242)."""
        if self.ref is not None:
            return self.ref.packsell_spmv(self.M, x)[self.r0:]
        import oracle as O
        return O.spmv(self.M, x)

    def nbytes(self, xsz, touched):
        """SURVEY §8d bytes of the slab's SpMV (x counted over the columns it touches)."""
        n_sl = len(self.offset) - 1
        b = 4 * int(self.pack.size) * (2 if self.pack.dtype.itemsize == 8 else 1) + 8 * (n_sl + 1)
        b += xsz * touched + xsz * self.n
        if self.perm is not None:
            b += self.perm.dtype.itemsize * self.n
        return b


def _slab_parity(P, A, vals, x, expect, preset):
    """Compare the CPU implementation's slab with the GPU's production matrix over the same rows.

    `expect` holds the GPU side: sha256 of the pack words / rebased offsets / perm of the
    slab's slices in the full device build, and the device REF_ORDER and FMA SpMV outputs
    on those rows for the same x (SURVEY §8c parity rules 1-3)."""
    import oracle as O
    f16 = x.dtype == np.float16
    y_ref = P.spmv(x)
    y_wide = P.spmv(x.astype(np.float32)) if f16 else y_ref
    q = np.abs(O.quantize(O.preset(preset), vals))
    anorm = float(np.max(np.add.reduceat(q, A.row_ptr[:-1]))) if A.nnz else 0.0
    lmax = int(np.diff(P.offset).max() // 32)
    e = float(np.abs(expect["y_fma"].astype(np.float64) - y_wide.astype(np.float64)).max()) / max(
        anorm * float(np.abs(x.astype(np.float64)).max()), 1e-300)
    bound = (2.0 ** -11 if f16 else 0.0) + 2 * lmax * 2.0 ** -24
    res = {"against": P.kind, "pack": _digest(P.pack) == expect["pack_sha"],
           "offset": _digest(P.offset) == expect["offset_sha"],
           "perm": _digest(P.perm) == expect["perm_sha"],
           "k_left": P.k_left == expect["k_left"],
           "spmv_ref_order_bitwise": bool(np.array_equal(y_ref.view(np.uint8), expect["y_ref"].view(np.uint8))),
           "spmv_fma_e_rel": e, "spmv_fma_bound": bound}
    ok = all(res[k] for k in ("pack", "offset", "perm", "k_left", "spmv_ref_order_bitwise")) and e <= bound
    res["status"] = "bitwise" if ok else "MISMATCH"
    res["words_compared"] = int(P.offset[-1])
    return res


def _cpu_slab(cfg, r0, r1):
    """Host CSR rows [r0, r1) of a config matrix with the reference's scaling (matrix.py:294-316)."""
    from paper_2604_13433_b200.stencil import stencil_rows
    if cfg["kind"] == "powerlaw":
        from paper_2604_13433_b200.stencil import powerlaw_rows
        A = powerlaw_rows(cfg["n"], cfg["seed"], r0, r1)
    elif cfg["kind"] == "powerlaw_far":
        from paper_2604_13433_b200.stencil import powerlaw_far_rows
        A = powerlaw_far_rows(cfg["n"], cfg["seed"], r0, r1)
    else:
        A = stencil_rows(cfg["kind"], cfg["nx"], r0, r1)
    vals = A.values
    if cfg["scale"] == "rowsum":
        rows = np.repeat(np.arange(A.n_rows), A.row_lengths())
        s = np.zeros(A.n_rows)
        np.add.at(s, rows, np.abs(vals))
        vals = vals / s[rows]
    return A, vals


def _cpu_worker(conn, cfg, r0, r1, k_left, seed, expect=None):
    os.environ["OMP_NUM_THREADS"] = "1"
    A, vals = _cpu_slab(cfg, r0, r1)
    t0 = time.perf_counter()
    P = CpuPath(cfg, A, vals, r0, k_left)
    t_build = time.perf_counter() - t0
    xsz = np.dtype(cfg["xdt"]).itemsize
    touched = int(A.col_idx.max()) - int(A.col_idx.min()) + 1 if A.nnz else 0
    nbytes = P.nbytes(xsz, touched)
    x = np.random.default_rng(seed).uniform(-1, 1, A.n_cols).astype(cfg["xdt"])
    parity = None if expect is None else _slab_parity(P, A, vals, x, expect, cfg["preset"])
    conn.send(("ready", nbytes, A.nnz, parity, P.kind, t_build))
    while True:
        msg = conn.recv()
        if msg == "stop":
            break
        t0 = time.perf_counter()
        P.spmv(x)
        conn.send(time.perf_counter() - t0)


def cpu_reference(cfg, workers: int, rows_per_worker: int, steps: int, warmup: int, expect=None):
    """Oracle port of packsell_spmv on `workers` host cores, disjoint slab samples.

    With `expect` (one worker, rows 0..rows_per_worker), the worker also checks the
    GPU's production matrix and SpMV outputs over its slab against its own build."""
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    n = cfg_rows(cfg)
    kl = stencil_k_left(cfg["kind"], cfg["nx"])
    rows_per_worker = max(cfg["sigma"], min(rows_per_worker, n) // cfg["sigma"] * cfg["sigma"])
    workers = max(1, min(workers, n // rows_per_worker))
    procs, conns = [], []
    stride = (n // workers) // cfg["sigma"] * cfg["sigma"]
    if reference_pkg() is not None:
        # the reference has no row origin: a slab at r0 > 0 would carry r0 empty rows whose
        # per-row work (y, the output index) is not the sample's; every worker runs the
        # matrix's first rows instead (interior stencil rows are all alike)
        stride = 0
    for w in range(workers):
        a, b = mp.Pipe()
        r0 = w * stride
        p = ctx.Process(target=_cpu_worker, args=(b, cfg, r0, min(n, r0 + rows_per_worker), kl, 7 + w,
                                                  expect if w == 0 else None))
        p.start()
        procs.append(p)
        conns.append(a)
    tot_bytes, tot_nnz, parity, kind, t_build = 0, 0, None, "port", 0.0
    for c in conns:
        _, nb, nz, par, kind, tb = c.recv()
        tot_bytes += nb
        tot_nnz += nz
        parity = parity or par
        t_build = max(t_build, tb)
    times = []
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        for c in conns:
            c.send("go")
        for c in conns:
            c.recv()
        if it >= warmup:
            times.append(time.perf_counter() - t0)
    for c in conns:
        c.send("stop")
    for p in procs:
        p.join()
    t = float(np.mean(times))
    return dict(gbs=tot_bytes / t / 1e9, gflops=2 * tot_nnz / t / 1e9, sec_per_step=t, workers=workers,
                rows=rows_per_worker, bytes=tot_bytes, nnz=tot_nnz, parity=parity, kind=kind, build_s=t_build,
                sec_min=float(np.min(times)))


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    r = cpu_reference(cfg, cores, args.ref_rows, args.steps, args.warmup)
    what = ("the reference's own packsell.packsell_spmv (baseline/_ref, pure numpy)" if r["kind"] == "reference"
            else "oracle port of packsell_spmv (numpy)")
    where = ("each on rows 0..%d" % (r["rows"] - 1)) if r["kind"] == "reference" else "on disjoint sigma-aligned slabs"
    sample = (f"{r['workers']} worker processes x {r['rows']} rows ({r['nnz']} nnz total) of the same matrix, "
              f"{where}, global k_left; {what}, 1 thread each; os.cpu_count() = {cores}")
    line = {
        "metric": METRIC, "value": r["gbs"], "unit": "GB/s", "impl": "reference",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["sec_per_step"] * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dtype_label(cfg, "reference"),
        "data": "synthetic", "config": {"workload": cfg["workload"], "cpu_sample": sample},
        "gflops": r["gflops"],
        "cpu_baseline": {"value": r["gbs"], "unit": "GB/s", "cores": r["workers"], "kind": r["kind"],
                         "sample": sample, "ms_per_step_min": r["sec_min"] * 1e3, "build_s_per_worker": r["build_s"]},
        "e2e": {"value": r["gbs"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- PCG (config 5)
def pcg_bytes(M, n_local, nnz_local, n_glob_touched):
    """Algorithmic bytes of one inner and one outer iteration."""
    inner = M.spmv_bytes(4, 4, with_perm=True, x_elems=n_glob_touched) + 36 * n_local
    csr64 = 8 * (n_local + 1) + 12 * nnz_local + 8 * n_glob_touched + 8 * n_local
    outer = csr64 + 168 * n_local
    return inner, outer


def pcg_cpu_baseline(args, nx, rep_io, rep64, t_io, t_64):
    """Config 5 on the host CPU as BASELINE.md §3 plans it, with the reference's own solvers
    (baseline/_ref: packsell.iocg / pcg, pure numpy, one core) when installed, else the
    oracle port: full solves at 64^3 (and 128^3 with --pcg-cpu-full: ~8 min), and at the
    GPU's grid a fixed window -- 3 inner PCG iterations on the PackSELL e8m14 operator and
    2 FP64 PCG iterations -- extrapolated by the GPU run's own iteration counts
    (labelled "extrapolated")."""
    R = reference_pkg()
    kind = "reference" if R is not None else "port"
    from paper_2604_13433_b200 import solvers as S

    def problem(m):
        if R is not None:
            return R.sym_diag_scale(R.poisson3d(m))
        import paper_2604_13433_b200 as P
        return P.sym_diag_scale(P.poisson3d(m))

    def solve_full(m):
        A = problem(m)
        b = S.make_rhs_and_x0(A.n_rows, 42)[0]
        res = {"grid": f"{m}^3", "n": A.n_rows}
        if R is not None:
            t = time.perf_counter()
            r = R.iocg(A, b, R.SolveConfig(solver="iocg", tol=1e-9, m_in=args.pcg_m_in, a_backend="packsell-e8m14",
                                           max_outer=400))
            res["iocg"] = {"solve_s": time.perf_counter() - t, "outer_iters": r.outer_iters,
                           "inner_iters": r.total_inner_iters, "converged": r.converged,
                           "true_relres": r.final_true_relres}
            t = time.perf_counter()
            r = R.pcg(A, b, R.SolveConfig(tol=1e-9, max_outer=5000))
            res["fp64_pcg"] = {"solve_s": time.perf_counter() - t, "iters": r.outer_iters, "converged": r.converged,
                               "true_relres": r.final_true_relres}
        else:
            import oracle as O
            OM = O.build(A.row_ptr, A.col_idx, A.values, A.n_cols, 32, 256, O.preset("e8m14"), "implicit")
            ap64 = lambda v: O.csr_spmv(A.row_ptr, A.col_idx, A.values, v, np.float64)  # noqa: E731
            t = time.perf_counter()
            r = O.iocg(ap64, lambda v: O.spmv(OM, v), b, 1e-9, 400, args.pcg_m_in)
            res["iocg"] = {"solve_s": time.perf_counter() - t, "outer_iters": r["outer_iters"],
                           "inner_iters": r["total_inner_iters"], "converged": r["converged"]}
            t = time.perf_counter()
            r = O.pcg(ap64, b, 1e-9, 5000)
            res["fp64_pcg"] = {"solve_s": time.perf_counter() - t, "iters": r["outer_iters"],
                               "converged": r["converged"]}
        return res

    out = {"kind": kind, "cores": 1, "os_cpu_count": os.cpu_count(),
           "what": ("the reference's own packsell.iocg / packsell.pcg (baseline/_ref)" if R is not None
                    else "the oracle port of iocg / pcg"),
           "full": [solve_full(m) for m in ([64, 128] if args.pcg_cpu_full else [64])]}
    def window(m, k_in=3, k_pcg=4):
        """(s per inner PCG iteration, s per FP64 PCG iteration, gen s, build s) at m^3."""
        t0 = time.perf_counter()
        A = problem(m)
        b = S.make_rhs_and_x0(A.n_rows, 42)[0]
        t_gen = time.perf_counter() - t0
        ts = []
        if R is not None:
            from packsell import solvers as RS
            t0 = time.perf_counter()
            be = RS.make_backend(A, "packsell-e8m14")
            t_build = time.perf_counter() - t0
            RS._inner_pcg(be.apply, b, 1, lambda r: r, np.float32)  # builds the SpMV plan cache
            t0 = time.perf_counter()
            RS._inner_pcg(be.apply, b, k_in, lambda r: r, np.float32)
            t_in = (time.perf_counter() - t0) / k_in
            del be
            for k in (1, 1 + k_pcg):
                t0 = time.perf_counter()
                R.pcg(A, b, R.SolveConfig(tol=1e-300, max_outer=k))
                ts.append(time.perf_counter() - t0)
        else:
            import oracle as O
            t0 = time.perf_counter()
            OM = O.build(A.row_ptr, A.col_idx, A.values, A.n_cols, 32, 256, O.preset("e8m14"), "implicit")
            t_build = time.perf_counter() - t0
            t0 = time.perf_counter()
            O.inner_pcg(lambda v: O.spmv(OM, v), b, k_in)
            t_in = (time.perf_counter() - t0) / k_in
            ap64 = lambda v: O.csr_spmv(A.row_ptr, A.col_idx, A.values, v, np.float64)  # noqa: E731
            for k in (1, 1 + k_pcg):
                t0 = time.perf_counter()
                O.pcg(ap64, b, 1e-300, k)
                ts.append(time.perf_counter() - t0)
        return t_in, (ts[1] - ts[0]) / k_pcg, t_gen, t_build

    def extrap(t_in, t64, inner, outer, iters64):
        return inner * t_in + (outer + 1) * t64, iters64 * t64

    # the window model checked against the full 64^3 solves, then applied at the GPU's grid
    f64 = out["full"][0]
    w = window(64)
    e_io, e_64 = extrap(w[0], w[1], f64["iocg"]["inner_iters"], f64["iocg"]["outer_iters"],
                        f64["fp64_pcg"]["iters"])
    out["window_model_check_64"] = {"iocg_extrapolated_over_measured": e_io / f64["iocg"]["solve_s"],
                                    "fp64_pcg_extrapolated_over_measured": e_64 / f64["fp64_pcg"]["solve_s"]}
    if nx <= 256:
        t_in, t_it64, t_gen, t_build = window(nx) if nx != 64 else w
        io_s, p64_s = extrap(t_in, t_it64, rep_io.total_inner_iters, rep_io.outer_iters, rep64.outer_iters)
        out["window"] = {
            "grid": f"{nx}^3", "label": "extrapolated",
            "how": f"3 inner PCG iterations (f32, PackSELL e8m14 operator) and 4 FP64 PCG iterations timed at "
                   f"{nx}^3; IO-CG = GPU inner iterations x t_inner + (GPU outer iterations + 1) x "
                   f"t_fp64_iteration; FP64 PCG = GPU iterations x t_fp64_iteration (model checked at 64^3: "
                   f"window_model_check_64)",
            "s_per_inner_iter": t_in, "s_per_fp64_iter": t_it64, "gen_s": t_gen, "build_s": t_build,
            "iocg_solve_s_extrapolated": io_s, "fp64_pcg_solve_s_extrapolated": p64_s,
            "gpu_speedup_iocg": io_s / t_io, "gpu_speedup_fp64_pcg": p64_s / t_64}
    return out


def run_pcg(args, world, rank, comm, peak):
    """Config 5: mixed-precision IO-CG on sym-scaled 7-pt 256^3, PackSELL e8m14 inner, vs FP64 PCG."""
    import torch
    import paper_2604_13433_b200 as P
    from paper_2604_13433_b200 import dist as D
    from paper_2604_13433_b200 import solvers as S
    from paper_2604_13433_b200.packed import lower_bandwidth
    nx = args.pcg_nx
    n = nx ** 3
    slabs = D.equal_row_slabs(n, world, 256)
    D.check_equal(slabs)
    r0, r1 = slabs[rank]
    A = P.stencil_device("poisson3d", nx, scale="sym", row_begin=r0, row_end=r1)
    b = S.make_rhs_and_x0(n, 42)[0][r0:r1]
    kl = lower_bandwidth(A)
    if comm is not None:
        kl = comm.allreduce_max(kl)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    be = S.make_backend(A, "packsell-e8m14", k_left=kl)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    cfg = S.SolveConfig(solver="iocg", tol=1e-9, m_in=args.pcg_m_in, a_backend="packsell-e8m14", max_outer=400)

    def timed(fn):
        if comm is not None:
            comm.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        rep = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        if comm is not None:
            tt = torch.tensor([dt], dtype=torch.float64, device="cuda" if comm.nccl else "cpu")
            comm.dist.all_reduce(tt, op=comm.dist.ReduceOp.MAX)
            dt = tt.item()
        return rep, dt

    S.iocg(A, b, S.SolveConfig(solver="iocg", tol=1e-9, m_in=args.pcg_m_in, a_backend="packsell-e8m14",
                               max_outer=1), backend=be, comm=comm)  # warm-up (graph capture)
    rep, t_io = timed(lambda: S.iocg(A, b, cfg, backend=be, comm=comm))
    # warm-up of the FP64 PCG's kernels (first launches load their modules lazily)
    S.pcg(A, b, S.SolveConfig(tol=1e-9, max_outer=2), comm=comm)
    rep64, t_64 = timed(lambda: S.pcg(A, b, S.SolveConfig(tol=1e-9, max_outer=5000), comm=comm))
    rep32 = t_32 = None
    sell_spmv_bytes = 0
    if world == 1:  # FP32 IO-CG comparator: SELL-C-sigma f32 inner operator, same protocol
        be32 = S.make_backend(A, "sell32")
        cfg32 = S.SolveConfig(solver="iocg", tol=1e-9, m_in=args.pcg_m_in, a_backend="sell32", max_outer=400)
        S.iocg(A, b, S.SolveConfig(solver="iocg", tol=1e-9, m_in=args.pcg_m_in, a_backend="sell32", max_outer=1),
               backend=be32)
        rep32, t_32 = timed(lambda: S.iocg(A, b, cfg32, backend=be32))
        Ms = be32.matrix  # SELL bytes per inner SpMV: f32 value + int32 column per stored entry
        sell_spmv_bytes = (8 * Ms.n_stored + 8 * (Ms.n_slices + 1) + (Ms.n_rows if Ms.mode == "implicit" else 0)
                           + 4 * n + 4 * (r1 - r0))
        del be32, Ms
    touched = n if world == 1 else (r1 - r0) + 2 * nx * nx
    ib, ob = pcg_bytes(be.matrix, r1 - r0, A.nnz, touched)
    io_bytes = rep.total_inner_iters * ib + (rep.outer_iters + 1) * ob
    csr64 = 8 * (r1 - r0 + 1) + 12 * A.nnz + 16 * (r1 - r0)
    p64_bytes = rep64.outer_iters * (csr64 + 8 * touched - 8 * (r1 - r0) + 80 * (r1 - r0))
    agg = lambda v: v * world  # equal slabs: every rank moves the same bytes  # noqa: E731
    out = {
        "problem": f"config 5: sym-scaled 7-point Laplacian {nx}^3 (n={n}), b = make_rhs_and_x0(n, 42), tol 1e-9",
        "iocg": {"inner": "PackSELL e8m14 (D=8), f32 vectors, m_in=%d, CUDA-graph inner loop" % args.pcg_m_in,
                 "solve_s": t_io, "outer_iters": rep.outer_iters, "inner_iters": rep.total_inner_iters,
                 "converged": rep.converged, "true_relres": rep.final_true_relres,
                 "ms_per_inner_iter": 1e3 * t_io / max(rep.total_inner_iters, 1),
                 "roofline_s": agg(io_bytes) / (peak * world * 1e9),
                 "frac_of_roofline": (agg(io_bytes) / (peak * world * 1e9)) / t_io,
                 "bytes_per_inner_iter": int(agg(ib))},
        "fp64_pcg": {"solve_s": t_64, "iters": rep64.outer_iters, "converged": rep64.converged,
                     "true_relres": rep64.final_true_relres,
                     "roofline_s": agg(p64_bytes) / (peak * world * 1e9),
                     "frac_of_roofline": agg(p64_bytes) / (peak * world * 1e9) / t_64},
        "fp32_sell_iocg": None if rep32 is None else {
            "inner": "SELL-C-sigma (C=32, sigma=256) f32 values + int32 columns, f32 vectors, m_in=%d" % args.pcg_m_in,
            "solve_s": t_32, "outer_iters": rep32.outer_iters, "inner_iters": rep32.total_inner_iters,
            "converged": rep32.converged, "true_relres": rep32.final_true_relres,
            # the same roofline accounting as the PackSELL IO-CG (inner SpMV bytes + 36 B/row of
            # vectors per inner iteration, the outer iterations as there)
            "roofline_s": (rep32.total_inner_iters * (sell_spmv_bytes + 36 * (r1 - r0))
                           + (rep32.outer_iters + 1) * ob) / (peak * 1e9),
            "frac_of_roofline": (rep32.total_inner_iters * (sell_spmv_bytes + 36 * (r1 - r0))
                                 + (rep32.outer_iters + 1) * ob) / (peak * 1e9) / t_32},
        "speedup_iocg_vs_fp64_pcg": t_64 / t_io,
        # the comparator runs at a lower fraction of its own roofline than the IO-CG, so the
        # measured speed-up overstates the format's advantage: the roofline-to-roofline ratio
        # is the one a perfectly tuned FP64 PCG would see
        "speedup_iocg_vs_fp64_pcg_roofline_to_roofline": (agg(p64_bytes) / agg(io_bytes)),
        "speedup_iocg_vs_fp32_sell_iocg": None if t_32 is None else t_32 / t_io,
        "speedup_iocg_vs_fp32_sell_iocg_roofline_to_roofline": None if t_32 is None else (
            (rep32.total_inner_iters * (sell_spmv_bytes + 36 * (r1 - r0)) + (rep32.outer_iters + 1) * ob)
            / agg(io_bytes)),
        "build_s": t_build,
        "collectives": "none" if world == 1 else (
            "peer-memory transport (K8, csrc/peer.cu): one kernel per halo exchange pushes p's halo (f32 inner, "
            "f64 outer) into the peers' vectors over NVLink; the inner iteration's two FP64 dot all-reduces run in "
            "the last CTA of the SpMV and of the r update (push to every peer's arena, flag, rank-ordered sum; "
            + ("fused; the halo pushed by the direction kernel: 3 launches per inner iteration"
               if os.environ.get("PSELL_PEER_FUSED", "1") != "0"
               else "PSELL_PEER_FUSED=0: separate exchange kernels, 9 launches per inner iteration")
            + "); the distributed inner iteration is one CUDA graph per outer step"
            if comm.peer(n) is not None else
            "torch.distributed: point-to-point halo exchange of p (K7 pack/unpack, dist.Halo) + all-gather of the "
            "FP64 per-rank dot sums (rank-ordered), eager"),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = pcg_cpu_baseline(args, nx, rep, rep64, t_io, t_64)
    return out


# ----------------------------------------------------------------------------- GPU side
def _event_ms(fn, reps=20):
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    v0.record()
    for _ in range(reps):
        fn()
    v1.record()
    torch.cuda.synchronize()
    return v0.elapsed_time(v1) / reps


def vendor_baselines(S, xt, dev, cfg):
    """The paper's vendor comparators on the same matrix, one GPU (§V):
    cuSPARSE SELL ("cuSELL": SELL-C-sigma, C = 32, sigma = 256, rows explicitly sigma-reordered,
    values and vectors in x's dtype, FP32 compute) and cuSPARSE CSR (torch.sparse_csr_tensor @ x)."""
    import numpy as np
    import torch
    out = {}
    try:
        from paper_2604_13433_b200.vendor import CuSell
        V = CuSell(S, 32, 256, np.float16 if xt == torch.float16 else np.float32)
        V.x.copy_((torch.rand(S.n_cols, device=dev) * 2 - 1).to(xt))
        out["cusparse_sell"] = {"what": "cuSPARSE SELL-C-sigma SpMV (cusparseCreateSlicedEll + SELL_ALG1, "
                                        "preprocessed), C=32, sigma=256 sorted rows, values/x/y in x dtype",
                                "ms_per_step": _event_ms(V.spmv)}
        V.close()
        del V
    except Exception as e:  # noqa: BLE001
        out["cusparse_sell"] = {"unavailable": repr(e)[:200]}
    torch.cuda.empty_cache()
    try:
        Acsr = torch.sparse_csr_tensor(S.row_ptr.to(torch.int32), S.col_idx, S.values.to(xt), (S.n_rows, S.n_cols))
        xv = (torch.rand(Acsr.shape[1], device=dev) * 2 - 1).to(xt).unsqueeze(1)
        out["cusparse_csr"] = {"what": "cuSPARSE CSR SpMV via torch.sparse_csr_tensor @ x (values in x dtype)",
                               "ms_per_step": _event_ms(lambda: Acsr @ xv)}
        del Acsr, xv
    except Exception as e:  # noqa: BLE001
        out["cusparse_csr"] = {"unavailable": repr(e)[:200]}
    torch.cuda.empty_cache()
    return out


def gpu_slab_expect(M, cfg, rows, seed):
    """GPU side of the bench-line parity block: digests of the production matrix over
    storage rows 0..rows-1 and the device SpMV outputs on those rows for the CPU
    sample's x (generated identically on the host)."""
    import torch
    from paper_2604_13433_b200 import _dev
    import paper_2604_13433_b200 as P
    s1 = rows // M.c
    off = M.offset
    x = np.random.default_rng(seed).uniform(-1, 1, M.n_cols).astype(cfg["xdt"])
    xd = torch.from_numpy(x).cuda()
    y_ref = P.packsell_spmv(M, xd, ref_order=True)[:rows].cpu().numpy()
    y_fma = P.packsell_spmv(M, xd)[:rows].cpu().numpy()
    return {"pack_sha": _digest(_dev.download(M.d_pack[:off[s1]], M.fmt.word_dtype)),
            "offset_sha": _digest(off[:s1 + 1]),
            "perm_sha": _digest(M.perm[:rows]),
            "k_left": M.k_left, "y_ref": y_ref, "y_fma": y_fma}


def seg_launches(seg, kernel_name):
    """Launches per SpMV and the kernel label of a segmented (power-law) matrix: the long
    slices' segments run in one grid with the short slices (spmv_dual_seg_kernel) unless
    PSELL_SEGMERGE=0 splits them into their own launch; a combine kernel adds them up."""
    if seg is None:
        return 1, kernel_name
    if os.environ.get("PSELL_DSTATIC", "1") != "0" and os.environ.get("PSELL_AFF", "0") == "0":
        return 1 + (seg["n_long"] > 0), ("spmv_dual_static_kernel (one CTA per SM: its segments, then a "
                                         "contiguous word-balanced range of short-slice pairs) + seg_combine_kernel")
    merged = seg["n_seg"] > 0 and os.environ.get("PSELL_SEGMERGE", "1") != "0"
    if merged:
        return 1 + (seg["n_long"] > 0), "spmv_dual_seg_kernel (segments + short slices in one grid) + seg_combine_kernel"
    return 1 + (seg["n_seg"] > 0) + (seg["n_long"] > 0), kernel_name + " + spmv_seg_kernel + seg_combine_kernel"


EXTRA_CONFIGS = ("c3", "c3-e8m10", "c4", "c4b")


def config_summary(args, name, peak):
    """One GPU, whole matrix: the SpMV of another BASELINE config measured inside the default
    run (build, K timed steps by CUDA events, roofline, vendor comparators and a bitwise
    parity sample against the reference's own code), so that the driver's record carries
    every config, not only the headline."""
    import torch
    import paper_2604_13433_b200 as P
    from paper_2604_13433_b200 import _dev, _lib
    from paper_2604_13433_b200.packed import _seg_schedule, lower_bandwidth
    cfg = CONFIGS[name]
    dev = torch.device("cuda", torch.cuda.current_device())
    n = cfg_rows(cfg)
    S = make_slab(cfg, 0, n)
    kl = lower_bandwidth(S)
    t0 = time.perf_counter()
    M = P.build_packsell(S, cfg["c"], cfg["sigma"], P.parse_format(cfg["preset"]), cfg["mode"], _k_left_override=kl)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    xt = getattr(torch, cfg["xdt"])
    nnz = int(S.nnz)
    vendor = None if args.no_vendor else vendor_baselines(S, xt, dev, cfg)
    del S
    torch.cuda.empty_cache()
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    x = (torch.rand(n, generator=g, device=dev, dtype=torch.float32) * 2 - 1).to(xt)
    y = torch.empty(M.n_rows, dtype=xt, device=dev)
    xsz = x.element_size()
    kernel = _lib.lib().psell_spmv_kernel_name(M.desc(), _dev.T_DT_CODE[x.dtype], M.spmv_flags()).decode()
    seg = _seg_schedule(M)
    kernel = seg_launches(seg, kernel)[1]
    for _ in range(max(3, args.warmup)):
        P.packsell_spmv(M, x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        P.packsell_spmv(M, x, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    nbytes = M.spmv_bytes(xsz, xsz, with_perm=True, x_elems=n)
    gbs = nbytes / (ms * 1e-3) / 1e9
    out = {"workload": cfg["workload"], "n": n, "nnz": nnz, "n_stored": int(M.n_stored), "counts": list(M.counts),
           "k_left": int(kl), "kernel": kernel, "steps": args.steps, "ms_per_step": ms, "bytes_per_step": int(nbytes),
           "value": gbs, "unit": "GB/s", "gflops": 2 * nnz / (ms * 1e-3) / 1e9,
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "frac": gbs / peak,
                        "traffic": ncu_traffic(name)[0], "traffic_source": ncu_traffic(name)[1]},
           "build_s": build_s}
    if cfg["kind"].startswith("powerlaw"):
        try:
            from paper_2604_13433_b200.vendor import gather_ceiling
            ceil = gather_ceiling(1 << 23, xsz)
            bound_ms = nnz / ceil * 1e3
            out["roofline"]["gather"] = {"bound": "l2_random_gather", "ceiling_gathers_per_s": ceil,
                                         "bound_ms": bound_ms, "frac": bound_ms / ms}
        except Exception as e:  # noqa: BLE001
            out["roofline"]["gather"] = {"unavailable": repr(e)[:200]}
    if vendor:
        for v in vendor.values():
            if "ms_per_step" in v:
                v["speedup_packsell"] = v["ms_per_step"] / ms
        out["vendor_baseline"] = vendor
    if not args.no_cpu_baseline:
        rows = max(cfg["sigma"], min(args.extra_cpu_rows, M.n_rows) // cfg["sigma"] * cfg["sigma"])
        expect = gpu_slab_expect(M, cfg, rows, 7)
        r = cpu_reference(cfg, 1, rows, 1, 0, expect=expect)
        out["parity"] = r["parity"]
        out["parity"]["sample"] = f"rows 0..{rows - 1}: GPU production build + SpMV vs the {r['kind']} on the same rows"
        out["cpu_baseline"] = {"value": r["gbs"], "unit": "GB/s", "cores": 1, "kind": r["kind"],
                               "sample": f"{rows} rows, one SpMV"}
    del M, x, y
    torch.cuda.empty_cache()
    return out


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    import paper_2604_13433_b200 as P
    from paper_2604_13433_b200.packed import lower_bandwidth

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PSELL_SHARE_GPU=1 + PSELL_DIST_BACKEND=gloo: every rank on cuda:0 over gloo, to
    # exercise the multi-rank bench path on a single GPU (the real run uses NCCL)
    # More ranks than visible GPUs (e.g. --gpus 2 on a one-GPU box): the same shared mode,
    # chosen automatically and labelled in the line, instead of an invalid-device error.
    shared = bool(os.environ.get("PSELL_SHARE_GPU")) or (world > 1 and world > torch.cuda.device_count())
    if shared:
        local = 0
        os.environ.setdefault("PSELL_XPORT", "peer")  # CUDA IPC works between ranks on one GPU
    backend = os.environ.get("PSELL_DIST_BACKEND", "gloo" if shared and not os.environ.get("PSELL_SHARE_GPU")
                             else "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def allreduce(v, op):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=op)
        return t.item()

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    n = cfg_rows(cfg)
    sig = cfg["sigma"]
    r0, r1 = partition(cfg, world)[rank]
    fmt = P.parse_format(cfg["preset"])

    t_b0 = time.perf_counter()
    S = make_slab(cfg, r0, r1)
    kl = int(allreduce(lower_bandwidth(S), dist.ReduceOp.MAX if world > 1 else None))
    torch.cuda.synchronize()
    t_b1 = time.perf_counter()
    M = P.build_packsell(S, cfg["c"], sig, fmt, cfg["mode"], _k_left_override=kl)
    torch.cuda.synchronize()
    t_b2 = time.perf_counter()
    # the first build pays the device allocations (pack, workspace) and module
    # loading; a second, warm build -- its pack reusing the first one's freed memory --
    # is the packing cost proper
    del M
    M = P.build_packsell(S, cfg["c"], sig, fmt, cfg["mode"], _k_left_override=kl)
    torch.cuda.synchronize()
    t_b3 = time.perf_counter()
    if world == 1:
        touched = n
    elif cfg["kind"].startswith("powerlaw"):
        touched = int(torch.unique(S.col_idx).numel())  # distinct x entries this slab gathers
    else:
        # stencil rows are ascending with ascending columns: the slab's x footprint
        # runs from its first stored column to its last
        touched = int(S.col_idx[-1].item()) - int(S.col_idx[0].item()) + 1 if S.nnz else 0
    nnz_local = S.nnz
    xt = getattr(torch, cfg["xdt"])
    # vendor baseline on the same matrix (one GPU): cuSPARSE CSR SpMV through
    # torch.sparse_csr_tensor @ x, CSR values in x's precision (the paper's cuCSR comparison)
    vendor = None
    if world == 1 and S.nnz < 2 ** 31 and not args.no_vendor:
        vendor = vendor_baselines(S, xt, dev, cfg)
    del S
    torch.cuda.empty_cache()

    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    x = (torch.rand(n, generator=g, device=dev, dtype=torch.float32) * 2 - 1).to(xt)
    y = torch.empty(M.n_rows, dtype=xt, device=dev)
    xsz = x.element_size()
    from paper_2604_13433_b200 import _dev, _lib
    from paper_2604_13433_b200.packed import _seg_schedule
    kernel_name = _lib.lib().psell_spmv_kernel_name(M.desc(), _dev.T_DT_CODE[x.dtype], M.spmv_flags()).decode()
    seg = _seg_schedule(M)  # long power-law slices: + segments (merged grid by default) + combine
    launches_per_step, kernel_name = seg_launches(seg, kernel_name)
    bytes_local = M.spmv_bytes(xsz, xsz, with_perm=True, x_elems=touched)
    bytes_noperm = M.spmv_bytes(xsz, xsz, with_perm=False, x_elems=touched)
    st = torch.cuda.current_stream()

    for _ in range(max(3, args.warmup)):
        P.packsell_spmv(M, x, out=y)
    torch.cuda.synchronize()
    # soak so the clock sampler sees the kernel under load around the timed region
    gpu_uuid = str(torch.cuda.get_device_properties(dev).uuid)
    gpu_id = gpu_uuid if gpu_uuid.startswith("GPU-") else f"GPU-{gpu_uuid}"
    sampler = ClockSampler(gpu_id)
    with sampler:
        t_end = time.perf_counter() + 1.0
        while time.perf_counter() < t_end:
            for _ in range(20):
                P.packsell_spmv(M, x, out=y)
            torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.steps):
            P.packsell_spmv(M, x, out=y)
        e1.record(st)
        torch.cuda.synchronize()
        barrier()
        t_end = time.perf_counter() + 0.5
        while time.perf_counter() < t_end:
            for _ in range(20):
                P.packsell_spmv(M, x, out=y)
            torch.cuda.synchronize()
    ms_local = e0.elapsed_time(e1) / args.steps
    # A/B: the persistent TMA bulk-copy stream variant (not the headline)
    torch.cuda.synchronize()
    for _ in range(3):
        P.packsell_spmv(M, x, out=y, _pipe=1)
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(st)
    for _ in range(args.steps):
        P.packsell_spmv(M, x, out=y, _pipe=1)
    g1.record(st)
    torch.cuda.synchronize()
    ms_regpipe = g0.elapsed_time(g1) / args.steps
    ms = allreduce(ms_local, dist.ReduceOp.MAX if world > 1 else None)
    bytes_all = allreduce(float(bytes_local), dist.ReduceOp.SUM if world > 1 else None)
    nnz_all = allreduce(float(nnz_local), dist.ReduceOp.SUM if world > 1 else None)
    value = bytes_all / (ms * 1e-3) / 1e9
    gflops = 2 * nnz_all / (ms * 1e-3) / 1e9

    # e2e through the public API with host buffers (pinned), copies in the timed region
    xh = x.cpu().pin_memory()
    yh = torch.empty(M.n_rows, dtype=xt, pin_memory=True)
    for _ in range(2):
        P.packsell_spmv(M, xh, out=yh)
    barrier()
    torch.cuda.synchronize()
    k_e2e = max(3, min(args.steps, 50))
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    f0.record(st)
    for _ in range(k_e2e):
        P.packsell_spmv(M, xh, out=yh)
    f1.record(st)
    torch.cuda.synchronize()
    wall_e2e = (time.perf_counter() - w0) / k_e2e * 1e3
    ms_sync_local = max(f0.elapsed_time(f1) / k_e2e, wall_e2e)
    ms_sync = allreduce(ms_sync_local, dist.ReduceOp.MAX if world > 1 else None)
    # headline e2e: the pipelined public API (x_{i+1} H2D || SpMV_i || y_{i-1} D2H);
    # every step still uploads its x from pinned host memory and downloads its y
    xs = [xh, xh.clone().pin_memory()]
    ys = [yh, torch.empty_like(yh).pin_memory()]
    P.packsell_spmv_stream(M, [xs[i & 1] for i in range(4)], [ys[i & 1] for i in range(4)])
    # three timed runs of k_e2e steps, the median reported (host DMA rates wander run to
    # run on a shared host: one driver run read 1.32 ms against 0.75 ms on the next box)
    e2e_runs = []
    for _ in range(3):
        barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        P.packsell_spmv_stream(M, [xs[i & 1] for i in range(k_e2e)], [ys[i & 1] for i in range(k_e2e)])
        torch.cuda.synchronize()
        e2e_runs.append(allreduce((time.perf_counter() - w0) / k_e2e * 1e3, dist.ReduceOp.MAX if world > 1 else None))
    ms_e2e = sorted(e2e_runs)[1]
    e2e_value = bytes_all / (ms_e2e * 1e-3) / 1e9
    # the literal drop-in call: numpy x in, numpy y out (packed.py:242 signature), one call per step
    x_np = xh.numpy().copy()
    for _ in range(2):
        P.packsell_spmv(M, x_np)
    barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for _ in range(k_e2e):
        P.packsell_spmv(M, x_np)
    ms_np = allreduce((time.perf_counter() - w0) / k_e2e * 1e3, dist.ReduceOp.MAX if world > 1 else None)
    del x_np
    # the e2e bound: pinned H2D of x and D2H of y on two copy engines, no compute
    s_a, s_b = torch.cuda.Stream(), torch.cuda.Stream()
    xd_b, yd_b = torch.empty_like(x), torch.empty_like(y)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for _ in range(k_e2e):
        with torch.cuda.stream(s_a):
            xd_b.copy_(xh, non_blocking=True)
        with torch.cuda.stream(s_b):
            yh.copy_(yd_b, non_blocking=True)
    torch.cuda.synchronize()
    ms_pcie = (time.perf_counter() - w0) / k_e2e * 1e3
    del xd_b, yd_b

    peak, peak_kind = measured_peak()
    achieved = bytes_local / (ms_local * 1e-3) / 1e9
    gather_roof = None
    if cfg["kind"].startswith("powerlaw"):
        # irregular rows: the x gathers (one per real word; dummy / padding words issue
        # none) land on unrelated 32-B sectors of the L2-resident x, so the binding roof
        # is the GPU's random-gather rate, measured here by the probe kernel
        try:
            from paper_2604_13433_b200.vendor import gather_ceiling
            ceil = gather_ceiling(1 << 23, xsz)
            bound_ms = nnz_local / ceil * 1e3
            gather_roof = {"bound": "l2_random_gather", "gathers_per_step": int(nnz_local),
                           "ceiling_gathers_per_s": ceil, "bound_ms": bound_ms, "frac": bound_ms / ms_local,
                           "hbm_bound_ms": bytes_local / (peak * 1e9) * 1e3,
                           "ceiling_how": "csrc/vendor/probe.cu: 16 independent hashed gathers per thread, 8 CTAs/SM, "
                                          "2^23-element x (L2-resident), CUDA events"}
        except Exception as e:  # noqa: BLE001
            gather_roof = {"unavailable": repr(e)[:200]}
    clocks = sampler.summary()

    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rows = max(sig, min(args.cpu_rows, M.n_rows) // sig * sig)
        expect = gpu_slab_expect(M, cfg, rows, 7)
        r = cpu_reference(cfg, 1, args.cpu_rows, 3, 1, expect=expect)
        parity = r["parity"]
        who = "the reference's own build_packsell / packsell_spmv" if r["kind"] == "reference" else "the oracle port"
        parity["sample"] = (f"rows 0..{rows - 1} of the benchmarked matrix: the GPU production build's words / "
                            f"offsets / perm over those slices and its SpMV outputs on those rows vs {who} on the "
                            f"same rows (global k_left)")
        cpu = {"value": r["gbs"], "unit": "GB/s", "cores": 1, "kind": r["kind"],
               "sample": f"{r['rows']} rows (rows 0..{r['rows'] - 1}, {r['nnz']} nnz) of the same matrix, "
                         f"global k_left; {who}, numpy single thread; {r['gflops']:.4f} GFLOP/s; "
                         f"build {r['build_s']:.2f} s; os.cpu_count() = {os.cpu_count()}",
               "ms_per_step_min": r["sec_min"] * 1e3}

    # every collective runs on all ranks, before the rank-0-only report
    bytes_noperm_all = allreduce(float(bytes_noperm), dist.ReduceOp.SUM if world > 1 else None)
    pcg = None
    m_info = (M.n_stored, list(M.counts))
    h2d_b, d2h_b = int(xh.numel() * xh.element_size()), int(yh.numel() * yh.element_size())
    do_extra = world == 1 and args.config == "c2" and not args.no_extra
    if do_extra or not args.no_pcg:
        M = x = y = xh = yh = None  # noqa: F841 (free the headline matrix before the next ones)
        torch.cuda.empty_cache()
    extra = None
    if do_extra:
        extra = {}
        for name in EXTRA_CONFIGS:
            try:
                extra[name] = config_summary(args, name, peak)
            except Exception as e:  # noqa: BLE001
                extra[name] = {"error": repr(e)[:300]}
    if not args.no_pcg:
        from paper_2604_13433_b200 import dist as D
        comm = D.Comm() if world > 1 else None
        try:
            pcg = run_pcg(args, world, rank, comm, peak)
        except Exception as e:  # noqa: BLE001
            if comm is None or os.environ.get("PSELL_XPORT") == "nccl":
                raise
            # the peer-memory transport failed on this node (IPC mapping refused, or a wait
            # timed out on every rank alike): rerun the solves over torch.distributed
            comm.close()
            os.environ["PSELL_XPORT"] = "nccl"
            comm = D.Comm()
            pcg = run_pcg(args, world, rank, comm, peak)
            pcg["transport_fallback"] = f"peer transport failed ({repr(e)[:160]}); solved over torch.distributed"
        if comm is not None:
            comm.close()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": dtype_label(cfg, "ours"), "data": "synthetic",
            "config": {"workload": cfg["workload"], "n": n, "nnz": int(nnz_all),
                       **({"shared_gpu": f"{world} ranks on one GPU ({torch.cuda.device_count()} visible): "
                                         "a functional run of the multi-rank path, not a scaling number"}
                          if shared and world > 1 else {}),
                       "n_stored_rank0": m_info[0], "counts_rank0": m_info[1], "k_left": kl,
                       "partition": "sigma-aligned row slabs, x replicated (no collective in the step)",
                       "l2": f"inputs larger than L2: {m_info[0] * 4 / 1e9:.2f} GB of packed words stream per "
                             f"SpMV on rank 0 (126 MB L2); x ({n * np.dtype(cfg['xdt']).itemsize / 1e6:.1f} MB) "
                             "is L2-resident by design and counted once"},
            "pct_hbm_peak": value / (peak * world),
            "gflops": gflops,
            "bytes_per_step": int(bytes_all),
            "bytes_per_step_without_perm": int(bytes_noperm_all),
            "build_s": t_b2 - t_b1, "build_warm_s": t_b3 - t_b2, "gen_s": t_b1 - t_b0,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(args.config)[0],
                         "traffic_source": ncu_traffic(args.config)[1],
                         "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                         "kernel": f"{kernel_name} ({launches_per_step} launch(es) per step; traffic = ncu "
                                   "DRAM bytes per launch of the SpMV kernel)",
                         "gather": gather_roof},
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": {"value": e2e_value, "unit": "GB/s", "ms_per_step": ms_e2e,
                    "h2d_bytes_per_step": h2d_b,
                    "d2h_bytes_per_step": d2h_b,
                    "api": "paper_2604_13433_b200.packsell_spmv_stream(M, [x_pinned]*K, [y_pinned]*K) "
                           "(copy-in / compute / copy-out streams overlapped across steps)",
                    "runs_ms_per_step": e2e_runs, "of_runs": "median of 3 timed runs of %d steps" % k_e2e,
                    "pcie_bound": {"ms_per_step": ms_pcie, "frac": ms_pcie / ms_e2e,
                                   "what": "x H2D || y D2H from / to pinned host memory alone (no SpMV)"},
                    "numpy_per_call": {"value": bytes_all / (ms_np * 1e-3) / 1e9, "ms_per_step": ms_np,
                                       "api": "y = packsell_spmv(M, x_numpy) (the reference signature; "
                                              "pageable H2D, D2H into cached page-locked memory)"},
                    "sync_per_call": {"value": bytes_all / (ms_sync * 1e-3) / 1e9, "ms_per_step": ms_sync,
                                      "api": "packsell_spmv(M, x_pinned_cpu, out=y_pinned_cpu), one blocking call per step"}},
            "gpu_launches": args.steps * launches_per_step,
            "variants_ms": {"register_pipeline (headline)": ms_local, "tma_bulk_stream": ms_regpipe},
            "vendor_baseline": None if vendor is None else {
                k: dict(v, **({"speedup_packsell": v["ms_per_step"] / ms} if "ms_per_step" in v else {}))
                for k, v in vendor.items()},
            "clocks": clocks,
            "other_configs": extra,
            "pcg": pcg,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(n: int) -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)  # >= 1000 timed reps
    ap.add_argument("--warmup", type=int, default=100)  # 100 warm-ups
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--sigma", type=int, default=0, help="override the sorting window")
    ap.add_argument("--ref-rows", type=int, default=131072, help="rows per CPU worker (reference arm)")
    ap.add_argument("--cpu-rows", type=int, default=1048576, help="rows of the cpu_baseline sample (~10 s of CPU work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pcg", action="store_true", help="skip the config-5 PCG time-to-solution")
    ap.add_argument("--no-vendor", action="store_true", help="skip the cuSPARSE CSR comparison")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the other configs' SpMV summaries (other_configs) of the default c2 run")
    ap.add_argument("--extra-cpu-rows", type=int, default=262144, help="rows of each other config's parity sample")
    ap.add_argument("--pcg-nx", type=int, default=256)
    ap.add_argument("--pcg-m-in", type=int, default=50)
    ap.add_argument("--pcg-cpu-full", action="store_true",
                    help="also run the full 128^3 CPU solves of the config-5 baseline (~8 min)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N`: one process per GPU, launched here the way the
        # driver launches N > 1 (torch.distributed.run, rendezvous on 127.0.0.1)
        sys.exit(spawn_ranks(args.gpus))
    cfg = dict(CONFIGS[args.config])
    if args.sigma:
        cfg["sigma"] = args.sigma
        cfg["workload"] += f" [sigma overridden to {args.sigma}]"
    if args.config in ("c4", "c4b") and not args.no_pcg:
        args.no_pcg = True  # the PCG time-to-solution belongs to the stencil configs (config 5)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
