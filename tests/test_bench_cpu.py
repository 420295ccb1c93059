"""bench.py host logic on CPU: config table vs BASELINE.json, k_left formulas vs the oracle,
partitions, the reference arm's CPU sample (oracle port) and its JSON contract."""

import json
import os

import pytest

import bench
import oracle as O
from paper_2604_13433_b200 import stencil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_metric_matches_baseline_json():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        base = json.load(f)
    assert bench.METRIC == base["metric"]
    assert {"c1", "c2", "c3", "c4"} <= set(bench.CONFIGS)


@pytest.mark.parametrize("kind,nx", [("stencil27", 8), ("poisson3d", 8), ("poisson2d", 16)])
def test_stencil_k_left_matches_oracle(kind, nx):
    A = {"stencil27": stencil.stencil27, "poisson3d": stencil.poisson3d, "poisson2d": stencil.poisson2d}[kind](nx)
    assert bench.stencil_k_left(kind, nx) == O.lower_bandwidth(A.row_ptr, A.col_idx)


def test_partitions_cover_rows():
    for key in ("c1", "c2", "c3"):
        cfg = bench.CONFIGS[key]
        n = bench.cfg_rows(cfg)
        for world in (1, 2, 8):
            slabs = bench.partition(cfg, world)
            assert slabs[0][0] == 0 and slabs[-1][1] == n
            assert all(b == c for (_, b), (c, _) in zip(slabs, slabs[1:]))
            assert all(a % cfg["sigma"] == 0 for a, _ in slabs)


def test_reference_arm_sample_runs(capsys):
    """The CPU reference arm on a tiny sample prints the contract's JSON line."""
    cfg = dict(bench.CONFIGS["c1"])

    class A:
        gpus, steps, warmup, ref_rows = 1, 1, 0, 4096
    os.environ.pop("RANK", None)
    r = bench.cpu_reference(cfg, 2, 4096, 1, 0)
    assert r["gbs"] > 0 and r["workers"] == 2 and r["nnz"] > 0
    bench.run_reference(A, cfg)
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    # the reference's own code when baseline/_ref is installed, else the oracle port
    want = "reference" if bench.reference_pkg() is not None else "port"
    assert line["cpu_baseline"]["kind"] == want and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["metric"] == bench.METRIC and line["higher_is_better"] is True


def test_bench_spawns_ranks_for_gpus_n():
    """`python bench.py --gpus 2` without torchrun launches 2 ranks itself (the driver's
    command form); the printed line reports the actual world size."""
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0", "--config", "c1", "--ref-rows", "4096"],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"


def test_cpu_path_reference_equals_oracle_on_a_slab():
    """The reference arm's slab trick (r0 empty rows, global k_left) reproduces the oracle's
    slab build with a row origin byte for byte, and the same REF SpMV."""
    import numpy as np
    if bench.reference_pkg() is None:
        pytest.skip("reference not installed in baseline/_ref")
    cfg = dict(bench.CONFIGS["c2"], nx=16)
    A, vals = bench._cpu_slab(cfg, 256, 1024)
    kl = bench.stencil_k_left("stencil27", 16)
    Pr = bench.CpuPath(cfg, A, vals, 256, kl)
    Po = bench.CpuPath(cfg, A, vals, 256, kl, prefer_reference=False)
    assert Pr.kind == "reference" and Po.kind == "port"
    assert np.array_equal(Pr.pack, Po.pack) and np.array_equal(Pr.offset, Po.offset)
    assert np.array_equal(Pr.perm, Po.perm) and Pr.counts == Po.counts
    x = np.random.default_rng(0).uniform(-1, 1, A.n_cols).astype(np.float16)
    assert np.array_equal(Pr.spmv(x).view(np.uint16), Po.spmv(x).view(np.uint16))
