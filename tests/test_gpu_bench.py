"""bench.py end to end on the GPU at small sizes: the JSON line the driver parses carries every
key of the contract (roofline, cpu_baseline, parity, e2e, clocks, pcg) and a bitwise parity
block, so a regression in the benchmark harness shows up in the GPU suite, not at round end."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_small():
    d = _run("--config", "c1", "--steps", "5", "--warmup", "3", "--pcg-nx", "32", "--cpu-rows", "65536")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks", "pcg"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["achieved"] > 0 and r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["parity"]["status"] == "bitwise"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= d["steps"]
    p = d["pcg"]
    assert p["iocg"]["converged"] and p["fp64_pcg"]["converged"]
    assert p["iocg"]["inner_iters"] == 50 * p["iocg"]["outer_iters"]


def test_bench_reference_arm_small():
    d = _run("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1", "--ref-rows", "32768")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0
