"""GPU: .psell container straight to/from HBM, K6 backward error, bench_spmv, and the CLI.

Parity bar: container bytes identical to the reference's (container_golden.npz),
backward errors bit-identical to metrics.backward_error (metrics_golden.*), CLI
JSON schema and values as the reference CLI (reference tests/test_cli.py).
"""

import io
import json
import os

import numpy as np
import pytest

import paper_2604_13433_b200 as P
from paper_2604_13433_b200 import cli
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden_container():
    z = np.load(os.path.join(GOLDEN, "container_golden.npz"))
    with open(os.path.join(GOLDEN, "container_golden.json")) as f:
        return z, json.load(f)


def _csr(z, p, m):
    return P.CsrMatrix(m["n_rows"], m["n_cols"], z[p + "row_ptr"], z[p + "col_idx"], z[p + "values"])


def _equal(a, b):
    return (a.n_rows == b.n_rows and a.n_cols == b.n_cols and a.c == b.c and a.sigma == b.sigma
            and a.mode == b.mode and a.fmt == b.fmt and a.k_left == b.k_left and tuple(a.counts) == tuple(b.counts)
            and np.array_equal(a.offset, b.offset) and np.array_equal(a.pack, b.pack)
            and ((a.perm is None and b.perm is None)
                 or (a.perm is not None and b.perm is not None and a.perm.dtype == b.perm.dtype
                     and np.array_equal(a.perm, b.perm))))


def test_container_bytes_identical_to_reference(golden_container):
    z, meta = golden_container
    for i, m in enumerate(meta["cases"]):
        p = f"k{i}_"
        M = P.build_packsell(_csr(z, p, m), m["c"], m["sigma"], P.parse_format(m["preset"]), m["mode"])
        buf = io.BytesIO()
        P.write_psell(M, buf)  # words streamed straight out of HBM (no host pack cached yet)
        assert buf.getvalue() == z[p + "bytes"].tobytes(), i


def test_container_read_to_device_and_spmv(golden_container, tmp_path):
    z, meta = golden_container
    for i, m in enumerate(meta["cases"]):
        p = f"k{i}_"
        raw = z[p + "bytes"].tobytes()
        R = P.read_psell(io.BytesIO(raw))
        assert R.d_pack.is_cuda and R.d_offset.is_cuda
        M = P.build_packsell(_csr(z, p, m), m["c"], m["sigma"], P.parse_format(m["preset"]), m["mode"])
        assert _equal(M, R), i
        x = np.random.default_rng(i).uniform(-1, 1, M.n_cols).astype(np.float32)
        assert np.array_equal(P.packsell_spmv(M, x, ref_order=True), P.packsell_spmv(R, x, ref_order=True))
        f = tmp_path / f"m{i}.psell"
        P.write_psell(R, f)  # and back out again from a matrix that came in through the container
        assert f.read_bytes() == raw


def test_container_stable_and_perm_width(rng):
    from conftest import random_csr_arrays
    rp, ci, v = random_csr_arrays(rng, 600, 64, 0.05)
    A = P.CsrMatrix(600, 64, rp, ci, v)
    for sigma, dt in ((256, np.uint8), (512, np.uint16)):
        M = P.build_packsell(A, 8, sigma, P.parse_format("e8m20"), "implicit")
        b1, b2 = io.BytesIO(), io.BytesIO()
        P.write_psell(M, b1)
        _ = M.pack  # host copy cached: the second write takes the host path, same bytes
        P.write_psell(M, b2)
        assert b1.getvalue() == b2.getvalue()
        b1.seek(0)
        R = P.read_psell(b1)
        assert R.perm.dtype == dt and np.array_equal(R.perm, M.perm)


@pytest.fixture(scope="module")
def golden_metrics():
    z = np.load(os.path.join(GOLDEN, "metrics_golden.npz"))
    with open(os.path.join(GOLDEN, "metrics_golden.json")) as f:
        return z, json.load(f)


def test_backward_error_bitwise_vs_reference(golden_metrics):
    z, meta = golden_metrics
    for i, m in enumerate(meta):
        p = f"m{i}_"
        rp = z[p + "row_ptr"]
        A = P.CsrMatrix(len(rp) - 1, len(z[p + "x"]), rp, z[p + "col_idx"], z[p + "values"])
        assert P.backward_error(A, z[p + "x"], z[p + "y"]) == m["backward_error"], i
        assert P.inf_norm_matrix(A) == m["inf_norm"], i


def test_backward_error_reference_cases(rng):
    A = P.CsrMatrix(1, 1, [0, 1], [0], [1.0])
    assert P.backward_error(A, np.array([1.0]), np.array([1.0 + 2.0 ** -11])) == 2.0 ** -11
    with pytest.raises(ValueError, match="zero"):
        P.backward_error(A, np.zeros(1), np.ones(1))
    with pytest.raises(ValueError, match="dimension"):
        P.backward_error(A, np.ones(2), np.ones(1))
    assert np.isnan(P.backward_error(A, np.array([1.0]), np.array([np.nan])))
    from conftest import random_csr_arrays
    rp, ci, v = random_csr_arrays(rng, 50, 50, 0.2)
    B = P.CsrMatrix(50, 50, rp, ci, v)
    x = rng.uniform(-1, 1, 50)
    assert P.backward_error(B, x, P.csr_spmv(B, x)) == 0.0


def test_bench_spmv_reports(rng):
    from conftest import random_csr_arrays
    rp, ci, v = random_csr_arrays(rng, 300, 200, 0.04)
    A = P.CsrMatrix(300, 200, rp, ci, v)
    M = P.build_packsell(A, 32, 32, P.PackFormat(32, 1, "e8my"), "implicit")
    assert M.counts.n_dummy > 0
    x = np.ones(200, dtype=np.float32)
    rep = P.bench_spmv(M, x, reps=5, warmup=1, source=A)
    assert rep.format_name == "packsell-e8m21" and rep.elapsed_per_call > 0
    assert rep.gflops == pytest.approx(2 * A.nnz / rep.elapsed_per_call / 1e9)
    assert rep.y.dtype == np.float32 and rep.y.shape == (300,)
    assert rep.backward_error == P.backward_error(A, x, rep.y)
    assert rep.bytes_touched_estimate == 4 * M.n_stored + 8 * (M.n_slices + 1) + 300 + 4 * M.n_stored + 4 * 300
    assert set(rep.to_dict()) == {"format", "reps", "warmup", "elapsed_per_call", "gflops", "backward_error",
                                  "bytes_touched_estimate"}
    r1 = P.bench_spmv(A, x.astype(np.float64), reps=2, warmup=0)
    S = P.build_sell(A, 4, 8, "implicit")
    r2 = P.bench_spmv(S, x.astype(np.float64), reps=2, warmup=0, source=A)
    assert r1.format_name == "csr" and r2.format_name == "sell64"
    assert np.array_equal(r1.y, r2.y) and r1.backward_error == r2.backward_error
    with pytest.raises(ValueError):
        P.bench_spmv(M, x, reps=1, warmup=0)
    with pytest.raises(ValueError):
        P.bench_spmv(A, x, reps=0)


def _run(capsys, *argv):
    code = cli.main(list(argv))
    out, err = capsys.readouterr()
    return code, out, err


@pytest.fixture
def poisson_file(tmp_path, capsys):
    p = str(tmp_path / "p.mtx")
    _run(capsys, "gen", "--stencil", "poisson2d", "--dims", "12x12", p)
    return p


def test_cli_convert_round_trip(capsys, tmp_path, poisson_file):
    out = str(tmp_path / "p.psell")
    code, o, _ = _run(capsys, "convert", poisson_file, out, "--codec", "e8my", "--d", "8", "--json")
    rep = json.loads(o)
    assert code == 0 and rep["format"] == "e8m14" and rep["nnz"] == 12 * 12 * 5 - 4 * 12
    A = P.to_csr(P.load_matrix_market(poisson_file))
    M = P.build_packsell(A, 32, 256, P.parse_format("e8m14"), "implicit")
    buf = io.BytesIO()
    P.write_psell(M, buf)
    with open(out, "rb") as f:
        assert f.read() == buf.getvalue()
    code, o, _ = _run(capsys, "convert", poisson_file, out, "--codec", "fp16", "--d", "14")
    assert code == 1


def test_cli_spmv_and_container(capsys, tmp_path, poisson_file):
    code, o, _ = _run(capsys, "spmv", poisson_file, "--format", "packsell-fp16", "--reps", "20", "--warmup", "2",
                      "--x", "random:1")
    rep = json.loads(o)
    assert code == 0 and rep["format"] == "packsell-fp16" and rep["gflops"] > 0 and "footprint_ratio" in rep
    assert rep["backward_error"] < 1e-3
    code, o, _ = _run(capsys, "spmv", poisson_file, "--reps", "3", "--warmup", "0")
    rep = json.loads(o)
    assert code == 0 and rep["format"] == "csr" and rep["backward_error"] == 0.0
    out = str(tmp_path / "p.psell")
    _run(capsys, "convert", poisson_file, out)
    code, o, _ = _run(capsys, "spmv", out, "--reps", "3", "--warmup", "1")
    rep = json.loads(o)
    assert code == 0 and rep["format"] == "packsell-fp16" and rep["backward_error"] <= 2.0 ** -10
    code, o, e = _run(capsys, "spmv", poisson_file, "--reps", "0")
    assert code == 1 and o == "" and "reps" in e


def test_cli_footprint_and_solve(capsys, tmp_path, poisson_file):
    code, o, _ = _run(capsys, "footprint", poisson_file, "--sweep-d", "2..4", "--json")
    rep = json.loads(o)
    assert code == 0 and [r["d"] for r in rep["rows"]] == [2, 3, 4] and rep["dense_band_limit_ratio"] == 0.5
    dummies = [r["n_dummy"] for r in rep["rows"]]
    assert dummies == sorted(dummies, reverse=True)
    code, o, e = _run(capsys, "footprint", poisson_file, "--codec", "fp16", "--sweep-d", "1..3")
    assert code == 1 and "D=15" in e
    code, o, _ = _run(capsys, "solve", poisson_file, "--solver", "pcg", "--tol", "1e-9")
    rep = json.loads(o)
    assert code == 0 and rep["converged"] and rep["final_true_relres"] < 1e-9
    code, o, _ = _run(capsys, "solve", poisson_file, "--solver", "iocg", "--backend", "packsell-e8m14",
                      "--m-in", "10", "--residual-csv", str(tmp_path / "r.csv"))
    rep = json.loads(o)
    assert code == 0 and rep["converged"] and rep["total_inner_iters"] == 10 * rep["outer_iters"]
    lines = (tmp_path / "r.csv").read_text().splitlines()
    assert lines[0] == "iteration,relative_residual" and len(lines) == len(rep["residual_history"]) + 1
    code, o, e = _run(capsys, "solve", poisson_file, "--max-outer", "2")
    assert code == 1 and json.loads(o)["converged"] is False and "did not converge" in e


def test_integration_ctypes_stub_runs():
    """The reference-side ctypes binding shown in INTEGRATION.md §3 works as written."""
    import os
    import re
    import types
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "INTEGRATION.md")).read()
    sec = text[text.index("## 3. The C ABI directly"):]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    code = code.replace('ctypes.CDLL("paper_2604_13433_b200/libpsell.so")',
                        'ctypes.CDLL(os.path.join(ROOT, "paper_2604_13433_b200", "libpsell.so"))')
    ns = {"os": os, "ROOT": root}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    rng = np.random.default_rng(3)
    from conftest import random_csr_arrays
    rp, ci, v = random_csr_arrays(rng, 300, 280, 0.05)
    A = P.CsrMatrix(300, 280, rp, ci, v)
    M = P.build_packsell(A, 32, 256, P.parse_format("e8m14"), "implicit")
    ref_like = types.SimpleNamespace(fmt=M.fmt, c=M.c, sigma=M.sigma, mode=M.mode, n_rows=M.n_rows,
                                     n_cols=M.n_cols, k_left=M.k_left, counts=M.counts, pack=M.pack,
                                     offset=M.offset, perm=M.perm)
    x = rng.uniform(-1, 1, 280).astype(np.float32)
    y = ns["packsell_spmv_b200"](ref_like, x)
    assert np.array_equal(y, P.packsell_spmv(M, x))


def test_footprint_bits_vs_reference():
    """footprint_bits (packed.py:306-327) equals the reference on 15 fixtures (all modes, C, sigma, codecs)."""
    z = np.load(os.path.join(GOLDEN, "footprint_golden.npz"))
    with open(os.path.join(GOLDEN, "footprint_golden.json")) as f:
        meta = json.load(f)
    for i, m in enumerate(meta):
        p = f"f{i}_"
        A = P.CsrMatrix(m["n_rows"], m["n_cols"], z[p + "row_ptr"], z[p + "col_idx"], z[p + "values"])
        M = P.build_packsell(A, m["c"], m["sigma"], P.parse_format(m["preset"]), m["mode"])
        fp = P.footprint_bits(M)
        assert (fp.pack_bits, fp.sell_equiv_bits) == (m["pack_bits"], m["sell_equiv_bits"]), i
        assert fp.ratio == m["ratio"], i


def test_host_device_staging_round_trip():
    """_dev.upload's threaded page-locked path (>= 16 MiB, ragged chunk tail, unsigned
    types re-viewed as signed, `out=`) and download's page-locked view: bit-exact."""
    import torch
    from paper_2604_13433_b200 import _dev
    rng = np.random.default_rng(21)
    for dt, n in ((np.float64, 5_000_003), (np.uint32, 4_194_305), (np.float16, 9_000_001)):
        a = (rng.standard_normal(n) * 100).astype(dt) if dt != np.uint32 else rng.integers(0, 2**32, n, dtype=np.uint32)
        t = _dev.upload(a)
        assert t.is_cuda and t.numel() == n
        back = _dev.download(t, dt)
        assert back.dtype == dt and np.array_equal(back.view(np.uint8), a.view(np.uint8))
        out = torch.empty_like(t)
        assert _dev.upload(a, out=out) is out and torch.equal(out, t)
    with pytest.raises(ValueError):
        _dev.upload(np.zeros(5_000_000), out=torch.empty(10, dtype=torch.float64, device="cuda"))


def _corrupt(M, *, pack=None, perm=None):
    """A .psell byte string of M with its pack / perm replaced (header and offsets kept)."""
    buf = io.BytesIO()
    P.write_psell(M, buf)
    raw = bytearray(buf.getvalue())
    hdr = len(P.container.header_bytes(M)) + 8 * (M.n_slices + 1)
    if perm is not None:
        pb = np.ascontiguousarray(perm).tobytes()
        raw[hdr:hdr + len(pb)] = pb
    if pack is not None:
        start = hdr + (M.perm.dtype.itemsize * M.n_rows if M.mode == "implicit" else 0)
        pk = np.ascontiguousarray(pack).tobytes()
        raw[start:start + len(pk)] = pk
    return io.BytesIO(bytes(raw))


def test_container_rejects_streams_the_device_cannot_run(rng):
    """a container whose perm leaves its sigma-block or whose deltas run past
    n_cols is rejected with ContainerError instead of reaching the kernels."""
    from conftest import random_csr_arrays
    rp, ci, v = random_csr_arrays(rng, 300, 280, 0.05)
    A = P.CsrMatrix(300, 280, rp, ci, v)
    M = P.build_packsell(A, 32, 64, P.parse_format("fp16"), "implicit")
    assert _equal(P.read_psell(_corrupt(M)), M)  # untouched bytes read back
    bad_perm = M.perm.copy()
    bad_perm[-1] = 200  # last sigma-block holds 300 - 256 = 44 rows
    with pytest.raises(P.ContainerError, match="perm"):
        P.read_psell(_corrupt(M, perm=bad_perm))
    pack = M.pack.copy()
    real = np.nonzero(pack & 1)[0][0]
    pack[real] |= np.uint32(0x7FFF) << np.uint32(1)  # delta 32767: far past n_cols
    with pytest.raises(P.ContainerError, match="beyond n_cols"):
        P.read_psell(_corrupt(M, pack=pack))


def test_fp16_with_64bit_words_rejected_on_device():
    """PackFormat(64, 47, 'fp16') is a valid reference format whose reference decode reads
    its values from delta bits (codec.py:242); the device path refuses it loudly."""
    A = P.poisson2d(8)
    fmt = P.PackFormat(64, 47, "fp16")
    with pytest.raises(ValueError, match="32-bit words"):
        P.build_packsell(A, 32, 64, fmt, "implicit")
