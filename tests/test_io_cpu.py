"""Host-side I/O around the path, CPU only: .psell header validation, Matrix Market, CLI plumbing.

Pinned by fixtures written by the real reference (tests/golden/make_golden.py:
container_golden.*, mm_golden.json).  Every container error below is raised
before any device upload, so it runs without a GPU.
"""

import io
import json
import os

import numpy as np
import pytest

import paper_2604_13433_b200 as P
from paper_2604_13433_b200 import cli
from paper_2604_13433_b200.container import ContainerError, read_psell
from conftest import GOLDEN


@pytest.fixture(scope="module")
def golden_container():
    z = np.load(os.path.join(GOLDEN, "container_golden.npz"))
    with open(os.path.join(GOLDEN, "container_golden.json")) as f:
        return z, json.load(f)


def _corrupt(raw: bytes, name: str) -> bytes:
    """The corruptions of make_golden.container_fixture (reference tests/test_container.py:66-104)."""
    b = bytearray(raw)
    if name == "bad_magic":
        b[0] ^= 0xFF
    elif name == "truncated_payload":
        b = b[:-3]
    elif name == "truncated_header":
        b = b[:20]
    elif name == "unknown_codec":
        b[10] = 99
    elif name == "unknown_mode":
        b[11] = 7
    elif name == "invalid_format":
        b[8] = 16
    elif name == "count_mismatch":
        pos = 8 + 4 + 8 + 24
        b[pos:pos + 8] = (2 ** 40).to_bytes(8, "little")
    elif name == "offset_not_zero":
        pos = 8 + 4 + 8 + 7 * 8
        b[pos:pos + 8] = (5).to_bytes(8, "little")
    elif name == "empty":
        b = bytearray()
    return bytes(b)


@pytest.mark.parametrize("name", ["bad_magic", "truncated_payload", "truncated_header", "unknown_codec",
                                  "unknown_mode", "invalid_format", "count_mismatch", "offset_not_zero", "empty"])
def test_container_errors_match_reference(golden_container, name):
    z, meta = golden_container
    exc, msg = meta["errors"][name]
    data = _corrupt(z["small_bytes"].tobytes(), name)
    with pytest.raises(ContainerError) as ei:
        read_psell(io.BytesIO(data))
    assert type(ei.value).__name__ == exc and str(ei.value) == msg
    assert isinstance(ei.value, ValueError)


def test_container_errors_from_path(golden_container, tmp_path):
    z, _ = golden_container
    p = tmp_path / "t.psell"
    p.write_bytes(_corrupt(z["small_bytes"].tobytes(), "truncated_payload"))
    with pytest.raises(ContainerError, match="truncated"):
        read_psell(str(p))


@pytest.fixture(scope="module")
def golden_mm():
    with open(os.path.join(GOLDEN, "mm_golden.json")) as f:
        return json.load(f)


def test_matrix_market_read_matches_reference(golden_mm):
    for case in golden_mm:
        if case["error"] is not None:
            with pytest.raises(ValueError) as ei:
                P.load_matrix_market(case["text"].encode())
            assert [type(ei.value).__name__, str(ei.value)] == case["error"], case["text"][:80]
            continue
        co = P.load_matrix_market(case["text"].encode())
        assert (co.n_rows, co.n_cols) == (case["n_rows"], case["n_cols"])
        assert co.rows.tolist() == case["rows"] and co.cols.tolist() == case["cols"]
        assert [repr(v) for v in co.values.tolist()] == case["values"]
        buf = io.StringIO()
        P.write_matrix_market(co, buf)
        assert buf.getvalue() == case["written"]


def test_matrix_market_sources(golden_mm, tmp_path):
    txt = next(c["text"] for c in golden_mm if c["error"] is None)
    p = tmp_path / "a.mtx"
    p.write_text(txt)
    a, b, c = P.load_matrix_market(str(p)), P.load_matrix_market(io.StringIO(txt)), P.load_matrix_market(p)
    assert np.array_equal(a.values, b.values) and np.array_equal(a.cols, c.cols)


def _run(capsys, *argv):
    code = cli.main(list(argv))
    out, err = capsys.readouterr()
    return code, out, err


def test_cli_gen_info(capsys, tmp_path):
    p = str(tmp_path / "p.mtx")
    code, out, _ = _run(capsys, "gen", "--stencil", "poisson2d", "--dims", "3x3", p, "--json")
    assert code == 0 and out.count("\n") == 1
    rep = json.loads(out)
    assert rep == {"schema": 1, "stencil": "poisson2d", "dims": [3, 3], "n": 9, "nnz": 33, "out": p}
    code, out, _ = _run(capsys, "info", p, "--json")
    rep = json.loads(out)
    assert code == 0 and rep["symmetric"] is True and rep["nnz"] == 33
    assert rep["lower_bandwidth"] == rep["upper_bandwidth"] == 3
    code, out, _ = _run(capsys, "gen", "--stencil", "poisson3d", "--dims", "2", str(tmp_path / "q.mtx"), "--json")
    assert code == 0 and json.loads(out)["dims"] == [2, 2, 2] and json.loads(out)["n"] == 8


def test_cli_errors_go_to_stderr(capsys, tmp_path):
    code, out, err = _run(capsys, "gen", "--stencil", "poisson2d", "--dims", "3x3x3", str(tmp_path / "x.mtx"))
    assert code == 1 and out == "" and "dims" in err
    code, out, err = _run(capsys, "info", str(tmp_path / "missing.mtx"))
    assert code == 1 and out == "" and "ERROR" in err
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n")
    code, out, err = _run(capsys, "info", str(bad))
    assert code == 1 and "outside declared" in err


def test_cli_parser_defaults():
    p = cli.build_parser()
    a = p.parse_args(["spmv", "m.mtx"])
    assert (a.format, a.reps, a.warmup, a.x, a.c, a.sigma) == ("csr", 10000, 100, "ones", 32, 256)
    a = p.parse_args(["solve", "m.mtx"])
    assert (a.solver, a.backend, a.m_in, a.tol, a.scale, a.max_outer) == ("pcg", "csr64", 50, 1e-9, "sym", 1000)
    a = p.parse_args(["footprint", "m.mtx", "--sweep-d", "3..5"])
    assert a.sweep_d == (3, 5)
    assert cli._working_dtype("packsell-e8m14") == np.float32 and cli._working_dtype("sell16") == np.float16
    assert np.array_equal(cli._make_x("random:3", 4, np.float32),
                          np.random.Generator(np.random.PCG64(3)).random(4).astype(np.float32))
