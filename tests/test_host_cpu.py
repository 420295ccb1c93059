"""Host-side logic and the C ABI surface (CPU only, no kernel launches)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2604_13433_b200 as P
from paper_2604_13433_b200 import _lib
from paper_2604_13433_b200.sell import _check_layout_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _raises_like(fn, golden):
    if golden["exc"] is None:
        fn()
        return
    with pytest.raises(Exception) as ei:
        fn()
    assert type(ei.value).__name__ == golden["exc"]
    assert str(ei.value) == golden["msg"]


@pytest.mark.parametrize("w,d,cd", [(16, 4, "fp16"), (32, 0, "e8my"), (32, 31, "e8my"), (32, 14, "fp16"),
                                    (64, 15, "e8my"), (32, 22, "e8my"), (32, 15, "fp32embed"),
                                    (64, 40, "fp32embed"), (32, 15, "bogus")])
def test_packformat_validation_messages(golden_errors, w, d, cd):
    _raises_like(lambda: P.PackFormat(w, d, cd), golden_errors[f"fmt_{w}_{d}_{cd}"])


@pytest.mark.parametrize("name", ["q5", "e8mx", "E8M14", "FP16"])
def test_parse_format(golden_errors, name):
    _raises_like(lambda: P.parse_format(name), golden_errors[f"parse_{name}"])


def test_presets():
    assert P.parse_format("fp16") == P.PackFormat(32, 15, "fp16")
    assert P.parse_format("e8m14") == P.PackFormat(32, 8, "e8my")
    assert P.parse_format("e8m14").name == "e8m14"
    assert P.parse_format("fp32embed").word_dtype == np.uint64
    f = P.PackFormat()
    assert (f.max_delta, f.max_dummy_delta, f.v) == (2 ** 15 - 1, 2 ** 31 - 1, 16)


@pytest.mark.parametrize("name,c,sigma,mode", [("bad_mode", 1, 1, "sorted"), ("bad_c", 0, 1, "none"),
                                               ("bad_sigma", 4, 6, "implicit"), ("big_sigma", 4, 65540, "implicit")])
def test_layout_param_messages(golden_errors, name, c, sigma, mode):
    _raises_like(lambda: _check_layout_params(c, sigma, mode), golden_errors[name])


def test_leftmost_offset_and_delta_stream():
    assert P.leftmost_offset(300, 256, 10) == 246
    assert P.leftmost_offset(300, 256, 256) == 0
    fmt = P.PackFormat(32, 2, "e8my")
    s = P.build_delta_stream([1, 5], [1.0, 2.0], 0, fmt)
    assert s == [P.DeltaEntry(1, 1.0), P.DeltaEntry(4, None), P.DeltaEntry(0, 2.0)]
    gap = 2 ** 31 + 5
    s = P.build_delta_stream([0, gap], [1.0, 2.0], 0, P.PackFormat())
    assert sum(e.delta for e in s if e.value is None) == gap


def test_host_generators_shapes():
    A = P.stencil27(6)
    assert A.nnz == (3 * 6 - 2) ** 3
    assert np.all(np.diff(A.col_idx[A.row_ptr[0]:A.row_ptr[1]]) > 0)
    assert np.all(A.values[A.col_idx == np.repeat(np.arange(A.n_rows), A.row_lengths())] == 26.0)
    B = P.poisson3d(5)
    assert B.nnz == 5 ** 3 * 7 - 6 * 5 ** 2
    C = P.powerlaw(4096, seed=3)
    assert C.n_rows == 4096 and C.nnz > 4096
    lens = C.row_lengths()
    assert lens.max() > 10 * lens.mean()


def test_csr_validation():
    with pytest.raises(ValueError):
        P.CsrMatrix(2, 2, [0, 1], [0], [1.0])
    with pytest.raises(ValueError):
        P.CsrMatrix(2, 2, [0, 2, 1], [0, 1], [1.0, 2.0])


def _header_functions():
    src = open(os.path.join(ROOT, "include", "psell.h")).read()
    return sorted(set(re.findall(r"PSELL_API\s+[\w\s\*]+?\b(psell_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    """libpsell.so loads (no GPU needed) and exports every function include/psell.h declares."""
    lib = ctypes.CDLL(_lib.LIB_PATH)
    decl = _header_functions()
    assert len(decl) >= 30
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(_lib.exported_symbols()) == decl
    l2 = _lib.load(require_gpu=False)
    assert l2.psell_abi_version() == 1
    assert b"sm_100a" in l2.psell_version()


def test_workspace_sizing_is_host_only():
    l = _lib.load(require_gpu=False)
    d = _lib.PsellDesc()
    d.w, d.d, d.codec, d.c, d.sigma, d.mode = 32, 15, 0, 32, 256, 2
    d.n_rows, d.n_cols, d.row0, d.k_left, d.nnz = 1 << 24, 1 << 24, 0, -1, 449455096
    ws = l.psell_build_workspace_bytes(d)
    assert 3 * 4 * (1 << 24) <= ws < 64 * (1 << 24)
    # persistent TMA grid: SMs x CTAs/SM (148 x 6 when no device is visible)
    assert 1 <= l.psell_spmv_dot_partials(d, 0) <= (1 << 24) // 256


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.encode_values(P.PackFormat(), [1.0])


def test_multiply_high_division_identity():
    """Host mirror of magic_div / fast_div (csrc/spmv.cu): n / d == (umulhi(n, m) + n) >> l for n < 2^31."""
    rng = np.random.default_rng(5)
    for d in list(range(1, 300)) + [32 * k for k in range(1, 2048, 7)] + [65535, 65536]:
        l = 0
        while (1 << l) < d:
            l += 1
        m = ((1 << 32) * ((1 << l) - d)) // d + 1
        assert m < (1 << 32)
        ns = np.concatenate([np.arange(0, 4096), rng.integers(0, 2 ** 31, 2000),
                             [2 ** 31 - 1, 2 ** 31 - 2, d - 1, d, d + 1, 2 ** 31 - 1 - (2 ** 31 - 1) % d]])
        for n in ns.tolist():
            assert (((n * m) >> 32) + n) >> l == n // d, (d, n)


# packsell 0.1.0 public names (reference pkg/src/packsell/__init__.py:24-45)
REFERENCE_ALL = [
    "CodecError", "E8MY", "FP16", "FP32EMBED", "PackFormat", "UnpackedEntry",
    "decode_value", "encode_value", "pack", "parse_format", "quantize", "unpack",
    "ContainerError", "read_psell", "write_psell",
    "CooMatrix", "CsrMatrix", "MatrixFormatError", "MatrixStats",
    "compute_stats", "csr_spmv", "load_matrix_market", "permute_rows",
    "row_sum_scale", "sym_diag_scale", "to_coo", "to_csr", "write_matrix_market",
    "SpmvReport", "backward_error", "bench_spmv",
    "DeltaEntry", "FootprintReport", "PackSellMatrix", "StorageCounts",
    "build_delta_stream", "build_packsell", "footprint_bits",
    "leftmost_offset", "packsell_spmv", "packsell_to_csr",
    "SellMatrix", "build_sell", "row_sort_order", "sell_spmv",
    "SolveConfig", "SolveReport", "SpmvBackend", "fcg", "iocg",
    "make_backend", "make_rhs_and_x0", "pcg",
    "poisson2d", "poisson3d",
    "__version__",
]


def test_public_api_covers_reference():
    """Every public name of the reference package exists here (drop-in import)."""
    missing = [n for n in REFERENCE_ALL if not hasattr(P, n)]
    assert not missing, missing
    assert P.__version__ == "0.1.0"
    from paper_2604_13433_b200 import cli, container, metrics, sell
    assert callable(cli.main) and callable(container.read_psell) and callable(metrics.bench_spmv)
    assert sell.build_sell is P.build_sell


@pytest.mark.parametrize("lang,std", [("c", "c99"), ("c++", "c++17")])
def test_header_is_plain_c_abi(lang, std, tmp_path):
    """include/psell.h compiles warning-free as C99 and C++17 (the boundary is a C ABI)."""
    import shutil
    import subprocess
    cc = shutil.which("gcc" if lang == "c" else "g++")
    if cc is None:
        pytest.skip("no host compiler")
    src = tmp_path / ("t.c" if lang == "c" else "t.cc")
    src.write_text('#include "psell.h"\nint main(void) { psell_desc d; psell_error e; (void)d; (void)e; '
                   'return psell_abi_version() == PSELL_ABI_VERSION ? 0 : 1; }\n')
    r = subprocess.run([cc, "-std=" + std, "-Wall", "-Wextra", "-Werror", "-fsyntax-only",
                        "-I", os.path.join(ROOT, "include"), str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_plain_c_program_links_and_calls_the_abi(tmp_path):
    """A C program (no Python) links libpsell.so and calls its host-only entry points."""
    import shutil
    import subprocess
    cc = shutil.which("gcc")
    if cc is None:
        pytest.skip("no host compiler")
    src = tmp_path / "abi.c"
    src.write_text(r'''
#include <stdio.h>
#include "psell.h"
int main(void) {
  psell_desc d = {32, 15, PSELL_FP16, 32, 256, PSELL_MODE_IMPLICIT, 1 << 20, 1 << 20, 0, -1, 27000000};
  size_t ws = psell_build_workspace_bytes(&d);
  printf("%s %zu\n", psell_version(), ws);
  return (psell_abi_version() == PSELL_ABI_VERSION && ws > 0) ? 0 : 1;
}
''')
    libdir = os.path.dirname(_lib.LIB_PATH)
    exe = tmp_path / "abi"
    r = subprocess.run([cc, "-std=c99", "-Wall", "-I", os.path.join(ROOT, "include"), str(src), "-L", libdir,
                        "-lpsell", "-Wl,-rpath," + libdir, "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    env = dict(os.environ)
    import torch  # noqa: F401  (makes the bundled libcudart discoverable like the Python path does)
    cudart = [p for p in os.environ.get("LD_LIBRARY_PATH", "").split(":") if p]
    try:
        import nvidia.cuda_runtime as ncr
        cudart.append(os.path.join(os.path.dirname(ncr.__file__), "lib"))
    except ImportError:
        pass
    cudart.append("/usr/local/cuda/lib64")
    env["LD_LIBRARY_PATH"] = ":".join(cudart)
    run = subprocess.run([str(exe)], capture_output=True, text=True, env=env)
    assert run.returncode == 0, run.stderr
    assert "sm_100a" in run.stdout


def test_powerlaw_far_rows_properties():
    """Config-4b host generator: sorted unique columns in [0, n), Pareto row lengths, the
    lower bandwidth ~ n (far entries push k_left so every d_i = 0)."""
    import oracle as O
    from paper_2604_13433_b200.stencil import powerlaw_far_k_left, powerlaw_far_rows
    n = 1 << 16
    A = powerlaw_far_rows(n, 9)
    rp, ci = A.row_ptr, A.col_idx
    assert rp[0] == 0 and rp[-1] == A.nnz and np.all(np.diff(rp) >= 1)
    assert ci.min() >= 0 and ci.max() < n
    row = np.repeat(np.arange(n), np.diff(rp))
    same = row[1:] == row[:-1]
    assert np.all(ci[1:][same] > ci[:-1][same])
    kl = O.lower_bandwidth(rp, ci)
    assert kl == powerlaw_far_k_left(n, 9) and kl > n - 4096
    B = powerlaw_far_rows(n, 9, 1000, 3000)
    assert np.array_equal(B.col_idx, ci[rp[1000]:rp[3000]]) and np.array_equal(B.values, A.values[rp[1000]:rp[3000]])


def test_fused_peer_entry_points_validate_before_launch():
    """The fused distributed entry points refuse a bad peer group on the host (no launch,
    no CUDA call): ranks out of range, G outside [1, 64] (or < 2 for the halo push), missing
    arena table or halo ranges."""
    import ctypes
    l = _lib.load(require_gpu=False)
    EARG = 4
    lo = (ctypes.c_int64 * 2)(0, 0)
    hi = (ctypes.c_int64 * 2)(4, 0)
    dst = (ctypes.c_int32 * 2)(1, 0)
    fake = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    # halo push: G must be >= 2, rank in range, peers non-null, <= 2 ranges, dst a peer
    assert l.psell_ipcg_direction_x_push(8, fake, fake, fake, fake, fake, 1, 0, fake, 0, 0, 1, lo, hi, dst, 1, None) == EARG
    assert l.psell_ipcg_direction_x_push(8, fake, fake, fake, fake, fake, 2, 2, fake, 0, 0, 1, lo, hi, dst, 1, None) == EARG
    assert l.psell_ipcg_direction_x_push(8, fake, fake, fake, fake, fake, 2, 0, None, 0, 0, 1, lo, hi, dst, 1, None) == EARG
    assert l.psell_ipcg_direction_x_push(8, fake, fake, fake, fake, fake, 2, 0, fake, 0, 0, 3, lo, hi, dst, 1, None) == EARG
    assert l.psell_ipcg_direction_x_push(8, fake, fake, fake, fake, fake, 2, 1, fake, 0, 0, 1, lo, hi, dst, 1, None) == EARG
    # the fused dot all-reduce of the update: same group checks
    assert l.psell_ipcg_update_beta_peer(8, None, fake, fake, fake, fake, None, fake, fake, fake, fake,
                                         65, 0, fake, 1, None) == EARG
    assert l.psell_ipcg_update_beta_peer(8, None, fake, fake, fake, fake, None, fake, fake, fake, fake,
                                         2, 0, None, 1, None) == EARG
    assert l.psell_ipcg_update_beta_peer(8, None, fake, fake, fake, fake, None, fake, fake, fake, None,
                                         2, 0, fake, 1, None) == EARG
    # the FP64 PCG fused entry points: missing scalars / gate / ticket
    assert l.psell_pcg_update_status(8, fake, fake, fake, fake, None, fake, 1.0, 1e-9, fake, fake, fake, None) == EARG
    err = _lib.PsellError()
    assert l.psell_csr_spmv_dot_alpha(8, fake, fake, fake, fake, fake, fake, fake, None, fake, fake, None,
                                      ctypes.byref(err)) == EARG
    d = _lib.PsellDesc()
    d.w, d.d, d.codec, d.c, d.sigma, d.mode = 32, 8, 1, 32, 256, 2
    d.n_rows, d.n_cols, d.row0, d.k_left, d.nnz = 4096, 4096, 0, 256, 28672
    for G, rank, peers in ((0, 0, fake), (2, 2, fake), (2, 0, None), (65, 0, fake)):
        assert l.psell_spmv_dot_alpha_peer(d, fake, fake, fake, fake, fake, fake, fake, fake, fake, fake, 4, G, rank,
                                           peers, 1, None, ctypes.byref(err)) == EARG, (G, rank)
