"""GPU parity: the CUDA path (through the C ABI) vs the reference fixtures and the oracle.

Bar: pack / offset / perm / k_left / counts byte-identical;
REF_ORDER SpMV bitwise equal to the reference; production FMA SpMV within
    e_rel = ||y - y_ref||_inf / (||A_q||_inf ||x||_inf) <= 2 * L_max * 2^-24  (f32 / f64 x),
    e_rel <= 2^-11 + 2 * L_max * 2^-24 vs the f32-widened reference       (f16 x),
with L_max the maximum stored words per row.
"""

import numpy as np
import pytest

import oracle as O
import paper_2604_13433_b200 as P
from conftest import case_csr, golden_x, random_csr_arrays

pytestmark = pytest.mark.gpu


def _csr(z, i, m):
    rp, ci, v = case_csr(z, i)
    return P.CsrMatrix(m["n_rows"], m["n_cols"], rp, ci, v)


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def test_build_bit_exact_vs_reference(golden_build):
    z, meta = golden_build
    for i, m in enumerate(meta):
        A = _csr(z, i, m)
        M = P.build_packsell(A, m["c"], m["sigma"], P.parse_format(m["preset"]), m["mode"],
                             _k_left_override=m["k_left_override"])
        assert M.pack.dtype == z[f"c{i}_pack"].dtype
        assert np.array_equal(M.pack, z[f"c{i}_pack"]), i
        assert np.array_equal(M.offset, z[f"c{i}_offset"]), i
        if m["perm_dtype"]:
            assert M.perm.dtype.name == m["perm_dtype"] and np.array_equal(M.perm, z[f"c{i}_perm"]), i
        else:
            assert M.perm is None
        assert M.k_left == m["k_left"] and list(M.counts) == m["counts"], i
        assert (M.n_slices, M.n_stored) == (m["n_slices"], m["n_stored"])


def test_decode_vs_reference(golden_build):
    z, meta = golden_build
    for i, m in enumerate(meta):
        M = P.build_packsell(_csr(z, i, m), m["c"], m["sigma"], P.parse_format(m["preset"]), m["mode"],
                             _k_left_override=m["k_left_override"])
        R = P.packsell_to_csr(M)
        assert np.array_equal(R.row_ptr, z[f"c{i}_dec_row_ptr"]), i
        assert np.array_equal(R.col_idx, z[f"c{i}_dec_col_idx"]), i
        assert np.array_equal(_bits(R.values), _bits(z[f"c{i}_dec_values"])), i


def test_spmv_ref_order_bitwise_and_fma_tolerance(golden_build):
    z, meta = golden_build
    for i, m in enumerate(meta):
        A = _csr(z, i, m)
        fmt = P.parse_format(m["preset"])
        M = P.build_packsell(A, m["c"], m["sigma"], fmt, m["mode"], _k_left_override=m["k_left_override"])
        lmax = max(1, int(np.max(np.diff(M.offset) // m["c"])) if M.n_slices else 1)
        aq = np.abs(P.quantize(fmt, A.values)) if A.nnz else np.zeros(0)
        rows = np.repeat(np.arange(A.n_rows), A.row_lengths())
        anorm = np.bincount(rows, aq, minlength=A.n_rows).max() if A.nnz else 0.0
        for dt in (np.float16, np.float32, np.float64):
            x = golden_x(i, m["n_cols"], dt)
            want = z[f"c{i}_y_{np.dtype(dt).name}"]
            y = P.packsell_spmv(M, x, ref_order=True)
            assert y.dtype == want.dtype and np.array_equal(_bits(y), _bits(want)), (i, dt)
            yf = P.packsell_spmv(M, x)
            assert yf.dtype == want.dtype
            if A.nnz == 0 or anorm == 0:
                assert not np.any(yf)
                continue
            xw = x.astype(np.float32) if dt == np.float16 else x
            ref = P.packsell_spmv(M, xw, ref_order=True).astype(np.float64)
            den = anorm * max(np.abs(x.astype(np.float64)).max(), 1e-300)
            err = np.abs(yf.astype(np.float64) - ref).max() / den
            bound = 2 * lmax * 2.0 ** -24 + (2.0 ** -11 if dt == np.float16 else 0.0)
            assert err <= bound, (i, dt, err, bound)


def test_csr_spmv_bitwise(golden_build):
    z, meta = golden_build
    for i, m in enumerate(meta):
        A = _csr(z, i, m)
        for dt in (np.float16, np.float32, np.float64):
            x = golden_x(i, m["n_cols"], dt)
            y = P.csr_spmv(A, x, dt)
            assert np.array_equal(_bits(y), _bits(z[f"c{i}_csr_{np.dtype(dt).name}"])), (i, dt)


def test_csr_spmv_pipelined_bitwise_large():
    """K4's persistent path at a size with many more 256-row blocks than resident
    CTAs (each shared-memory stage refilled ~200 times), empty rows, and blocks
    whose entries exceed one stage (the synchronous fallback): bitwise vs the oracle."""
    rng = np.random.default_rng(7)
    n = 300_000
    lens = rng.integers(0, 12, n)
    lens[rng.integers(0, n, 200)] = rng.integers(300, 3000, 200)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = rng.integers(0, n, int(rp[-1])).astype(np.int32)
    v = rng.standard_normal(int(rp[-1]))
    A = P.CsrMatrix(n, n, rp, ci, v)
    for dt in (np.float32, np.float64):
        x = rng.standard_normal(n).astype(dt)
        y = P.csr_spmv(A, x, dt)
        assert np.array_equal(_bits(y), _bits(O.csr_spmv(rp, ci, v, x, dt))), dt


def test_csr_spmv_dot_fused():
    """psell_csr_spmv_dot (FP64 PCG's q = A p with p.q): y bitwise equal to csr_spmv,
    the dot within FP64 summation error of the exact one, identical run to run."""
    import torch
    from paper_2604_13433_b200 import _lib
    rng = np.random.default_rng(8)
    n = 250_000
    lens = rng.integers(0, 10, n)
    lens[rng.integers(0, n, 50)] = 2500
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = rng.integers(0, n, int(rp[-1])).astype(np.int32)
    A = P.CsrMatrix(n, n, rp, ci, rng.standard_normal(int(rp[-1])))
    x = rng.standard_normal(n)
    want = O.csr_spmv(rp, ci, A.values, x, np.float64)
    D = A.to_device()
    xd = torch.tensor(x, device="cuda")
    outs = []
    for _ in range(2):
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        parts = torch.zeros(8192, dtype=torch.float64, device="cuda")
        dot = torch.zeros(1, dtype=torch.float64, device="cuda")
        err = _lib.PsellError()
        rc = _lib.lib().psell_csr_spmv_dot(n, _lib.ptr(D.row_ptr), _lib.ptr(D.col_idx), _lib.ptr(D.values),
                                           xd.data_ptr(), y.data_ptr(), xd.data_ptr(), parts.data_ptr(),
                                           dot.data_ptr(), _lib.stream_handle(), err)
        _lib.check(rc, err)
        assert np.array_equal(_bits(y.cpu().numpy()), _bits(want))
        outs.append(float(dot.item()))
    exact = float(np.sum(x * want))
    assert abs(outs[0] - exact) <= 1e-12 * float(np.sum(np.abs(x * want)))
    assert outs[0] == outs[1]


def test_errors_match_reference(golden_errors):
    def check(name, fn):
        g = golden_errors[name]
        if g["exc"] is None:
            fn()
            return
        with pytest.raises(Exception) as ei:
            fn()
        assert type(ei.value).__name__ == g["exc"], name
        assert str(ei.value) == g["msg"], name

    fp16, e14, e20, f32 = (P.parse_format(s) for s in ("fp16", "e8m14", "e8m20", "fp32embed"))
    A = P.to_csr(P.CooMatrix(3, 300, [0, 1, 2], [0, 0, 1], [1.0, 2.0, 3.0]))
    check("first_gap", lambda: P.build_packsell(A, 1, 1, fp16, "implicit", _k_left_override=0))
    B = P.to_csr(P.CooMatrix(600, 600, [300, 301, 599], [0, 3, 10], [1.0, 2.0, 3.0]))
    check("first_gap_argmin", lambda: P.build_packsell(B, 4, 8, e14, "implicit", _k_left_override=5))
    C = P.CsrMatrix(2, 5, [0, 2, 3], [0, 3, 1], [1.0, np.nan, np.inf])
    check("nonfinite", lambda: P.build_packsell(C, 1, 1, fp16, "none"))
    D = P.CsrMatrix(2, 5, [0, 2, 3], [0, 3, 1], [1.0, 7e4, 1e6])
    check("overflow_fp16", lambda: P.build_packsell(D, 1, 1, fp16, "none"))
    E = P.CsrMatrix(2, 5, [0, 2, 3], [0, 3, 1], [1.0, 3.5e38, 1e300])
    check("overflow_e8m20", lambda: P.build_packsell(E, 1, 1, e20, "none"))
    check("overflow_fp32", lambda: P.build_packsell(E, 1, 1, f32, "none"))
    F = P.CsrMatrix(2, 5, [0, 2, 3], [0, 3, 1], [1e6, np.nan, 1.0])
    check("nonfinite_before_overflow", lambda: P.build_packsell(F, 1, 1, fp16, "none"))
    check("layout_before_codec", lambda: P.build_packsell(
        P.CsrMatrix(2, 9, [0, 1, 2], [0, 0], [np.nan, 1.0]), 1, 1, fp16, "implicit", _k_left_override=0))
    G = P.to_csr(P.CooMatrix(2, 2 ** 31 - 1, [0, 0], [0, 2 ** 31 - 2], [1.0, 2.0]))
    check("no_gap_range_w32", lambda: P.build_packsell(G, 1, 1, fp16, "none"))
    check("bad_mode", lambda: P.build_packsell(A, 1, 1, fp16, "sorted"))
    check("bad_sigma", lambda: P.build_packsell(A, 4, 6, fp16, "implicit"))
    check("encode_nan", lambda: P.encode_values(e14, [1.0, float("nan")]))
    check("encode_over", lambda: P.encode_values(fp16, [1.0, 2.0, -1e9]))
    check("spmv_len", lambda: P.packsell_spmv(P.build_packsell(A, 1, 1, fp16, "none"), np.ones(3, np.float32)))


@pytest.mark.parametrize("name", ["fp16", "fp32embed"] + [f"e8m{y}" for y in range(1, 22)])
def test_codec_vs_reference(golden_codec, name):
    fmt = P.parse_format(name)
    pat = P.encode_values(fmt, golden_codec[f"{name}_values"])
    want = golden_codec[f"{name}_patterns"]
    assert pat.dtype == want.dtype and np.array_equal(pat, want)
    dec = P.decode_patterns(fmt, pat)
    assert np.array_equal(_bits(dec), _bits(O.decode(O.preset(name), want)))
    v, d, fl = P.unpack_words(fmt, golden_codec[f"{name}_words"])
    assert np.array_equal(_bits(v), _bits(golden_codec[f"{name}_unpack_values"]))
    assert np.array_equal(d, golden_codec[f"{name}_unpack_deltas"]) and d.dtype == fmt.word_dtype
    assert np.array_equal(fl, golden_codec[f"{name}_unpack_flags"])
    n = len(pat)
    deltas = np.arange(n) % (fmt.max_delta + 1)
    w = P.pack_words(fmt, pat, deltas, np.ones(n, bool))
    assert np.array_equal(w, O.pack_words(O.preset(name), pat, deltas, np.ones(n, bool)))


def test_scalar_pack_unpack_goldens():
    fmt = P.PackFormat(32, 15, "fp16")
    assert P.pack(fmt, 1.0, 3) == 0x3C000007
    assert P.unpack(fmt, 0x3C000007) == P.UnpackedEntry(1.0, 3, True)
    assert P.pack(fmt, None, 70000) == 0x000222E0
    assert P.unpack(fmt, 0) == P.UnpackedEntry(0.0, 0, False)
    assert P.encode_value(P.PackFormat(32, 2, "e8my"), 0.1) << 3 == 0x3DCCCCD0


def test_random_sweep_vs_oracle(rng):
    """c03-style sweep: modes x C x sigma x codecs, bit-exact build + REF SpMV vs the oracle."""
    presets = ["fp16", "e8m14", "e8m20", "e8m3", "fp32embed"]
    for it in range(80):
        n = int(rng.integers(1, 600))
        m = int(rng.integers(1, 600))
        dens = float(np.exp(rng.uniform(np.log(0.001), np.log(0.2))))
        rp, ci, v = random_csr_arrays(rng, n, m, dens, banded=(it % 3 == 0))
        A = P.CsrMatrix(n, m, rp, ci, v)
        mode = ["none", "explicit", "implicit"][it % 3]
        c = [1, 2, 4, 16, 32, 64][it % 6]
        sigma = c * [1, 8, 2][it % 3]
        if sigma > 65536:
            sigma = c
        pre = presets[it % len(presets)]
        M = P.build_packsell(A, c, sigma, P.parse_format(pre), mode)
        OM = O.build(rp, ci, v, m, c, sigma, O.preset(pre), mode)
        assert np.array_equal(M.pack, OM.pack) and np.array_equal(M.offset, OM.offset), it
        assert M.k_left == OM.k_left and tuple(M.counts) == OM.counts
        if mode == "implicit":
            assert np.array_equal(M.perm, OM.perm)
        x = rng.uniform(-1, 1, m).astype(np.float32)
        assert np.array_equal(_bits(P.packsell_spmv(M, x, ref_order=True)), _bits(O.spmv(OM, x))), it


@pytest.mark.parametrize("sigma", [1, 3, 32, 256, 1024, 2048, 4096, 65536])
def test_row_sort_order_vs_oracle(rng, sigma):
    n = 200_000
    counts = rng.integers(0, 40, n) * (rng.random(n) < 0.9) + (rng.random(n) < 0.01) * 5000
    assert np.array_equal(P.row_sort_order(counts, sigma), O.sort_order(counts, sigma))


@pytest.mark.parametrize("kind,dims,scale", [("poisson2d", (9, 7), None), ("poisson3d", (6, 5, 4), "sym"),
                                             ("stencil27", (7, 6, 5), None), ("stencil27", (5, 5, 5), "rowsum"),
                                             ("poisson3d", (10, 10, 10), None)])
def test_device_generators_equal_host(kind, dims, scale):
    host = {"poisson2d": P.poisson2d, "poisson3d": P.poisson3d, "stencil27": P.stencil27}[kind](*dims)
    if scale == "sym":
        host = P.sym_diag_scale(host)
    elif scale == "rowsum":
        host = P.row_sum_scale(host)
    D = P.stencil_device(kind, *dims, scale=scale).to_host()
    assert np.array_equal(D.row_ptr, host.row_ptr)
    assert np.array_equal(D.col_idx, host.col_idx)
    assert np.array_equal(_bits(D.values), _bits(host.values))
    n = host.n_rows
    r0, r1 = n // 3, 2 * n // 3
    S = P.stencil_device(kind, *dims, scale=scale, row_begin=r0, row_end=r1).to_host()
    assert np.array_equal(S.row_ptr, host.row_ptr[r0:r1 + 1] - host.row_ptr[r0])
    assert np.array_equal(S.col_idx, host.col_idx[host.row_ptr[r0]:host.row_ptr[r1]])


def test_slab_builds_concatenate_to_global(rng):
    """Rank slabs (sigma-aligned row ranges, global k_left) concatenate to the global pack."""
    A = P.stencil27(12)
    fmt = P.parse_format("fp16")
    G = P.build_packsell(A, 32, 256, fmt, "implicit")
    n = A.n_rows
    bounds = [0, 256, 768, n]
    packs, perms, base = [], [], 0
    x = rng.uniform(-1, 1, n).astype(np.float32)
    yg = P.packsell_spmv(G, x, ref_order=True)
    for a, b in zip(bounds[:-1], bounds[1:]):
        S = P.stencil_device("stencil27", 12, row_begin=a, row_end=b)
        M = P.build_packsell(S, 32, 256, fmt, "implicit", _k_left_override=G.k_left)
        packs.append(M.pack)
        perms.append(M.perm)
        k0 = a // 32
        assert np.array_equal(M.offset + base, G.offset[k0:k0 + M.n_slices + 1])
        base += M.n_stored
        ys = P.packsell_spmv(M, x, ref_order=True)
        assert np.array_equal(_bits(ys), _bits(yg[a:b]))
    assert np.array_equal(np.concatenate(packs), G.pack)
    assert np.array_equal(np.concatenate(perms), G.perm)


@pytest.mark.parametrize("n,r0,r1", [(5000, 0, 5000), (2 ** 23, 0, 40_000), (2 ** 23, 2 ** 22, 2 ** 22 + 30_000)])
def test_powerlaw_device_equals_host(n, r0, r1):
    from paper_2604_13433_b200.stencil import powerlaw_device, powerlaw_rows
    H = powerlaw_rows(n, 2604, r0, r1)
    D = powerlaw_device(n, 2604, row_begin=r0, row_end=r1).to_host()
    assert np.array_equal(D.row_ptr, H.row_ptr)
    assert np.array_equal(D.col_idx, H.col_idx)
    assert np.array_equal(_bits(D.values), _bits(H.values))


def test_powerlaw_build_vs_oracle():
    """Config-4 family (irregular widths, sigma up to 65536) through K1/K2 vs the oracle."""
    from paper_2604_13433_b200.stencil import powerlaw_rows
    A = powerlaw_rows(1 << 16, 7)
    x = np.random.default_rng(1).uniform(-1, 1, A.n_cols).astype(np.float32)
    for sigma in (256, 4096, 65536):
        for pre in ("fp16", "e8m14"):
            M = P.build_packsell(A, 32, sigma, P.parse_format(pre), "implicit")
            OM = O.build(A.row_ptr, A.col_idx, A.values, A.n_cols, 32, sigma, O.preset(pre), "implicit")
            assert np.array_equal(M.pack, OM.pack) and np.array_equal(M.perm, OM.perm)
            assert np.array_equal(M.offset, OM.offset) and tuple(M.counts) == OM.counts
            assert np.array_equal(_bits(P.packsell_spmv(M, x, ref_order=True)), _bits(O.spmv(OM, x)))


@pytest.mark.parametrize("sigma,pre,dt", [(256, "fp16", np.float16), (4096, "e8m14", np.float32),
                                          (65536, "fp16", np.float32)])
def test_long_slice_segmentation(monkeypatch, sigma, pre, dt):
    """Power-law rows wider than SEG_LEN run as checkpointed segments; result within the FMA bound.
    The static SM-affine grid (default), the merged segment + short-slice grid and the
    two-launch form are bitwise equal."""
    from paper_2604_13433_b200 import _lib
    from paper_2604_13433_b200.packed import SEG_LEN, _seg_schedule
    from paper_2604_13433_b200.stencil import powerlaw_rows
    A = powerlaw_rows(1 << 17, 11)
    M = P.build_packsell(A, 32, sigma, P.parse_format(pre), "implicit")
    s = _seg_schedule(M)
    assert s is not None and s["n_long"] > 0
    x = np.random.default_rng(2).uniform(-1, 1, A.n_cols).astype(dt)
    y = P.packsell_spmv(M, x)
    for env in ({"PSELL_DSTATIC": "0"}, {"PSELL_DSTATIC": "0", "PSELL_SEGMERGE": "0"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        _lib.lib().psell_reload_env()
        y2 = P.packsell_spmv(M, x)
        for k in env:
            monkeypatch.delenv(k)
        _lib.lib().psell_reload_env()
        assert np.array_equal(_bits(y), _bits(y2)), env
    y = y.astype(np.float64)
    ref = P.packsell_spmv(M, x.astype(np.float32), ref_order=True).astype(np.float64)
    lmax = int(np.max(np.diff(M.offset) // 32))
    aq = np.abs(P.quantize(P.parse_format(pre), A.values))
    anorm = np.bincount(np.repeat(np.arange(A.n_rows), A.row_lengths()), aq, minlength=A.n_rows).max()
    err = np.abs(y - ref).max() / (anorm * np.abs(x.astype(np.float64)).max())
    assert err <= 2 * lmax * 2.0 ** -24 + (2.0 ** -11 if dt == np.float16 else 0.0), err
    assert lmax > SEG_LEN


def test_spmv_stream_equals_per_call(rng):
    """The pipelined host-buffer API returns exactly the per-call results."""
    import torch
    A = P.stencil27(14)
    M = P.build_packsell(A, 32, 256, P.parse_format("fp16"), "implicit")
    xs = [torch.from_numpy(rng.uniform(-1, 1, A.n_cols).astype(np.float16)).pin_memory() for _ in range(5)]
    outs = P.packsell_spmv_stream(M, xs)
    for x, y in zip(xs, outs):
        assert np.array_equal(_bits(y.numpy()), _bits(P.packsell_spmv(M, x.numpy())))
    ys = P.packsell_spmv_stream(M, [x.numpy() for x in xs], ref_order=True)
    for x, y in zip(xs, ys):
        assert np.array_equal(_bits(y.numpy()), _bits(P.packsell_spmv(M, x.numpy(), ref_order=True)))


@pytest.mark.parametrize("sigma,nnz_per_row", [(96, 7), (160, 7), (224, 27), (32 * 1023, 5), (96, 27)])
@pytest.mark.parametrize("mode", ["implicit", "explicit", "none"])
def test_production_kernels_non_pow2_sigma(rng, sigma, nnz_per_row, mode):
    """Dual / pair / persistent-pair kernels with sigma not a power of two (multiply-high division of
    base offsets and output rows): FMA SpMV within the bound of the REF_ORDER result, which is bitwise
    the oracle's; build bit-exact."""
    n = 4096 + 96 * 7
    rows = np.repeat(np.arange(n), nnz_per_row)
    cols = np.clip(rows + rng.integers(-600, 600, rows.size), 0, n - 1)
    order = np.lexsort((cols, rows))
    r, c = rows[order], cols[order]
    keep = np.ones(r.size, bool)
    keep[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    r, c = r[keep], c[keep]
    v = rng.uniform(0.01, 1, r.size) * rng.choice([-1.0, 1.0], r.size)
    rp = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=n))]).astype(np.int64)
    A = P.CsrMatrix(n, n, rp, c.astype(np.int32), v)
    for pre, dt in (("fp16", np.float16), ("e8m14", np.float32)):
        M = P.build_packsell(A, 32, sigma, P.parse_format(pre), mode)
        OM = O.build(rp, c.astype(np.int32), v, n, 32, sigma, O.preset(pre), mode)
        assert np.array_equal(M.pack, OM.pack) and np.array_equal(M.offset, OM.offset)
        x = rng.uniform(-1, 1, n).astype(dt)
        yr = P.packsell_spmv(M, x.astype(np.float32), ref_order=True)
        assert np.array_equal(_bits(yr), _bits(O.spmv(OM, x.astype(np.float32))))
        yf = P.packsell_spmv(M, x).astype(np.float64)
        lmax = int(np.max(np.diff(M.offset) // 32))
        anorm = np.bincount(np.repeat(np.arange(n), np.diff(rp)), np.abs(P.quantize(P.parse_format(pre), v))).max()
        err = np.abs(yf - yr.astype(np.float64)).max() / (anorm * np.abs(x.astype(np.float64)).max())
        assert err <= 2 * lmax * 2.0 ** -24 + (2.0 ** -11 if dt == np.float16 else 0.0), (pre, err)


@pytest.mark.parametrize("kind,nx", [("poisson3d", 24), ("poisson2d", 200)])
def test_tile_tma_kernel_equals_pair_kernel(monkeypatch, kind, nx):
    """A/B kernel (PSELL_TILE=1: TMA producer/consumer ring) gives the production kernel's bits,
    plain and with the fused p.q."""
    from paper_2604_13433_b200 import _lib
    S = P.stencil_device(kind, nx, scale="sym")
    M = P.build_packsell(S, 32, 256, P.parse_format("e8m14"), "implicit")
    assert M.spmv_flags() & 4  # narrow slices
    import torch
    x = torch.rand(M.n_cols, device="cuda") * 2 - 1
    lib = _lib.lib()
    res = {}
    for tile in ("0", "1"):
        monkeypatch.setenv("PSELL_TILE", tile)
        lib.psell_reload_env()  # the launchers cache their knobs
        from paper_2604_13433_b200 import _dev
        assert lib.psell_spmv_kernel_name(M.desc(), _dev.T_DT_CODE[x.dtype], M.spmv_flags()).decode().startswith(
            "spmv_tile" if tile == "1" else ("spmv_pair", "spmv_narrow"))
        y = P.packsell_spmv(M, x)
        npart = lib.psell_spmv_dot_partials(M.desc(), M.spmv_flags())
        part = torch.zeros(npart, dtype=torch.float64, device="cuda")
        q = torch.empty_like(x)
        err = _lib.PsellError()
        rc = lib.psell_spmv_dot(M.desc(), _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                                x.data_ptr(), q.data_ptr(), x.data_ptr(), part.data_ptr(), None, M.spmv_flags(),
                                _lib.stream_handle(), err)
        _lib.check(rc, err)
        res[tile] = (y.clone(), q.clone(), float(part.sum()))
    monkeypatch.delenv("PSELL_TILE")
    lib.psell_reload_env()
    assert torch.equal(res["0"][0], res["1"][0]) and torch.equal(res["0"][1], res["1"][1])
    assert res["0"][2] == pytest.approx(res["1"][2], rel=1e-12)


def test_spmv_argument_validation(rng):
    """Bad x / out shapes, dtypes and devices raise instead of reading or writing out of bounds."""
    import torch
    rp, ci, v = random_csr_arrays(rng, 100, 90, 0.1)
    M = P.build_packsell(P.CsrMatrix(100, 90, rp, ci, v), 32, 256, P.parse_format("fp16"), "implicit")
    x = torch.rand(90, device="cuda")
    with pytest.raises(ValueError):
        P.packsell_spmv(M, torch.rand(91, device="cuda"))
    with pytest.raises(ValueError):
        P.packsell_spmv(M, torch.rand(90, 2, device="cuda"))
    with pytest.raises(ValueError):
        P.packsell_spmv(M, x, out=torch.empty(99, device="cuda"))
    with pytest.raises(ValueError):
        P.packsell_spmv(M, x, out=torch.empty(100, dtype=torch.float16, device="cuda"))
    with pytest.raises(ValueError):
        P.packsell_spmv(M, np.ones((90, 2), np.float32))
    with pytest.raises(TypeError):
        P.packsell_spmv(M, x.to(torch.int32))
    xs = torch.rand(180, device="cuda")[::2]  # strided view: made contiguous, same result
    assert torch.equal(P.packsell_spmv(M, xs), P.packsell_spmv(M, xs.contiguous()))


def test_persistent_pair_kernel_at_scale(rng):
    """The persistent pair kernel over many grid-stride trips per warp (1.2 M rows, far
    more slice pairs than resident warps), narrow slices of mixed widths (tails split
    at 9 steps, both slices reaching it or not) plus some wider than 12 steps (full
    chunks and the longer slice's remainder): FMA SpMV within the bound of the
    REF_ORDER kernel, in e8m14 / f32 x and fp16 / f16 x."""
    n = 1_200_000
    lens = rng.integers(3, 10, n)
    lens[rng.integers(0, n, 3000)] = rng.integers(12, 20, 3000)
    rows = np.repeat(np.arange(n), lens)
    cols = np.clip(rows + rng.integers(-120, 120, rows.size), 0, n - 1)
    order = np.lexsort((cols, rows))
    r, c = rows[order], cols[order]
    keep = np.ones(r.size, bool)
    keep[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    r, c = r[keep], c[keep]
    v = rng.uniform(0.01, 1, r.size) * rng.choice([-1.0, 1.0], r.size)
    rp = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=n))]).astype(np.int64)
    A = P.CsrMatrix(n, n, rp, c.astype(np.int32), v)
    for pre, dt in (("e8m14", np.float32), ("fp16", np.float16)):
        M = P.build_packsell(A, 32, 256, P.parse_format(pre), "implicit")
        assert M.spmv_flags() & 4, "expected the narrow (pair-kernel) path"
        x = rng.uniform(-1, 1, n).astype(dt)
        yr = P.packsell_spmv(M, x.astype(np.float32), ref_order=True).astype(np.float64)
        yf = P.packsell_spmv(M, x).astype(np.float64)
        lmax = int(np.max(np.diff(M.offset) // 32))
        anorm = np.bincount(r, np.abs(P.quantize(P.parse_format(pre), v)), minlength=n).max()
        err = np.abs(yf - yr).max() / (anorm * np.abs(x.astype(np.float64)).max())
        assert err <= 2 * lmax * 2.0 ** -24 + (2.0 ** -11 if dt == np.float16 else 0.0), (pre, err)


@pytest.mark.parametrize("n,r0,r1", [(5000, 0, 5000), (2 ** 23, 0, 30_000), (2 ** 23, 2 ** 23 - 20_000, 2 ** 23)])
def test_powerlaw_far_device_equals_host(n, r0, r1):
    """Config-4b generator (SURVEY §8d's far columns): device == host mirror, bit for bit."""
    from paper_2604_13433_b200.stencil import powerlaw_device, powerlaw_far_rows
    H = powerlaw_far_rows(n, 2604, r0, r1)
    D = powerlaw_device(n, 2604, row_begin=r0, row_end=r1, far=True).to_host()
    assert np.array_equal(D.row_ptr, H.row_ptr)
    assert np.array_equal(D.col_idx, H.col_idx)
    assert np.array_equal(_bits(D.values), _bits(H.values))


@pytest.mark.parametrize("sigma", [256, 65536])
def test_powerlaw_far_build_and_spmv_vs_oracle(sigma):
    """The dummy-heavy far-gap regime (k_left ~ n, every d_i = 0) through K1/K2 vs the oracle,
    including the segmented path and its SM-affine short-slice kernel (bitwise equal to the
    block-linear one)."""
    import os
    from paper_2604_13433_b200 import _lib
    from paper_2604_13433_b200.stencil import powerlaw_far_rows
    A = powerlaw_far_rows(1 << 17, 5)
    M = P.build_packsell(A, 32, sigma, P.parse_format("fp16"), "implicit")
    OM = O.build(A.row_ptr, A.col_idx, A.values, A.n_cols, 32, sigma, O.preset("fp16"), "implicit")
    assert M.k_left == OM.k_left > (1 << 17) - 2 * sigma
    assert np.array_equal(M.pack, OM.pack) and np.array_equal(M.perm, OM.perm)
    assert np.array_equal(M.offset, OM.offset) and tuple(M.counts) == OM.counts
    assert OM.counts[1] > A.nnz // 20  # dummy heavy (27 % of nnz at the full n = 2^23)
    x = np.random.default_rng(3).uniform(-1, 1, A.n_cols).astype(np.float16)
    assert np.array_equal(_bits(P.packsell_spmv(M, x, ref_order=True)), _bits(O.spmv(OM, x)))
    ys = {}
    for aff in ("0", "1"):
        os.environ["PSELL_AFF"] = aff
        _lib.lib().psell_reload_env()
        ys[aff] = P.packsell_spmv(M, x)
    os.environ.pop("PSELL_AFF")
    _lib.lib().psell_reload_env()
    assert np.array_equal(_bits(ys["0"]), _bits(ys["1"]))
    ref = O.spmv(OM, x.astype(np.float32)).astype(np.float64)
    lmax = int(np.max(np.diff(OM.offset) // 32))
    aq = np.abs(O.quantize(O.preset("fp16"), A.values))
    anorm = np.bincount(np.repeat(np.arange(A.n_rows), A.row_lengths()), aq, minlength=A.n_rows).max()
    err = np.abs(ys["0"].astype(np.float64) - ref).max() / (anorm * np.abs(x.astype(np.float64)).max())
    assert err <= 2.0 ** -11 + 2 * lmax * 2.0 ** -24, err


def _narrow_csr(rng, n, lmin, lmax, spread):
    lens = rng.integers(lmin, lmax + 1, n)
    rows = np.repeat(np.arange(n), lens)
    cols = np.clip(rows + rng.integers(-spread, spread + 1, rows.size), 0, n - 1)
    order = np.lexsort((cols, rows))
    r, c = rows[order], cols[order]
    keep = np.ones(r.size, bool)
    keep[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    r, c = r[keep], c[keep]
    v = rng.uniform(0.01, 1, r.size) * rng.choice([-1.0, 1.0], r.size)
    rp = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=n))]).astype(np.int64)
    return P.CsrMatrix(n, n, rp, c.astype(np.int32), v)


@pytest.mark.parametrize("matrix", ["poisson3d-37", "ragged-narrow"])
@pytest.mark.parametrize("sigma,mode", [(256, "implicit"), (512, "implicit"), (96, "implicit"), (256, "explicit"),
                                        (1, "none")])
def test_narrow_kernel_equals_pair_kernel(monkeypatch, rng, matrix, sigma, mode):
    """The narrow kernels (default for slices <= 12 steps: words staged through shared memory
    by cp.async.bulk; PSELL_NARROW_TMA=0: words loaded per lane) give the persistent pair
    kernel's bits (same FMAs in the same order): plain SpMV for every codec / x dtype they
    serve and the fused SpMV + p.q, with u8 / u16 / no perm, power-of-two and other sigma, tail
    steps past 9 and a ragged last slice pair."""
    import torch
    from paper_2604_13433_b200 import _dev, _lib
    if matrix == "poisson3d-37":
        A = P.sym_diag_scale(P.poisson3d(37))                 # 50653 rows: odd slice count, ragged last slice
    else:
        A = _narrow_csr(rng, 200_003, 3, 11, 100)             # widths up to 12: the [9, 12) tail path
    lib = _lib.lib()
    variants = {"pair": ("0", "0", "spmv_pair"), "narrow": ("1", "0", "spmv_narrow_kernel"),
                "narrow_tma": ("1", "1", "spmv_narrow_tma")}
    for pre, dt in (("e8m14", torch.float32), ("fp16", torch.float16), ("fp16", torch.float32),
                    ("e8m14", torch.float16)):
        M = P.build_packsell(A, 32, sigma, P.parse_format(pre), mode)
        assert M.spmv_flags() & 12 == 12, "expected narrow slices of <= 12 steps"
        x = (torch.rand(M.n_cols, device="cuda") * 2 - 1).to(dt)
        res = {}
        for key, (nar, tma, kname) in variants.items():
            monkeypatch.setenv("PSELL_NARROW", nar)
            monkeypatch.setenv("PSELL_NARROW_TMA", tma)
            lib.psell_reload_env()
            name = lib.psell_spmv_kernel_name(M.desc(), _dev.T_DT_CODE[x.dtype], M.spmv_flags()).decode()
            assert name.startswith(kname), name
            y = P.packsell_spmv(M, x)
            out = [y.clone()]
            if dt == torch.float32:
                npart = lib.psell_spmv_dot_partials(M.desc(), M.spmv_flags())
                part = torch.zeros(npart, dtype=torch.float64, device="cuda")
                q = torch.empty_like(x)
                err = _lib.PsellError()
                rc = lib.psell_spmv_dot(M.desc(), _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                                        x.data_ptr(), q.data_ptr(), x.data_ptr(), part.data_ptr(), None,
                                        M.spmv_flags(), _lib.stream_handle(), err)
                _lib.check(rc, err)
                out += [q.clone(), float(part.sum())]
            res[key] = out
        monkeypatch.delenv("PSELL_NARROW")
        monkeypatch.delenv("PSELL_NARROW_TMA")
        lib.psell_reload_env()
        for key in ("narrow", "narrow_tma"):
            assert torch.equal(res["pair"][0], res[key][0]), (matrix, pre, dt, key)
            if dt == torch.float32:
                assert torch.equal(res["pair"][1], res[key][1]), (matrix, pre, key)
                assert res[key][2] == pytest.approx(res["pair"][2], rel=1e-12)


@pytest.mark.parametrize("n", [1, 3, 255, 257, 5000])
def test_csr_spmv_bulk_edges(n):
    """K4's bulk-staged path on ragged small matrices: a single partial block, spans that
    start and end off the 16-byte grid (tail entries in registers), empty rows and rows
    longer than one stage; bitwise vs the oracle in every working precision."""
    rng = np.random.default_rng(n)
    lens = rng.integers(0, 12, n)
    lens[rng.integers(0, n, max(1, n // 500))] = rng.integers(0, 2500, max(1, n // 500))
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = rng.integers(0, n, int(rp[-1])).astype(np.int32)
    v = rng.standard_normal(int(rp[-1]))
    A = P.CsrMatrix(n, n, rp, ci, v)
    for dt in (np.float16, np.float32, np.float64):
        x = rng.standard_normal(n).astype(dt)
        y = P.csr_spmv(A, x, dt)
        assert np.array_equal(_bits(y), _bits(O.csr_spmv(rp, ci, v, x, dt))), dt


@pytest.mark.parametrize("matrix", ["stencil27-21", "ragged-wide"])
@pytest.mark.parametrize("sigma,mode", [(256, "implicit"), (96, "implicit"), (65536, "implicit"), (1, "none")])
def test_wide_kernel_equals_dual_kernel(monkeypatch, rng, matrix, sigma, mode):
    """The wide TMA kernel (PSELL_WIDE=1, slices of <= 32 steps staged by cp.async.bulk) and the
    staged dual kernel (PSELL_DSTAGE=1, 8-step chunks staged two ahead) give the dual kernel's bits: plain SpMV over the codec / x dtypes it serves and the fused
    SpMV + p.q, u8 / u16 / no perm, power-of-two and other sigma, a ragged last slice."""
    import torch
    from paper_2604_13433_b200 import _dev, _lib
    if matrix == "stencil27-21":
        A = P.stencil27(21)                                  # 9261 rows: ragged last slice
    else:
        A = _narrow_csr(rng, 100_003, 13, 27, 400)          # 13..27 entries + dummies-free widths <= 32
    lib = _lib.lib()
    for pre, dt in (("fp16", torch.float16), ("e8m10", torch.float32), ("fp16", torch.float32),
                    ("e8m14", torch.float16)):
        M = P.build_packsell(A, 32, sigma, P.parse_format(pre), mode)
        if not M.spmv_flags() & 16:
            continue  # a slice wider than 32 steps (dummies): the wide kernel does not apply
        assert not M.spmv_flags() & 4
        x = (torch.rand(M.n_cols, device="cuda") * 2 - 1).to(dt)
        res = {}
        for wide, kname in (("0", "spmv_dual_kernel"), ("1", "spmv_wide_tma"), ("s", "spmv_dual_stage")):
            monkeypatch.setenv("PSELL_WIDE", "1" if wide == "1" else "0")
            monkeypatch.setenv("PSELL_DSTAGE", "1" if wide == "s" else "0")
            lib.psell_reload_env()
            name = lib.psell_spmv_kernel_name(M.desc(), _dev.T_DT_CODE[x.dtype], M.spmv_flags()).decode()
            assert name.startswith(kname), name
            out = [P.packsell_spmv(M, x).clone()]
            if dt == torch.float32:  # the fused SpMV + p.q is the f32 inner-PCG operator
                npart = lib.psell_spmv_dot_partials(M.desc(), M.spmv_flags())
                part = torch.zeros(npart, dtype=torch.float64, device="cuda")
                q = torch.empty_like(x)
                err = _lib.PsellError()
                rc = lib.psell_spmv_dot(M.desc(), _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                                        x.data_ptr(), q.data_ptr(), x.data_ptr(), part.data_ptr(), None,
                                        M.spmv_flags(), _lib.stream_handle(), err)
                _lib.check(rc, err)
                out += [q.clone(), float(part.sum())]
            res[wide] = out
        monkeypatch.delenv("PSELL_WIDE")
        monkeypatch.delenv("PSELL_DSTAGE")
        lib.psell_reload_env()
        for v in ("1", "s"):
            assert torch.equal(res["0"][0], res[v][0]), (matrix, pre, dt, v)
            if dt == torch.float32:
                assert torch.equal(res["0"][1], res[v][1]), (matrix, pre, dt, v)
                assert res[v][2] == pytest.approx(res["0"][2], rel=1e-12)
