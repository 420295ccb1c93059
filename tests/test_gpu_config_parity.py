"""Byte-exact parity at the BASELINE config sizes (VERDICT r01 "next" #1).

The production matrices of BASELINE.json's configs are generated and packed in
HBM at their full size; the CPU oracle (the pinned restatement of
packed.py:176-271) builds sigma-aligned slabs of the same matrices -- the first,
a middle and the last 2^20 rows -- from host CSR rows with the *global* k_left
and the slab's global row origin.  For every slab:

* the device CSR rows equal the host rows (generator + scaling, bitwise);
* the full device build's ``pack`` words, rebased ``offset`` and ``perm`` over
  the slab's slices equal the oracle's byte for byte (packed.py:176-239);
* a device *slab* build (the multi-GPU path: ``stencil_device(row_begin=..)``
  + ``_k_left_override``) equals the oracle too, ``counts`` included;
* REF_ORDER SpMV of the full matrix is bitwise equal to the oracle's
  ``packsell_spmv`` on the slab's rows (packed.py:242-271);
* the production FMA SpMV is within the SURVEY §8c bound of the oracle:
  e_rel <= 2*L_max*2^-24 (f32 x) and <= 2^-11 + 2*L_max*2^-24 (f16 x, oracle
  fed the f32-widened x).

Config 1 (5-point 512^2, the reference's CPU-runnable case) is compared whole.
The oracle slabs are built in forked worker processes while the GPU works.
"""

from __future__ import annotations

import multiprocessing as mp
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SLAB = 1 << 20
X_SEED = 4321

# (id, generator kind, nx, scale, preset, x dtype, global k_left)
CASES = [
    ("c2-fp16", "stencil27", 256, None, "fp16", "float16", 65_793),
    ("c3-e8m10", "stencil27", 256, "rowsum", "e8m10", "float32", 65_793),
    ("c3-e8m11", "stencil27", 256, "rowsum", "e8m11", "float32", 65_793),
    ("c3-e8m20", "stencil27", 256, "rowsum", "e8m20", "float32", 65_793),
    ("c3-e8m21", "stencil27", 256, "rowsum", "e8m21", "float32", 65_793),
    ("c5-e8m14", "poisson3d", 256, "sym", "e8m14", "float32", 65_536),
    ("c5-fp16", "poisson3d", 256, "sym", "fp16", "float32", 65_536),
]


def host_rows(kind, nx, scale, r0, r1):
    """Host CSR rows [r0, r1) with the reference's scaling formulas (matrix.py:294-316)."""
    from paper_2604_13433_b200.stencil import stencil_rows
    A = stencil_rows(kind, nx, r0, r1)
    v = A.values
    if scale == "rowsum":
        rows = np.repeat(np.arange(A.n_rows), A.row_lengths())
        s = np.zeros(A.n_rows)
        np.add.at(s, rows, np.abs(v))
        v = v / s[rows]
    elif scale == "sym":
        # every stencil row stores its diagonal (6 for the 7-point Laplacian), so g is uniform
        g = np.sqrt(np.abs(6.0 if kind == "poisson3d" else 4.0))
        v = v / (g * g)
    return A.row_ptr, A.col_idx, v, A.n_cols


def global_x(n, xdt):
    return np.random.default_rng(X_SEED).uniform(-1, 1, n).astype(xdt)


def oracle_slab(kind, nx, scale, preset, xdt, k_left, r0, r1):
    """Worker: oracle build + REF SpMV (+ widened-x SpMV for f16) of one slab."""
    import oracle as O
    rp, ci, v, n_cols = host_rows(kind, nx, scale, r0, r1)
    f = O.preset(preset)
    M = O.build(rp, ci, v, n_cols, 32, 256, f, "implicit", k_left=k_left, row0=r0)
    x = global_x(n_cols, xdt)
    y_ref = O.spmv(M, x)
    y_wide = O.spmv(M, x.astype(np.float32)) if xdt == "float16" else y_ref
    q = np.abs(O.quantize(f, v))
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    rs = np.zeros(len(rp) - 1)
    np.add.at(rs, rows, q)
    lmax = int(np.diff(M.offset).max() // 32)
    return dict(rp=rp, ci=ci, v=v, pack=M.pack, offset=M.offset, perm=M.perm, counts=M.counts,
                k_left=M.k_left, y_ref=y_ref, y_wide=y_wide, anorm=float(rs.max()), lmax=lmax)


def _slabs(n):
    mid = (n // 2) // 256 * 256
    return [(0, SLAB), (mid, mid + SLAB), (n - SLAB, n)]


@pytest.fixture(scope="module")
def pool():
    ex = ProcessPoolExecutor(max_workers=3, mp_context=mp.get_context("fork"))
    yield ex
    ex.shutdown()


def _dl(t, dt):
    from paper_2604_13433_b200 import _dev
    return _dev.download(t, dt)


def _check_fma(y, ref, anorm, x, lmax, f16):
    xmax = float(np.abs(x.astype(np.float64)).max())
    e = float(np.abs(y.astype(np.float64) - ref.astype(np.float64)).max()) / (anorm * xmax)
    bound = (2.0 ** -11 if f16 else 0.0) + 2 * lmax * 2.0 ** -24
    assert e <= bound, (e, bound)
    return e


@pytest.mark.parametrize("cid,kind,nx,scale,preset,xdt,k_left", CASES, ids=[c[0] for c in CASES])
def test_config_slabs_byte_exact(pool, cid, kind, nx, scale, preset, xdt, k_left):
    import torch

    import paper_2604_13433_b200 as P
    from paper_2604_13433_b200.packed import lower_bandwidth

    n = nx ** 3
    slabs = _slabs(n)
    futs = [pool.submit(oracle_slab, kind, nx, scale, preset, xdt, k_left, r0, r1) for r0, r1 in slabs]

    fmt = P.parse_format(preset)
    wdt = fmt.word_dtype
    A = P.stencil_device(kind, nx, scale=scale)
    assert lower_bandwidth(A) == k_left
    M = P.build_packsell(A, 32, 256, fmt, "implicit")
    assert M.k_left == k_left
    x = global_x(n, xdt)
    xd = torch.from_numpy(x).cuda()
    y_ref = P.packsell_spmv(M, xd, ref_order=True).cpu().numpy()
    y_fma = P.packsell_spmv(M, xd).cpu().numpy()
    off = M.offset
    for (r0, r1), fut in zip(slabs, futs):
        o = fut.result()
        s0, s1 = r0 // 32, r1 // 32
        # the generator's rows (device) equal the host rows the oracle packed
        rp = _dl(A.row_ptr[r0:r1 + 1], np.int64)
        assert np.array_equal(rp - rp[0], o["rp"]), (cid, r0)
        assert np.array_equal(_dl(A.col_idx[rp[0]:rp[-1]], np.int32), o["ci"]), (cid, r0)
        assert np.array_equal(_dl(A.values[rp[0]:rp[-1]], np.float64).view(np.uint64),
                              o["v"].view(np.uint64)), (cid, r0)
        # the production matrix's bytes over the slab
        assert o["k_left"] == k_left
        assert np.array_equal(off[s0:s1 + 1] - off[s0], o["offset"]), (cid, r0)
        assert np.array_equal(_dl(M.d_pack[off[s0]:off[s1]], wdt), o["pack"]), (cid, r0)
        assert np.array_equal(M.perm[r0:r1], o["perm"]), (cid, r0)
        # the multi-GPU slab build of the same rows
        S = P.stencil_device(kind, nx, scale=scale, row_begin=r0, row_end=r1)
        Ms = P.build_packsell(S, 32, 256, fmt, "implicit", _k_left_override=k_left)
        assert np.array_equal(Ms.offset, o["offset"]) and np.array_equal(Ms.pack, o["pack"]), (cid, r0)
        assert np.array_equal(Ms.perm, o["perm"]) and tuple(Ms.counts) == tuple(o["counts"]), (cid, r0)
        del S, Ms
        # SpMV: REF_ORDER bitwise, production FMA within the bound
        assert np.array_equal(y_ref[r0:r1].view(np.uint8), o["y_ref"].view(np.uint8)), (cid, r0)
        _check_fma(y_fma[r0:r1], o["y_wide"], o["anorm"], x, o["lmax"], xdt == "float16")
    torch.cuda.synchronize()


def test_config1_whole_byte_exact():
    """Config 1 (5-point 512^2, fp16, f16 x): the whole matrix against the oracle."""
    import oracle as O
    import paper_2604_13433_b200 as P
    A = P.poisson2d(512)
    M = P.build_packsell(A, 32, 256, P.parse_format("fp16"), "implicit")
    OM = O.build(A.row_ptr, A.col_idx, A.values, A.n_cols, 32, 256, O.preset("fp16"), "implicit")
    assert np.array_equal(M.pack, OM.pack) and np.array_equal(M.offset, OM.offset)
    assert np.array_equal(M.perm, OM.perm) and tuple(M.counts) == OM.counts and M.k_left == OM.k_left == 512
    D = P.stencil_device("poisson2d", 512)
    Md = P.build_packsell(D, 32, 256, P.parse_format("fp16"), "implicit")
    assert np.array_equal(Md.pack, OM.pack) and np.array_equal(Md.offset, OM.offset)
    x = global_x(A.n_cols, "float16")
    assert np.array_equal(P.packsell_spmv(M, x, ref_order=True).view(np.uint16), O.spmv(OM, x).view(np.uint16))
    anorm = float(np.max(np.add.reduceat(np.abs(O.quantize(O.preset("fp16"), A.values)), A.row_ptr[:-1])))
    _check_fma(P.packsell_spmv(M, x), O.spmv(OM, x.astype(np.float32)), anorm, x,
               int(np.diff(OM.offset).max() // 32), True)
