"""Synthetic matrix generators for the BASELINE configs.

Host generators return a `CsrMatrix` (numpy) identical to what the reference
builds for the same problem:

* `poisson2d` / `poisson3d` — Dirichlet Laplacians, diagonal 2*ndim, -1
  neighbours, row-major ordering (reference stencil.py:10-52);
* `stencil27` — the HPCG 27-point box stencil (diag 26, off -1), the paper's
  HPCG_k_k_k matrices (BASELINE config 2/3);
* `powerlaw` — the config-4 irregular matrix (SURVEY.md §8d proposal).

Device generators write the same CSR directly into HBM (psell_gen_stencil),
optionally only the row range of one rank's slab and optionally with the
sym_diag_scale / row_sum_scale preprocessing fused — bitwise equal to the
host generator followed by the host scaling (tests/test_gpu_generators.py).
"""

from __future__ import annotations

import numpy as np

from .matrix import CsrMatrix


def _grid_stencil(dims, box: bool, diag: float, row_begin: int = 0, row_end: int = None) -> CsrMatrix:
    dims = [int(d) for d in dims]
    if any(d < 1 for d in dims):
        raise ValueError(f"grid dimensions must be positive, got {dims}")
    n = int(np.prod(dims))
    if n > 2**31 - 1:
        raise ValueError(f"grid of {n} points overflows 32-bit indexing")
    if row_begin != 0 or (row_end is not None and row_end != n):
        return _grid_rows(dims, box, diag, int(row_begin), n if row_end is None else int(row_end))
    nd = len(dims)
    # neighbour offsets in lexicographic order => ascending column order per row
    strides = np.cumprod([1] + dims[::-1][:-1])[::-1].astype(np.int64)
    if box:
        offs = np.array(np.meshgrid(*([[-1, 0, 1]] * nd), indexing="ij")).reshape(nd, -1).T
    else:
        eye = np.eye(nd, dtype=np.int64)
        offs = np.concatenate([-eye, np.zeros((1, nd), np.int64), eye])
    # ascending flat column delta => ascending columns in every row
    offs = offs[np.argsort(offs @ strides, kind="stable")]
    coords = np.stack(np.meshgrid(*[np.arange(d) for d in dims], indexing="ij"), -1).reshape(-1, nd)
    cols, vals, lens = [], [], np.zeros(n, dtype=np.int64)
    for o in offs:
        nb = coords + o
        ok = np.all((nb >= 0) & (nb < np.array(dims)), axis=1)
        c = np.where(ok, nb @ strides, -1)
        v = diag if not np.any(o) else -1.0
        cols.append(c)
        vals.append(np.where(ok, v, 0.0))
        lens += ok
    C = np.stack(cols, 1)
    V = np.stack(vals, 1)
    keep = C >= 0
    row_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return CsrMatrix(n, n, row_ptr, C[keep].astype(np.int32), V[keep])


def _grid_rows(dims, box, diag, r0, r1) -> CsrMatrix:
    """Rows [r0, r1) of the stencil as a local CSR (n_cols global) — a rank slab / CPU sample."""
    nd = len(dims)
    n = int(np.prod(dims))
    strides = np.cumprod([1] + dims[::-1][:-1])[::-1].astype(np.int64)
    if box:
        offs = np.array(np.meshgrid(*([[-1, 0, 1]] * nd), indexing="ij")).reshape(nd, -1).T
    else:
        eye = np.eye(nd, dtype=np.int64)
        offs = np.concatenate([-eye, np.zeros((1, nd), np.int64), eye])
    offs = offs[np.argsort(offs @ strides, kind="stable")]
    coords = np.stack(np.unravel_index(np.arange(r0, r1, dtype=np.int64), dims), -1)
    cols, vals = [], []
    lens = np.zeros(r1 - r0, dtype=np.int64)
    for o in offs:
        nb = coords + o
        ok = np.all((nb >= 0) & (nb < np.array(dims)), axis=1)
        cols.append(np.where(ok, nb @ strides, -1))
        vals.append(np.where(ok, diag if not np.any(o) else -1.0, 0.0))
        lens += ok
    C = np.stack(cols, 1)
    V = np.stack(vals, 1)
    keep = C >= 0
    row_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return CsrMatrix(r1 - r0, n, row_ptr, C[keep].astype(np.int32), V[keep])


def stencil_rows(kind: str, nx: int, row_begin: int, row_end: int) -> CsrMatrix:
    """Host rows [row_begin, row_end) of poisson2d/poisson3d/stencil27 on an nx^d grid."""
    if kind == "poisson2d":
        return _grid_rows([nx, nx], False, 4.0, row_begin, row_end)
    if kind == "poisson3d":
        return _grid_rows([nx, nx, nx], False, 6.0, row_begin, row_end)
    if kind == "stencil27":
        return _grid_rows([nx, nx, nx], True, 26.0, row_begin, row_end)
    raise ValueError(f"unknown stencil {kind!r}")


def poisson2d(nx: int, ny: int = None) -> CsrMatrix:
    """5-point Laplacian, diagonal 4 (reference stencil.py:45-47)."""
    return _grid_stencil([nx, nx if ny is None else ny], box=False, diag=4.0)


def poisson3d(nx: int, ny: int = None, nz: int = None) -> CsrMatrix:
    """7-point Laplacian, diagonal 6 (reference stencil.py:50-52)."""
    return _grid_stencil([nx, nx if ny is None else ny, nx if nz is None else nz], box=False, diag=6.0)


def stencil27(nx: int, ny: int = None, nz: int = None) -> CsrMatrix:
    """HPCG 27-point box stencil on nx*ny*nz, z slowest (diag 26, off-diagonal -1)."""
    return _grid_stencil([nx, nx if ny is None else ny, nx if nz is None else nz], box=True, diag=26.0)


_U64 = np.uint64


def _smix(z):
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic), = smix in csrc/gen.cu."""
    with np.errstate(over="ignore"):
        z = z + _U64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> _U64(30))) * _U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _U64(27))) * _U64(0x94D049BB133111EB)
    return z ^ (z >> _U64(31))


def powerlaw_rows(n: int = 2**23, seed: int = 2604, row_begin: int = 0, row_end: int = None) -> CsrMatrix:
    """Rows [row_begin, row_end) of the config-4 power-law matrix (host mirror of
    psell_gen_powerlaw_*; the generator law is documented in csrc/gen.cu).

    Counter-based hashing makes every row independent, so a CPU sample or a
    rank slab is generated without the rest of the matrix and equals the GPU's.
    """
    r1 = n if row_end is None else int(row_end)
    r0 = int(row_begin)
    rows = np.arange(r0, r1, dtype=np.int64)
    with np.errstate(over="ignore"):
        hr = _smix(_U64(seed) ^ (rows.astype(_U64) * _U64(0xD1B54A32D192ED03)))

    def draw(stream, j, h):
        return _smix(h ^ (_U64(stream) << _U64(56)) ^ _U64(j))

    u = (draw(0, 0, hr) >> _U64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    thr = powerlaw_thresholds()
    # number of leading (non-increasing) thresholds >= u  ==  binary search in gen.cu
    L = np.maximum(np.searchsorted(-thr, -u, side="right"), 1).astype(np.int64)
    G2 = (2 * np.maximum(1, 8192 // L)).astype(_U64)
    far = np.maximum(n // (8 * L), 1).astype(_U64)
    c = np.maximum(rows - 4096, 0)
    out_r, out_j, out_c, out_v = [], [], [], []
    act = np.nonzero((L > 0) & (c < n))[0]
    j = 0
    while act.size:
        h = hr[act]
        out_r.append(act)
        out_j.append(np.full(act.size, j, dtype=np.int64))
        out_c.append(c[act].copy())
        m = 0.01 + 0.99 * ((draw(4, j, h) >> _U64(11)).astype(np.float64) * (1.0 / 9007199254740992.0))
        out_v.append(np.where((draw(3, j, h) & _U64(1)) != 0, -m, m))
        step = 1 + (draw(1, j, h) % G2[act]).astype(np.int64)
        jump = np.where(draw(2, j, h) % _U64(5) == 0, (draw(5, j, h) % far[act]).astype(np.int64), 0)
        c[act] += step + jump
        j += 1
        act = act[(j < L[act]) & (c[act] < n)]
    if out_r:
        rr = np.concatenate(out_r)
        o = np.lexsort((np.concatenate(out_j), rr))
        cols = np.concatenate(out_c)[o].astype(np.int32)
        vals = np.concatenate(out_v)[o]
        counts = np.bincount(rr, minlength=r1 - r0)
    else:
        cols, vals, counts = np.zeros(0, np.int32), np.zeros(0), np.zeros(r1 - r0, np.int64)
    row_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return CsrMatrix(r1 - r0, n, row_ptr, cols, vals)


def powerlaw_far_rows(n: int = 2**23, seed: int = 2604, row_begin: int = 0, row_end: int = None) -> CsrMatrix:
    """Rows [row_begin, row_end) of the config-4b far-column power-law matrix (host mirror
    of psell_gen_powerlaw_far_*; law in csrc/gen.cu): a near-diagonal walk and a walk
    spread uniformly over [0, n), merged into sorted unique columns."""
    r1 = n if row_end is None else int(row_end)
    r0 = int(row_begin)
    rows = np.arange(r0, r1, dtype=np.int64)
    with np.errstate(over="ignore"):
        hr = _smix(_U64(seed) ^ (rows.astype(_U64) * _U64(0xD1B54A32D192ED03)))

    def draw(stream, j, h):
        return _smix(h ^ (_U64(stream) << _U64(56)) ^ _U64(j))

    u = (draw(0, 0, hr) >> _U64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    L = np.maximum(np.searchsorted(-powerlaw_thresholds(), -u, side="right"), 1).astype(np.int64)
    mf = np.zeros(len(rows), np.int64)
    act = np.arange(len(rows))
    j = 0
    while act.size:
        mf[act] += (draw(2, j, hr[act]) % _U64(5) == 0)
        j += 1
        act = act[j < L[act]]
    mn = L - mf
    G2 = (2 * np.maximum(1, 8192 // np.maximum(mn, 1))).astype(_U64)
    S = np.maximum(n // (mf + 1), 1).astype(_U64)
    out_r, out_c = [], []

    def walk(c, count, stream, step_mod):
        act = np.nonzero((count > 0) & (c < n))[0]
        k = 0
        while act.size:
            out_r.append(act)
            out_c.append(c[act].copy())
            c[act] += 1 + (draw(stream, k, hr[act]) % step_mod[act]).astype(np.int64)
            k += 1
            act = act[(k < count[act]) & (c[act] < n)]

    walk(np.maximum(rows - 4096, 0) + (draw(6, 0, hr) % _U64(1024)).astype(np.int64), mn, 1, G2)
    walk((draw(5, 0, hr) % S).astype(np.int64), mf, 7, _U64(2) * S)
    if out_r:
        rr = np.concatenate(out_r)
        cc = np.concatenate(out_c)
        o = np.lexsort((cc, rr))
        rr, cc = rr[o], cc[o]
        keep = np.ones(len(rr), bool)
        keep[1:] = (rr[1:] != rr[:-1]) | (cc[1:] != cc[:-1])
        rr, cc = rr[keep], cc[keep]
        h = hr[rr]
        m = 0.01 + 0.99 * ((draw(4, 0, h ^ cc.astype(_U64)) >> _U64(11)).astype(np.float64)
                           * (1.0 / 9007199254740992.0))
        vals = np.where((draw(3, 0, h ^ cc.astype(_U64)) & _U64(1)) != 0, -m, m)
        counts = np.bincount(rr, minlength=r1 - r0)
        cols = cc.astype(np.int32)
    else:
        cols, vals, counts = np.zeros(0, np.int32), np.zeros(0), np.zeros(r1 - r0, np.int64)
    row_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return CsrMatrix(r1 - r0, n, row_ptr, cols, vals)


def powerlaw_thresholds() -> np.ndarray:
    """T_k = (4/k)^1.5, k = 1..8192: L >= k  <=>  u <= T_k (Pareto alpha 1.5)."""
    return (4.0 / np.arange(1, 8193, dtype=np.float64)) ** 1.5


def powerlaw(n: int = 2**23, seed: int = 2604) -> CsrMatrix:
    """The whole config-4 power-law matrix on the host (see powerlaw_rows)."""
    return powerlaw_rows(n, seed)


def powerlaw_far_k_left(n: int = 2**23, seed: int = 2604) -> int:
    """Lower bandwidth of the whole config-4b matrix from each row's first column only
    (the smaller of the two walks' starts), on the host: max_i(i - first_col_i)."""
    rows = np.arange(n, dtype=np.int64)
    with np.errstate(over="ignore"):
        hr = _smix(_U64(seed) ^ (rows.astype(_U64) * _U64(0xD1B54A32D192ED03)))

    def draw(stream, j, h):
        return _smix(h ^ (_U64(stream) << _U64(56)) ^ _U64(j))

    u = (draw(0, 0, hr) >> _U64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    L = np.maximum(np.searchsorted(-powerlaw_thresholds(), -u, side="right"), 1).astype(np.int64)
    mf = np.zeros(n, np.int64)
    act = np.arange(n)
    j = 0
    while act.size:
        mf[act] += (draw(2, j, hr[act]) % _U64(5) == 0)
        j += 1
        act = act[j < L[act]]
    big = np.int64(1) << 62
    near = np.where(L - mf > 0, np.maximum(rows - 4096, 0) + (draw(6, 0, hr) % _U64(1024)).astype(np.int64), big)
    far = np.where(mf > 0, (draw(5, 0, hr) % np.maximum(n // (mf + 1), 1).astype(_U64)).astype(np.int64), big)
    first = np.minimum(near, far)
    ok = first < n
    return int(max(0, int(np.max(rows[ok] - first[ok])))) if ok.any() else 0


def powerlaw_row_lengths(n: int = 2**23, seed: int = 2604, far: bool = False) -> np.ndarray:
    """Row lengths of the whole config-4 (4b: far=True) matrix (device count pass only) — partition weights."""
    import ctypes
    from . import _dev, _lib
    lib = _lib.lib()
    thr = _dev.upload(powerlaw_thresholds())
    ws = _dev.workspace(lib.psell_gen_workspace_bytes(n))
    row_ptr = _dev.empty(n + 1, np.int64)
    nnz = ctypes.c_int64(0)
    err = _lib.PsellError()
    plan = lib.psell_gen_powerlaw_far_plan if far else lib.psell_gen_powerlaw_plan
    rc = plan(n, seed, _lib.ptr(thr), 0, n, _lib.ptr(ws), ws.numel(), _lib.ptr(row_ptr), ctypes.byref(nnz),
              _lib.stream_handle(), err)
    _lib.check(rc, err)
    return np.diff(_dev.download(row_ptr, np.int64))


def powerlaw_device(n: int = 2**23, seed: int = 2604, *, row_begin: int = 0, row_end: int = None,
                    far: bool = False):
    """Rows [row_begin, row_end) of the config-4 matrix (config 4b with far=True) generated in
    HBM (DeviceCsrMatrix)."""
    import ctypes
    from . import _dev, _lib
    from .matrix import DeviceCsrMatrix
    lib = _lib.lib()
    r1 = n if row_end is None else int(row_end)
    r0 = int(row_begin)
    thr = _dev.upload(powerlaw_thresholds())
    ws = _dev.workspace(lib.psell_gen_workspace_bytes(r1 - r0))
    row_ptr = _dev.empty(r1 - r0 + 1, np.int64)
    nnz = ctypes.c_int64(0)
    err = _lib.PsellError()
    st = _lib.stream_handle()
    plan = lib.psell_gen_powerlaw_far_plan if far else lib.psell_gen_powerlaw_plan
    fill = lib.psell_gen_powerlaw_far_fill if far else lib.psell_gen_powerlaw_fill
    rc = plan(n, seed, _lib.ptr(thr), r0, r1, _lib.ptr(ws), ws.numel(), _lib.ptr(row_ptr), ctypes.byref(nnz), st, err)
    _lib.check(rc, err)
    col = _dev.empty(nnz.value, np.int32)
    val = _dev.empty(nnz.value, np.float64)
    rc = fill(n, seed, _lib.ptr(thr), r0, r1, _lib.ptr(row_ptr), _lib.ptr(col), _lib.ptr(val), st, err)
    _lib.check(rc, err)
    return DeviceCsrMatrix(r1 - r0, n, row_ptr, col, val, row0=r0)


_SCALES = {None: 0, "none": 0, "sym": 1, "rowsum": 2}


def stencil_device(kind: str, nx: int, ny: int = None, nz: int = None, *, scale=None,
                   row_begin: int = 0, row_end: int = None):
    """Generate rows [row_begin, row_end) of a stencil matrix directly in HBM.

    kind: "poisson2d" (5-pt, diag 4), "poisson3d" (7-pt, diag 6) or "stencil27"
    (27-pt box, diag 26).  scale: None, "sym" (sym_diag_scale) or "rowsum"
    (row_sum_scale).  Returns a DeviceCsrMatrix whose row0 = row_begin and whose
    n_cols is the global matrix size.
    """
    import ctypes
    from . import _dev, _lib
    from .matrix import DeviceCsrMatrix
    lib = _lib.lib()
    if kind == "poisson2d":
        dims, box, diag = (1, nx, nx if ny is None else ny), 0, 4.0
    elif kind == "poisson3d":
        dims, box, diag = (nx, nx if ny is None else ny, nx if nz is None else nz), 0, 6.0
    elif kind == "stencil27":
        dims, box, diag = (nx, nx if ny is None else ny, nx if nz is None else nz), 1, 26.0
    else:
        raise ValueError(f"unknown stencil {kind!r}")
    n = int(np.prod(dims))
    if n > 2**31 - 1:
        raise ValueError(f"grid of {n} points overflows 32-bit indexing")
    r1 = n if row_end is None else int(row_end)
    r0 = int(row_begin)
    rows = r1 - r0
    ws = _dev.workspace(lib.psell_gen_workspace_bytes(rows))
    row_ptr = _dev.empty(rows + 1, np.int64)
    nnz = ctypes.c_int64(0)
    err = _lib.PsellError()
    st = _lib.stream_handle()
    rc = lib.psell_gen_stencil_plan(dims[0], dims[1], dims[2], box, diag, r0, r1, _lib.ptr(ws),
                                    ws.numel(), _lib.ptr(row_ptr), ctypes.byref(nnz), st, err)
    _lib.check(rc, err)
    col = _dev.empty(nnz.value, np.int32)
    val = _dev.empty(nnz.value, np.float64)
    rc = lib.psell_gen_stencil_fill(dims[0], dims[1], dims[2], box, diag, _SCALES[scale], r0, r1,
                                    _lib.ptr(row_ptr), _lib.ptr(col), _lib.ptr(val), st, err)
    _lib.check(rc, err)
    return DeviceCsrMatrix(rows, n, row_ptr, col, val, row0=r0)


__all__ = ["poisson2d", "poisson3d", "stencil27", "powerlaw", "stencil_device"]
