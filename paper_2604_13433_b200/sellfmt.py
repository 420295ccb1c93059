"""SELL-C-sigma comparator format — drop-in for reference `packsell.sell`
(SellMatrix / build_sell / sell_spmv, sell.py:49-204).

The FP64 / FP32 / FP16 sliced-ELL baseline the paper compares PackSELL against
and the reference uses for `make_backend("sell64"|"sell32"|"sell16")` (the
FP32 IO-CG comparator of test_acceptance c08).  Built on the GPU with the
PackSELL plan (a format that cannot emit dummies gives plain row lengths) plus
a SELL fill kernel; the SpMV reproduces sell_spmv's rounding bit for bit.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from .sell import _check_layout_params, perm_dtype


class SellMatrix:
    """HBM-resident sliced ELL: val / col column-major per slice, int64 offsets, perm (sell.py:49-111)."""

    def __init__(self, n_rows, n_cols, c, sigma, mode, d_val, d_col, d_offset, d_perm=None,
                 nnz=None, n_padding=None, value_dtype=np.float64):
        self.n_rows, self.n_cols, self.c, self.sigma, self.mode = int(n_rows), int(n_cols), int(c), int(sigma), mode
        self.d_val, self.d_col, self.d_offset, self.d_perm = d_val, d_col, d_offset, d_perm
        self.nnz = None if nnz is None else int(nnz)
        self.n_padding = None if n_padding is None else int(n_padding)
        self.value_dtype = np.dtype(value_dtype)
        self._h = {}

    def _get(self, key, t, dt):
        if key not in self._h:
            from . import _dev
            self._h[key] = None if t is None else _dev.download(t, dt)
        return self._h[key]

    @property
    def val(self) -> np.ndarray:
        return self._get("val", self.d_val, self.value_dtype)

    @property
    def col(self) -> np.ndarray:
        return self._get("col", self.d_col, np.int32)

    @property
    def offset(self) -> np.ndarray:
        return self._get("offset", self.d_offset, np.int64)

    @property
    def perm(self) -> Optional[np.ndarray]:
        return self._get("perm", self.d_perm, perm_dtype(self.sigma))

    @property
    def n_slices(self) -> int:
        return int(self.d_offset.numel()) - 1

    @property
    def n_stored(self) -> int:
        return int(self.d_val.numel())

    def desc(self):
        from . import _lib
        d = _lib.PsellDesc()
        d.w, d.d, d.codec = 64, 31, _lib.CODEC_IDS["fp32embed"]
        d.c, d.sigma, d.mode = self.c, self.sigma, _lib.MODE_IDS[self.mode]
        d.n_rows, d.n_cols, d.row0, d.k_left, d.nnz = self.n_rows, self.n_cols, 0, 0, self.nnz or 0
        return d


def build_sell(A, c: int = 32, sigma: int = 256, mode: str = "implicit", value_dtype=np.float64) -> SellMatrix:
    """Sliced storage from CSR on the GPU (sell.py:114-178).

    `explicit` stores rows in sorted order without perm (== the reference's
    permute-then-build), `implicit` keeps the per-block perm, `none` no sort.
    """
    from . import _dev, _lib
    _check_layout_params(c, sigma, mode)
    vdt = np.dtype(value_dtype)
    if vdt not in _dev.DT_CODE:
        raise TypeError(f"unsupported value dtype {vdt}")
    lib = _lib.lib()
    D = A.to_device()
    d = _lib.PsellDesc()
    d.w, d.d, d.codec = 64, 31, _lib.CODEC_IDS["fp32embed"]  # no dummy words: counts = row lengths
    d.c, d.sigma, d.mode = int(c), int(sigma), _lib.MODE_IDS[mode]
    d.n_rows, d.n_cols, d.row0, d.k_left, d.nnz = D.n_rows, D.n_cols, 0, -1, D.nnz
    ws = _dev.workspace(lib.psell_build_workspace_bytes(d))
    ns = -(-D.n_rows // int(c))
    offset = _dev.empty(ns + 1, np.int64)
    perm = _dev.empty(D.n_rows, perm_dtype(sigma)) if mode == "implicit" else None
    out = (ctypes.c_int64 * 3)()
    err = _lib.PsellError()
    st = _lib.stream_handle()
    rc = lib.psell_build_plan(d, _lib.ptr(D.row_ptr), _lib.ptr(D.col_idx), _lib.ptr(ws), ws.numel(),
                              _lib.ptr(offset), _lib.ptr(perm), out, st, err)
    _lib.check(rc, err)
    n_stored = int(out[1])
    val = _dev.empty(n_stored, vdt)
    col = _dev.empty(n_stored, np.int32)
    rc = lib.psell_sell_fill(d, _lib.ptr(D.row_ptr), _lib.ptr(D.col_idx), _lib.ptr(D.values), _lib.ptr(ws),
                             _lib.ptr(offset), _dev.DT_CODE[vdt], _lib.ptr(val), _lib.ptr(col), st, err)
    _lib.check(rc, err)
    return SellMatrix(D.n_rows, D.n_cols, c, sigma, mode, val, col, offset, perm, nnz=D.nnz,
                      n_padding=n_stored - D.nnz, value_dtype=vdt)


def sell_spmv(M: SellMatrix, x, *, out=None):
    """y = M x in x's precision, numpy rounding order (sell.py:181-204).

    `out` (device x only): contiguous CUDA tensor of n_rows entries in x's dtype."""
    import torch
    from . import _dev, _lib
    lib = _lib.lib()
    on_dev = isinstance(x, torch.Tensor) and x.is_cuda
    if len(x) != M.n_cols:
        raise ValueError(f"x has length {len(x)}, expected {M.n_cols}")
    if on_dev:
        xd = x.contiguous()
        wd = _dev.T2NP.get(x.dtype)
    else:
        x = np.asarray(x)
        wd = x.dtype
        xd = _dev.upload(x)
    if wd not in _dev.DT_CODE:
        raise TypeError(f"unsupported x dtype {wd}")
    if out is not None:
        if not on_dev or not (out.is_cuda and out.is_contiguous() and out.numel() == M.n_rows
                              and out.dtype == xd.dtype and out.device == xd.device):
            raise ValueError("sell_spmv: out must be a contiguous CUDA tensor of n_rows entries in x's dtype")
        y = out
    else:
        y = _dev.empty(M.n_rows, wd)
    err = _lib.PsellError()
    rc = lib.psell_sell_spmv(M.desc(), _lib.ptr(M.d_val), _dev.DT_CODE[M.value_dtype], _lib.ptr(M.d_col),
                             _lib.ptr(M.d_offset), _lib.ptr(M.d_perm), _lib.ptr(xd), _dev.DT_CODE[wd], _lib.ptr(y),
                             _lib.stream_handle(), err)
    _lib.check(rc, err)
    return y if on_dev else _dev.download(y, wd)


__all__ = ["SellMatrix", "build_sell", "sell_spmv"]
