"""Sliced-ELL helpers the PackSELL builder shares with the SELL-C-sigma format
(reference sell.py:19-46).

`row_sort_order` runs the builder's device sort (psell_sort_order: stable
descending sort inside sigma blocks, one CTA per block).  The SELL-C-sigma
baseline format itself (SellMatrix / build_sell / sell_spmv) is the FP32/FP64
comparator of SURVEY.md §8 f2 and lives in `sellfmt.py`.
"""

from __future__ import annotations

import numpy as np

MODES = ("none", "explicit", "implicit")


def _check_layout_params(c: int, sigma: int, mode: str) -> None:
    """sell.py:33-42, same order and messages."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    if c < 1:
        raise ValueError(f"slice size must be >= 1, got {c}")
    if mode != "none":
        if sigma < 1 or sigma % c != 0:
            raise ValueError(f"sigma ({sigma}) must be a positive multiple of the slice size ({c})")
        if sigma > 65536:
            raise ValueError("sigma above 65536 is not supported (perm entries are at most 16-bit)")


def perm_dtype(sigma: int) -> np.dtype:
    """u8 perm entries for sigma <= 256, u16 otherwise (sell.py:45-46)."""
    return np.dtype(np.uint8) if sigma <= 256 else np.dtype(np.uint16)


def row_sort_order(counts, sigma: int) -> np.ndarray:
    """Storage order: descending count inside each sigma block, stable (sell.py:22-30)."""
    from . import _dev, _lib
    lib = _lib.lib()
    c = np.asarray(counts)
    n = len(c)
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    if c.min() < 0 or c.max() > 0xFFFFFFFF:
        raise ValueError("counts must fit in 32 unsigned bits")
    dc = _dev.upload(c.astype(np.uint32))
    order = _dev.empty(n, np.int32)
    ws = _dev.workspace(lib.psell_sort_workspace_bytes(n, int(sigma)))
    err = _lib.PsellError()
    rc = lib.psell_sort_order(_lib.ptr(dc), n, int(sigma), _lib.ptr(order), _lib.ptr(ws), ws.numel(),
                              _lib.stream_handle(), err)
    _lib.check(rc, err)
    return _dev.download(order, np.int32).astype(np.int64)


def __getattr__(name):
    """`sell.SellMatrix / build_sell / sell_spmv` as in the reference module (sell.py:49-204);
    they live in sellfmt (device containers), loaded lazily to keep this module import-light."""
    if name in ("SellMatrix", "build_sell", "sell_spmv"):
        from . import sellfmt
        return getattr(sellfmt, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
