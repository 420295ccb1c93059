"""`.psell` binary container, read into and written from HBM (reference container.py:1-103).

Same bytes as the reference: the 8-byte magic, the 68-byte little-endian
header (W, D, codec id, mode id as u8; C, sigma as u32; n_rows, n_cols,
k_left, nnz_real, n_dummy, n_padding, n_slices as u64), then the u64 slice
offsets, the perm (implicit mode only, u8 when sigma <= 256 else u16) and the
packed words (u32 / u64) — container.py:3-13, 39-53.  `write_psell` of a
device-resident matrix streams the packed words straight out of HBM through
one pinned staging buffer; `read_psell` reads the payload into pinned host
memory, validates it exactly as the reference does (same checks, same order,
same `ContainerError` messages, container.py:64-103) and uploads it with one
H2D copy per array, returning an HBM-resident `PackSellMatrix` that the CUDA
SpMV can run immediately.  Reading needs a CUDA device (the matrix lives in
HBM; there is no host-side matrix type to fall back to) — every validation
error is raised before the upload.
"""

from __future__ import annotations

import struct
from pathlib import Path
from typing import BinaryIO, Union

import numpy as np

from .codec import E8MY, FP16, FP32EMBED, PackFormat
from .packed import PackSellMatrix, StorageCounts
from .sell import perm_dtype

MAGIC = b"PSELL\x00v1"
_HEADER = struct.Struct("<BBBBIIQQQQQQQ")
_CODEC_IDS = {FP16: 1, E8MY: 2, FP32EMBED: 3}
_CODEC_NAMES = {v: k for k, v in _CODEC_IDS.items()}
_MODE_IDS = {"none": 0, "explicit": 1, "implicit": 2}
_MODE_NAMES = {v: k for k, v in _MODE_IDS.items()}


class ContainerError(ValueError):
    """Malformed or inconsistent .psell content (container.py:36-37)."""


def _pinned(nbytes: int) -> np.ndarray:
    """Host staging buffer: page-locked when a CUDA device is present (full-speed DMA)."""
    try:
        import torch
        if torch.cuda.is_available() and nbytes > 0:
            return torch.empty(nbytes, dtype=torch.uint8, pin_memory=True).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.empty(nbytes, dtype=np.uint8)


def _device_bytes(t, nbytes: int) -> np.ndarray:
    """D2H of a device tensor's raw bytes into pinned memory (no dtype round trip)."""
    import torch
    host = _pinned(nbytes)
    if nbytes:
        src = t.contiguous().view(torch.uint8)
        torch.from_numpy(host).copy_(src, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    return host


def header_bytes(M: PackSellMatrix) -> bytes:
    """Magic + header of M exactly as the reference writes them (container.py:43-48)."""
    return MAGIC + _HEADER.pack(
        M.fmt.w, M.fmt.d, _CODEC_IDS[M.fmt.codec], _MODE_IDS[M.mode],
        M.c, M.sigma, M.n_rows, M.n_cols, M.k_left,
        M.counts.nnz_real, M.counts.n_dummy, M.counts.n_padding, M.n_slices)


def write_psell(M: PackSellMatrix, dest: Union[str, Path, BinaryIO]) -> None:
    """Serialise M (container.py:39-53); identical bytes for identical matrices."""
    if not isinstance(M, PackSellMatrix):
        raise TypeError(f"write_psell expects a PackSellMatrix, got {type(M).__name__}")
    own = isinstance(dest, (str, Path))
    f = open(dest, "wb") if own else dest
    try:
        f.write(header_bytes(M))
        # offsets are non-negative int64: their bytes are the reference's '<u8' bytes
        f.write(np.ascontiguousarray(M.offset, dtype="<i8").tobytes())
        if M.mode == "implicit":
            pdt = perm_dtype(M.sigma).newbyteorder("<")
            if "perm" in M._h and M._h["perm"] is not None:
                f.write(np.ascontiguousarray(M._h["perm"]).astype(pdt).tobytes())
            else:
                f.write(memoryview(_device_bytes(M.d_perm, M.n_rows * pdt.itemsize)))
        wbytes = M.n_stored * M.fmt.word_dtype.itemsize
        if "pack" in M._h:
            f.write(np.ascontiguousarray(M._h["pack"]).astype(M.fmt.word_dtype.newbyteorder("<")).tobytes())
        else:
            f.write(memoryview(_device_bytes(M.d_pack, wbytes)))
    finally:
        if own:
            f.close()


def _read_exact(f: BinaryIO, n: int, what: str, into: np.ndarray = None):
    """n bytes or ContainerError "truncated container ..." (container.py:56-60)."""
    if into is None:
        data = f.read(n)
        got = len(data)
    else:
        got = 0
        mv = memoryview(into)
        readinto = getattr(f, "readinto", None)
        while got < n:
            if readinto is not None:
                k = readinto(mv[got:n])
            else:
                chunk = f.read(n - got)
                k = len(chunk)
                mv[got:got + k] = chunk
            if not k:
                break
            got += k
        data = into
    if got != n:
        raise ContainerError(f"truncated container: expected {n} bytes for {what}, got {got}")
    return data


def read_psell(source: Union[str, Path, BinaryIO]) -> PackSellMatrix:
    """Parse and validate a .psell container into an HBM-resident PackSellMatrix (container.py:63-103)."""
    own = isinstance(source, (str, Path))
    f = open(source, "rb") if own else source
    try:
        if _read_exact(f, len(MAGIC), "magic") != MAGIC:
            raise ContainerError("not a .psell container (bad magic)")
        fields = _HEADER.unpack(_read_exact(f, _HEADER.size, "header"))
        w, d, codec_id, mode_id, c, sigma, n_rows, n_cols, k_left, nnz, n_dummy, n_pad, n_slices = fields
        if codec_id not in _CODEC_NAMES:
            raise ContainerError(f"unknown codec id {codec_id}")
        if mode_id not in _MODE_NAMES:
            raise ContainerError(f"unknown mode id {mode_id}")
        try:
            fmt = PackFormat(w, d, _CODEC_NAMES[codec_id])
        except ValueError as e:
            raise ContainerError(f"invalid format in header: {e}") from None
        mode = _MODE_NAMES[mode_id]

        offset = np.frombuffer(_read_exact(f, 8 * (n_slices + 1), "offset array"), dtype="<u8").astype(np.int64)
        if len(offset) and (offset[0] != 0 or np.any(np.diff(offset) < 0)):
            raise ContainerError("offset array is not a non-decreasing prefix starting at 0")
        perm_raw = None
        if mode == "implicit":
            pdt = perm_dtype(sigma)
            perm_raw = _read_exact(f, pdt.itemsize * n_rows, "perm array", into=_pinned(pdt.itemsize * n_rows))
        n_words = int(offset[-1]) if len(offset) else 0
        _check_device_safe(fmt, c, sigma, mode, n_rows, n_cols, k_left, n_slices, offset, perm_raw)
        wdt = fmt.word_dtype
        pack_raw = _read_exact(f, wdt.itemsize * n_words, "pack array", into=_pinned(wdt.itemsize * n_words))
        if nnz + n_dummy + n_pad != n_words:
            raise ContainerError(
                f"header counts ({nnz} + {n_dummy} + {n_pad}) do not sum to the stored word count {n_words}")
    finally:
        if own:
            f.close()
    M = _upload(n_rows, n_cols, c, sigma, mode, fmt, pack_raw, offset, perm_raw, k_left,
                StorageCounts(nnz, n_dummy, n_pad))
    _check_stream_columns(M)
    return M


def _check_device_safe(fmt, c, sigma, mode, n_rows, n_cols, k_left, n_slices, offset, perm_raw):
    """Layout facts the reference's builder guarantees and the device kernels rely on.

    The reference reader checks only the counts (container.py:96-98) and its numpy
    SpMV would raise IndexError on a corrupt perm or column; on the device the same
    file would read or write out of bounds, so it is rejected here."""
    if fmt.codec == "fp16" and fmt.w != 32:
        raise ContainerError("fp16 values need 32-bit words on the device")
    if c < 1 or n_rows < 0 or n_cols < 0 or k_left < 0:
        raise ContainerError("header has a negative size or slice height")
    if n_rows >= 2 ** 31 or n_cols >= 2 ** 31:
        raise ContainerError(f"matrix of {n_rows} x {n_cols} exceeds 32-bit row / column indexing")
    if n_slices != -(-n_rows // c):
        raise ContainerError(f"header has {n_slices} slices, {n_rows} rows need {-(-n_rows // c)} of height {c}")
    if len(offset) and np.any(offset % c):
        raise ContainerError(f"offset array holds a slice start that is not a multiple of C = {c}")
    if perm_raw is not None and n_rows:
        perm = np.frombuffer(perm_raw, dtype=perm_dtype(sigma)).astype(np.int64)
        lim = np.minimum(sigma, n_rows - (np.arange(n_rows) // sigma) * sigma)
        bad = np.nonzero(perm >= lim)[0]
        if bad.size:
            raise ContainerError(f"perm[{bad[0]}] = {perm[bad[0]]} points outside its sigma-block")


def _check_stream_columns(M):
    """Every real word's column < n_cols (one device pass, psell_max_column)."""
    import ctypes
    from . import _dev, _lib
    if M.n_stored == 0:
        return
    ws = _dev.workspace(8)
    out = ctypes.c_int64(0)
    err = _lib.PsellError()
    rc = _lib.lib().psell_max_column(M.desc(), _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                                     ctypes.byref(out), _lib.ptr(ws), _lib.stream_handle(), err)
    _lib.check(rc, err, M.fmt)
    if M.counts.nnz_real and out.value >= M.n_cols:
        raise ContainerError(f"packed stream addresses column {out.value}, beyond n_cols = {M.n_cols}")


def _upload(n_rows, n_cols, c, sigma, mode, fmt, pack_raw, offset, perm_raw, k_left, counts):
    """Pinned staging -> HBM (one async H2D per array), then the device matrix."""
    import torch
    from . import _dev, _lib
    _lib.lib()  # loud failure without libpsell / a CUDA device (no host matrix fallback)

    def up(raw, np_dtype):
        t = _dev.empty(len(raw) // np.dtype(np_dtype).itemsize, np_dtype)
        if len(raw):
            t.view(torch.uint8).copy_(torch.from_numpy(raw), non_blocking=True)
        return t

    d_pack = up(pack_raw, fmt.word_dtype)
    d_offset = _dev.upload(offset)
    d_perm = up(perm_raw, perm_dtype(sigma)) if perm_raw is not None else None
    torch.cuda.current_stream().synchronize()  # staging buffers may be reused by the caller
    return PackSellMatrix(n_rows, n_cols, c, sigma, mode, fmt, d_pack, d_offset, d_perm, k_left, counts)


__all__ = ["MAGIC", "ContainerError", "read_psell", "write_psell", "header_bytes"]
