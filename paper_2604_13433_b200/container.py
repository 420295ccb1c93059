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

import contextlib
import struct
from pathlib import Path
from typing import BinaryIO, NamedTuple, Union

import numpy as np

from . import codec as _codec
from .codec import PackFormat
from .packed import PackSellMatrix, StorageCounts
from .sell import perm_dtype as _perm_dtype

MAGIC = b"PSELL\x00v1"


class _Header(NamedTuple):
    """The fixed little-endian header after the magic (container.py:27-36): u8 W, D, codec id,
    mode id; u32 C, sigma; u64 n_rows, n_cols, k_left, nnz, n_dummy, n_padding, n_slices."""
    w: int
    d: int
    codec_id: int
    mode_id: int
    c: int
    sigma: int
    n_rows: int
    n_cols: int
    k_left: int
    nnz: int
    n_dummy: int
    n_pad: int
    n_slices: int


_LAYOUT = struct.Struct("<4B2I7Q")
_CODECS = (None, _codec.FP16, _codec.E8MY, _codec.FP32EMBED)  # id -> codec (id 0 unused)
_MODES = ("none", "explicit", "implicit")                       # id -> mode


@contextlib.contextmanager
def _stream(target, mode: str):
    """A path is opened (and closed) here; a file object is used as is."""
    if isinstance(target, (str, Path)):
        with open(target, mode) as f:
            yield f
    else:
        yield target


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
    h = _Header(M.fmt.w, M.fmt.d, _CODECS.index(M.fmt.codec), _MODES.index(M.mode), M.c, M.sigma, M.n_rows,
                M.n_cols, M.k_left, M.counts.nnz_real, M.counts.n_dummy, M.counts.n_padding, M.n_slices)
    return MAGIC + _LAYOUT.pack(*h)


def write_psell(M: PackSellMatrix, dest: Union[str, Path, BinaryIO]) -> None:
    """Serialise M (container.py:39-53); identical bytes for identical matrices."""
    if not isinstance(M, PackSellMatrix):
        raise TypeError(f"write_psell expects a PackSellMatrix, got {type(M).__name__}")
    le_word = M.fmt.word_dtype.newbyteorder("<")
    sections = [header_bytes(M), np.ascontiguousarray(M.offset, dtype="<i8").tobytes()]  # offsets >= 0: '<u8' bytes
    if M.mode == "implicit":
        le_perm = _perm_dtype(M.sigma).newbyteorder("<")
        host_perm = M._h.get("perm")
        sections.append(np.ascontiguousarray(host_perm).astype(le_perm).tobytes() if host_perm is not None
                        else memoryview(_device_bytes(M.d_perm, M.n_rows * le_perm.itemsize)))
    sections.append(np.ascontiguousarray(M._h["pack"]).astype(le_word).tobytes() if "pack" in M._h
                    else memoryview(_device_bytes(M.d_pack, M.n_stored * le_word.itemsize)))
    with _stream(dest, "wb") as f:
        for part in sections:
            f.write(part)


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
    """Parse and validate a .psell container into an HBM-resident PackSellMatrix (container.py:63-103).

    The reference's checks in its order and words; the arrays land in page-locked
    buffers and go to HBM in one copy each."""
    with _stream(source, "rb") as f:
        if _read_exact(f, len(MAGIC), "magic") != MAGIC:
            raise ContainerError("not a .psell container (bad magic)")
        h = _Header(*_LAYOUT.unpack(_read_exact(f, _LAYOUT.size, "header")))
        if not 1 <= h.codec_id < len(_CODECS):
            raise ContainerError(f"unknown codec id {h.codec_id}")
        if h.mode_id >= len(_MODES):
            raise ContainerError(f"unknown mode id {h.mode_id}")
        try:
            fmt = PackFormat(h.w, h.d, _CODECS[h.codec_id])
        except ValueError as e:
            raise ContainerError(f"invalid format in header: {e}") from None
        mode = _MODES[h.mode_id]
        raw_off = _read_exact(f, 8 * (h.n_slices + 1), "offset array")
        offset = np.frombuffer(raw_off, dtype="<u8").astype(np.int64)
        if offset.size and (offset[0] != 0 or (offset[1:] < offset[:-1]).any()):
            raise ContainerError("offset array is not a non-decreasing prefix starting at 0")
        perm_raw = None
        if mode == "implicit":
            nb = _perm_dtype(h.sigma).itemsize * h.n_rows
            perm_raw = _read_exact(f, nb, "perm array", into=_pinned(nb))
        n_words = int(offset[-1]) if offset.size else 0
        _check_device_safe(fmt, h.c, h.sigma, mode, h.n_rows, h.n_cols, h.k_left, h.n_slices, offset, perm_raw)
        nb = fmt.word_dtype.itemsize * n_words
        pack_raw = _read_exact(f, nb, "pack array", into=_pinned(nb))
        if h.nnz + h.n_dummy + h.n_pad != n_words:
            raise ContainerError(f"header counts ({h.nnz} + {h.n_dummy} + {h.n_pad}) do not sum to the "
                                 f"stored word count {n_words}")
    M = _upload(h.n_rows, h.n_cols, h.c, h.sigma, mode, fmt, pack_raw, offset, perm_raw, h.k_left,
                StorageCounts(h.nnz, h.n_dummy, h.n_pad))
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
        perm = np.frombuffer(perm_raw, dtype=_perm_dtype(sigma)).astype(np.int64)
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
    d_perm = up(perm_raw, _perm_dtype(sigma)) if perm_raw is not None else None
    torch.cuda.current_stream().synchronize()  # staging buffers may be reused by the caller
    return PackSellMatrix(n_rows, n_cols, c, sigma, mode, fmt, d_pack, d_offset, d_perm, k_left, counts)


__all__ = ["MAGIC", "ContainerError", "read_psell", "write_psell", "header_bytes"]
