"""W-bit word layout and value codecs — drop-in for reference `packsell.codec`.

Same names, signatures, validation messages and exception classes as the
reference (codec.py:33-269).  `PackFormat`/`parse_format` are host metadata;
every array operation (encode, decode, pack, unpack, quantize) runs on the GPU
through libpsell (`psell_encode`, `psell_decode`, `psell_pack_words`,
`psell_unpack_words`), the same device functions the builder and SpMV kernels
inline.  There is no numpy fallback.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np

FP16 = "fp16"
E8MY = "e8my"
FP32EMBED = "fp32embed"

_WORD_DTYPES = {32: np.dtype(np.uint32), 64: np.dtype(np.uint64)}


class CodecError(ValueError):
    """A value cannot be represented (non-finite input or overflow after rounding)."""


@dataclass(frozen=True)
class PackFormat:
    """(W, D, codec): word width, delta bits, value encoding (codec.py:37-99)."""

    w: int = 32
    d: int = 15
    codec: str = FP16

    def __post_init__(self):
        # the reference's checks, in its order and with its messages (codec.py:45-62)
        problem = self._problem()
        if problem is not None:
            raise ValueError(problem)

    def _problem(self) -> Optional[str]:
        w, d, c = self.w, self.d, self.codec
        if w not in _WORD_DTYPES:
            return f"word width must be 32 or 64, got {w}"
        if d < 1 or d > w - 2:
            return f"delta bits must be in [1, {w - 2}], got {d}"
        if c == FP16:
            return None if self.v == 16 else f"fp16 codec needs 16 value bits, got V={self.v} (use D={w - 17})"
        if c == E8MY:
            if w != 32:
                return "e8my codec requires 32-bit words"
            m = self.mantissa_bits
            return None if m >= 1 else f"e8my needs at least 1 mantissa bit (D={d} leaves {m})"
        if c == FP32EMBED:
            return None if (w == 64 and self.v >= 32) else "fp32embed codec requires 64-bit words and V >= 32"
        return f"unknown codec {c!r}"

    def __eq__(self, other):
        # a reference PackFormat with the same (W, D, codec) is the same format: a
        # patched reference installation (integration.py) compares its own formats
        # with the ones the B200 objects carry (the dataclass __eq__ would say False)
        if all(hasattr(other, f) for f in ("w", "d", "codec")):
            return (self.w, self.d, self.codec) == (other.w, other.d, other.codec)
        return NotImplemented

    def __hash__(self):
        return hash((self.w, self.d, self.codec))

    # derived layout (codec.py:64-99): V value bits, Y mantissa bits of e8mY, the largest
    # real / dummy delta, the numpy word and decoded value types, the preset name
    v = property(lambda self: self.w - self.d - 1)
    mantissa_bits = property(lambda self: self.v - 9)
    max_delta = property(lambda self: (1 << self.d) - 1)
    max_dummy_delta = property(lambda self: (1 << (self.w - 1)) - 1)
    word_dtype = property(lambda self: _WORD_DTYPES[self.w])
    value_dtype = property(lambda self: np.dtype(np.float16 if self.codec == FP16 else np.float32))

    @property
    def name(self) -> str:
        return {FP16: "fp16", FP32EMBED: "fp32embed"}.get(self.codec) or f"e8m{self.mantissa_bits}"


def parse_format(name: str) -> PackFormat:
    """Preset name -> PackFormat (codec.py:102-115)."""
    key = name.lower()
    if key == "fp16":
        return PackFormat(32, 15, FP16)
    if key == "fp32embed":
        return PackFormat(64, 31, FP32EMBED)
    if key.startswith("e8m"):
        try:
            y = int(key[3:])
        except ValueError:
            raise ValueError(f"unknown format preset {name.lower()!r}") from None
        return PackFormat(32, 22 - y, E8MY)
    raise ValueError(f"unknown format preset {key!r}")


class UnpackedEntry(NamedTuple):
    value: float
    delta: int
    has_value: bool


# ----------------------------------------------------------------------------
# device-backed array codecs
# ----------------------------------------------------------------------------

def _run(fmt: PackFormat):
    from . import _lib
    return _lib.lib(), _lib.desc_for_format(fmt)


def encode_values(fmt: PackFormat, values) -> np.ndarray:
    """Finite reals -> right-aligned V-bit patterns (codec.py:173-181), on device."""
    import torch
    from . import _dev, _lib
    lib, desc = _run(fmt)
    v = np.asarray(values, dtype=np.float64).reshape(-1)
    dv = _dev.upload(v)
    out = _dev.empty(len(v), fmt.word_dtype)
    ws = torch.empty(2, dtype=torch.int64, device=_dev.DEVICE)
    err = _lib.PsellError()
    rc = lib.psell_encode(desc, _lib.ptr(dv), len(v), _lib.ptr(out), _lib.ptr(ws),
                          _lib.stream_handle(), err)
    _lib.check(rc, err, fmt)
    pat = _dev.download(out, fmt.word_dtype)
    # the reference returns uint32 patterns for both 32-bit codecs, uint64 for fp32embed
    return pat


def decode_patterns(fmt: PackFormat, patterns) -> np.ndarray:
    """Right-aligned patterns -> codec's natural float dtype (codec.py:184-192)."""
    from . import _dev, _lib
    lib, desc = _run(fmt)
    wt = np.uint64 if fmt.codec == FP32EMBED else np.uint32
    p = np.asarray(patterns).astype(wt).reshape(-1)
    dp = _dev.upload(p)
    out = _dev.empty(len(p), fmt.value_dtype)
    err = _lib.PsellError()
    rc = lib.psell_decode(desc, _lib.ptr(dp), len(p), _lib.ptr(out), _lib.stream_handle(), err)
    _lib.check(rc, err, fmt)
    return _dev.download(out, fmt.value_dtype)


def encode_value(fmt: PackFormat, value: float) -> int:
    return int(encode_values(fmt, [value])[0])


def decode_value(fmt: PackFormat, pattern: int) -> float:
    return float(decode_patterns(fmt, [pattern])[0])


def quantize(fmt: PackFormat, values) -> np.ndarray:
    """decode(encode(v)) in float64 (codec.py:205-207)."""
    return decode_patterns(fmt, encode_values(fmt, values)).astype(np.float64)


def pack_words(fmt: PackFormat, patterns, deltas, flags) -> np.ndarray:
    """Assemble words (codec.py:210-224); deltas reduce modulo 2^W like numpy."""
    from . import _dev, _lib
    lib, desc = _run(fmt)
    wt = fmt.word_dtype
    pat = np.asarray(patterns).astype(wt).reshape(-1)
    n = len(pat)
    dl = np.asarray(deltas)
    # numpy's astype(uint) of the reference, then reinterpret as int64 for the ABI
    dl = dl.astype(wt).astype(np.uint64).view(np.int64).reshape(-1)
    fl = np.asarray(flags).astype(bool).astype(np.uint8).reshape(-1)
    dpat, ddl, dfl = _dev.upload(pat), _dev.upload(dl), _dev.upload(fl)
    out = _dev.empty(n, wt)
    err = _lib.PsellError()
    rc = lib.psell_pack_words(desc, _lib.ptr(dpat), _lib.ptr(ddl), _lib.ptr(dfl), n, _lib.ptr(out),
                              _lib.stream_handle(), err)
    _lib.check(rc, err, fmt)
    return _dev.download(out, wt)


def unpack_words(fmt: PackFormat, words):
    """Branch-free unpack (codec.py:227-250) -> (values, deltas, flags)."""
    from . import _dev, _lib
    lib, desc = _run(fmt)
    wt = fmt.word_dtype
    w = np.asarray(words, dtype=wt).reshape(-1)
    n = len(w)
    dw = _dev.upload(w)
    vals = _dev.empty(n, fmt.value_dtype)
    dl = _dev.empty(n, np.uint64)
    fl = _dev.empty(n, np.uint8)
    err = _lib.PsellError()
    rc = lib.psell_unpack_words(desc, _lib.ptr(dw), n, _lib.ptr(vals), _lib.ptr(dl), _lib.ptr(fl),
                                _lib.stream_handle(), err)
    _lib.check(rc, err, fmt)
    return (_dev.download(vals, fmt.value_dtype),
            _dev.download(dl, np.uint64).astype(wt),
            _dev.download(fl, np.uint8).astype(bool))


def pack(fmt: PackFormat, value: Optional[float], delta: int) -> int:
    """One (value, delta) pair; value None -> dummy/padding word (codec.py:253-262)."""
    if delta < 0:
        raise ValueError(f"delta must be non-negative, got {delta}")
    if value is None:
        if delta > fmt.max_dummy_delta:
            raise ValueError(f"dummy delta {delta} exceeds {fmt.max_dummy_delta}")
        return int(pack_words(fmt, [0], [delta], [False])[0])
    if delta > fmt.max_delta:
        raise ValueError(f"delta {delta} exceeds {fmt.max_delta} (needs a dummy word)")
    return int(pack_words(fmt, encode_values(fmt, [value]), [delta], [True])[0])


def unpack(fmt: PackFormat, word: int) -> UnpackedEntry:
    """Total on every W-bit pattern (codec.py:265-269)."""
    values, deltas, flags = unpack_words(fmt, [word])
    return UnpackedEntry(float(values[0]), int(deltas[0]), bool(flags[0]))
