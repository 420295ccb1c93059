"""PackSELL format: builder, SpMV, decode — drop-in for reference `packsell.packed`.

Same names and signatures as the reference (packed.py:23-327).  The matrix
lives in HBM; `build_packsell` runs the K1 CUDA pipeline (psell_build_plan +
psell_build_fill), `packsell_spmv` the K2 kernel, `packsell_to_csr` the K5
decode.  `PackSellMatrix` exposes the reference's numpy fields (`pack`,
`offset`, `perm` with the reference dtypes) as lazily downloaded, cached
host copies so reference-style tests and the .psell container keep working,
and accepts host arrays in its constructor (uploaded once).
"""

from __future__ import annotations

import ctypes
from typing import NamedTuple, Optional

import numpy as np

from . import codec
from .matrix import CsrMatrix
from .sell import _check_layout_params, perm_dtype

MODES = ("none", "explicit", "implicit")


class DeltaEntry(NamedTuple):
    delta: int
    value: Optional[float]  # None marks a dummy word


class StorageCounts(NamedTuple):
    nnz_real: int
    n_dummy: int
    n_padding: int


class FootprintReport(NamedTuple):
    pack_bits: int
    sell_equiv_bits: int
    ratio: float


def leftmost_offset(i: int, sigma: int, k_left: int) -> int:
    """Eq. 4 base column of row i (packed.py:40-47)."""
    start = (i // sigma) * sigma
    return start - k_left if k_left < start else 0


def _leftmost_offsets(n: int, sigma: int, k_left: int, row0: int = 0) -> np.ndarray:
    start = ((np.arange(n, dtype=np.int64) + row0) // sigma) * sigma
    return np.where(k_left < start, start - k_left, 0)


def build_delta_stream(row_cols, row_vals, d_i: int, fmt: codec.PackFormat) -> list:
    """Per-row delta stream with dummy insertion (packed.py:55-80), scalar test helper."""
    cols = [int(c) for c in row_cols]
    if cols and cols[0] < d_i:
        raise ValueError(
            f"first column {cols[0]} is left of the row base offset {d_i}; "
            "the lower bandwidth used to derive the offset is inconsistent"
        )
    out: list = []
    prev = d_i
    for col, val in zip(cols, row_vals):
        gap = col - prev
        if gap >= 1 << fmt.d:
            while gap > fmt.max_dummy_delta:
                out.append(DeltaEntry(fmt.max_dummy_delta, None))
                gap -= fmt.max_dummy_delta
            out.append(DeltaEntry(gap, None))
            gap = 0
        out.append(DeltaEntry(gap, float(val)))
        prev = col
    return out


def _is_tensor(a) -> bool:
    try:
        import torch
        return isinstance(a, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


class PackSellMatrix:
    """HBM-resident packed words + slice offsets + perm + bandwidth metadata (packed.py:83-142).

    `pack`, `offset`, `perm` are host numpy views (downloaded on first access);
    `d_pack`, `d_offset`, `d_perm` are the device tensors the kernels read.
    `row0` is the global index of local storage row 0 for a rank's slab.
    """

    def __init__(self, n_rows, n_cols, c, sigma, mode, fmt, pack, offset,
                 perm=None, k_left=0, counts=StorageCounts(0, 0, 0), *, row0: int = 0):
        from . import _dev
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.c = int(c)
        self.sigma = int(sigma)
        self.mode = mode
        self.fmt = fmt
        self.k_left = int(k_left)
        self.counts = StorageCounts(*counts)
        self.row0 = int(row0)
        self._h = {}
        if _is_tensor(pack):
            self.d_pack = pack
        else:
            p = np.asarray(pack, dtype=fmt.word_dtype)
            self._h["pack"] = p
            self.d_pack = _dev.upload(p)
        if _is_tensor(offset):
            self.d_offset = offset
        else:
            o = np.asarray(offset, dtype=np.int64)
            self._h["offset"] = o
            self.d_offset = _dev.upload(o)
        self._perm_dtype = None
        if perm is None:
            self.d_perm = None
            self._h["perm"] = None
        elif _is_tensor(perm):
            self.d_perm = perm
            self._perm_dtype = perm_dtype(self.sigma)
        else:
            pp = np.asarray(perm)
            self._h["perm"] = pp
            self._perm_dtype = pp.dtype
            self.d_perm = _dev.upload(pp.astype(perm_dtype(self.sigma)))
        self._out_idx = None
        self._seg = 0  # long-slice schedule: 0 = not built yet, None = none needed
        self._n_stored = int(self.d_pack.numel())
        self._n_slices = int(self.d_offset.numel()) - 1

    # -- reference numpy fields (lazy host copies)
    @property
    def pack(self) -> np.ndarray:
        if "pack" not in self._h:
            from . import _dev
            self._h["pack"] = _dev.download(self.d_pack, self.fmt.word_dtype)
        return self._h["pack"]

    @property
    def offset(self) -> np.ndarray:
        if "offset" not in self._h:
            from . import _dev
            self._h["offset"] = _dev.download(self.d_offset, np.int64)
        return self._h["offset"]

    @property
    def perm(self) -> Optional[np.ndarray]:
        if "perm" not in self._h:
            from . import _dev
            self._h["perm"] = _dev.download(self.d_perm, self._perm_dtype)
        return self._h["perm"]

    @property
    def n_slices(self) -> int:
        return self._n_slices

    @property
    def n_stored(self) -> int:
        return self._n_stored

    @property
    def effective_sigma(self) -> int:
        return 1 if self.mode == "none" else self.sigma

    def output_index(self) -> np.ndarray:
        """Original row of each storage row (packed.py:128-136)."""
        if self._out_idx is None:
            s = np.arange(self.n_rows, dtype=np.int64)
            if self.mode == "implicit":
                self._out_idx = (s // self.sigma) * self.sigma + self.perm[:self.n_rows].astype(np.int64)
            else:
                self._out_idx = s
        return self._out_idx

    def storage_base_offsets(self) -> np.ndarray:
        """Block-uniform base offsets per storage row (packed.py:138-142)."""
        return _leftmost_offsets(self.n_slices * self.c, self.effective_sigma, self.k_left, self.row0)

    # -- device side
    def desc(self):
        """The C descriptor (built once: the matrix is immutable)."""
        d = self.__dict__.get("_desc_cache")
        if d is not None:
            return d
        from . import _lib
        d = _lib.PsellDesc()
        d.w, d.d, d.codec = self.fmt.w, self.fmt.d, _lib.CODEC_IDS[self.fmt.codec]
        d.c, d.sigma, d.mode = self.c, self.sigma, _lib.MODE_IDS[self.mode]
        d.n_rows, d.n_cols, d.row0 = self.n_rows, self.n_cols, self.row0
        d.k_left, d.nnz = self.k_left, self.counts.nnz_real
        self.__dict__["_desc_cache"] = d
        return d

    def spmv_flags(self) -> int:
        """Kernel-shape hint for psell_spmv / psell_spmv_dot: PSELL_SPMV_NARROW when the
        mean slice width is <= 12 steps (7-point rows), so one 12-step chunk covers a slice;
        NARROW12 / W32 when every slice is <= 12 / 32 steps (the staged kernels' slots)."""
        if self.n_slices == 0:
            return 0
        f = self.__dict__.get("_flags_cache")
        if f is None:
            import torch
            f = 0
            wmax = int(torch.max(self.d_offset[1:] - self.d_offset[:-1]).item()) // self.c
            if self.n_stored <= 12 * self.c * self.n_slices:
                f = 4  # PSELL_SPMV_NARROW
                if wmax <= 12:
                    f |= 8  # PSELL_SPMV_NARROW12: every slice fits the slot kernel's 12 steps
            if self.c == 32 and wmax <= 32:
                f |= 16  # PSELL_SPMV_W32: every slice fits the wide TMA kernel's 32-step slot
            self.__dict__["_flags_cache"] = f
        return f

    def spmv_bytes(self, x_itemsize: int, y_itemsize: Optional[int] = None, with_perm: bool = True,
                   x_elems: Optional[int] = None) -> int:
        """Algorithmic bytes of one SpMV: words + slice offsets + x once + y (+ perm)."""
        y_itemsize = x_itemsize if y_itemsize is None else y_itemsize
        b = (self.fmt.w // 8) * self.n_stored + 8 * (self.n_slices + 1)
        b += x_itemsize * (self.n_cols if x_elems is None else x_elems) + y_itemsize * self.n_rows
        if with_perm and self.mode == "implicit":
            b += np.dtype(perm_dtype(self.sigma)).itemsize * self.n_rows
        return int(b)


def lower_bandwidth(A, c: int = 32, sigma: int = 256, mode: str = "implicit") -> int:
    """Device k_left of a (slab) CSR: max(0, max_i(row0 + i - first_col_i)) (matrix.py:334-339).

    Ranks of a row-partitioned build all-reduce MAX of this value and pass it
    as `_k_left_override` so every slab uses the global lower bandwidth.
    """
    from . import _dev, _lib
    lib = _lib.lib()
    D = A.to_device()
    d = _lib.PsellDesc()
    d.w, d.d, d.codec = 32, 15, 0
    d.c, d.sigma, d.mode = int(c), int(sigma), _lib.MODE_IDS[mode]
    d.n_rows, d.n_cols, d.row0, d.k_left, d.nnz = D.n_rows, D.n_cols, D.row0, -1, D.nnz
    ws = _dev.workspace(lib.psell_build_workspace_bytes(d))
    out = ctypes.c_int64(0)
    err = _lib.PsellError()
    rc = lib.psell_lower_bandwidth(d, _lib.ptr(D.row_ptr), _lib.ptr(D.col_idx), _lib.ptr(ws), ws.numel(),
                                   ctypes.byref(out), _lib.stream_handle(), err)
    _lib.check(rc, err)
    return int(out.value)


def build_packsell(A, c: int = 32, sigma: int = 256,
                   fmt: codec.PackFormat = codec.PackFormat(),
                   mode: str = "implicit", _k_left_override: Optional[int] = None) -> PackSellMatrix:
    """CSR -> PackSELL on the GPU (packed.py:176-239), byte-identical to the reference.

    `A` is a CsrMatrix (uploaded once and cached on the matrix) or a
    DeviceCsrMatrix (used in place; a rank slab when its row0 > 0, in which
    case pass the global k_left as `_k_left_override`).
    """
    from . import _dev, _lib
    _check_layout_params(c, sigma, mode)
    lib = _lib.lib()
    D = A.to_device()
    if _k_left_override is not None and int(_k_left_override) < 0:
        raise ValueError("negative k_left override is not supported")
    d = _lib.PsellDesc()
    d.w, d.d, d.codec = fmt.w, fmt.d, _lib.CODEC_IDS[fmt.codec]
    d.c, d.sigma, d.mode = int(c), int(sigma), _lib.MODE_IDS[mode]
    d.n_rows, d.n_cols, d.row0 = D.n_rows, D.n_cols, D.row0
    d.k_left = -1 if _k_left_override is None else int(_k_left_override)
    d.nnz = D.nnz
    ws = _dev.workspace(lib.psell_build_workspace_bytes(d))
    n_slices = -(-D.n_rows // int(c))
    offset = _dev.empty(n_slices + 1, np.int64)
    perm = _dev.empty(D.n_rows, perm_dtype(sigma)) if mode == "implicit" else None
    out = (ctypes.c_int64 * 3)()
    err = _lib.PsellError()
    st = _lib.stream_handle()
    rc = lib.psell_build_plan(d, _lib.ptr(D.row_ptr), _lib.ptr(D.col_idx), _lib.ptr(ws), ws.numel(),
                              _lib.ptr(offset), _lib.ptr(perm), out, st, err)
    _lib.check(rc, err, fmt)
    k_left, n_stored, n_dummy = int(out[0]), int(out[1]), int(out[2])
    d.k_left = k_left
    pack = _dev.empty(n_stored, fmt.word_dtype)
    rc = lib.psell_build_fill(d, _lib.ptr(D.row_ptr), _lib.ptr(D.col_idx), _lib.ptr(D.values),
                              _lib.ptr(ws), ws.numel(), _lib.ptr(offset), _lib.ptr(pack), st, err)
    _lib.check(rc, err, fmt)
    nnz = D.nnz
    counts = StorageCounts(nnz, n_dummy, n_stored - nnz - n_dummy)
    return PackSellMatrix(D.n_rows, D.n_cols, c, sigma, mode, fmt, pack, offset, perm, k_left,
                          counts, row0=D.row0)


SEG_LEN = 256  # steps per segment of a long slice (32 KB of words)


def _seg_dtypes():
    import torch
    return (torch.float16, torch.float32)


class _LazyDtypes:
    def __contains__(self, dt):
        return dt in _seg_dtypes()


_SEG_DTYPES = _LazyDtypes()


def _seg_schedule(M: PackSellMatrix):
    """Segments of the slices wider than SEG_LEN steps, with device cursor checkpoints.

    Built once per matrix from the int64 slice offsets (metadata only); the
    checkpoints come from psell_spmv_seg_checkpoints.  None when the matrix
    has no long slices or the layout is not segmentable (C != 32, W != 32).
    """
    if getattr(M, "_seg", 0) != 0:
        return M._seg
    M._seg = None
    if M.c != 32 or M.fmt.w != 32 or M.n_slices == 0:
        return None
    from . import _dev, _lib
    w = np.diff(M.offset) // M.c
    long_ = np.nonzero(w > SEG_LEN)[0]
    if long_.size == 0:
        return None
    per = -(-w[long_] // SEG_LEN)
    seg0 = np.concatenate([[0], np.cumsum(per)]).astype(np.int32)
    n_seg = int(seg0[-1])
    seg_slice = np.repeat(long_, per).astype(np.int32)
    seg_q0 = ((np.arange(n_seg) - np.repeat(seg0[:-1], per)) * SEG_LEN).astype(np.int32)
    G = _lib.sm_count()
    # static SM-affine ranges (PSELL_DSTATIC A/B): G contiguous slice-pair ranges balanced by the
    # words of the short slices (the long ones run as segments)
    ws = np.where(w > SEG_LEN, 0, w).astype(np.int64)
    ws = np.concatenate([ws, np.zeros(len(ws) % 2, np.int64)])
    pw = np.cumsum(ws[0::2] + ws[1::2])
    npairs = len(pw)
    NC = 2 * G  # word-balanced chunks: two per SM (psell: one 1024- or two 768-thread CTAs per SM)
    cut = np.searchsorted(pw, (pw[-1] * np.arange(1, NC)) // NC, side="right") if npairs else np.zeros(NC - 1, np.int64)
    ranges = np.concatenate([[0], np.minimum(cut, npairs), [npairs]]).astype(np.uint32)
    sched = np.concatenate([np.zeros(G + 1, np.uint32), ranges])
    s = dict(n_seg=n_seg, n_long=int(long_.size), seg_slice=_dev.upload(seg_slice), seg_q0=_dev.upload(seg_q0),
             long_slice=_dev.upload(long_.astype(np.int32)), long_seg0=_dev.upload(seg0),
             seg_c2=_dev.empty(n_seg * 32, np.uint32),
             # SM-affine scheduler counters of the short-slice kernel (left zeroed by every launch),
             # then the static ranges
             sched=_dev.upload(sched), sched_chunks=-G)  # < 0: the static chunk table follows
    lib = _lib.lib()
    err = _lib.PsellError()
    rc = lib.psell_spmv_seg_checkpoints(M.desc(), _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), SEG_LEN, n_seg,
                                        _lib.ptr(s["seg_slice"]), _lib.ptr(s["seg_q0"]), s["n_long"],
                                        _lib.ptr(s["long_slice"]), _lib.ptr(s["long_seg0"]),
                                        _lib.ptr(s["seg_c2"]), _lib.stream_handle(), err)
    _lib.check(rc, err, M.fmt)
    M._seg = s
    return s


_MODS = None


def _mods():
    """(_dev, _lib), imported on first use (they pull in torch / the library)."""
    global _MODS
    if _MODS is None:
        from . import _dev, _lib
        _MODS = (_dev, _lib)
    return _MODS


def _spmv_device(M: PackSellMatrix, xd, y, ref_order: bool, pipe: int = 0):
    _dev, _lib = _mods()
    lib = _lib.lib()
    err = _lib.PsellError()
    if not ref_order and not pipe and M.fmt.codec != codec.FP32EMBED and xd.dtype in _SEG_DTYPES:
        s = _seg_schedule(M)
        if s is not None:
            import torch
            part = torch.empty(s["n_seg"] * 32, dtype=torch.float32, device=xd.device)
            rc = lib.psell_spmv_segmented(M.desc(), _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                                          _lib.ptr(xd), _dev.T_DT_CODE[xd.dtype], _lib.ptr(y), SEG_LEN, s["n_seg"],
                                          _lib.ptr(s["seg_slice"]), _lib.ptr(s["seg_q0"]), _lib.ptr(s["seg_c2"]),
                                          _lib.ptr(part), s["n_long"], _lib.ptr(s["long_slice"]),
                                          _lib.ptr(s["long_seg0"]), _lib.ptr(s["sched"]), s["sched_chunks"],
                                          _lib.stream_handle(), err)
            _lib.check(rc, err, M.fmt)
            return y
    rc = lib.psell_spmv(M.desc(), _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                        _lib.ptr(xd), _dev.T_DT_CODE[xd.dtype], _lib.ptr(y),
                        (_lib.SPMV_REF_ORDER if ref_order else 0) | (2 if pipe else 0) | M.spmv_flags(),
                        _lib.stream_handle(), err)
    _lib.check(rc, err, M.fmt)
    return y


def packsell_spmv(M: PackSellMatrix, x, *, ref_order: bool = False, out=None, _pipe: int = 0):
    """y = M x with on-the-fly unpacking (packed.py:242-271), y in x's dtype.

    x: numpy array (returns numpy, the reference call), CUDA tensor (returns a
    CUDA tensor, no host traffic), or CPU tensor (ideally pinned; copied in,
    result copied back into `out` or a new CPU tensor, stream synchronised).
    Accumulation is FP32 FMA (FP64 for f64 x); `ref_order=True` reproduces the
    reference's numpy rounding bit for bit.
    """
    import torch
    _dev = _mods()[0]
    if isinstance(x, torch.Tensor):
        if x.dim() != 1:
            raise ValueError(f"x must be one-dimensional, got shape {tuple(x.shape)}")
        if x.shape[0] != M.n_cols:
            raise ValueError(f"x has length {x.shape[0]}, expected {M.n_cols}")
        if x.dtype not in _dev.T_DT_CODE:
            raise TypeError(f"unsupported x dtype {x.dtype}")
        if out is not None and (not isinstance(out, torch.Tensor) or out.dim() != 1 or out.shape[0] != M.n_rows
                                or out.dtype != x.dtype or not out.is_contiguous()):
            raise ValueError(f"out must be a contiguous {x.dtype} tensor of {M.n_rows} entries")
        if x.is_cuda:
            # device indices (ints) rather than torch.device objects: this is the
            # per-call path of small SpMVs, which are host-bound
            xi = x.get_device()
            if xi != M.d_pack.get_device():
                raise ValueError(f"x is on {x.device}, the matrix on {M.d_pack.device}")
            if out is not None and out.get_device() != xi:
                raise ValueError(f"out must be on {x.device}")
            y = out if out is not None else torch.empty(M.n_rows, dtype=x.dtype, device=x.device)
            return _spmv_device(M, x.contiguous(), y, ref_order, _pipe)
        xd = x.to(M.d_pack.device, non_blocking=True).contiguous()
        yd = torch.empty(M.n_rows, dtype=x.dtype, device=M.d_pack.device)
        _spmv_device(M, xd, yd, ref_order, _pipe)
        if out is None:
            out = torch.empty(M.n_rows, dtype=x.dtype, pin_memory=True)
        elif out.is_cuda:
            raise ValueError("out must be a host tensor for a host x")
        out.copy_(yd, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out
    x = np.asarray(x)
    if x.ndim != 1:
        raise ValueError(f"x must be one-dimensional, got shape {x.shape}")
    if len(x) != M.n_cols:
        raise ValueError(f"x has length {len(x)}, expected {M.n_cols}")
    if x.dtype not in _dev.DT_CODE:
        raise TypeError(f"unsupported x dtype {x.dtype}")
    xd = _dev.upload(x)
    y = _dev.empty(M.n_rows, x.dtype)
    _spmv_device(M, xd, y, ref_order, _pipe)
    return _dev.download(y, x.dtype)


def packsell_spmv_stream(M: PackSellMatrix, xs, outs=None, *, ref_order: bool = False):
    """Pipelined SpMVs over a sequence of host vectors: y_i = M x_i.

    The host<->device copies of consecutive calls overlap the SpMVs: x_{i+1}
    uploads on a copy-in stream while y_i = M x_i computes and y_{i-1}
    downloads on a copy-out stream (double-buffered device vectors, CUDA
    events between the three streams).  `xs` are CPU tensors (pinned for
    full-duplex DMA) or numpy arrays; results go to `outs` (CPU tensors) or
    new pinned tensors.  Returns the list of outputs after a final sync.
    """
    import torch
    from . import _dev
    xs = [torch.from_numpy(np.ascontiguousarray(x)) if not _is_tensor(x) else x for x in xs]
    if not xs:
        return []
    dt = xs[0].dtype
    if dt not in _dev.T_DT_CODE:
        raise TypeError(f"unsupported x dtype {dt}")
    for x in xs:
        if len(x) != M.n_cols:
            raise ValueError(f"x has length {len(x)}, expected {M.n_cols}")
    if outs is None:
        outs = [torch.empty(M.n_rows, dtype=dt, pin_memory=True) for _ in xs]
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    xd = [torch.empty(M.n_cols, dtype=dt, device=_dev.DEVICE) for _ in range(2)]
    yd = [torch.empty(M.n_rows, dtype=dt, device=_dev.DEVICE) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_cmp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    for i, x in enumerate(xs):
        b = i & 1
        with torch.cuda.stream(s_in):
            if i >= 2:
                s_in.wait_event(ev_cmp[b])        # x buffer b free (SpMV i-2 done)
            xd[b].copy_(x, non_blocking=True)
            ev_in[b].record(s_in)
        comp.wait_event(ev_in[b])
        if i >= 2:
            comp.wait_event(ev_out[b])             # y buffer b drained (D2H i-2 done)
        _spmv_device(M, xd[b], yd[b], ref_order)
        ev_cmp[b].record(comp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_cmp[b])
            outs[i].copy_(yd[b], non_blocking=True)
            ev_out[b].record(s_out)
    s_out.synchronize()
    comp.wait_stream(s_out)
    return outs


def packsell_to_csr(M: PackSellMatrix) -> CsrMatrix:
    """Decode every delta chain back to the quantised CSR, logical row order (packed.py:274-303)."""
    return _to_csr_device(M).to_host()


def _decoded_row_lengths(M: PackSellMatrix) -> np.ndarray:
    """Real entries per logical row (the decode's row pointer, packed.py:274-303) on the host."""
    from . import _dev, _lib
    lib = _lib.lib()
    d = M.desc()
    ws = _dev.workspace(lib.psell_to_csr_workspace_bytes(d))
    row_ptr = _dev.empty(M.n_rows + 1, np.int64)
    nnz = ctypes.c_int64(0)
    err = _lib.PsellError()
    rc = lib.psell_to_csr_plan(d, _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                               _lib.ptr(ws), ws.numel(), _lib.ptr(row_ptr), ctypes.byref(nnz),
                               _lib.stream_handle(), err)
    _lib.check(rc, err, M.fmt)
    return np.diff(_dev.download(row_ptr, np.int64))


def _to_csr_device(M: PackSellMatrix):
    """K5 decode into an HBM-resident CSR (DeviceCsrMatrix; row0 = M.row0)."""
    from . import _dev, _lib
    from .matrix import DeviceCsrMatrix
    lib = _lib.lib()
    d = M.desc()
    ws = _dev.workspace(lib.psell_to_csr_workspace_bytes(d))
    row_ptr = _dev.empty(M.n_rows + 1, np.int64)
    nnz = ctypes.c_int64(0)
    err = _lib.PsellError()
    st = _lib.stream_handle()
    rc = lib.psell_to_csr_plan(d, _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                               _lib.ptr(ws), ws.numel(), _lib.ptr(row_ptr), ctypes.byref(nnz), st, err)
    _lib.check(rc, err, M.fmt)
    col = _dev.empty(nnz.value, np.int32)
    val = _dev.empty(nnz.value, np.float64)
    rc = lib.psell_to_csr_fill(d, _lib.ptr(M.d_pack), _lib.ptr(M.d_offset), _lib.ptr(M.d_perm),
                               _lib.ptr(row_ptr), _lib.ptr(col), _lib.ptr(val), st, err)
    _lib.check(rc, err, M.fmt)
    return DeviceCsrMatrix(M.n_rows, M.n_cols, row_ptr, col, val, row0=M.row0)


def footprint_bits(M: PackSellMatrix) -> FootprintReport:
    """Packed vs like-for-like sliced storage bits (packed.py:306-327).

    The sliced side needs only the decoded row lengths: its padding is the
    SELL-C-sigma layout of those lengths (sell.py:124-147), computed here from
    the K5 decode's row pointer.
    """
    value_bits = 16 if M.fmt.codec == codec.FP16 else 32
    perm_bits = 0 if M.perm is None else M.perm.dtype.itemsize * 8 * len(M.perm)
    pack_bits = M.fmt.w * M.n_stored + 64 * (M.n_slices + 1) + perm_bits
    lens = _decoded_row_lengths(M)  # K5 count pass only: no column / value decode or download
    sell_mode = "none" if M.mode == "explicit" else M.mode
    n = M.n_rows
    if sell_mode == "none":
        ordered = lens
    else:
        from .sell import row_sort_order
        ordered = lens[row_sort_order(lens, M.sigma)]
    n_sl = -(-n // M.c)
    padded = np.zeros(n_sl * M.c, dtype=np.int64)
    padded[:n] = ordered
    sell_stored = int((padded.reshape(n_sl, M.c).max(axis=1) * M.c).sum()) if n_sl else 0
    sell_perm_bits = 8 * np.dtype(perm_dtype(M.sigma)).itemsize * n if sell_mode == "implicit" else 0
    sell_bits = (value_bits + 32) * sell_stored + 64 * (n_sl + 1) + sell_perm_bits
    ratio = pack_bits / sell_bits if sell_bits else 1.0
    return FootprintReport(int(pack_bits), int(sell_bits), float(ratio))
