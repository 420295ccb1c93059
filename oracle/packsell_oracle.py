"""CPU oracle: a plain-numpy restatement of the reference PackSELL path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites the
reference file:line it restates; paths are relative to
/root/reference/pkg/src/packsell/.  The code is written from the algorithm
description, not copied: sorting uses one
`np.lexsort` instead of a per-block loop, SpMV walks storage steps across all
slices at once instead of width groups, and so on.  Numerics (rounding points,
dtype promotion, reduction order of the solvers) follow the reference exactly
so the oracle is bit-identical to it; that is pinned by
tests/test_oracle_golden.py against fixtures produced by the reference itself.
"""

from __future__ import annotations

from typing import NamedTuple, Optional

import numpy as np

__all__ = [
    "Fmt", "OracleError", "OracleCodecError", "check_format", "preset", "fmt_v",
    "encode", "decode", "quantize", "pack_words", "unpack_words",
    "lower_bandwidth", "base_offsets", "OracleMatrix", "build", "spmv",
    "to_csr", "csr_spmv", "sort_order", "dot", "pcg", "fcg", "inner_pcg",
    "iocg", "format_error", "spmv_bytes",
]

FP16, E8MY, FP32EMBED = "fp16", "e8my", "fp32embed"


class Fmt(NamedTuple):
    """(W, D, codec) — codec.py:37-44."""
    w: int = 32
    d: int = 15
    codec: str = FP16


class OracleError(ValueError):
    """Layout/parameter error with the reference's payload (kind, index, aux, value)."""

    def __init__(self, kind: str, index: int = -1, aux: int = 0, value: float = 0.0):
        super().__init__(kind)
        self.kind, self.index, self.aux, self.value = kind, int(index), int(aux), float(value)


class OracleCodecError(OracleError):
    pass


def fmt_v(f: Fmt) -> int:
    """V = W - D - 1 (codec.py:64-67)."""
    return f.w - f.d - 1


def check_format(w: int, d: int, codec: str) -> Fmt:
    """Validation rules of PackFormat.__post_init__ (codec.py:45-62)."""
    if w not in (32, 64):
        raise ValueError("w")
    if d < 1 or d > w - 2:
        raise ValueError("d")
    v = w - d - 1
    if codec == FP16:
        if v != 16:
            raise ValueError("fp16 V")
    elif codec == E8MY:
        if w != 32 or v - 9 < 1:
            raise ValueError("e8my")
    elif codec == FP32EMBED:
        if w != 64 or v < 32:
            raise ValueError("fp32embed")
    else:
        raise ValueError("codec")
    return Fmt(w, d, codec)


def preset(name: str) -> Fmt:
    """Preset table of parse_format (codec.py:102-115)."""
    name = name.lower()
    table = {"fp16": (32, 15, FP16), "fp32embed": (64, 31, FP32EMBED)}
    if name in table:
        return check_format(*table[name])
    if name[:3] == "e8m" and name[3:].lstrip("-").isdigit():
        return check_format(32, 22 - int(name[3:]), E8MY)
    raise ValueError(name)


def _wt(f: Fmt):
    return np.uint32 if f.w == 32 else np.uint64


# ----------------------------------------------------------------------------
# value codecs (codec.py:124-181)
# ----------------------------------------------------------------------------

def encode(f: Fmt, values) -> np.ndarray:
    """f64 -> right-aligned V-bit patterns, raising on non-finite then overflow.

    Follows encode_values (codec.py:173-181): _check_finite first (124-127),
    then the codec: direct f64->f16 RNE (130-138); e8my = f64->f32 RNE,
    subnormal flush, snap to the 2^(e-24+D+1) grid with round-half-away
    (141-160); fp32embed = f32 bits << (V-32) (163-170).
    """
    v = np.asarray(values, dtype=np.float64)
    nf = np.nonzero(~np.isfinite(v))[0]
    if nf.size:
        raise OracleCodecError("nonfinite", nf[0], value=v[nf[0]])
    with np.errstate(over="ignore", invalid="ignore"):
        if f.codec == FP16:
            h = v.astype(np.float16)
            bad = np.nonzero(np.isinf(h))[0]
            if bad.size:
                raise OracleCodecError("overflow", bad[0], value=v[bad[0]])
            return h.view(np.uint16).astype(np.uint32)
        if f.codec == E8MY:
            s = v.astype(np.float32)
            sub = (np.abs(s) < np.float32(2.0 ** -126)) & (s != 0)
            s = np.where(sub, np.copysign(np.float32(0), s), s)
            e = np.frexp(s)[1].astype(np.int64)
            step = np.ldexp(1.0, e + (f.d - 23))          # 2^(e - 24 + D + 1)
            ratio = s.astype(np.float64) / step
            snapped = np.trunc(ratio + np.copysign(0.5, ratio)) * step
            q = snapped.astype(np.float32)
            bad = np.nonzero(np.isinf(q))[0]
            if bad.size:
                raise OracleCodecError("overflow", bad[0], value=v[bad[0]])
            return q.view(np.uint32) >> np.uint32(f.d + 1)
        s = v.astype(np.float32)
        bad = np.nonzero(np.isinf(s))[0]
        if bad.size:
            raise OracleCodecError("overflow", bad[0], value=v[bad[0]])
        return s.view(np.uint32).astype(np.uint64) << np.uint64(fmt_v(f) - 32)


def decode(f: Fmt, patterns) -> np.ndarray:
    """Patterns -> codec's natural float dtype (codec.py:184-192)."""
    if f.codec == FP16:
        return np.asarray(patterns).astype(np.uint16).view(np.float16)
    if f.codec == E8MY:
        return (np.asarray(patterns).astype(np.uint32) << np.uint32(f.d + 1)).view(np.float32)
    p = np.asarray(patterns).astype(np.uint64) >> np.uint64(fmt_v(f) - 32)
    return p.astype(np.uint32).view(np.float32)


def quantize(f: Fmt, values) -> np.ndarray:
    """decode(encode(v)) in f64 (codec.py:205-207)."""
    return decode(f, encode(f, values)).astype(np.float64)


def pack_words(f: Fmt, patterns, deltas, flags) -> np.ndarray:
    """Word assembly (codec.py:210-224): flag=1 -> pat<<(D+1)|delta<<1|1, else delta<<1.

    Deltas are reduced modulo 2^W exactly like numpy's astype of int64.
    """
    wt = _wt(f)
    pat = np.asarray(patterns).astype(wt)
    dl = np.asarray(deltas).astype(np.int64).astype(wt)
    fl = np.asarray(flags).astype(bool)
    real = (pat << wt(f.d + 1)) | (dl << wt(1)) | wt(1)
    return np.where(fl, real, dl << wt(1)).astype(wt)


def unpack_words(f: Fmt, words):
    """Branch-free unpack (codec.py:227-250) -> (values, deltas, flags)."""
    wt = _wt(f)
    w = np.asarray(words).astype(wt)
    flag = w & wt(1)
    sh = flag * wt(fmt_v(f))
    deltas = (w << sh) >> (sh + wt(1))
    if f.codec == FP16:
        vals = ((w >> wt(16)).astype(np.uint16) * flag.astype(np.uint16)).view(np.float16)
    elif f.codec == E8MY:
        vals = ((w & ~wt((1 << (f.d + 1)) - 1)) * flag).view(np.float32)
    else:
        hi = (w >> wt(f.d + 1)) * flag
        vals = (hi >> np.uint64(fmt_v(f) - 32)).astype(np.uint32).view(np.float32)
    return vals, deltas, flag.astype(bool)


# ----------------------------------------------------------------------------
# structure (matrix.py:319-349, packed.py:40-52, sell.py:22-46)
# ----------------------------------------------------------------------------

def lower_bandwidth(row_ptr, col_idx, row0: int = 0) -> int:
    """k_left = max(0, max_i(i - first_col_i)) over non-empty rows (matrix.py:334-339).

    `row0` shifts local row indices to global ones for slab builds.
    """
    rp = np.asarray(row_ptr, dtype=np.int64)
    lens = np.diff(rp)
    ne = np.nonzero(lens > 0)[0]
    if ne.size == 0:
        return 0
    first = np.asarray(col_idx)[rp[ne]].astype(np.int64)
    return int(max(0, int(np.max(ne + row0 - first))))


def base_offsets(n: int, sigma_eff: int, k_left: int, row0: int = 0) -> np.ndarray:
    """Eq. 4 leftmost offsets d_i (packed.py:40-52), for global rows row0..row0+n-1."""
    start = ((np.arange(n, dtype=np.int64) + row0) // sigma_eff) * sigma_eff
    return np.where(start > k_left, start - k_left, 0)


def sort_order(counts, sigma: int) -> np.ndarray:
    """Stable descending order inside sigma blocks (sell.py:22-30), one lexsort."""
    counts = np.asarray(counts, dtype=np.int64)
    idx = np.arange(len(counts), dtype=np.int64)
    return np.lexsort((idx, -counts, idx // sigma)).astype(np.int64)


class OracleMatrix(NamedTuple):
    """Fields of PackSellMatrix (packed.py:83-100) needed by the oracle."""
    n_rows: int
    n_cols: int
    c: int
    sigma: int
    mode: str
    fmt: Fmt
    pack: np.ndarray
    offset: np.ndarray
    perm: Optional[np.ndarray]
    k_left: int
    counts: tuple
    row0: int = 0

    @property
    def sigma_eff(self) -> int:
        return 1 if self.mode == "none" else self.sigma

    def out_index(self) -> np.ndarray:
        """packed.py:128-136."""
        s = np.arange(self.n_rows, dtype=np.int64)
        if self.mode == "implicit":
            return (s // self.sigma) * self.sigma + self.perm.astype(np.int64)
        return s


def build(row_ptr, col_idx, values, n_cols: int, c: int = 32, sigma: int = 256,
          f: Fmt = Fmt(), mode: str = "implicit", k_left: Optional[int] = None,
          row0: int = 0) -> OracleMatrix:
    """CSR -> PackSELL, restating build_packsell (packed.py:176-239).

    Order of checks: layout params (sell.py:33-42), first gap < 0
    (packed.py:159-164, reporting the row of the most negative first gap),
    any gap > 2^(W-1)-1 (166-170), then the codec (226).  `row0` builds the
    slab of global rows row0.. of a larger matrix (multi-GPU partitions);
    it must be sigma-aligned (C-aligned for mode none).
    """
    if mode not in ("none", "explicit", "implicit"):
        raise OracleError("mode")
    if c < 1:
        raise OracleError("c")
    if mode != "none":
        if sigma < 1 or sigma % c:
            raise OracleError("sigma")
        if sigma > 65536:
            raise OracleError("sigma_max")
    rp = np.asarray(row_ptr, dtype=np.int64)
    ci = np.asarray(col_idx, dtype=np.int32)
    vals = np.asarray(values, dtype=np.float64)
    n = len(rp) - 1
    nnz = int(rp[-1]) if n >= 0 else 0
    se = 1 if mode == "none" else sigma
    kl = lower_bandwidth(rp, ci, row0) if k_left is None else int(k_left)
    d_row = base_offsets(n, se, kl, row0)

    lens = np.diff(rp)
    row_of = np.repeat(np.arange(n, dtype=np.int64), lens)
    j_in_row = np.arange(nnz, dtype=np.int64) - rp[row_of]
    prev = np.empty(nnz, dtype=np.int64)
    if nnz:
        prev[1:] = ci[:-1]
        first = j_in_row == 0
        prev[first] = d_row[row_of[first]]
    gap = ci.astype(np.int64) - prev
    if nnz:
        fg = np.where(j_in_row == 0, gap, np.iinfo(np.int64).max)
        kmin = int(np.argmin(fg))
        if fg[kmin] < 0:
            r = int(row_of[kmin])
            raise OracleError("first_gap", r + row0, aux=int(ci[rp[r]]))
        if int(gap.max()) > (1 << (f.w - 1)) - 1:
            raise OracleError("gap_range")
    is_dummy = gap >= (1 << f.d)
    # dummies up to and including entry k, counted inside its row
    cz = np.concatenate([[0], np.cumsum(is_dummy.astype(np.int64))])
    q = j_in_row + cz[1:] - cz[rp[:-1]][row_of]
    stored = lens + (cz[rp[1:]] - cz[rp[:-1]])

    order = np.arange(n, dtype=np.int64) if mode == "none" else sort_order(stored, sigma)
    inv = np.empty(n, dtype=np.int64)
    inv[order] = np.arange(n, dtype=np.int64)
    n_slices = -(-n // c)
    scount = np.zeros(n_slices * c, dtype=np.int64)
    scount[:n] = stored[order]
    width = scount.reshape(n_slices, c).max(axis=1) if n_slices else np.zeros(0, np.int64)
    offset = np.concatenate([[0], np.cumsum(width * c)]).astype(np.int64)

    patterns = encode(f, vals)
    wt = _wt(f)
    pack = np.zeros(int(offset[-1]), dtype=wt)
    s = inv[row_of]
    slot = offset[s // c] + s % c
    pack[slot + q * c] = pack_words(f, patterns, np.where(is_dummy, 0, gap), np.ones(nnz, bool))
    dk = np.nonzero(is_dummy)[0]
    pack[slot[dk] + (q[dk] - 1) * c] = pack_words(f, np.zeros(dk.size), gap[dk], np.zeros(dk.size, bool))

    perm = None
    if mode == "implicit":
        perm = (order - (np.arange(n) // sigma) * sigma).astype(np.uint8 if sigma <= 256 else np.uint16)
    nd = int(is_dummy.sum())
    counts = (nnz, nd, int(offset[-1]) - nnz - nd)
    return OracleMatrix(n, int(n_cols), c, sigma, mode, f, pack, offset, perm, kl, counts, row0)


def _steps(M: OracleMatrix):
    """Yield (storage rows, word positions) per step q over all slices with width > q."""
    width = np.diff(M.offset) // M.c
    n_storage = len(width) * M.c
    srow = np.arange(n_storage, dtype=np.int64)
    w_row = np.repeat(width, M.c)
    base = M.offset[srow // M.c] + srow % M.c
    for q in range(int(width.max()) if width.size else 0):
        act = np.nonzero(w_row > q)[0]
        yield act, base[act] + q * M.c


def spmv(M: OracleMatrix, x) -> np.ndarray:
    """y = A x in x's dtype with reference rounding (packed.py:242-271).

    Decoded values are cast to x's dtype, every product and running sum is
    rounded in that dtype (no FMA), the cursor starts at
    min(d_s, n_cols-1) for storage row s (packed.py:257).
    """
    x = np.asarray(x)
    if len(x) != M.n_cols:
        raise ValueError("x length")
    wd = x.dtype
    n_storage = (len(M.offset) - 1) * M.c
    cursor = np.minimum(base_offsets(n_storage, M.sigma_eff, M.k_left, M.row0), max(M.n_cols - 1, 0))
    acc = np.zeros(n_storage, dtype=wd)
    for act, pos in _steps(M):
        v, dl, _ = unpack_words(M.fmt, M.pack[pos])
        cursor[act] += dl.astype(np.int64)
        acc[act] = acc[act] + v.astype(wd) * x[cursor[act]]
    y = np.zeros(M.n_rows, dtype=wd)
    y[M.out_index()] = acc[:M.n_rows]
    return y


def to_csr(M: OracleMatrix):
    """Decode every chain back to (row_ptr, col_idx, f64 values) in logical order (packed.py:274-303)."""
    n_storage = (len(M.offset) - 1) * M.c
    cursor = base_offsets(n_storage, M.sigma_eff, M.k_left, M.row0).copy()
    rows, cols, vals, seq = [], [], [], []
    for q, (act, pos) in enumerate(_steps(M)):
        v, dl, fl = unpack_words(M.fmt, M.pack[pos])
        cursor[act] += dl.astype(np.int64)
        keep = fl & (act < M.n_rows)
        rows.append(act[keep]); cols.append(cursor[act][keep]); vals.append(v[keep].astype(np.float64))
        seq.append(np.full(int(keep.sum()), q))
    out = M.out_index()
    if rows:
        r = out[np.concatenate(rows)]; cc = np.concatenate(cols); vv = np.concatenate(vals)
        o = np.lexsort((cc, r))
        r, cc, vv = r[o], cc[o], vv[o]
    else:
        r = cc = np.zeros(0, np.int64); vv = np.zeros(0)
    rp = np.zeros(M.n_rows + 1, dtype=np.int64)
    np.add.at(rp, r + 1, 1)
    return np.cumsum(rp), cc.astype(np.int32), vv


def csr_spmv(row_ptr, col_idx, values, x, dtype=np.float64) -> np.ndarray:
    """Row-sequential CSR SpMV in `dtype`, one rounding per op (matrix.py:272-291)."""
    wd = np.dtype(dtype)
    rp = np.asarray(row_ptr, dtype=np.int64)
    ci = np.asarray(col_idx, dtype=np.int64)
    xv = np.asarray(x).astype(wd)
    vv = np.asarray(values).astype(wd)
    n = len(rp) - 1
    lens = np.diff(rp)
    y = np.zeros(n, dtype=wd)
    live = np.nonzero(lens > 0)[0]
    if live.size:
        y[live] = vv[rp[live]] * xv[ci[rp[live]]]
    for j in range(1, int(lens.max()) if n else 0):
        r = np.nonzero(lens > j)[0]
        k = rp[r] + j
        y[r] = y[r] + vv[k] * xv[ci[k]]
    return y


def spmv_bytes(M: OracleMatrix, x_itemsize: int, y_itemsize: int, with_perm: bool = True) -> int:
    """Algorithmic bytes per SpMV."""
    b = (M.fmt.w // 8) * int(M.offset[-1]) + 8 * len(M.offset) + x_itemsize * M.n_cols \
        + y_itemsize * M.n_rows
    if with_perm and M.perm is not None:
        b += M.perm.dtype.itemsize * M.n_rows
    return int(b)


# ----------------------------------------------------------------------------
# solvers (solvers.py:87-333)
# ----------------------------------------------------------------------------

def dot(a, b) -> float:
    """f64 product then numpy pairwise add.reduce (solvers.py:87-89)."""
    return float(np.add.reduce(np.asarray(a).astype(np.float64) * np.asarray(b).astype(np.float64)))


def _nrm(a) -> float:
    return float(np.sqrt(dot(a, a)))


def _audit(res: dict, true_apply64, b, tol):
    """solvers.py:152-168."""
    bn = _nrm(b)
    if bn == 0.0:
        res["final_true_relres"] = 0.0
        return res
    res["final_true_relres"] = _nrm(b - true_apply64(res["x"])) / bn
    if res["converged"] and not res["final_true_relres"] < 10.0 * tol:
        res["converged"] = False
    return res


def pcg(apply, b, tol=1e-9, max_outer=1000, precond=None, true_apply64=None, x0=None) -> dict:
    """f64 PCG on the recurred residual (solvers.py:171-217)."""
    b = np.asarray(b, dtype=np.float64)
    P = precond or (lambda r: r)
    x = np.zeros_like(b) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
    bn = _nrm(b)
    if bn == 0.0:
        return dict(converged=True, outer_iters=0, history=[], x=x, final_true_relres=0.0)
    r = b - apply(x) if x.any() else b.copy()
    hist = [_nrm(r) / bn]
    z = P(r)
    p = z.copy()
    rz = dot(r, z)
    conv, it, reason = False, 0, None
    while it < max_outer:
        if hist[-1] < tol:
            conv = True
            break
        q = apply(p)
        pq = dot(p, q)
        if pq <= 0.0 or not np.isfinite(pq):
            reason = "breakdown"
            break
        a = rz / pq
        x += a * p
        r -= a * q
        it += 1
        hist.append(_nrm(r) / bn)
        z = P(r)
        rzn = dot(r, z)
        beta = rzn / rz
        rz = rzn
        p = z + beta * p
    if not conv and hist[-1] < tol:
        conv = True
    res = dict(converged=conv, outer_iters=it, history=hist, x=x, reason=reason)
    return _audit(res, true_apply64 or apply, b, tol)


def fcg(apply64, b, inner, tol=1e-9, max_outer=1000) -> dict:
    """Truncated flexible CG, one retained direction (solvers.py:220-275)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    bn = _nrm(b)
    if bn == 0.0:
        return dict(converged=True, outer_iters=0, history=[], x=x, final_true_relres=0.0)
    r = b.copy()
    hist = [_nrm(r) / bn]
    conv, it, p, r_old, zr_old, reason = False, 0, None, None, None, None
    while it < max_outer:
        if hist[-1] < tol:
            conv = True
            break
        z = inner(r)
        if p is None:
            p = z.copy()
        else:
            p = z + (dot(z, r - r_old) / zr_old) * p
        zr_old = dot(z, r)
        r_old = r.copy()
        q = apply64(p)
        pq = dot(p, q)
        if pq <= 0.0 or not np.isfinite(pq):
            reason = "breakdown"
            break
        a = dot(p, r) / pq
        x += a * p
        r -= a * q
        it += 1
        hist.append(_nrm(r) / bn)
    if not conv and hist[-1] < tol:
        conv = True
    res = dict(converged=conv, outer_iters=it, history=hist, x=x, reason=reason)
    return _audit(res, apply64, b, tol)


def inner_pcg(apply, r64, m_in, dtype=np.float32, precond=None):
    """Fixed-count reduced-precision PCG from zero (solvers.py:278-308)."""
    P = precond or (lambda r: r)
    rhs = np.asarray(r64).astype(dtype)
    x = np.zeros_like(rhs)
    r = rhs.copy()
    z = P(r)
    p = z.copy()
    rz = dot(r, z)
    done = 0
    for _ in range(m_in):
        q = apply(p)
        pq = dot(p, q)
        if pq <= 0.0 or not np.isfinite(pq) or rz == 0.0:
            break
        a = rz / pq
        x += a * p       # numpy weak-scalar promotion: a is rounded to dtype
        r -= a * q
        done += 1
        z = P(r)
        rzn = dot(r, z)
        beta = rzn / rz
        rz = rzn
        p = z + beta * p
    return x.astype(np.float64), done


def iocg(apply64, apply_inner, b, tol=1e-9, max_outer=1000, m_in=50, dtype=np.float32,
         precond=None) -> dict:
    """Inner-outer CG (solvers.py:311-333)."""
    total = [0]

    def inner(r):
        z, k = inner_pcg(apply_inner, r, m_in, dtype, precond)
        total[0] += k
        return z

    res = fcg(apply64, b, inner, tol, max_outer)
    res["total_inner_iters"] = total[0]
    return res


def format_error(err: OracleError, fmt: Fmt) -> str:
    """Message text the reference raises for each error kind (packed.py:159-170, codec.py:124-170)."""
    k = err.kind
    if k == "first_gap":
        return (f"row {err.index}: first column {err.aux} is left of its base offset; "
                "lower bandwidth metadata is inconsistent")
    if k == "gap_range":
        return (f"a column gap exceeds the dummy delta range 2**{fmt.w - 1} - 1; "
                "matrices this wide are not supported")
    v = repr(np.float64(err.value))
    if k == "nonfinite":
        return f"non-finite value {v} at position {err.index}"
    if fmt.codec == FP16:
        return f"value {v} overflows FP16 (|v| beyond 65504) at position {err.index}"
    if fmt.codec == E8MY:
        return f"value {v} rounds to infinity in e8m{22 - fmt.d} at position {err.index}"
    return f"value {v} overflows FP32 at position {err.index}"
