"""Patch a reference `packsell` installation in place so its own callers run the B200 path
(INTEGRATION.md §2).

The reference modules import the path functions by name (solvers.py:26-27,
metrics.py:16-18, cli.py:25-27, container.py:25), so every importing module is
patched, plus the package namespace.  At the boundary the wrappers

* adopt reference `CsrMatrix` objects (same fields, host arrays) on the way in, so
  reference code and tests pass their own matrices; the B200 `PackSellMatrix` /
  `CsrMatrix` come back out and expose the reference's numpy fields;
* raise the reference's own exception classes (`codec.CodecError`,
  `container.ContainerError`, `matrix.MatrixFormatError`; the message is the B200
  one, equal to the reference's), so `except packsell.CodecError` keeps working;
* run `packsell_spmv` in the reference's rounding order (`ref_order=True`, bit for
  bit numpy, packed.py:264-268): the reference promises bit-reproducible SpMV
  against its CSR oracle (package docstring, test_packed.py:160-180), and a patched
  installation keeps that contract.  Callers after speed call
  `paper_2604_13433_b200.packsell_spmv` directly (FP32 FMA, within the stated bound).

    import packsell
    from paper_2604_13433_b200.integration import patch_reference
    patch_reference(packsell)      # returns the list of "module.name" it replaced
"""

from __future__ import annotations

import functools
import importlib

from . import codec as _codec
from . import container as _container
from . import matrix as _matrix
from . import metrics as _metrics
from . import packed as _packed
from . import solvers as _solvers
from .matrix import CsrMatrix, DeviceCsrMatrix


def adopt(A):
    """A reference CsrMatrix (or anything with its fields) as this package's CsrMatrix."""
    if isinstance(A, (CsrMatrix, DeviceCsrMatrix, _solvers.SpmvBackend)) or A is None:
        return A
    if all(hasattr(A, f) for f in ("n_rows", "n_cols", "row_ptr", "col_idx", "values")):
        return CsrMatrix(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values)
    return A


def _errors_of(pkg):
    """(B200 exception class, the reference's class) pairs for translation."""
    pairs = []
    for mod, name, mine in (("codec", "CodecError", _codec.CodecError),
                            ("container", "ContainerError", _container.ContainerError),
                            ("matrix", "MatrixFormatError", _matrix.MatrixFormatError)):
        try:
            theirs = getattr(importlib.import_module(f"{pkg.__name__}.{mod}"), name)
        except (ImportError, AttributeError):
            continue
        pairs.append((mine, theirs))
    return pairs


def _wrap(fn, errors, n_adopt: int = 0, kw=("A", "source", "matrix"), **fixed):
    """fn with its first n_adopt positional arguments (and the named keywords) adopted,
    `fixed` keywords applied, and B200 exceptions re-raised as the reference's classes."""
    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        args = tuple(adopt(a) if i < n_adopt else a for i, a in enumerate(args))
        for k in kw:
            if k in kwargs:
                kwargs[k] = adopt(kwargs[k])
        for k, v in fixed.items():
            kwargs.setdefault(k, v)
        try:
            return fn(*args, **kwargs)
        except tuple(m for m, _ in errors) as e:
            for mine, theirs in errors:
                if isinstance(e, mine):
                    raise theirs(str(e)) from e
            raise
    wrapped.__b200__ = True
    return wrapped


def _to_reference_csr(pkg, fn):
    """fn returning this package's CsrMatrix -> the reference's CsrMatrix (same arrays), so
    reference code downstream (its csr_spmv, permute_rows, ...) accepts it."""
    Ref = importlib.import_module(f"{pkg.__name__}.matrix").CsrMatrix

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        A = fn(*args, **kwargs)
        return Ref(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values) if isinstance(A, CsrMatrix) else A
    return wrapped


def _unless_foreign(fn, original):
    """fn, except for a matrix type of the reference's own that this package does not take
    (its SellMatrix: the comparator formats stay on the reference's CPU code)."""
    from .packed import PackSellMatrix
    from .sellfmt import SellMatrix

    @functools.wraps(fn)
    def wrapped(matrix, *args, **kwargs):
        ours = isinstance(matrix, (PackSellMatrix, SellMatrix, CsrMatrix, DeviceCsrMatrix)) or \
            type(matrix).__name__ == "CsrMatrix"
        return fn(matrix, *args, **kwargs) if ours or original is None else original(matrix, *args, **kwargs)
    return wrapped


def replacements(pkg) -> dict:
    """The B200 implementation of every reference name on the path and either side of it."""
    E = _errors_of(pkg)
    ref_metrics = importlib.import_module(f"{pkg.__name__}.metrics")
    return {
        "build_packsell": _wrap(_packed.build_packsell, E, 1),
        "packsell_spmv": _wrap(_packed.packsell_spmv, E, 0, ref_order=True),
        "packsell_to_csr": _to_reference_csr(pkg, _wrap(_packed.packsell_to_csr, E)),
        "footprint_bits": _wrap(_packed.footprint_bits, E),
        "encode_values": _wrap(_codec.encode_values, E),
        "decode_patterns": _wrap(_codec.decode_patterns, E),
        "pack_words": _wrap(_codec.pack_words, E),
        "unpack_words": _wrap(_codec.unpack_words, E),
        "quantize": _wrap(_codec.quantize, E),
        "make_backend": _wrap(_solvers.make_backend, E, 1),
        "pcg": _wrap(_solvers.pcg, E, 1),
        "fcg": _wrap(_solvers.fcg, E, 1),
        "iocg": _wrap(_solvers.iocg, E, 1),
        "backward_error": _wrap(_metrics.backward_error, E, 1),
        "bench_spmv": _unless_foreign(_wrap(_metrics.bench_spmv, E, 1), getattr(ref_metrics, "bench_spmv", None)),
        "read_psell": _wrap(_container.read_psell, E),
        "write_psell": _wrap(_container.write_psell, E),
    }


_MODULES = ("", ".codec", ".packed", ".solvers", ".metrics", ".container", ".cli")


def patch_reference(pkg) -> list:
    """Replace the reference's path functions by the B200 ones in every module that holds
    them (the package itself and codec / packed / solvers / metrics / container / cli)."""
    R = replacements(pkg)
    done = []
    for suffix in _MODULES:
        try:
            mod = importlib.import_module(pkg.__name__ + suffix) if suffix else pkg
        except ImportError:
            continue
        for name, impl in R.items():
            if hasattr(mod, name):
                setattr(mod, name, impl)
                done.append(f"{mod.__name__}.{name}")
    return done


__all__ = ["adopt", "patch_reference", "replacements"]
