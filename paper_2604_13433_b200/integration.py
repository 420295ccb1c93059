"""Patch a reference `packsell` installation in place so its own callers run the B200 path
(INTEGRATION.md §2).

The reference modules import the path functions by name (solvers.py:26-27,
metrics.py:16-18, cli.py:25-27, container.py:25), so every importing module is
patched, plus the package namespace.  Reference `CsrMatrix` objects are adopted
(same fields, host arrays) on the way in, so reference code and tests can pass
their own matrices; the B200 `PackSellMatrix` / `CsrMatrix` come back out and
expose the reference's numpy fields.

    import packsell
    from paper_2604_13433_b200.integration import patch_reference
    patch_reference(packsell)      # returns the list of "module.name" it replaced
"""

from __future__ import annotations

import functools
import importlib

from . import codec as _codec
from . import container as _container
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


def _adopting(fn, n_args: int = 1, kw=("A", "source", "matrix")):
    """fn with its first n_args positional arguments (and the named keywords) adopted."""
    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        args = tuple(adopt(a) if i < n_args else a for i, a in enumerate(args))
        for k in kw:
            if k in kwargs:
                kwargs[k] = adopt(kwargs[k])
        return fn(*args, **kwargs)
    wrapped.__b200__ = True
    return wrapped


# the B200 implementation of every reference name on the path and either side of it
REPLACEMENTS = {
    "build_packsell": _adopting(_packed.build_packsell),
    "packsell_spmv": _packed.packsell_spmv,
    "packsell_to_csr": _packed.packsell_to_csr,
    "footprint_bits": _packed.footprint_bits,
    "PackSellMatrix": _packed.PackSellMatrix,
    "encode_values": _codec.encode_values,
    "decode_patterns": _codec.decode_patterns,
    "pack_words": _codec.pack_words,
    "unpack_words": _codec.unpack_words,
    "quantize": _codec.quantize,
    "make_backend": _adopting(_solvers.make_backend),
    "pcg": _adopting(_solvers.pcg),
    "fcg": _adopting(_solvers.fcg),
    "iocg": _adopting(_solvers.iocg),
    "backward_error": _adopting(_metrics.backward_error),
    "bench_spmv": _adopting(_metrics.bench_spmv),
    "read_psell": _container.read_psell,
    "write_psell": _container.write_psell,
}

_MODULES = ("", ".codec", ".packed", ".solvers", ".metrics", ".container", ".cli")


def patch_reference(pkg) -> list:
    """Replace the reference's path functions by the B200 ones in every module that holds
    them (the package itself and codec / packed / solvers / metrics / container / cli)."""
    done = []
    for suffix in _MODULES:
        try:
            mod = importlib.import_module(pkg.__name__ + suffix) if suffix else pkg
        except ImportError:
            continue
        for name, impl in REPLACEMENTS.items():
            if hasattr(mod, name):
                setattr(mod, name, impl)
                done.append(f"{mod.__name__}.{name}")
    return done


__all__ = ["adopt", "patch_reference", "REPLACEMENTS"]
