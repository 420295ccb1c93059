"""ctypes binding of libpsell.so (the C ABI in include/psell.h).

The shared library is built in-tree (`paper_2604_13433_b200/libpsell.so`, see
csrc/Makefile or `__graft_entry__.build()`).  There is no CPU fallback: if the
library is missing, or no CUDA device is visible, every compute entry point
raises instead of silently computing on the host.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char, c_double, c_int32, c_int64, c_size_t, c_uint8, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# PSELL_LIB selects an alternative in-tree build for A/B runs (csrc/Makefile `alt` target)
LIB_PATH = os.path.join(_HERE, os.environ.get("PSELL_LIB", "libpsell.so"))

PSELL_OK, PSELL_EVALUE, PSELL_ECODEC, PSELL_ECUDA, PSELL_EARG = 0, 1, 2, 3, 4
KIND_NONE, KIND_FIRST_GAP, KIND_GAP_RANGE, KIND_NONFINITE, KIND_OVERFLOW, KIND_PARAM, KIND_CUDA = range(7)
CODEC_IDS = {"fp16": 0, "e8my": 1, "fp32embed": 2}
MODE_IDS = {"none": 0, "explicit": 1, "implicit": 2}
DT_F16, DT_F32, DT_F64 = 0, 1, 2
SPMV_REF_ORDER = 1
RED_BLOCKS = 1184


class PsellDesc(ctypes.Structure):
    _fields_ = [("w", c_int32), ("d", c_int32), ("codec", c_int32),
                ("c", c_int32), ("sigma", c_int32), ("mode", c_int32),
                ("n_rows", c_int64), ("n_cols", c_int64), ("row0", c_int64),
                ("k_left", c_int64), ("nnz", c_int64)]


class PsellError(ctypes.Structure):
    _fields_ = [("code", c_int32), ("kind", c_int32), ("index", c_int64), ("aux", c_int64),
                ("value", c_double), ("msg", c_char * 256)]


class LibpsellError(RuntimeError):
    """A CUDA/runtime failure inside libpsell (not a reference-level error)."""


_P = c_void_p
_D = POINTER(PsellDesc)
_E = POINTER(PsellError)

# name -> (restype, argtypes); must match include/psell.h
_SIGS = {
    "psell_version": (ctypes.c_char_p, []),
    "psell_abi_version": (c_int32, []),
    "psell_reload_env": (c_int32, []),
    "psell_build_workspace_bytes": (c_size_t, [_D]),
    "psell_lower_bandwidth": (c_int32, [_D, _P, _P, _P, c_size_t, POINTER(c_int64), _P, _E]),
    "psell_build_plan": (c_int32, [_D, _P, _P, _P, c_size_t, _P, _P, POINTER(c_int64), _P, _E]),
    "psell_build_fill": (c_int32, [_D, _P, _P, _P, _P, c_size_t, _P, _P, _P, _E]),
    "psell_sort_workspace_bytes": (c_size_t, [c_int64, c_int32]),
    "psell_sort_order": (c_int32, [_P, c_int64, c_int32, _P, _P, c_size_t, _P, _E]),
    "psell_spmv": (c_int32, [_D, _P, _P, _P, _P, c_int32, _P, c_int32, _P, _E]),
    "psell_spmv_kernel_name": (ctypes.c_char_p, [_D, c_int32, c_int32]),
    "psell_spmv_seg_checkpoints": (c_int32, [_D, _P, _P, c_int32, c_int64, _P, _P, c_int64, _P, _P, _P, _P, _E]),
    "psell_spmv_segmented": (c_int32, [_D, _P, _P, _P, _P, c_int32, _P, c_int32, c_int64, _P, _P, _P, _P,
                                       c_int64, _P, _P, _P, c_int32, _P, _E]),
    "psell_spmv_dot_partials": (c_int64, [_D, c_int32]),
    "psell_spmv_dot": (c_int32, [_D, _P, _P, _P, _P, _P, _P, _P, _P, c_int32, _P, _E]),
    "psell_to_csr_workspace_bytes": (c_size_t, [_D]),
    "psell_to_csr_plan": (c_int32, [_D, _P, _P, _P, _P, c_size_t, _P, POINTER(c_int64), _P, _E]),
    "psell_to_csr_fill": (c_int32, [_D, _P, _P, _P, _P, _P, _P, _P, _E]),
    "psell_max_column": (c_int32, [_D, _P, _P, _P, POINTER(c_int64), _P, _P, _E]),
    "psell_encode": (c_int32, [_D, _P, c_int64, _P, _P, _P, _E]),
    "psell_decode": (c_int32, [_D, _P, c_int64, _P, _P, _E]),
    "psell_pack_words": (c_int32, [_D, _P, _P, _P, c_int64, _P, _P, _E]),
    "psell_unpack_words": (c_int32, [_D, _P, c_int64, _P, _P, _P, _P, _E]),
    "psell_csr_spmv": (c_int32, [c_int64, _P, _P, _P, _P, c_int32, _P, _P, _E]),
    "psell_csr_spmv_dot": (c_int32, [c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _E]),
    "psell_halo_pack": (c_int32, [c_int64, _P, _P, _P, c_int32, _P]),
    "psell_halo_unpack": (c_int32, [c_int64, _P, _P, _P, c_int32, _P]),
    "psell_peer_arena_bytes": (c_size_t, [c_int64]),
    "psell_peer_vec_offset": (c_int64, [c_int64, c_int32]),
    "psell_peer_alloc": (c_int32, [c_size_t, POINTER(c_void_p), _P]),
    "psell_peer_open": (c_int32, [_P, POINTER(c_void_p)]),
    "psell_peer_close": (c_int32, [_P]),
    "psell_peer_free": (c_int32, [_P]),
    "psell_peer_exchange": (c_int32, [c_int32, c_int32, _P, c_int64, _P, _P, c_int64, _P, c_int32, c_int64, _P,
                                      c_int32, _P, c_int64, _P]),
    "psell_peer_error": (c_int32, [_P, POINTER(c_int32)]),
    "psell_backward_error": (c_int32, [c_int64, c_int64, _P, _P, _P, _P, c_int32, _P, c_int32, _P, _P, _E]),
    "psell_sum_partials": (c_int32, [_P, c_int64, c_int32, _P, _P, _P]),
    "psell_sum_strided": (c_int32, [_P, c_int32, c_int32, c_int32, _P, _P]),
    "psell_dot": (c_int32, [_P, _P, c_int32, c_int64, _P, _P, _P]),
    "psell_ipcg_begin": (c_int32, [c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "psell_ipcg_set_rz": (c_int32, [_P, c_int32, c_int32, _P, _P, _P]),
    "psell_ipcg_set_rz_gated": (c_int32, [_P, c_int32, c_int32, _P, _P, _P, _P]),
    "psell_ipcg_alpha": (c_int32, [_P, c_int32, c_int32, _P, _P, _P]),
    "psell_ipcg_update": (c_int32, [c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "psell_ipcg_beta": (c_int32, [_P, c_int32, c_int32, _P, _P, _P]),
    "psell_spmv_dot_alpha": (c_int32, [_D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, c_int32, _P, _E]),
    "psell_ipcg_update_beta": (c_int32, [c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "psell_spmv_dot_alpha_peer": (c_int32, [_D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, c_int32, c_int32, c_int32,
                                            _P, c_int64, _P, _E]),
    "psell_ipcg_direction_x_push": (c_int32, [c_int64, _P, _P, _P, _P, _P, c_int32, c_int32, _P, c_int64, c_int64,
                                              c_int32, _P, _P, _P, c_int64, _P]),
    "psell_ipcg_update_beta_peer": (c_int32, [c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, c_int32, c_int32, _P,
                                              c_int64, _P]),
    "psell_ipcg_direction_x": (c_int32, [c_int64, _P, _P, _P, _P, _P, _P]),
    "psell_ipcg_direction": (c_int32, [c_int64, _P, _P, _P, _P, _P]),
    "psell_ipcg_end": (c_int32, [c_int64, _P, _P, _P]),
    "psell_fcg_zr": (c_int32, [c_int64, _P, _P, _P, _P, _P, _P]),
    "psell_pq_pr": (c_int32, [c_int64, _P, _P, _P, _P, _P, _P]),
    "psell_axpy2": (c_int32, [c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "psell_xpby": (c_int32, [c_int64, _P, _P, _P, _P]),
    "psell_xpby_checked": (c_int32, [c_int64, _P, _P, _P, _P, _P]),
    "psell_resid": (c_int32, [c_int64, _P, _P, _P, _P, _P]),
    "psell_precond_dot": (c_int32, [c_int64, _P, _P, _P, _P, _P, _P]),
    "psell_scalar_div": (c_int32, [_P, _P, c_int32, c_int32, _P, _P, c_int32, _P]),
    "psell_pcg_status": (c_int32, [_P, _P, _P, c_double, c_double, _P, _P]),
    "psell_csr_spmv_dot_alpha": (c_int32, [c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _E]),
    "psell_pcg_update_status": (c_int32, [c_int64, _P, _P, _P, _P, _P, _P, c_double, c_double, _P, _P, _P, _P]),
    "psell_sell_fill": (c_int32, [_D, _P, _P, _P, _P, _P, c_int32, _P, _P, _P, _E]),
    "psell_sell_spmv": (c_int32, [_D, _P, c_int32, _P, _P, _P, _P, c_int32, _P, _P, _E]),
    "psell_sell_spmv_dot_partials": (c_int64, [_D]),
    "psell_sell_spmv_dot_alpha": (c_int32, [_D, _P, c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _E]),
    "psell_gen_workspace_bytes": (c_size_t, [c_int64]),
    "psell_gen_powerlaw_plan": (c_int32, [c_int64, c_uint64, _P, c_int64, c_int64, _P, c_size_t, _P,
                                          POINTER(c_int64), _P, _E]),
    "psell_gen_powerlaw_fill": (c_int32, [c_int64, c_uint64, _P, c_int64, c_int64, _P, _P, _P, _P, _E]),
    "psell_gen_powerlaw_far_plan": (c_int32, [c_int64, c_uint64, _P, c_int64, c_int64, _P, c_size_t, _P,
                                              POINTER(c_int64), _P, _E]),
    "psell_gen_powerlaw_far_fill": (c_int32, [c_int64, c_uint64, _P, c_int64, c_int64, _P, _P, _P, _P, _E]),
    "psell_gen_stencil_plan": (c_int32, [c_int64, c_int64, c_int64, c_int32, c_double, c_int64, c_int64,
                                         _P, c_size_t, _P, POINTER(c_int64), _P, _E]),
    "psell_gen_stencil_fill": (c_int32, [c_int64, c_int64, c_int64, c_int32, c_double, c_int32, c_int64,
                                         c_int64, _P, _P, _P, _P, _E]),
}

_lib = None


def exported_symbols():
    """Names the binding expects libpsell.so to export (for the ABI test)."""
    return sorted(_SIGS)


def load(require_gpu: bool = False):
    """Load libpsell.so once; raise loudly if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libpsell.so not found at {LIB_PATH}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.psell_abi_version() != 1:
            raise ImportError("libpsell ABI version mismatch")
        _lib = lib
    if require_gpu and not _gpu_ok:
        _check_gpu()
    return _lib


_gpu_ok = False


def _check_gpu():
    global _gpu_ok
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the PackSELL path runs on a CUDA (sm_100a) device only; "
                           "no CUDA device is visible and there is no CPU fallback")
    _gpu_ok = True  # checked once per process (the launch path is host-bound on small matrices)


def lib():
    if _lib is not None and _gpu_ok:
        return _lib
    return load(require_gpu=True)


_SMS = None


def sm_count() -> int:
    """Streaming multiprocessors of the current device (148 on B200), queried once."""
    global _SMS
    if _SMS is None:
        import torch
        _SMS = int(torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count)
    return _SMS


def ptr(t) -> int:
    """Device pointer of a torch tensor (or None -> NULL)."""
    return None if t is None else t.data_ptr()


_torch = None


def stream_handle():
    """The current CUDA stream of the current device, as a c_void_p.

    Uses torch's raw-stream query (0.1 us) instead of building a torch.cuda.Stream
    object (3.4 us measured): on small matrices the launch path is host-bound."""
    global _torch
    if _torch is None:
        import torch
        _torch = torch
    try:
        return c_void_p(_torch._C._cuda_getCurrentRawStream(_torch._C._cuda_getDevice()))
    except AttributeError:  # private API moved: the public path
        return c_void_p(_torch.cuda.current_stream().cuda_stream)


def check(rc: int, err: PsellError, fmt=None):
    """Turn a libpsell status into the reference's exception (or LibpsellError)."""
    if rc == PSELL_OK:
        return
    from . import codec as _codec
    if rc == PSELL_ECODEC:
        raise _codec.CodecError(_codec_message(err, fmt))
    if rc == PSELL_EVALUE:
        if err.kind == KIND_FIRST_GAP:
            raise ValueError(
                f"row {err.index}: first column {err.aux} is left of its base offset; "
                "lower bandwidth metadata is inconsistent")
        if err.kind == KIND_GAP_RANGE:
            raise ValueError(
                f"a column gap exceeds the dummy delta range 2**{fmt.w - 1} - 1; "
                "matrices this wide are not supported")
        raise ValueError(err.msg.decode(errors="replace"))
    raise LibpsellError(f"libpsell status {rc}: {err.msg.decode(errors='replace')}")


def _codec_message(err: PsellError, fmt) -> str:
    import numpy as np
    v = repr(np.float64(err.value))
    if err.kind == KIND_NONFINITE:
        return f"non-finite value {v} at position {err.index}"
    if fmt.codec == "fp16":
        return f"value {v} overflows FP16 (|v| beyond 65504) at position {err.index}"
    if fmt.codec == "e8my":
        return f"value {v} rounds to infinity in e8m{22 - fmt.d} at position {err.index}"
    return f"value {v} overflows FP32 at position {err.index}"


def check_launch(rc: int, what: str):
    if rc != PSELL_OK:
        raise LibpsellError(f"{what} failed with libpsell status {rc}")


def desc_for_format(fmt) -> PsellDesc:
    d = PsellDesc()
    d.w, d.d, d.codec = fmt.w, fmt.d, CODEC_IDS[fmt.codec]
    d.c, d.sigma, d.mode = 1, 1, 0
    d.n_rows = d.n_cols = d.row0 = d.nnz = 0
    d.k_left = 0
    return d


__all__ = ["load", "lib", "ptr", "check", "check_launch", "stream_handle", "PsellDesc", "PsellError",
           "LibpsellError", "exported_symbols", "desc_for_format", "LIB_PATH", "c_int64", "c_uint8",
           "c_uint64", "c_void_p"]
