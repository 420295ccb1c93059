"""Vendor comparators and measurement probes for the bench (NOT on the product path).

cuSPARSE sliced ELL ("cuSELL", the paper's primary vendor baseline,
PAPER.md §V) through libpsell_vendor.so (csrc/vendor/cusell.cu), on the
SELL-C-sigma storage of our own GPU builder (sellfmt.build_sell, implicit mode):
rows sigma-sorted and stored in sorted order — the paper's "explicitly
reordered rows" — with padded entries' columns set to -1 as cuSPARSE requires.
y comes back in storage order; `to_original` maps it back for checking.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_vlib = None


def vlib():
    global _vlib
    if _vlib is None:
        path = os.path.join(_HERE, "libpsell_vendor.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: build it with `make -C paper_2604_13433_b200/csrc vendor`")
        L = ctypes.CDLL(path)
        P = ctypes.c_void_p
        L.vendor_sell_prepare.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, P, P, P,
                                          ctypes.c_int32, P, P, P]
        L.vendor_cusell_create.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int32, P, P, P, ctypes.c_int32, ctypes.c_int32, P, P, P,
                                           ctypes.POINTER(P)]
        L.vendor_cusell_spmv.argtypes = [P]
        L.vendor_cusell_destroy.argtypes = [P]
        L.probe_gather.argtypes = [P, ctypes.c_int, ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P]
        _vlib = L
    return _vlib


class CuSell:
    """cuSPARSE SELL-C-sigma SpMV y_storage = A_sorted x (values and vectors in `dtype`,
    FP32 compute; FP64 for f64)."""

    def __init__(self, A, c: int = 32, sigma: int = 256, dtype=np.float32):
        import torch
        from . import _dev, _lib
        from .sellfmt import build_sell
        L = vlib()
        D = A.to_device()
        self.S = S = build_sell(D, c, sigma, "implicit", dtype)
        code = _dev.DT_CODE[np.dtype(dtype)]
        tdt = _dev.torch_dtype(dtype)
        self.off32 = torch.empty(S.n_slices + 1, dtype=torch.int32, device="cuda")
        pb = S.d_perm.element_size()
        st = _lib.stream_handle()
        if L.vendor_sell_prepare(S.n_rows, S.n_slices, c, sigma, S.d_offset.data_ptr(), D.row_ptr.data_ptr(),
                                 S.d_perm.data_ptr(), pb, S.d_col.data_ptr(), self.off32.data_ptr(), st):
            raise RuntimeError("vendor_sell_prepare failed")
        self.x = torch.zeros(S.n_cols, dtype=tdt, device="cuda")
        self.y = torch.zeros(S.n_slices * c, dtype=tdt, device="cuda")
        h = ctypes.c_void_p()
        rc = L.vendor_cusell_create(S.n_slices * c, S.n_cols, D.nnz, S.n_stored, c, self.off32.data_ptr(),
                                    S.d_col.data_ptr(), S.d_val.data_ptr(), code, code, self.x.data_ptr(),
                                    self.y.data_ptr(), st, ctypes.byref(h))
        if rc:
            raise RuntimeError(f"cusparse SELL setup failed (code {rc}) for {np.dtype(dtype).name}")
        self.h = h
        self.n_rows = S.n_rows
        self.bytes = S.n_stored * (np.dtype(dtype).itemsize + 4) + 4 * (S.n_slices + 1) + \
            np.dtype(dtype).itemsize * (S.n_cols + S.n_slices * c)

    def spmv(self):
        """y <- A x on the current stream (x, y are this object's bound device vectors)."""
        if vlib().vendor_cusell_spmv(self.h):
            raise RuntimeError("cusparseSpMV (SELL) failed")

    def to_original(self):
        """y in original row order (storage row s -> (s // sigma) * sigma + perm[s])."""
        import torch
        S = self.S
        s = torch.arange(S.n_rows, device="cuda")
        out_idx = (s // S.sigma) * S.sigma + S.d_perm.to(torch.int64) % (1 << (8 * S.d_perm.element_size()))
        y = torch.empty(S.n_rows, dtype=self.y.dtype, device="cuda")
        y[out_idx] = self.y[:S.n_rows]
        return y

    def close(self):
        if self.h:
            vlib().vendor_cusell_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def gather_ceiling(n_elems: int = 1 << 23, elem_bytes: int = 2, reps: int = 10) -> float:
    """Measured random-gather rate (gathers/s) of an L2-resident vector on this GPU: the
    ceiling of an SpMV whose x gathers land on unrelated 32-B sectors (config 4).  Every
    thread of a 8-CTA-per-SM grid issues 16 independent hashed gathers per round
    (csrc/vendor/probe.cu); scripts/probe/l2_gather.py sweeps the knobs (flat at ~289 G/s)."""
    import torch
    L = vlib()
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    grid, rounds, g = sms * 8, 64, 16
    x = torch.rand(n_elems, device="cuda").to(torch.float16 if elem_bytes == 2 else torch.float32)
    out = torch.zeros(grid * 256, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        L.probe_gather(x.data_ptr(), elem_bytes, n_elems, g, rounds, grid, out.data_ptr(), st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        L.probe_gather(x.data_ptr(), elem_bytes, n_elems, g, rounds, grid, out.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
    return grid * 256 * rounds * g / (e0.elapsed_time(e1) / reps * 1e-3)
