"""Device-memory plumbing: numpy <-> torch CUDA tensors with the reference dtypes.

torch has no arithmetic on unsigned 16/32/64-bit types, so unsigned words are
stored in same-width signed tensors and re-viewed as unsigned on the numpy
side; the kernels only ever see raw pointers.
"""

from __future__ import annotations

import numpy as np
import torch

_NP2T = {
    np.dtype(np.float16): torch.float16,
    np.dtype(np.float32): torch.float32,
    np.dtype(np.float64): torch.float64,
    np.dtype(np.int8): torch.int8,
    np.dtype(np.uint8): torch.uint8,
    np.dtype(np.int16): torch.int16,
    np.dtype(np.uint16): torch.int16,
    np.dtype(np.int32): torch.int32,
    np.dtype(np.uint32): torch.int32,
    np.dtype(np.int64): torch.int64,
    np.dtype(np.uint64): torch.int64,
    np.dtype(np.bool_): torch.uint8,
}
_SIGNED = {np.dtype(np.uint16): np.int16, np.dtype(np.uint32): np.int32,
           np.dtype(np.uint64): np.int64, np.dtype(np.bool_): np.uint8}

DEVICE = "cuda"


def torch_dtype(np_dtype) -> torch.dtype:
    return _NP2T[np.dtype(np_dtype)]


def upload(a: np.ndarray, device=None) -> torch.Tensor:
    """Copy a host array to the device (unsigned types as same-width signed)."""
    a = np.ascontiguousarray(a)
    s = _SIGNED.get(a.dtype)
    if s is not None:
        a = a.view(s)
    return torch.from_numpy(a).to(device or DEVICE)


def download(t: torch.Tensor, np_dtype) -> np.ndarray:
    """Device tensor -> host array re-viewed as np_dtype (same item size)."""
    h = t.detach().cpu().numpy()
    return h.view(np.dtype(np_dtype)) if h.dtype != np.dtype(np_dtype) else h


def empty(n: int, np_dtype, device=None) -> torch.Tensor:
    return torch.empty(int(n), dtype=torch_dtype(np_dtype), device=device or DEVICE)


def zeros(n: int, np_dtype, device=None) -> torch.Tensor:
    return torch.zeros(int(n), dtype=torch_dtype(np_dtype), device=device or DEVICE)


def workspace(nbytes: int, device=None) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device or DEVICE)


DT_CODE = {np.dtype(np.float16): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2}
T_DT_CODE = {torch.float16: 0, torch.float32: 1, torch.float64: 2}
T2NP = {torch.float16: np.dtype(np.float16), torch.float32: np.dtype(np.float32),
        torch.float64: np.dtype(np.float64)}
