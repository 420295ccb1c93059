"""Device-memory plumbing: numpy <-> torch CUDA tensors with the reference dtypes.

torch has no arithmetic on unsigned 16/32/64-bit types, so unsigned words are
stored in same-width signed tensors and re-viewed as unsigned on the numpy
side; the kernels only ever see raw pointers.
"""

from __future__ import annotations

import os

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


_PINNED_MIN = 4 << 20  # results from 4 MiB up land in page-locked memory


_CHUNK_MIN = int(os.environ.get("PSELL_H2D_CHUNK", str(1 << 20)))  # host-copy / DMA granule (bytes)
_UPLOAD_THREADED_MIN = 16 << 20  # below this the pageable copy is as fast (scripts/upload_sweep.py)
_pool = None


def _copy_pool():
    global _pool
    if _pool is None:
        from concurrent.futures import ThreadPoolExecutor
        nt = int(os.environ.get("PSELL_H2D_THREADS", "4"))
        _pool = ThreadPoolExecutor(max_workers=max(1, min(nt, os.cpu_count() or 1)), thread_name_prefix="psell-h2d")
    return _pool


def upload(a: np.ndarray, device=None, out: torch.Tensor = None) -> torch.Tensor:
    """Copy a host array to the device (unsigned types as same-width signed).

    From 16 MiB up the array is copied into a page-locked block of torch's
    caching host allocator by 4 threads (numpy releases the GIL for the copy),
    chunks of max(1 MiB, size / 32), each chunk's DMA queued as soon as its
    host copy lands.  A single-threaded copy (the driver's pageable bounce
    buffer or one staging memcpy) runs at ~12 GB/s on the B200 hosts, a
    quarter of PCIe: 134 MB 11.4 ms pageable vs 4.9 ms, 33.5 MB 1.6 vs 1.2 ms
    (profiles/r01/upload_sweep.txt; 8 or 16 threads were no faster).  The pinned block returns to the cache when
    its DMA has completed (the allocator records the copy's stream event), so
    the call does not synchronise the device; `a` is no longer read on return.
    """
    a = np.ascontiguousarray(a)
    s = _SIGNED.get(a.dtype)
    if s is not None:
        a = a.view(s)
    dev = device or DEVICE
    if a.nbytes < _UPLOAD_THREADED_MIN or not torch.cuda.is_available():
        t = torch.from_numpy(a).to(dev)
        if out is None:
            return t
        out.copy_(t.view(out.shape))
        return out
    if out is None:
        out = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device=dev)
    src = a.reshape(-1).view(np.uint8)
    dst = out.view(-1).view(torch.uint8)
    if dst.numel() != src.size:
        raise ValueError(f"upload: out has {dst.numel()} bytes, array {src.size}")
    h = torch.empty(src.size, dtype=torch.uint8, pin_memory=True)
    hn = h.numpy()

    ck = max(_CHUNK_MIN, -(-src.size // 32) + 4095 & ~4095)

    def fill(off):
        hn[off:off + ck] = src[off:off + ck]

    offs = range(0, src.size, ck)
    futs = [_copy_pool().submit(fill, off) for off in offs]
    for off, f in zip(offs, futs):
        f.result()
        dst[off:off + ck].copy_(h[off:off + ck], non_blocking=True)
    return out


def download(t: torch.Tensor, np_dtype) -> np.ndarray:
    """Device tensor -> host array re-viewed as np_dtype (same item size).

    Large results are copied into a page-locked tensor from torch's caching host
    allocator and returned as a numpy view of it: full-PCIe D2H with no host
    bounce (33.5 MB: 0.6 ms vs 15.5 ms pageable; the pinned block returns to the
    cache when the array is released)."""
    t = t.detach()
    if t.is_cuda and t.numel() * t.element_size() >= _PINNED_MIN:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        h = h.numpy()
    else:
        h = t.cpu().numpy()
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
T2NP_ALL = {**T2NP, torch.int8: np.dtype(np.int8), torch.uint8: np.dtype(np.uint8), torch.int16: np.dtype(np.int16),
            torch.int32: np.dtype(np.int32), torch.int64: np.dtype(np.int64)}
