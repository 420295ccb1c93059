"""Host numpy -> device upload paths for a 134 MB f64 solver vector (b at 256^3), and the reverse."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_13433_b200 import _dev  # noqa: E402

n = 256 ** 3
a = np.random.default_rng(0).standard_normal(n)
out = torch.empty(n, dtype=torch.float64, device="cuda")


def t(f, reps=5):
    f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


print(f"host memcpy 134MB: {t(lambda: np.copyto(np.empty_like(a), a)):.2f} ms")
print(f"pageable upload  : {t(lambda: torch.from_numpy(a).cuda()):.2f} ms")
print(f"_dev.upload      : {t(lambda: _dev.upload(a)):.2f} ms")
x16 = a[:n].astype(np.float16)
print(f"_dev.upload 33.5MB f16: {t(lambda: _dev.upload(x16)):.2f} ms  (pageable {t(lambda: torch.from_numpy(x16).cuda()):.2f} ms)")
print(f"threaded pinned (into out): {t(lambda: _dev.upload(a, out=out)):.2f} ms")
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
print(f"pinned full (memcpy+dma): {t(lambda: (h.numpy().__setitem__(Ellipsis, a), out.copy_(h, non_blocking=True))):.2f} ms")
print(f"dma only from pinned: {t(lambda: out.copy_(h, non_blocking=True)):.2f} ms")
print(f"download (pinned alloc): {t(lambda: _dev.download(out, np.float64)):.2f} ms")
print(f"torch .cpu()           : {t(lambda: out.cpu().numpy()):.2f} ms")
