"""_dev.upload timing for 8.4 / 33.5 / 134 MB (env PSELL_H2D_THREADS / PSELL_H2D_CHUNK set by the caller)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_13433_b200 import _dev  # noqa: E402


def t(f, reps=7):
    f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


res = []
for nb in (8 << 20, 33554432, 134217728):
    a = np.random.default_rng(0).integers(0, 255, nb, dtype=np.uint8)
    res.append(f"{nb / 1e6:.1f}MB up {t(lambda: _dev.upload(a)):.2f} (pageable {t(lambda: torch.from_numpy(a).cuda()):.2f})")
print(f"threads={os.environ.get('PSELL_H2D_THREADS', '8')} chunk={os.environ.get('PSELL_H2D_CHUNK', '2097152')}: "
      + "; ".join(res), flush=True)
