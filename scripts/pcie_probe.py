"""Pinned host<->device copy bandwidth (the e2e bound): H2D alone, D2H alone, both concurrently."""
import time

import torch

n = 33554432  # bytes per direction per step (config 2: x and y, f16, 16.7 M entries)
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=20):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


for _ in range(2):
    a, b, c = run(True, False), run(False, True), run(True, True)
print(f"H2D {n / a / 1e9:.1f} GB/s  D2H {n / b / 1e9:.1f} GB/s  concurrent: {c * 1e3:.3f} ms per step "
      f"({2 * n / c / 1e9:.1f} GB/s total)")
