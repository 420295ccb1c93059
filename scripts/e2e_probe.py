"""e2e probe (config 2): pinned-buffer copy rates per buffer and the pipelined public API with
the same / alternating host buffers, repeated, plus the host's NUMA view of the GPU."""
import glob
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_13433_b200 as P  # noqa: E402

print("cpu_count", os.cpu_count(), "affinity", sorted(os.sched_getaffinity(0))[:4], "...", len(os.sched_getaffinity(0)))
for d in glob.glob("/sys/bus/pci/devices/*"):
    try:
        if open(d + "/vendor").read().strip() == "0x10de" and open(d + "/class").read().startswith("0x0302"):
            print(d, "numa", open(d + "/numa_node").read().strip(), "cpus", open(d + "/local_cpulist").read().strip())
    except OSError:
        pass
print("nodes", glob.glob("/sys/devices/system/node/node*"))

n = 1 << 24
xh = torch.empty(n, dtype=torch.float16, pin_memory=True)
xh.copy_(torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n).astype(np.float16)))
yh = torch.empty(n, dtype=torch.float16, pin_memory=True)
x2 = xh.clone().pin_memory()
y2 = torch.empty_like(yh).pin_memory()
xd = torch.empty(n, dtype=torch.float16, device="cuda")
s = torch.cuda.Stream()


def rate(h, h2d, reps=20):
    torch.cuda.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(s):
        for _ in range(reps):
            (xd.copy_(h, non_blocking=True) if h2d else h.copy_(xd, non_blocking=True))
    torch.cuda.synchronize()
    return h.numel() * 2 * reps / (time.perf_counter() - t) / 1e9


for name, h in (("xh", xh), ("x2=clone.pin", x2), ("yh", yh), ("y2=empty_like.pin", y2)):
    print(f"{name:20s} H2D {rate(h, True):6.1f} GB/s  D2H {rate(h, False):6.1f} GB/s")

S = P.stencil_device("stencil27", 256)
M = P.build_packsell(S, 32, 256, P.parse_format("fp16"), "implicit")
del S
K = 50
for rep in range(3):
    for label, xs, ys in (("same", [xh] * K, [yh] * K), ("alt", [(xh, x2)[i & 1] for i in range(K)],
                                                       [(yh, y2)[i & 1] for i in range(K)])):
        P.packsell_spmv_stream(M, xs[:4], ys[:4])
        torch.cuda.synchronize()
        t = time.perf_counter()
        P.packsell_spmv_stream(M, xs, ys)
        torch.cuda.synchronize()
        print(f"rep {rep} {label:5s} {(time.perf_counter() - t) / K * 1e3:.3f} ms/step")
