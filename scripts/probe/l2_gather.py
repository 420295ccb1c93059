"""Random-gather ceiling of an L2-resident vector on this GPU (the config-4 bound).

    python scripts/probe/l2_gather.py      (kernel: csrc/vendor/probe.cu in libpsell_vendor.so)

Prints gathers/s and the equivalent 32-B sector rate per (dtype, vector size, ILP,
CTAs per SM); the best f16 row at 2^23 elements (config 4's x) is the measured peak
the bench divides config 4's ncu lts__t_sectors rate by."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2604_13433_b200.vendor import vlib  # noqa: E402

L = vlib()
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.zeros(sms * 8 * 256, device="cuda")
rows = []
for dt in (torch.float16, torch.float32):
    for lg in (20, 23, 24):
        x = torch.rand(1 << lg, device="cuda").to(dt)
        for g in (8, 16):
            for per_sm in (4, 8):
                grid = sms * per_sm
                rounds = 64
                st = torch.cuda.current_stream().cuda_stream
                for _ in range(3):
                    L.probe_gather(x.data_ptr(), x.element_size(), 1 << lg, g, rounds, grid, out.data_ptr(), st)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                reps = 10
                for _ in range(reps):
                    L.probe_gather(x.data_ptr(), x.element_size(), 1 << lg, g, rounds, grid, out.data_ptr(), st)
                e1.record()
                torch.cuda.synchronize()
                s = e0.elapsed_time(e1) / reps * 1e-3
                n_g = grid * 256 * rounds * g
                r = {"dtype": str(dt).split(".")[1], "elems": 1 << lg, "MB": (1 << lg) * x.element_size() / 1e6,
                     "ilp": g, "ctas_per_sm": per_sm, "gathers_per_s": n_g / s, "sector_TBps": n_g * 32 / s / 1e12}
                rows.append(r)
                print(f"{r['dtype']:8s} 2^{lg} ({r['MB']:6.1f} MB) ilp {g:2d} ctas/SM {per_sm}: "
                      f"{r['gathers_per_s'] / 1e9:7.1f} G gathers/s = {r['sector_TBps']:6.2f} TB/s of 32-B sectors",
                      flush=True)
json.dump(rows, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/l2_gather.json", "w"), indent=1)
