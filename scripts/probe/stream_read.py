"""Read-only HBM streaming ceiling vs the copy rate (csrc/vendor/probe.cu probe_stream_read):
the denominator question for a read-dominated SpMV.  2 GiB buffer (config 2 streams 1.94 GB)."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
L = ctypes.CDLL(os.path.join(ROOT, "paper_2604_13433_b200", "libpsell_vendor.so"))
P = ctypes.c_void_p
L.probe_stream_read.argtypes = [P, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, P, P]
nbytes = 2 << 30
buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
buf.random_(0, 255)
out = torch.zeros(4, dtype=torch.int32, device="cuda")
dst = torch.empty_like(buf)
sms = torch.cuda.get_device_properties(0).multi_processor_count
st = torch.cuda.current_stream().cuda_stream


def t_ms(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms = t_ms(lambda: dst.copy_(buf))
print(f"copy (read+write bytes)   {2 * nbytes / ms / 1e6:8.1f} GB/s  ({ms * 1e3:.1f} us)")
for unroll in (2, 4, 8):
    for cps in (4, 8):
        ms = t_ms(lambda: L.probe_stream_read(buf.data_ptr(), nbytes, unroll, sms * cps, out.data_ptr(), st))
        print(f"read-only U={unroll} ctas/SM={cps}  {nbytes / ms / 1e6:8.1f} GB/s  ({ms * 1e3:.1f} us)")
