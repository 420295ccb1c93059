"""Warm PackSELL build of config 2 with the global k_left given (the bench path), per kernel."""
import sys, time, torch
sys.path.insert(0, ".")
import paper_2604_13433_b200 as P
from paper_2604_13433_b200.packed import lower_bandwidth
from torch.profiler import profile, ProfilerActivity
A = P.stencil_device("stencil27", 256)
kl = int(lower_bandwidth(A))
args = (32, 256, P.parse_format("fp16"), "implicit")
for _ in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    M = P.build_packsell(A, *args, _k_left_override=kl)
    torch.cuda.synchronize(); print(f"build(k_left given) {1e3*(time.perf_counter()-t0):.2f} ms"); del M
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    M = P.build_packsell(A, *args, _k_left_override=kl); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=8, max_name_column_width=40))
