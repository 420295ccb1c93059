"""Segmented power-law SpMV (configs 4 / 4b): the merged segment + dual grid (default) vs two
launches (PSELL_SEGMERGE=0).  CUDA-event time over 100 launches, digest of y (bitwise check).
usage: seg_ab.py [c4|c4b ...] [-- VAR=VAL[,..] ...]"""
import hashlib
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import torch
    sys.path.insert(0, ".")
    import bench  # noqa: E402
    import paper_2604_13433_b200 as P  # noqa: E402
    from paper_2604_13433_b200.packed import lower_bandwidth  # noqa: E402
    cfg = bench.CONFIGS[sys.argv[2]]
    S = bench.make_slab(cfg, 0, cfg["n"])
    M = P.build_packsell(S, 32, cfg["sigma"], P.parse_format(cfg["preset"]), "implicit",
                         _k_left_override=lower_bandwidth(S))
    del S
    g = torch.Generator(device="cuda")
    g.manual_seed(1234)
    x = (torch.rand(M.n_cols, generator=g, device="cuda") * 2 - 1).to(torch.float16)
    y = torch.empty(M.n_rows, dtype=torch.float16, device="cuda")
    for _ in range(10):
        P.packsell_spmv(M, x, out=y)
    torch.cuda.synchronize()
    h = hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest()[:16]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        e0.record()
        for _ in range(100):
            P.packsell_spmv(M, x, out=y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 100 * 1e3)
    print(f"  {sys.argv[2]:4s} {' '.join(f'{t:6.1f}' for t in ts)} us  y {h}", flush=True)
    sys.exit(0)

args = sys.argv[1:]
variants = ["PSELL_DSTATIC=0,PSELL_SEGMERGE=0", "PSELL_DSTATIC=0", "PSELL_DSTATIC=1"]
if "--" in args:
    variants = args[args.index("--") + 1:]
    args = args[:args.index("--")]
for name in args or ["c4", "c4b"]:
    for v in variants:
        env = dict(os.environ)
        for kv in v.split(","):
            if kv:
                env[kv.split("=", 1)[0]] = kv.split("=", 1)[1]
        print(f"  [{v}]", end="", flush=True)
        subprocess.run([sys.executable, __file__, "--child", name], env=env, check=False)
