"""Wide TMA kernel (PSELL_WIDE=1) vs the dual kernel on the 27-point 256^3 configs: CUDA-event
time over 100 launches and a digest of y (the two must be bitwise equal).  Each variant runs in
a fresh process; usage: wide_ab.py [config ...] (c2, c3, c3-e8m10)."""
import hashlib
import os
import subprocess
import sys

CFG = {"c2": ("fp16", "float16", None), "c3": ("e8m21", "float32", "rowsum"), "c3-e8m10": ("e8m10", "float32", "rowsum")}

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import torch
    sys.path.insert(0, ".")
    import paper_2604_13433_b200 as P  # noqa: E402
    from paper_2604_13433_b200 import _dev, _lib  # noqa: E402
    name = sys.argv[2]
    preset, xdt, scale = CFG[name]
    S = P.stencil_device("stencil27", 256, scale=scale)
    M = P.build_packsell(S, 32, 256, P.parse_format(preset), "implicit")
    del S
    xt = getattr(torch, xdt)
    g = torch.Generator(device="cuda")
    g.manual_seed(1234)
    x = (torch.rand(M.n_cols, generator=g, device="cuda") * 2 - 1).to(xt)
    y = torch.empty(M.n_rows, dtype=xt, device="cuda")
    kname = _lib.lib().psell_spmv_kernel_name(M.desc(), _dev.T_DT_CODE[xt], M.spmv_flags()).decode()
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
    nb = M.spmv_bytes(x.element_size(), x.element_size())
    print(f"  {name:9s} {kname[:28]:28s} {' '.join(f'{t:6.1f}' for t in ts)} us  {nb / min(ts) / 1e3:7.1f} GB/s  y {h}",
          flush=True)
    sys.exit(0)

# usage: wide_ab.py [configs ...] [-- VAR=VAL[,VAR=VAL] ...]  (default variants PSELL_WIDE=0 / 1)
args = sys.argv[1:]
variants = ["PSELL_WIDE=0", "PSELL_WIDE=1"]
if "--" in args:
    variants = args[args.index("--") + 1:]
    args = args[:args.index("--")]
for name in args or ["c2", "c3", "c3-e8m10"]:
    for v in variants:
        env = dict(os.environ)
        for kv in v.split(","):
            if kv:
                env[kv.split("=", 1)[0]] = kv.split("=", 1)[1]
        print(f"  [{v}]", end="", flush=True)
        subprocess.run([sys.executable, __file__, "--child", name], env=env, check=False)
