"""Randomised parity of the segmented (long-slice) SpMV: random power-law matrices with rows up
to a few thousand entries, random sigma / codec / x dtype: the static SM-affine grid (default) bitwise equal to the
merged segment grid and to the two-launch form, within the FMA bound of the oracle's
REF-order SpMV.  usage: fuzz_segments.py [n_cases] [seed]"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_2604_13433_b200 as P  # noqa: E402
from paper_2604_13433_b200 import _lib  # noqa: E402
from paper_2604_13433_b200.packed import _seg_schedule  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
lib = _lib.lib()
fails = segs = 0
for it in range(n_cases):
    n = int(rng.integers(2000, 40000))
    lens = np.minimum(n, (rng.pareto(1.2, n) * 3 + 1).astype(np.int64))
    lens[rng.integers(0, n, 3)] = rng.integers(300, min(n, 5000), 3)
    rows = np.repeat(np.arange(n), lens)
    cols = np.clip(rows + rng.integers(-3000, 3000, rows.size), 0, n - 1)
    order = np.lexsort((cols, rows))
    r, c = rows[order], cols[order]
    keep = np.ones(r.size, bool)
    keep[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    r, c = r[keep], c[keep]
    v = rng.uniform(0.01, 1, r.size) * rng.choice([-1.0, 1.0], r.size)
    rp = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=n))]).astype(np.int64)
    A = P.CsrMatrix(n, n, rp, c.astype(np.int32), v)
    sigma = int(rng.choice([32, 256, 992, 4096]))
    pre = str(rng.choice(["fp16", "e8m14", "e8m10"]))
    dt = [np.float16, np.float32][int(rng.integers(0, 2))]
    try:
        M = P.build_packsell(A, 32, sigma, P.parse_format(pre), "implicit")
        s = _seg_schedule(M)
        segs += s is not None and s["n_seg"] > 0
        x = rng.uniform(-1, 1, n).astype(dt)
        y1 = P.packsell_spmv(M, x)
        for env in ({"PSELL_DSTATIC": "0"}, {"PSELL_DSTATIC": "0", "PSELL_SEGMERGE": "0"}):
            os.environ.update(env)
            lib.psell_reload_env()
            y0 = P.packsell_spmv(M, x)
            for k in env:
                os.environ.pop(k)
            lib.psell_reload_env()
            assert np.array_equal(y1.view(np.uint8), y0.view(np.uint8)), f"static != {env}"
        OM = O.build(A.row_ptr, A.col_idx, A.values, A.n_cols, 32, sigma, O.preset(pre), "implicit")
        ref = O.spmv(OM, x.astype(np.float32)).astype(np.float64)
        lmax = int(np.max(np.diff(OM.offset) // 32))
        aq = np.abs(O.quantize(O.preset(pre), A.values))
        anorm = np.bincount(r, aq, minlength=n).max()
        err = np.abs(y1.astype(np.float64) - ref).max() / (anorm * np.abs(x.astype(np.float64)).max())
        bound = 2 * lmax * 2.0 ** -24 + (2.0 ** -11 if dt == np.float16 else 0.0)
        assert err <= bound, f"err {err} > {bound}"
    except AssertionError as e:
        fails += 1
        print(f"case {it}: n={n} sigma={sigma} {pre} {np.dtype(dt).name}: {e}", flush=True)
print(f"{n_cases} cases ({segs} segmented), {fails} failures")
sys.exit(1 if fails else 0)
