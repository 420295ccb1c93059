"""Randomised parity sweep (robustness, one-off): build byte-identical to the oracle, REF SpMV
bitwise, production (FMA) SpMV within the stated bound, decode bitwise, over many random
matrices / layouts / codecs / x dtypes.  usage: fuzz_parity.py [n_cases] [seed]"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle as O  # noqa: E402
import paper_2604_13433_b200 as P  # noqa: E402
from conftest import random_csr_arrays  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 500
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 11)
presets = ["fp16", "e8m14", "e8m20", "e8m3", "e8m10", "e8m21", "e8m1", "fp32embed", "e8m7"]
fails = 0
for it in range(n_cases):
    n = int(rng.integers(1, 3000))
    m = int(rng.integers(1, 3000))
    dens = float(np.exp(rng.uniform(np.log(0.0005), np.log(0.1))))
    rp, ci, v = random_csr_arrays(rng, n, m, dens, banded=bool(rng.integers(0, 2)))
    A = P.CsrMatrix(n, m, rp, ci, v)
    mode = ["none", "explicit", "implicit"][int(rng.integers(0, 3))]
    c = [1, 2, 4, 8, 16, 32, 32, 32, 64][int(rng.integers(0, 9))]
    sigma = c * int(rng.choice([1, 2, 3, 5, 8, 16]))
    if sigma > 65536:
        sigma = c
    pre = presets[int(rng.integers(0, len(presets)))]
    try:
        M = P.build_packsell(A, c, sigma, P.parse_format(pre), mode)
        OM = O.build(rp, ci, v, m, c, sigma, O.preset(pre), mode)
        assert np.array_equal(M.pack, OM.pack) and np.array_equal(M.offset, OM.offset), "pack/offset"
        assert M.k_left == OM.k_left and tuple(M.counts) == OM.counts, "counts"
        if mode == "implicit":
            assert np.array_equal(M.perm, OM.perm), "perm"
        for dt in (np.float32, np.float16, np.float64):
            x = rng.uniform(-1, 1, m).astype(dt)
            yr = P.packsell_spmv(M, x, ref_order=True)
            assert np.array_equal(yr.view(np.uint8), O.spmv(OM, x).view(np.uint8)), f"ref {np.dtype(dt).name}"
            yf = P.packsell_spmv(M, x).astype(np.float64)
            xw = x.astype(np.float32) if dt == np.float16 else x
            ref = P.packsell_spmv(M, xw, ref_order=True).astype(np.float64)
            if A.nnz:
                aq = np.abs(P.quantize(P.parse_format(pre), v))
                anorm = np.bincount(np.repeat(np.arange(n), np.diff(rp)), aq, minlength=n).max()
                lmax = max(1, int(np.max(np.diff(M.offset) // c)) if M.n_slices else 1)
                if anorm > 0:
                    err = np.abs(yf - ref).max() / (anorm * max(np.abs(x.astype(np.float64)).max(), 1e-300))
                    bound = 2 * lmax * 2.0 ** -24 + (2.0 ** -11 if dt == np.float16 else 0.0)
                    assert err <= bound, f"fma {np.dtype(dt).name} {err} > {bound}"
        D = P.packsell_to_csr(M)
        Or = O.to_csr(OM)
        assert np.array_equal(D.row_ptr, Or[0]) and np.array_equal(D.col_idx, Or[1]) and \
            np.array_equal(D.values, Or[2]), "decode"
    except AssertionError as e:
        fails += 1
        print(f"case {it}: n={n} m={m} nnz={A.nnz} c={c} sigma={sigma} mode={mode} {pre}: FAIL {e}", flush=True)
print(f"{n_cases} cases, {fails} failures")
sys.exit(1 if fails else 0)
