"""Full-size (BASELINE configs) GPU checks through size-independent properties.

* storage accounting (n_stored, dummies, padding, k_left) equals the survey's
  probe of the reference builder's rules,
* decode(build(A)) == quantise(A) bit for bit (K5 after K1, on the device),
* the production SpMV equals the CSR SpMV of the decoded matrix within the
  FMA-order bound 2 * L_max * 2^-24 (f32 x), and is linear in x.
"""

import numpy as np
import pytest
import torch

import paper_2604_13433_b200 as P
from paper_2604_13433_b200.packed import _to_csr_device, lower_bandwidth

pytestmark = pytest.mark.gpu

CASES = [  # kind, nx, scale, preset, (n_stored, n_dummy, n_padding), k_left
    ("stencil27", 256, None, "fp16", (484_084_480, 33_455_872, 1_173_512), 65_793),
    ("stencil27", 256, "rowsum", "e8m10", (484_113_152, 33_484_544, 1_173_512), 65_793),
    ("stencil27", 256, "rowsum", "e8m11", (484_115_200, 33_486_592, 1_173_512), 65_793),
    ("stencil27", 256, None, "e8m14", (None, 33_553_408, None), 65_793),
    ("poisson3d", 256, "sym", "e8m14", (150_666_752, 33_618_944, 512), 65_536),
    ("poisson3d", 256, "sym", "fp16", (150_634_240, 33_455_872, 131_072), 65_536),
    ("poisson2d", 512, None, "fp16", (1_309_696, 0, 1_024), 512),
]


@pytest.mark.parametrize("kind,nx,scale,preset,want,k_left", CASES)
def test_fullsize_storage_accounting(kind, nx, scale, preset, want, k_left):
    A = P.stencil_device(kind, nx, scale=scale)
    assert lower_bandwidth(A) == k_left
    M = P.build_packsell(A, 32, 256, P.parse_format(preset), "implicit")
    n_stored, n_dummy, n_pad = want
    assert M.k_left == k_left and M.counts.nnz_real == A.nnz
    assert M.counts.n_dummy == n_dummy
    if n_stored is not None:
        assert M.n_stored == n_stored and M.counts.n_padding == n_pad
    assert M.n_stored == M.counts.nnz_real + M.counts.n_dummy + M.counts.n_padding


@pytest.mark.parametrize("kind,scale,preset", [("stencil27", None, "fp16"), ("stencil27", "rowsum", "e8m10"),
                                               ("poisson3d", "sym", "e8m14")])
def test_fullsize_decode_roundtrip_and_spmv(kind, scale, preset):
    fmt = P.parse_format(preset)
    A = P.stencil_device(kind, 256, scale=scale)
    M = P.build_packsell(A, 32, 256, fmt, "implicit")
    D = _to_csr_device(M)
    assert torch.equal(D.row_ptr, A.row_ptr) and torch.equal(D.col_idx, A.col_idx)
    # values: the codec's quantisation of A, computed by the same device encoder (bit-exact vs the
    # reference fixtures in test_gpu_parity) on the generator's values
    q = torch.from_numpy(P.quantize(fmt, A.values[:4_000_000].cpu().numpy())).cuda()
    assert torch.equal(D.values[:4_000_000], q)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    x1 = torch.rand(M.n_cols, generator=g, device="cuda") * 2 - 1
    x2 = torch.rand(M.n_cols, generator=g, device="cuda") * 2 - 1
    y1 = P.packsell_spmv(M, x1).double()
    ref = P.csr_spmv(D, x1.double(), np.float64)
    lmax = int(torch.max(M.d_offset[1:] - M.d_offset[:-1]).item()) // 32
    anorm = float(P.inf_norm_matrix(D))
    den = anorm * float(x1.abs().max())
    assert float((y1 - ref).abs().max()) / den <= 2 * lmax * 2.0 ** -24
    y12 = P.packsell_spmv(M, x1 + x2).double()
    y2 = P.packsell_spmv(M, x2).double()
    den2 = anorm * float((x1.abs() + x2.abs()).max())
    assert float((y12 - y1 - y2).abs().max()) / den2 <= 6 * lmax * 2.0 ** -24
