"""Size-independent properties of the streaming kernels at BASELINE.json's FULL
sizes -- config 4 (20000 x 100000, 16 GB) and the row block one GPU holds of
config 5 at 8 GPUs (12500 x 200000, 20 GB), matrices drawn on the device:

* the single-pass HVP  y = A^T (d o (A v)) + shift v  against the two streaming
  passes gemv_n -> scale -> gemv_t on the same data (two independent kernels),
  its linearity, its symmetry  u.(H v) = v.(H u)  and  v.(H v) = sum d_i (a_i.v)^2;
* the one-pass ADMM tail (cluster stream) against gemv_n(k=2) + the row-wise
  loss kernel + gemv_t(k=3): T, w, row sums and the three A^T products.

(The solves at these sizes are pinned to the reference itself by
tests/test_gpu_solve.py: solve_cfg4.npz and solve_cfg5_shard.npz.)"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(20000, 100000), (12500, 200000)]


@pytest.fixture(scope="module")
def kx():
    from paper_2310_08333_b200.kernels import get_kernels

    return get_kernels()


def _matrix(kx, rows, n, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    A = kx.empty(rows, n)
    A.normal_(generator=g)
    A.mul_(1.0 / np.sqrt(n))
    return A, g


def _rel(a, b):
    return float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b).clamp_min(1e-300))


@pytest.mark.parametrize("rows,n", SHAPES)
def test_hvp_full_size_properties(kx, rows, n):
    A, g = _matrix(kx, rows, n, rows + n)
    v = kx.empty(n).normal_(generator=g)
    u = kx.empty(n).normal_(generator=g)
    d = kx.empty(rows).uniform_(0.05, 0.25, generator=g)
    shift = 0.37
    assert kx.hvp_plan_name(rows, n) != "hvp"  # the wide-row single-pass plans, not the two-pass fallback
    y, yu, pap = kx.empty(n), kx.empty(n), kx.zeros(1)
    kx.hvp(A, d, v, shift, y, pap)
    kx.hvp(A, d, u, shift, yu)
    # two independent streaming passes on the same data
    t = kx.empty(1, rows)
    kx.gemv(A, v.view(1, -1), t)
    av = t.view(-1).clone()
    t.view(-1).mul_(d)
    ref = kx.empty(1, n)
    kx.gemvT(A, t, ref)
    ref = ref.view(-1) + shift * v
    assert _rel(y, ref) < 1e-12
    # v.(H v) = sum d_i (a_i.v)^2 + shift ||v||^2 (the p.Ap the CG uses comes from the same pass)
    want = float(torch.dot(d, av * av) + shift * torch.dot(v, v))
    assert float(pap) == pytest.approx(want, rel=1e-12)
    assert float(torch.dot(v, y)) == pytest.approx(want, rel=1e-11)
    # symmetry and linearity
    assert float(torch.dot(u, y)) == pytest.approx(float(torch.dot(v, yu)), rel=1e-10)
    yc = kx.empty(n)
    kx.hvp(A, d, 0.75 * v - 1.5 * u, shift, yc)
    assert _rel(yc, 0.75 * y - 1.5 * yu) < 1e-12
    del A
    torch.cuda.empty_cache()


@pytest.mark.parametrize("rows,n", SHAPES)
def test_one_pass_tail_full_size_matches_two_passes(kx, rows, n):
    A, g = _matrix(kx, rows, n, 3 * rows + n)
    x = kx.empty(n).normal_(generator=g)
    z = x * (torch.rand(n, device=x.device, generator=g) < 0.01)  # a sparse prox output
    b = kx.empty(rows).normal_(generator=g)
    gb = kx.empty(1, n)
    kx.gemvT(A, b.view(1, -1), gb)
    T, w, AT, rs = kx.empty(3, rows), kx.empty(rows), kx.empty(3, n), kx.zeros(8)
    kx.ml_tail("square", A, x, z, b, T, w, AT, rs, gb=gb.view(-1))
    XZ = torch.stack([x, z]).contiguous()
    AXZ, T2, w2, AT2, rs2 = kx.empty(2, rows), kx.empty(3, rows), kx.empty(rows), kx.empty(3, n), kx.zeros(8)
    kx.gemv(A, XZ, AXZ)
    kx.ml_rowwise("square", AXZ[0], AXZ[1], b, T2[0], w2, T2[1], T2[2], rs2)
    kx.gemvT(A, T2, AT2)
    for j in range(3):
        assert _rel(T[j], T2[j]) < 1e-12
        assert _rel(AT[j], AT2[j]) < 1e-11
    assert torch.equal(w, w2)
    np.testing.assert_allclose(rs.cpu().numpy()[:5], rs2.cpu().numpy()[:5], rtol=1e-11, atol=1e-9)
    del A
    torch.cuda.empty_cache()


def test_one_pass_logistic_tail_full_size_matches_two_passes(kx):
    """The logistic epilogue of the cluster stream (config 2's loss at config 4's size)."""
    rows, n = 20000, 100000
    A, g = _matrix(kx, rows, n, 11)
    x = kx.empty(n).normal_(generator=g)
    z = x * (torch.rand(n, device=x.device, generator=g) < 0.3)
    b = kx.zeros(rows)
    T, w, AT, rs = kx.empty(3, rows), kx.empty(rows), kx.empty(3, n), kx.zeros(8)
    kx.ml_tail("logistic", A, x, z, b, T, w, AT, rs)
    XZ = torch.stack([x, z]).contiguous()
    AXZ, T2, w2, AT2, rs2 = kx.empty(2, rows), kx.empty(3, rows), kx.empty(rows), kx.empty(3, n), kx.zeros(8)
    kx.gemv(A, XZ, AXZ)
    kx.ml_rowwise("logistic", AXZ[0], AXZ[1], b, T2[0], w2, T2[1], T2[2], rs2)
    kx.gemvT(A, T2, AT2)
    for j in range(3):
        assert _rel(T[j], T2[j]) < 1e-12
        assert _rel(AT[j], AT2[j]) < 1e-11
    assert _rel(w, w2) < 1e-12
    np.testing.assert_allclose(rs.cpu().numpy()[:5], rs2.cpu().numpy()[:5], rtol=1e-11, atol=1e-9)
