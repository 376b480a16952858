"""Kernels of the general-operator engine on the B200: CSR SpMV / SpMV^T and the
device transpose, structured operators, spectrum probes and adaptive sizing,
each against the reference's outputs (tests/golden/kernels_*.npz) or NumPy.
Integer/index work (the transposed CSR) is checked bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from conftest import load_golden  # noqa: E402
import cases  # noqa: E402


@pytest.fixture(scope="module")
def nys():
    import paper_2310_08333_b200 as m

    return m


def _rand_csr(N, n, density, seed, long_row=False):
    import scipy.sparse as sp

    rng = np.random.default_rng(seed)
    D = np.where(rng.random((N, n)) < density, rng.standard_normal((N, n)), 0.0)
    if N > 3:
        D[1, :] = 0.0  # empty row
    if long_row:
        D[0, :] = rng.standard_normal(n)  # one dense row among sparse ones
    return sp.csr_matrix(D)


@pytest.mark.parametrize("N,n,density,long_row", [
    (1, 1, 1.0, False), (5, 3, 0.5, False), (300, 200, 0.05, False), (1000, 37, 0.3, True),
    (64, 5000, 0.002, True), (2000, 2000, 0.01, False), (4097, 129, 0.9, False), (50, 70000, 0.0005, True),
])
def test_csr_apply_and_adjoint(nys, N, n, density, long_row):
    A = _rand_csr(N, n, density, N * 7 + n, long_row)
    op = nys.SparseOperator(A)
    rng = np.random.default_rng(1)
    v = rng.standard_normal(n)
    t = rng.standard_normal(N)
    y = op.apply(v)
    z = op.apply_adjoint(t)
    ref_y, ref_z = A @ v, A.T @ t
    np.testing.assert_allclose(y, ref_y, rtol=1e-12, atol=1e-12 * max(1.0, np.abs(ref_y).max(initial=0)))
    np.testing.assert_allclose(z, ref_z, rtol=1e-12, atol=1e-12 * max(1.0, np.abs(ref_z).max(initial=0)))


@pytest.mark.parametrize("N,n,density", [(300, 200, 0.05), (1000, 37, 0.3), (17, 9000, 0.01), (5, 3, 0.0)])
def test_csr_transpose_is_exact(nys, N, n, density):
    """The device transpose equals scipy's A.T (canonical CSR) bit for bit:
    row pointer, column indices and values."""
    import torch

    A = _rand_csr(N, n, density, 99 + N)
    op = nys.SparseOperator(A)
    fwd, bwd = op.device_csr()
    T = A.T.tocsr()
    T.sort_indices()
    np.testing.assert_array_equal(bwd.rowptr.cpu().numpy(), T.indptr.astype(np.int64))
    nnz = T.nnz
    np.testing.assert_array_equal(bwd.col.cpu().numpy()[:nnz], T.indices)
    np.testing.assert_array_equal(bwd.val.cpu().numpy()[:nnz], T.data)
    # deterministic: a second build is identical
    op2 = nys.SparseOperator(A)
    _, bwd2 = op2.device_csr()
    assert torch.equal(bwd.col[:nnz], bwd2.col[:nnz]) and torch.equal(bwd.val[:nnz], bwd2.val[:nnz])


def test_csr_columns_and_reference_golden(nys):
    gold = load_golden("kernels_sparse.npz")
    A = cases._sparse_ml("square", 300, 200, 51)["A"]
    op = nys.SparseOperator(A)
    np.testing.assert_allclose(op.apply(gold["v"]), gold["Av"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(op.apply_adjoint(gold["t"]), gold["Atv"], rtol=1e-12, atol=1e-13)
    import torch

    V = torch.from_numpy(np.random.default_rng(3).standard_normal((200, 133))).cuda()
    Y = op.apply_columns_dev(V).cpu().numpy()
    np.testing.assert_allclose(Y, A @ V.cpu().numpy(), rtol=1e-12, atol=1e-12)
    W = torch.from_numpy(np.random.default_rng(4).standard_normal((300, 7))).cuda()
    from paper_2310_08333_b200.operators import adjoint_columns_dev

    Z = adjoint_columns_dev(op, W).cpu().numpy()
    np.testing.assert_allclose(Z, A.T @ W.cpu().numpy(), rtol=1e-12, atol=1e-12)


def test_structured_operators(nys):
    rng = np.random.default_rng(8)
    n, k = 40, 3
    d = rng.uniform(0.1, 2.0, n)
    F = rng.standard_normal((n, k))
    v = rng.standard_normal(n)
    P = nys.DiagPlusLowRank(d, F)
    np.testing.assert_allclose(P.apply(v), d * v + F @ (F.T @ v), rtol=1e-13, atol=1e-13)
    D = nys.DiagonalOperator(d)
    np.testing.assert_allclose(D.apply(v), d * v, rtol=0, atol=0)
    S = nys.stack_vertical([nys.OnesRowOperator(n), nys.IdentityOperator(n), nys.DenseOperator(F.T)])
    assert S.output_dim == 1 + n + k
    np.testing.assert_allclose(S.apply(v), np.concatenate([[v.sum()], v, F.T @ v]), rtol=1e-13, atol=1e-13)
    u = rng.standard_normal(1 + n + k)
    np.testing.assert_allclose(S.apply_adjoint(u), u[0] + u[1:n + 1] + F @ u[n + 1:], rtol=1e-13, atol=1e-13)
    # the known answer of test_operators.py:33-35
    op = nys.DiagPlusLowRank(np.array([1.0, 1.0]), np.array([[1.0], [1.0]]))
    np.testing.assert_allclose(op.to_dense(), [[2.0, 1.0], [1.0, 2.0]])
    # multi-column forms agree with the column-by-column definition
    import torch

    V = torch.from_numpy(rng.standard_normal((n, 9))).cuda()
    Vh = V.cpu().numpy()
    np.testing.assert_allclose(P.apply_columns_dev(V).cpu().numpy(), d[:, None] * Vh + F @ (F.T @ Vh),
                               rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(S.apply_columns_dev(V).cpu().numpy(),
                               np.vstack([Vh.sum(0, keepdims=True), Vh, F.T @ Vh]), rtol=1e-12, atol=1e-12)


def test_spectrum_probes_match_reference(nys):
    gold = load_golden("kernels_spectrum.npz")
    A = gold["A"]
    op = nys.DenseOperator(A)
    hi, lo = nys.estimate_extreme_eigs(op, iters=30, rng_seed=4)
    assert hi == pytest.approx(float(gold["eig_hi"]), rel=1e-10)
    assert lo == pytest.approx(float(gold["eig_lo"]), rel=1e-6)
    hi2, lo2 = nys.estimate_extreme_eigs(nys.DenseOperator(np.eye(10)), iters=10, rng_seed=0)
    assert hi2 == pytest.approx(1.0, rel=1e-12) and lo2 == pytest.approx(1.0, rel=1e-12)
    with pytest.raises(nys.DataError):
        nys.estimate_extreme_eigs(nys.DenseOperator(np.eye(3)), iters=1, rng_seed=0)
    S = nys.nystrom_sketch(op, 6, rng_seed=8)
    err = nys.estimate_error_norm(op, S, 20, rng_seed=9)
    assert err == pytest.approx(float(gold["err6"]), rel=1e-9)
    assert nys.condition_bound(S, err, 0.5) == pytest.approx(float(gold["cond6"]), rel=1e-9)
    for key, tgt in (("10", 10.0), ("30", 30.0), ("100", 100.0), ("1000", 1e3), ("inf", np.inf)):
        Sa = nys.adaptive_sketch(op, r0=2, r_max=32, nu=0.5, kappa_target=tgt, rng_seed=3)
        assert Sa.rank == int(gold[f"adapt_rank_{key}"])
        np.testing.assert_allclose(Sa.lambda_hat, gold[f"adapt_lam_{key}"], rtol=1e-9, atol=1e-10)
    with pytest.raises(nys.DataError):
        nys.adaptive_sketch(op, r0=4, r_max=2, nu=1.0, kappa_target=2.0, rng_seed=0)


def test_error_norm_zero_for_exact_sketch(nys):
    """test_sketch.py:150-154: a rank-r PSD matrix sketched at rank r."""
    rng = np.random.default_rng(11)
    A = cases.random_psd(20, rng, rank=4)
    op = nys.DenseOperator(A)
    S = nys.nystrom_sketch(op, 4, rng_seed=1)
    assert nys.estimate_error_norm(op, S, 10, rng_seed=2) <= 1e-8 * np.linalg.norm(A, 2)


def test_diagonal_reduce(nys):
    """(A + diag(d)) w = b via the unit-shift form (sketch.py:285-306)."""
    rng = np.random.default_rng(12)
    A = cases.random_psd(15, rng)
    d = rng.uniform(0.5, 2.0, 15)
    At, s = nys.diagonal_reduce(nys.DenseOperator(A), d)
    v = rng.standard_normal(15)
    ref = (A / np.sqrt(np.outer(d, d))) @ v
    np.testing.assert_allclose(At.apply(v), ref, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(s, 1.0 / np.sqrt(d), rtol=1e-15)
    with pytest.raises(nys.DataError):
        nys.diagonal_reduce(nys.DenseOperator(A), -d)
