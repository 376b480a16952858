"""Kernel-level parity of the C-ABI kernels against NumPy / the oracle.

Integer-free FP64 work: tolerances are stated per test (relative ~1e-12 for
single products, looser where the reference test uses looser ones)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from conftest import load_golden  # noqa: E402


@pytest.fixture(scope="module")
def kx():
    from paper_2310_08333_b200.kernels import get_kernels

    return get_kernels()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


SHAPES = [(1, 1), (3, 5), (7, 129), (64, 64), (1000, 2000), (37, 1001), (5000, 333), (130, 10000)]


@pytest.mark.parametrize("rows,n", SHAPES)
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_gemv_multi_rhs(kx, rows, n, k):
    g = np.random.default_rng(rows * 7 + n + k)
    A = g.standard_normal((rows, n))
    X = g.standard_normal((k, n))
    Y = kx.empty(k, rows)
    kx.gemv(dev(A), dev(X), Y)
    ref = X @ A.T
    np.testing.assert_allclose(Y.cpu().numpy(), ref, rtol=1e-12, atol=1e-12 * np.abs(A).sum(1).max())


@pytest.mark.parametrize("rows,n", SHAPES)
@pytest.mark.parametrize("k", [1, 3])
def test_gemvT_multi_rhs(kx, rows, n, k):
    g = np.random.default_rng(rows * 3 + n + k)
    A = g.standard_normal((rows, n))
    T = g.standard_normal((k, rows))
    Y = kx.empty(k, n)
    kx.gemvT(dev(A), dev(T), Y)
    ref = T @ A
    np.testing.assert_allclose(Y.cpu().numpy(), ref, rtol=1e-12, atol=1e-12 * np.abs(A).sum(0).max())


def test_gemv_odd_leading_dim(kx):
    g = np.random.default_rng(5)
    big = g.standard_normal((50, 77))
    At = dev(big)[:, :75]  # lda = 77 (odd), misaligned rows
    A = big[:, :75]
    x = g.standard_normal((2, 75))
    Y = kx.empty(2, 50)
    kx.gemv(At, dev(x), Y)
    np.testing.assert_allclose(Y.cpu().numpy(), x @ A.T, rtol=1e-12, atol=1e-12)
    t = g.standard_normal((1, 50))
    Z = kx.empty(1, 75)
    kx.gemvT(At, dev(t), Z)
    np.testing.assert_allclose(Z.cpu().numpy(), t @ A, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("rows,n", [(70, 45), (1000, 2000), (5000, 3000), (33, 7),
                                    # wide rows: column-strip kernel (csrc/hvp_strip.cu)
                                    (7, 20000), (301, 100000), (1001, 30002), (50, 250000), (2, 12802),
                                    # sub-segment cluster plan (L2 re-read for the axpy): config 5's width
                                    (37, 200000), (301, 150000), (3, 199998)])
def test_hvp_fused(kx, rows, n):
    g = np.random.default_rng(n)
    A = g.standard_normal((rows, n))
    d = g.uniform(0.1, 1.0, rows)
    v = g.standard_normal(n)
    y = kx.empty(n)
    pAp = kx.zeros(1)
    kx.hvp(dev(A), dev(d), dev(v), 0.7, y, pAp, True)
    ref = A.T @ (d * (A @ v)) + 0.7 * v
    np.testing.assert_allclose(y.cpu().numpy(), ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())
    assert abs(float(pAp) - v @ ref) <= 1e-11 * abs(v @ ref)
    # the shift without p.Ap (the CG's true-residual refresh, krylov.py:80-81)
    y1 = kx.empty(n)
    kx.hvp(dev(A), dev(d), dev(v), 0.7, y1, None, True)
    np.testing.assert_allclose(y1.cpu().numpy(), ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())
    # partial form (row shard) + finish
    y2 = kx.empty(n)
    kx.hvp(dev(A), None, dev(v), 0.0, y2, None, False)
    kx.shift_dot(dev(v), 0.3, y2, pAp)
    ref2 = A.T @ (A @ v) + 0.3 * v
    np.testing.assert_allclose(y2.cpu().numpy(), ref2, rtol=1e-11, atol=1e-11 * np.abs(ref2).max())


def test_hvp_matches_reference_golden(kx):
    """MLHessian.apply of the reference (problems.py:263-264) at a fixed point."""
    from cases import hvp_case
    from paper_2310_08333_b200 import MLProblem, builtin_loss
    from paper_2310_08333_b200.problems import MLHessian, ml_dual_gap, ml_gradient, ml_objective

    gold = load_golden("kernels_ml.npz")
    A, b, x, v = hvp_case()
    for loss in ("square", "logistic", "huber"):
        for lam2 in (0.0, 0.3):
            key = f"{loss}_{lam2}"
            p = MLProblem(builtin_loss(loss), A, b, 0.7, lam2)
            H = MLHessian(p, x)
            np.testing.assert_allclose(H.apply(v), gold[f"hvp_{key}"], rtol=1e-11, atol=1e-11)
            np.testing.assert_allclose(ml_gradient(p, x), gold[f"grad_{key}"], rtol=1e-11, atol=1e-11)
            assert abs(ml_objective(p, x) - gold[f"obj_{key}"]) <= 1e-12 * abs(gold[f"obj_{key}"])
            gg = float(gold[f"gap_{key}"])
            got = ml_dual_gap(p, x)
            if np.isfinite(gg):
                assert abs(got - gg) <= 1e-9 * max(1.0, abs(gg)), (key, got, gg)
            else:
                assert not np.isfinite(got)


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(5, 3, 7), (130, 70, 257), (1000, 133, 2000), (133, 133, 10000), (64, 64, 16)])
def test_dgemm_dmma(kx, ta, tb, M, N, K):
    g = np.random.default_rng(M + N + K + 10 * ta + tb)
    A = g.standard_normal((K, M) if ta else (M, K))
    B = g.standard_normal((N, K) if tb else (K, N))
    C0 = g.standard_normal((M, N))
    Cd = dev(C0)
    kx.gemm(ta, tb, M, N, K, 1.5, dev(A), A.shape[1], dev(B), B.shape[1], 0.5, Cd, N)
    ref = 1.5 * (A.T if ta else A) @ (B.T if tb else B) + 0.5 * C0
    np.testing.assert_allclose(Cd.cpu().numpy(), ref, rtol=1e-11, atol=1e-12 * np.sqrt(K) * 10)


@pytest.mark.parametrize("s", [1, 2, 5, 33, 133, 258])
def test_syevj(kx, s):
    g = np.random.default_rng(s)
    Q, _ = np.linalg.qr(g.standard_normal((s, s)))
    lam = np.concatenate([g.uniform(0.1, 10.0, s - s // 4), -g.uniform(0.1, 1.0, s // 4)])
    M = (Q * lam) @ Q.T
    M = 0.5 * (M + M.T)
    V = kx.empty(s, s)
    w = kx.empty(s)
    kx.syevj(dev(M), V, w)
    wn = w.cpu().numpy()
    Vn = V.cpu().numpy()
    np.testing.assert_allclose(wn, np.sort(lam)[::-1], rtol=1e-11, atol=1e-12 * 10)
    np.testing.assert_allclose(Vn.T @ Vn, np.eye(s), atol=1e-12 * s)
    np.testing.assert_allclose(M @ Vn, Vn * wn, atol=1e-11 * 10)


@pytest.mark.parametrize("kind", ["identity", "repeated", "diagonal", "rank1", "graded"])
@pytest.mark.parametrize("s", [3, 40, 133])
def test_syevj_degenerate_spectra(kx, kind, s):
    g = np.random.default_rng(7 * s)
    Q, _ = np.linalg.qr(g.standard_normal((s, s)))
    if kind == "identity":
        M = 2.5 * np.eye(s)
    elif kind == "repeated":
        lam = np.repeat([3.0, 1.0, 0.5], (s + 2) // 3)[:s]
        M = (Q * lam) @ Q.T
    elif kind == "diagonal":
        M = np.diag(np.linspace(5.0, 1.0, s))
    elif kind == "rank1":
        q = g.standard_normal(s)
        M = np.outer(q, q)
    else:
        M = (Q * np.logspace(0, -12, s)) @ Q.T
    M = 0.5 * (M + M.T)
    V = kx.empty(s, s)
    w = kx.empty(s)
    kx.syevj(dev(M), V, w)
    wn, Vn = w.cpu().numpy(), V.cpu().numpy()
    ref = np.sort(np.linalg.eigvalsh(M))[::-1]
    scale = np.abs(ref).max()
    np.testing.assert_allclose(wn, ref, atol=1e-12 * scale * s)
    np.testing.assert_allclose(Vn.T @ Vn, np.eye(s), atol=1e-10)
    np.testing.assert_allclose(M @ Vn, Vn * wn, atol=1e-11 * scale * s)


@pytest.mark.parametrize("shape", [0, 1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(5000, 133, 3000), (133, 133, 10000), (77, 45, 33), (300, 258, 1001)])
def test_dgemm_every_tile_shape(kx, shape, ta, tb, M, N, K):
    """Each CTA tile shape of the planner (nys_gemm_tile forces it), with
    split-K where the planner picks it, against NumPy FP64."""
    g = np.random.default_rng(M * 7 + N + K + shape)
    A = g.standard_normal((K, M) if ta else (M, K))
    B = g.standard_normal((N, K) if tb else (K, N))
    Cd = kx.empty(M, N)
    assert kx.L.nys_gemm_tile(shape) == 7
    try:
        kx.gemm(ta, tb, M, N, K, 1.0, dev(A), A.shape[1], dev(B), B.shape[1], 0.0, Cd, N)
    finally:
        kx.L.nys_gemm_tile(-1)
    ref = (A.T if ta else A) @ (B.T if tb else B)
    np.testing.assert_allclose(Cd.cpu().numpy(), ref, rtol=1e-11, atol=1e-12 * np.sqrt(K) * 10)


@pytest.mark.parametrize("s", [1, 7, 8, 9, 64, 133, 152, 153, 200])
def test_orthonormalize_cholinv_sizes(kx, s):
    """The fused Cholesky-inverse kernel (s <= 152) and the split path (s > 152)."""
    g = np.random.default_rng(s)
    n = max(4 * s, 50)
    Om = g.standard_normal((n, s))
    Q = kx.empty(n, s)
    kx.orthonormalize(dev(Om), Q)
    Qn = Q.cpu().numpy()
    np.testing.assert_allclose(Qn.T @ Qn, np.eye(s), atol=1e-13 * max(1, s // 16))
    np.testing.assert_allclose(Qn @ (Qn.T @ Om), Om, atol=1e-11)


def test_orthonormalize_singular_gram_falls_back(kx):
    """A rank-deficient Omega makes the Cholesky fail: the deferred check must
    catch it and the careful path must still return finite output."""
    g = np.random.default_rng(3)
    Om = g.standard_normal((500, 20))
    Om[:, 7] = Om[:, 3]  # exactly dependent columns
    Q = kx.empty(500, 20)
    kx.orthonormalize(dev(Om), Q)
    assert np.isfinite(Q.cpu().numpy()).all()


def test_orthonormalize_spans_omega(kx):
    g = np.random.default_rng(1)
    Om = g.standard_normal((2000, 70))
    Q = kx.empty(2000, 70)
    kx.orthonormalize(dev(Om), Q)
    Qn = Q.cpu().numpy()
    np.testing.assert_allclose(Qn.T @ Qn, np.eye(70), atol=1e-13)
    Qh, _ = np.linalg.qr(Om)
    # same range: projector equality
    np.testing.assert_allclose(Qn @ (Qn.T @ Om), Om, atol=1e-11)
    np.testing.assert_allclose(np.abs(Qh.T @ Qn).sum(0).min() >= 0.0, True)


def test_sketch_matches_reference_golden():
    """nystrom_sketch on the reference's fixture: eigenvalues to 1e-10 and the
    preconditioner apply (Eq. 11) to 1e-10 (test_sketch.py:113-120 tolerance)."""
    from cases import sketch_case
    from paper_2310_08333_b200 import DenseOperator, NystromPreconditioner, nystrom_sketch

    gold = load_golden("kernels_sketch.npz")
    M, r, seed = sketch_case()
    S = nystrom_sketch(DenseOperator(M), r, rng_seed=seed)
    np.testing.assert_allclose(S.lambda_hat, gold["lam"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(np.abs(S.U.T @ gold["U"]), np.eye(r), atol=1e-8)
    pc = NystromPreconditioner(S, nu=0.5)
    PV = np.column_stack([pc.apply(gold["V"][:, j]) for j in range(gold["V"].shape[1])])
    np.testing.assert_allclose(PV, gold["PV"], rtol=1e-10, atol=1e-10)


def test_pcg_matches_reference_golden():
    from cases import pcg_case
    from paper_2310_08333_b200 import DenseOperator, NystromPreconditioner, nystrom_sketch, pcg

    gold = load_golden("kernels_pcg.npz")
    H, b, x0 = pcg_case()
    S2 = nystrom_sketch(DenseOperator(H - 0.7 * np.eye(H.shape[0])), 6, rng_seed=4)
    pc2 = NystromPreconditioner(S2, nu=0.7)
    x1, rep1 = pcg(DenseOperator(H), b, x0=x0, tol_rel=1e-10)
    x2, rep2 = pcg(DenseOperator(H), b, x0=x0, Minv=pc2.apply, tol_rel=1e-10)
    assert rep1.iterations == int(gold["it_plain"])
    assert abs(rep2.iterations - int(gold["it_prec"])) <= 1
    np.testing.assert_allclose(x1, gold["x_plain"], rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(x2, gold["x_prec"], rtol=1e-8, atol=1e-10)


def test_precond_kat():
    """precond diag(2,1), nu = 1 applied to (1,1) -> (2/3, 1) (test_sketch.py:100-104)."""
    from paper_2310_08333_b200 import DenseOperator, NystromPreconditioner, nystrom_sketch, precond_apply

    S = nystrom_sketch(DenseOperator(np.diag([2.0, 1.0])), 2, rng_seed=0)
    P = NystromPreconditioner(S, nu=1.0)
    np.testing.assert_allclose(precond_apply(P, np.array([1.0, 1.0])), [2.0 / 3.0, 1.0], atol=1e-7)


def test_non_psd_sketch_rejected():
    from paper_2310_08333_b200 import DataError, DenseOperator, nystrom_sketch

    with pytest.raises(DataError):
        nystrom_sketch(DenseOperator(np.diag([1.0, -1.0, 0.5])), 3, rng_seed=0)


def test_exact_rank_recovery():
    from paper_2310_08333_b200 import DenseOperator, nystrom_sketch

    A = np.diag([3.0, 2.0, 0.0, 0.0])
    S = nystrom_sketch(DenseOperator(A), 2, rng_seed=0)
    assert np.allclose(sorted(S.lambda_hat, reverse=True), [3.0, 2.0], atol=1e-7)
    assert np.allclose(S.to_dense(), A, atol=1e-7)


def test_pcg_kats():
    from paper_2310_08333_b200 import DenseOperator, NotSPDError, pcg

    x, rep = pcg(DenseOperator(np.eye(3)), np.array([1.0, 2.0, 3.0]), tol_rel=1e-12)
    assert rep.iterations == 1 and rep.converged
    np.testing.assert_allclose(x, [1, 2, 3], atol=1e-12)
    x, rep = pcg(DenseOperator(np.diag([1.0, 100.0])), np.ones(2), tol_rel=1e-10)
    assert rep.iterations <= 2
    np.testing.assert_allclose(x, [1.0, 0.01], atol=1e-9)
    x, rep = pcg(DenseOperator(np.eye(4)), np.zeros(4))
    assert np.array_equal(x, np.zeros(4)) and rep.iterations == 0
    with pytest.raises(NotSPDError):
        pcg(DenseOperator(np.diag([1.0, -1.0])), np.ones(2), tol_rel=1e-12)


@pytest.mark.parametrize("seed,count", [(0, 1), (1, 70 * 2000), (7, 133 * 10000), (123456789, 5_000_003)])
def test_gaussian_matches_numpy_stream(kx, seed, count):
    """Omega drawn on the GPU equals np.random.default_rng(seed).standard_normal
    (sketch.py:97-98).  Bitwise except where CUDA's exp/log1p may differ from
    glibc by one ulp on the rare ziggurat rejection paths."""
    out = kx.empty(count)
    kx.gaussian(seed, out)
    got = out.cpu().numpy()
    ref = np.random.default_rng(seed).standard_normal(count)
    diff = got != ref
    assert diff.sum() <= max(1, count // 100000), diff.sum()
    np.testing.assert_allclose(got, ref, rtol=1e-15, atol=0)


@pytest.mark.parametrize("rank", [5, 40])
def test_sketch_low_rank_operator(rank):
    """A rank-deficient PSD operator: the core Cholesky may hit a tiny pivot
    (the pipelined sketch then re-runs the synchronous path with the eigh
    fallback of sketch.py:114-124); either way the Nystrom approximation of
    an exactly low-rank operator is exact and the extra eigenvalues vanish."""
    from paper_2310_08333_b200 import DenseOperator, nystrom_sketch

    g = np.random.default_rng(rank)
    B = g.standard_normal((200, rank))
    M = B @ B.T
    S = nystrom_sketch(DenseOperator(M), 20, rng_seed=rank)
    A_hat = (S.U * S.lambda_hat) @ S.U.T
    scale = np.linalg.norm(M, 2)
    assert np.isfinite(S.lambda_hat).all() and np.isfinite(S.U).all()
    if rank < 20:
        top = np.sort(np.linalg.eigvalsh(M))[::-1][:rank]
        np.testing.assert_allclose(S.lambda_hat[:rank], top, rtol=1e-8, atol=1e-10 * scale)
        np.testing.assert_allclose(A_hat, M, atol=1e-8 * scale)
        assert np.all(S.lambda_hat[rank:] <= 1e-9 * scale)
    else:
        # A_hat <= M in the Loewner order (test_sketch.py:57-67)
        assert np.linalg.eigvalsh(M - A_hat).min() >= -1e-8 * scale


@pytest.mark.parametrize("piece", [1000, 7919, 1 << 26])
def test_cfg5_block_generated_in_hbm_matches_host(kx, piece):
    """Config 5's row blocks generated on the GPU (devgen.py) equal the host
    recipe datagen.cfg5_block, including the noise drawn after the block; the
    pieces of one long stream chain exactly (draws consumed per piece)."""
    from paper_2310_08333_b200 import datagen, devgen

    rows, n = 6, 5000
    out = kx.empty(rows, n)
    noise = devgen.cfg5_block_into(kx, 3, out, rows, n, piece)
    A_ref, noise_ref = datagen.cfg5_block(3, rows, n)
    got = out.cpu().numpy()
    assert (got != A_ref).sum() <= 1
    np.testing.assert_allclose(got, A_ref, rtol=1e-15, atol=0)
    np.testing.assert_allclose(noise.cpu().numpy(), noise_ref, rtol=1e-15, atol=0)
    # the stacked generator with b = A x_true + noise (x_true from the host recipe)
    A2, b2, xt = devgen.cfg5_device(kx, [3], rows, n, piece)
    assert torch.equal(A2, out)
    np.testing.assert_allclose(b2.cpu().numpy(), A_ref @ xt.cpu().numpy() + noise_ref, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("host_b", [True, False])
def test_lasso_generated_in_hbm_matches_host(kx, host_b):
    """Configs 1/4's recipe with A generated on the GPU (devgen.lasso_device,
    used by bench.py for the 16 GB config 4): A bit-for-bit the host stream,
    the support / values / noise drawn after it from the continued host
    generator; with host_b, b and lambda bit-for-bit datagen.lasso_data."""
    from paper_2310_08333_b200 import datagen, devgen

    N, n, seed, frac = 300, 700, 3, 0.01
    A_ref, b_ref, lam_ref = datagen.lasso_data(N, n, seed, frac)
    A, b, lam, xt, A_host = devgen.lasso_device(kx, N, n, seed, frac, host_b=host_b)
    got = A.cpu().numpy()
    # the device ziggurat's tail (exp/log) may round one draw in 10^5 by an ulp
    assert (got != A_ref).sum() <= max(1, got.size // 100000)
    np.testing.assert_allclose(got, A_ref, rtol=1e-15, atol=0)
    if host_b:
        assert np.array_equal(A_host.numpy(), got)
        np.testing.assert_allclose(b, b_ref, rtol=1e-13, atol=1e-15)
        assert abs(lam - lam_ref) <= 1e-13 * lam_ref
    else:
        np.testing.assert_allclose(b, b_ref, rtol=1e-13, atol=1e-15)
        assert abs(lam - lam_ref) <= 1e-13 * lam_ref
    # a rank's rows of a sharded run: the same numbers
    A2, b2, lam2, _, _ = devgen.lasso_device(kx, N, n, seed, frac, rows=(100, 200), host_b=host_b)
    assert np.array_equal(A2.cpu().numpy(), got[100:200]) and np.array_equal(b2, b) and lam2 == lam


@pytest.mark.parametrize("rows,n,with_z,loss", [
    (300, 20000, True, "square"), (37, 100000, True, "square"), (301, 20002, False, "square"),
    (5, 14000, True, "square"),
    # every cluster size: C = 2 (config 2's width; the narrowest slices the plan
    # takes), 4, 8 and 16, with the logistic epilogue
    (400, 10000, True, "logistic"), (149, 7000, True, "logistic"), (64, 28000, True, "logistic"),
    (40, 50000, False, "logistic"), (23, 100000, True, "logistic")])
def test_ml_tail_one_pass(kx, rows, n, with_z, loss):
    """The one-pass ADMM tail (cluster stream over A): A{x,z}, the loss epilogue
    and A^T{l', w o Ax, nu} against NumPy, with the row sums of
    nys_ml_rowwise_f64 (problems.py:35-111 expressions)."""
    g = np.random.default_rng(rows + n)
    A = g.standard_normal((rows, n)) / np.sqrt(n)
    x, z, b = g.standard_normal(n), g.standard_normal(n), g.standard_normal(rows)
    T = kx.empty(3, rows)
    w = kx.empty(rows)
    K = 3 if with_z else 2
    AT = kx.empty(K, n)
    rs = kx.zeros(8)
    kx.ml_tail(loss, dev(A), dev(x), dev(z) if with_z else None, dev(b), T, w, AT, rs)
    ax = A @ x
    r1 = ax - b
    if loss == "square":
        tg, wr = r1, np.ones(rows)
        lval = lambda r: 0.5 * r * r  # noqa: E731
        conj = lambda y: 0.5 * y * y  # noqa: E731
    else:
        expit = lambda t: 1.0 / (1.0 + np.exp(-t))  # noqa: E731
        tg, wr = expit(r1), expit(r1) * expit(-r1)
        lval = lambda r: np.logaddexp(0.0, r)  # noqa: E731
        conj = lambda y: y * np.log(y) + (1.0 - y) * np.log1p(-y)  # noqa: E731
    thx = wr * ax
    Tn = T.cpu().numpy()
    np.testing.assert_allclose(Tn[0], tg, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(Tn[1], thx, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(w.cpu().numpy(), wr, rtol=1e-12, atol=1e-14)
    ref = [A.T @ tg, A.T @ thx]
    s = rs.cpu().numpy()
    assert s[0] == pytest.approx(np.sum(lval(r1)), rel=1e-12)
    if with_z:
        r2 = A @ z - b
        nu = r2 if loss == "square" else 1.0 / (1.0 + np.exp(-r2))
        np.testing.assert_allclose(Tn[2], nu, rtol=1e-12, atol=1e-12)
        ref.append(A.T @ nu)
        assert s[1] == pytest.approx(np.sum(lval(r2)), rel=1e-12)
        assert s[2] == pytest.approx(np.sum(conj(nu)), rel=1e-11)
        assert s[3] == 0.0
        assert s[4] == pytest.approx(b @ nu, rel=1e-11, abs=1e-11)
    ATn = AT.cpu().numpy()
    for j in range(K):
        np.testing.assert_allclose(ATn[j], ref[j], rtol=1e-11, atol=1e-11 * np.abs(ref[j]).max())


@pytest.mark.gpu
@pytest.mark.parametrize("loss", ["square", "logistic"])
@pytest.mark.parametrize("rows,n,dens", [
    (400, 10000, 0.01), (400, 10000, 0.085), (149, 7000, 0.0), (64, 28000, 0.03), (40, 50000, 0.07),
    (23, 100000, 0.005), (23, 100000, 0.0716), (300, 100000, 0.0065)])
def test_ml_tail_sparse_z(kx, rows, n, dens, loss):
    """The one-pass tail with a sparse z (the prox output): a CTA whose slice of z
    holds at most one nonzero per compute thread (448) forms a_i.z as one product
    per thread.  Densities below, around (CTAs of one cluster choosing
    differently) and above that limit, z = 0, both epilogues, with and without
    g_b; against NumPy and against the dense-z arithmetic on the same inputs."""
    g = np.random.default_rng(rows + n + int(1e4 * dens))
    A = g.standard_normal((rows, n)) / np.sqrt(n)
    x, b = g.standard_normal(n), g.standard_normal(rows)
    z = np.where(g.random(n) < dens, g.standard_normal(n), 0.0)
    az = A @ z
    r2 = az - b
    nu = r2 if loss == "square" else 1.0 / (1.0 + np.exp(-r2))
    for use_gb in ([False, True] if loss == "square" else [False]):
        T, w, AT, rs = kx.empty(3, rows), kx.empty(rows), kx.empty(3, n), kx.zeros(8)
        kw = {"gb": dev(A.T @ b)} if use_gb else {}
        kx.ml_tail(loss, dev(A), dev(x), dev(z), dev(b), T, w, AT, rs, **kw)
        Tn = T.cpu().numpy()
        np.testing.assert_allclose(Tn[2], nu, rtol=1e-12, atol=1e-12)
        ref = A.T @ nu
        scale = max(np.abs(ref).max(), np.abs(A.T @ b).max())
        np.testing.assert_allclose(AT.cpu().numpy()[2], ref, rtol=0, atol=1e-11 * scale)
        s = rs.cpu().numpy()
        lval = (lambda r: 0.5 * r * r) if loss == "square" else (lambda r: np.logaddexp(0.0, r))  # noqa: E731
        assert s[1] == pytest.approx(np.sum(lval(r2)), rel=1e-12)
        assert s[4] == pytest.approx(b @ nu, rel=1e-11, abs=1e-11)
        # the x side is untouched by the choice
        np.testing.assert_allclose(Tn[1], (np.ones(rows) if loss == "square" else
                                           (1.0 / (1.0 + np.exp(-(A @ x - b)))) * (1.0 / (1.0 + np.exp(A @ x - b)))) * (A @ x),
                                   rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("rows,n,dens", [
    (23, 200000, 0.005), (40, 150000, 0.01), (30, 120000, 0.0), (17, 229376, 0.02), (23, 200000, 0.2),
    (12, 200000, 1.0), (300, 200000, 0.004), (9, 114690, 0.03)])
def test_ml_tail_square_very_wide_rows(kx, rows, n, dens):
    """The one-pass square-loss tail for rows beyond the whole-slice plan
    (114688 < n <= 229376, config 5's n = 200000): x and the A^T(Az) accumulator
    in tensor memory, z through its compacted nonzeros (tail_q_kernel); sparse,
    empty, denser (several entries per thread) and dense z, every (Q, KQ) the
    plan picks; against NumPy."""
    g = np.random.default_rng(3 * rows + n + int(1e3 * dens))
    A = g.standard_normal((rows, n)) / np.sqrt(n)
    x, b = g.standard_normal(n), g.standard_normal(rows)
    z = np.where(g.random(n) < dens, g.standard_normal(n), 0.0)
    T, w, AT, rs = kx.empty(3, rows), kx.empty(rows), kx.empty(3, n), kx.zeros(8)
    kx.ml_tail("square", dev(A), dev(x), dev(z), dev(b), T, w, AT, rs, gb=dev(A.T @ b))
    ax, az = A @ x, A @ z
    r1, r2 = ax - b, az - b
    Tn = T.cpu().numpy()
    np.testing.assert_allclose(Tn[0], r1, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(Tn[1], ax, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(Tn[2], r2, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(w.cpu().numpy(), np.ones(rows))
    s = rs.cpu().numpy()
    assert s[0] == pytest.approx(0.5 * r1 @ r1, rel=1e-12)
    assert s[1] == pytest.approx(0.5 * r2 @ r2, rel=1e-12)
    assert s[4] == pytest.approx(b @ r2, rel=1e-11, abs=1e-11)
    ATn = AT.cpu().numpy()
    scale = max(np.abs(A.T @ ax).max(), np.abs(A.T @ b).max(), np.abs(A.T @ az).max())
    for j, ref in enumerate((A.T @ r1, A.T @ ax, A.T @ r2)):
        np.testing.assert_allclose(ATn[j], ref, rtol=0, atol=1e-12 * scale)


@pytest.mark.gpu
@pytest.mark.parametrize("rows,n", [(400, 10000), (149, 7000), (64, 28000), (40, 50000), (23, 100000)])
def test_ml_tail_square_two_products(kx, rows, n):
    """The square-loss one-pass tail given g_b = A^T b (nys_ml_tail_gb_f64):
    two streamed products A^T(Ax), A^T(Az), then A^T(Ax - b) = A^T(Ax) - g_b and
    A^T(Az - b) = A^T(Az) - g_b, against NumPy; every cluster size (2, 4, 8, 16)
    and both halves of the row outputs."""
    g = np.random.default_rng(7 * rows + n)
    A = g.standard_normal((rows, n)) / np.sqrt(n)
    x, z, b = g.standard_normal(n), g.standard_normal(n), g.standard_normal(rows)
    T, w, AT, rs = kx.empty(3, rows), kx.empty(rows), kx.empty(3, n), kx.zeros(8)
    gb = dev(A.T @ b)
    kx.ml_tail("square", dev(A), dev(x), dev(z), dev(b), T, w, AT, rs, gb=gb)
    ax, az = A @ x, A @ z
    r1, r2 = ax - b, az - b
    Tn = T.cpu().numpy()
    np.testing.assert_allclose(Tn[0], r1, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(Tn[1], ax, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(Tn[2], r2, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(w.cpu().numpy(), np.ones(rows))
    s = rs.cpu().numpy()
    assert s[0] == pytest.approx(0.5 * r1 @ r1, rel=1e-12)
    assert s[1] == pytest.approx(0.5 * r2 @ r2, rel=1e-12)
    assert s[4] == pytest.approx(b @ r2, rel=1e-11, abs=1e-11)
    ATn = AT.cpu().numpy()
    for j, ref in enumerate((A.T @ r1, A.T @ ax, A.T @ r2)):
        # the difference of two products: absolute error at the scale of the products
        scale = max(np.abs(A.T @ ax).max(), np.abs(A.T @ b).max(), np.abs(A.T @ az).max())
        np.testing.assert_allclose(ATn[j], ref, rtol=0, atol=1e-12 * scale)
