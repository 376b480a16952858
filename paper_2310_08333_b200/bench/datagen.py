"""Seeded problem generators of the reference benchmark suite
(``bench/datagen.py:26-193``), restated: the same NumPy PCG64 draws in the
same order, so a seed gives the reference's exact arrays."""

from __future__ import annotations

import numpy as np

from ..errors import DataError


def _unit_columns(X: np.ndarray) -> np.ndarray:
    X = X - X.mean(axis=0)
    return X / np.linalg.norm(X, axis=0)


def gen_regression_data(N: int, n: int, seed: int, nonzero_frac: float = 0.1, noise: float = 0.1):
    """Centred unit-norm columns, sparse truth, b = A x + noise (datagen.py:26-43)."""
    rng = np.random.default_rng(seed)
    A = _unit_columns(rng.standard_normal((N, n)))
    x = np.zeros(n)
    sup = rng.choice(n, size=max(1, round(nonzero_frac * n)), replace=False)
    x[sup] = rng.standard_normal(sup.size)
    return A, A @ x + noise * rng.standard_normal(N)


def gen_huber_data(n: int, seed: int):
    """N = n/2 samples, 10% support, 5% of responses shifted by +-10;
    lambda1 = 0.1 ||A'b||_inf (datagen.py:46-79)."""
    if n % 2 or n < 4:
        raise DataError("gen_huber_data requires even n >= 4")
    rng = np.random.default_rng(seed)
    N = n // 2
    A = _unit_columns(rng.standard_normal((N, n)))
    x = np.zeros(n)
    sup = rng.choice(n, size=round(n / 10), replace=False)
    x[sup] = rng.standard_normal(sup.size)
    b = A @ x + 0.1 * rng.standard_normal(N)
    k = round(N / 20)
    if k > 0:
        rows = rng.choice(N, size=k, replace=False)
        b[rows] += rng.choice([-10.0, 10.0], size=k)
    return A, b, 0.1 * float(np.max(np.abs(A.T @ b)))


def gen_portfolio_data(k: int, seed: int):
    """n = 100 k assets, d ~ U[0, sqrt(k)], half-dense N(0,1) factors, mu ~ N(0,1),
    gamma = 1 (datagen.py:82-101)."""
    if k < 1:
        raise DataError("gen_portfolio_data requires k >= 1")
    rng = np.random.default_rng(seed)
    n = 100 * k
    d = rng.uniform(0.0, np.sqrt(k), size=n)
    F = rng.standard_normal((n, k))
    F[rng.random((n, k)) < 0.5] = 0.0
    return d, F, rng.standard_normal(n), 1.0


def gen_bounded_ls(N: int, seed: int):
    """min 1/2 ||Ax - b||^2 over [0, 1]^(N/2) as a dense QP (datagen.py:104-122)."""
    from ..operators import DenseOperator, IdentityOperator
    from ..problems import QPProblem
    from ..prox import Box

    if N % 2 or N < 4:
        raise DataError("gen_bounded_ls requires even N >= 4")
    rng = np.random.default_rng(seed)
    n = N // 2
    A = rng.standard_normal((N, n))
    xr = rng.uniform(-0.2, 1.2, size=n)
    b = A @ xr + 0.1 * rng.standard_normal(N)
    return QPProblem(DenseOperator(A.T @ A), -A.T @ b, IdentityOperator(n), Box(np.zeros(n), np.ones(n)))


def gen_logistic_data(N: int, n: int, seed: int):
    """Margin matrix -label_i * features_i, lambda1 = 0.05 ||A'1||_inf (datagen.py:125-141)."""
    rng = np.random.default_rng(seed)
    feats = _unit_columns(rng.standard_normal((N, n)))
    x = np.zeros(n)
    sup = rng.choice(n, size=max(1, round(0.1 * n)), replace=False)
    x[sup] = rng.standard_normal(sup.size)
    labels = np.where(rng.random(N) < 1.0 / (1.0 + np.exp(-(feats @ x))), 1.0, -1.0)
    A = -labels[:, None] * feats
    return A, 0.05 * float(np.max(np.abs(A.T @ np.ones(N))))


def portfolio_equivalent_qp(d, F, mu, gamma: float):
    """Lifted QP over (x, y = F'x): diagonal P and a sparse constraint map
    [F' -I; 1' 0; I 0] (datagen.py:148-177)."""
    import scipy.sparse as sp

    from ..operators import DiagonalOperator, SparseOperator
    from ..problems import QPProblem
    from ..prox import Box

    d, F, mu = (np.asarray(a, dtype=float) for a in (d, F, mu))
    n, k = F.shape
    M = sp.bmat([[sp.csr_matrix(F.T), -sp.eye(k)], [sp.csr_matrix(np.ones((1, n))), None], [sp.eye(n), None]])
    lo = np.concatenate([np.zeros(k), [1.0], np.zeros(n)])
    hi = np.concatenate([np.zeros(k), [1.0], np.full(n, np.inf)])
    P = DiagonalOperator(np.concatenate([gamma * d, gamma * np.ones(k)]))
    return QPProblem(P, np.concatenate([-mu, np.zeros(k)]), SparseOperator(M.tocsr()), Box(lo, hi))


def portfolio_operator_qp(d, F, mu, gamma: float):
    """Diagonal-plus-low-rank P with the stacked budget / long-only map
    [1'; I] (datagen.py:180-193)."""
    from ..operators import DiagPlusLowRank, IdentityOperator, OnesRowOperator, stack_vertical
    from ..problems import QPProblem
    from ..prox import Box

    d, F, mu = (np.asarray(a, dtype=float) for a in (d, F, mu))
    n = d.size
    M = stack_vertical([OnesRowOperator(n), IdentityOperator(n)])
    lo = np.concatenate([[1.0], np.zeros(n)])
    hi = np.concatenate([[1.0], np.full(n, np.inf)])
    return QPProblem(DiagPlusLowRank(gamma * d, np.sqrt(gamma) * F), -mu, M, Box(lo, hi))


def portfolio_generic_problem(d, F, mu, gamma: float, prox_tol: float = 1e-8):
    """The splitting form with the simplex handled by direct projection
    (datagen.py:184-214): f(x) = (gamma/2) x'(D + F F')x - mu'x with a
    diagonal-plus-low-rank Hessian, g the simplex indicator with an inexact
    (bisection) projection as its prox."""
    import torch

    from ..operators import ConstantHessian, DiagPlusLowRank, IdentityOperator, device_fn, like_input, to_device
    from ..problems import GenericProblem
    from ..prox import simplex_indicator, simplex_project

    d, F, mu = (np.asarray(a, dtype=float) for a in (d, F, mu))
    n = d.size
    P = DiagPlusLowRank(gamma * d, np.sqrt(gamma) * F)

    @device_fn
    def f(x):
        xt = to_device(x)
        return 0.5 * float(torch.dot(xt, P._apply_dev(xt))) - float(torch.dot(to_device(mu), xt))

    @device_fn
    def grad(x):
        xt = to_device(x)
        return like_input(P._apply_dev(xt) - to_device(mu), x)

    return GenericProblem(n=n, m=n, f=f, grad_f=grad, hess=ConstantHessian(P), g=device_fn(lambda z: simplex_indicator(z)),
                          prox_g=device_fn(lambda v, rho, tol: simplex_project(v, min(tol, prox_tol))),
                          M=IdentityOperator(n), c=np.zeros(n), is_quadratic=True, full_rank=True, prox_inexact=True)
