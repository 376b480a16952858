"""Seeded synthetic inputs for the five BASELINE.json configs.

The recipe follows the reference generator conventions
(``/root/reference/pkg/src/nysopt/bench/datagen.py:28-137``): one
``np.random.default_rng(seed)`` stream consumed in the order A, support,
support values, noise/labels.  Config 5 is generated in 8 fixed row blocks of
12500 rows (``default_rng([4, j])``) so 1/2/4/8-GPU shards are unions of whole
blocks.  No public dataset is involved: BASELINE.json names none; these
seeded inputs stand in for the paper's YearMSD/real-sim data.

Everything here is host NumPy: it builds inputs, it is not on the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

# (rows N, features n, sketch rank r, seed) per config, BASELINE.json "configs"
CONFIGS = {
    1: dict(kind="lasso", N=1000, n=2000, rank=50, seed=0, nnz_frac=0.10),
    2: dict(kind="logistic", N=5000, n=10000, rank=100, seed=1, nnz_frac=0.05),
    3: dict(kind="boxqp", N=20000, n=10000, rank=100, seed=2),
    4: dict(kind="lasso", N=20000, n=100000, rank=200, seed=3, nnz_frac=0.01),
    5: dict(kind="lasso", N=100000, n=200000, rank=300, seed=4, nnz_frac=0.005),
}

CFG5_BLOCKS = 8


@dataclass
class ConfigData:
    """Inputs of one config.  ML configs fill A/b/lambda1/lambda2/loss; the box
    QP fills P/q/lo/hi (and keeps A/b for reference)."""

    cfg: int
    kind: str
    loss: Optional[str]
    A: Optional[np.ndarray]
    b: Optional[np.ndarray]
    lambda1: float = 0.0
    lambda2: float = 0.0
    P: Optional[np.ndarray] = None
    q: Optional[np.ndarray] = None
    lo: Optional[np.ndarray] = None
    hi: Optional[np.ndarray] = None
    rank: int = 50
    seed: int = 0


def _lasso(N, n, seed, nnz_frac, scale_rows=None):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((N, n)) * (1.0 / np.sqrt(N if scale_rows is None else scale_rows))
    k = max(1, int(round(nnz_frac * n)))
    support = rng.choice(n, size=k, replace=False)
    x_true = np.zeros(n)
    x_true[support] = rng.standard_normal(k)
    b = A @ x_true + 0.01 * rng.standard_normal(N)
    return A, b


def lasso_data(N, n, seed, nnz_frac):
    """Configs 1 and 4: A_ij ~ N(0, 1/N), x_true with nnz_frac nonzeros N(0,1),
    b = A x_true + 0.01 N(0,1), lambda = 0.1 ||A'b||_inf."""
    A, b = _lasso(N, n, seed, nnz_frac)
    lam = 0.1 * float(np.max(np.abs(A.T @ b)))
    return A, b, lam


def logistic_data(N, n, seed, nnz_frac=0.05):
    """Config 2: rows N(0, I/n), columns centred and scaled to unit l2 norm
    (reference convention, datagen.py:127-129), w_true 5% nonzeros N(0, 4),
    labels y ~ Bernoulli(sigmoid(F w)), margin matrix A = -diag(y) F, b = 0
    (datagen.py:133-135), lambda1 = 0.05 ||A'1||_inf / 2 as BASELINE.json writes it."""
    rng = np.random.default_rng(seed)
    F = rng.standard_normal((N, n)) * (1.0 / np.sqrt(n))
    F -= F.mean(axis=0)
    F /= np.linalg.norm(F, axis=0)
    k = max(1, int(round(nnz_frac * n)))
    support = rng.choice(n, size=k, replace=False)
    w_true = np.zeros(n)
    w_true[support] = 2.0 * rng.standard_normal(k)
    margin = F @ w_true
    y = np.where(rng.random(N) < 1.0 / (1.0 + np.exp(-margin)), 1.0, -1.0)
    A = -y[:, None] * F
    lam1 = 0.05 * float(np.max(np.abs(A.T @ np.ones(N)))) / 2.0
    return A, np.zeros(N), lam1


def boxqp_data(N, n, seed):
    """Config 3: A_ij ~ N(0, 1/N), x0 ~ U[-0.5, 1.5] clipped to [0, 1],
    b = A x0 + 0.01 N(0,1); P = A'A, q = -A'b, box [0, 1]^n (datagen.py:99-116)."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((N, n)) * (1.0 / np.sqrt(N))
    x0 = np.clip(rng.uniform(-0.5, 1.5, size=n), 0.0, 1.0)
    b = A @ x0 + 0.01 * rng.standard_normal(N)
    P = A.T @ A
    q = -(A.T @ b)
    return A, b, P, q


def cfg5_block(j, rows_per_block=12500, n=200000):
    """Config 5 row block j (of 8): A block then its noise from default_rng([4, j])."""
    g = np.random.default_rng([4, j])
    Ab = g.standard_normal((rows_per_block, n))
    Ab *= 1.0 / np.sqrt(100000)  # in place: same values as the product, half the peak memory
    noise = 0.01 * g.standard_normal(rows_per_block)
    return Ab, noise


def cfg5_truth(n=200000, nnz_frac=0.005):
    g = np.random.default_rng([4, 1000])
    k = int(round(nnz_frac * n))
    support = g.choice(n, size=k, replace=False)
    x = np.zeros(n)
    x[support] = g.standard_normal(k)
    return x


def make_config(cfg: int, scale: float = 1.0) -> ConfigData:
    """Build config ``cfg``.  ``scale`` < 1 shrinks N and n proportionally
    (test-sized variants of the same recipe); the published configs use 1."""
    c = CONFIGS[cfg]
    N = max(8, int(round(c["N"] * scale)))
    n = max(8, int(round(c["n"] * scale)))
    rank = max(1, min(int(round(c["rank"] * max(scale, 0.05))), n))
    if c["kind"] == "lasso":
        if cfg == 5 and scale == 1.0:
            raise ValueError("config 5 is generated per shard: use cfg5_block()")
        A, b, lam = lasso_data(N, n, c["seed"], c["nnz_frac"])
        return ConfigData(cfg, "lasso", "square", A, b, lam, 0.0, rank=rank, seed=c["seed"])
    if c["kind"] == "logistic":
        A, b, lam1 = logistic_data(N, n, c["seed"], c["nnz_frac"])
        return ConfigData(cfg, "logistic", "logistic", A, b, lam1, 1e-3, rank=rank, seed=c["seed"])
    A, b, P, q = boxqp_data(N, n, c["seed"])
    return ConfigData(
        cfg, "boxqp", None, A, b, P=P, q=q, lo=np.zeros(n), hi=np.ones(n), rank=rank, seed=c["seed"]
    )
