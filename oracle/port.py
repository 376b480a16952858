"""CPU oracle: a NumPy restatement of the reference inexact-ADMM hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` leg may import this module,
and only as the checker (or the timed CPU baseline), never as the product.
The product path (``paper_2310_08333_b200``) never imports it and fails
loudly when its CUDA library is missing.

Scope: the north-star path of SURVEY.md §8(a) -- dense ML problems (square,
logistic, huber losses; M = I, c = 0) and box-constrained QPs with a dense P
and M = I -- and the §8(f) rows built after it: sparse (scipy CSR) data,
structured P (diagonal-plus-low-rank), a general constraint map M with the
composite sketch target, the Lanczos rank probe and the adaptive sketch.  Every function cites the reference ``file:line`` it restates
(paths relative to ``/root/reference/pkg/src/nysopt``).  The arithmetic is
written in the same operation order as the reference so that, on identical
inputs, the oracle agrees with the reference bit for bit; this is pinned by
``tests/test_oracle_pins.py`` against ``tests/golden/*.npz``, which
``tests/golden/make_golden.py`` produced by running the reference itself.
"""

from __future__ import annotations

import math
import time
from collections import deque
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np
import scipy.linalg
from scipy.special import expit

EPS = float(np.finfo(float).eps)


class OracleError(Exception):
    pass


class OracleDataError(OracleError):
    pass


class OracleNotSPD(OracleError):
    pass


class OracleNumerical(OracleError):
    pass


# --------------------------------------------------------------------------
# losses  (problems.py:53-111)


def loss_value(kind: str, w):
    if kind == "square":  # problems.py:57
        return 0.5 * w**2
    if kind == "logistic":  # problems.py:82
        return np.logaddexp(0.0, w)
    if kind == "huber":  # problems.py:95-97
        w = np.asarray(w, dtype=float)
        return np.where(np.abs(w) <= 1.0, w**2, 2.0 * np.abs(w) - 1.0)
    raise OracleDataError(kind)


def loss_deriv(kind: str, w):
    w = np.asarray(w, dtype=float)
    if kind == "square":  # problems.py:58
        return w.copy()
    if kind == "logistic":  # problems.py:83
        return expit(w)
    if kind == "huber":  # problems.py:99-101
        return np.where(np.abs(w) <= 1.0, 2.0 * w, 2.0 * np.sign(w))
    raise OracleDataError(kind)


def loss_deriv2(kind: str, w):
    w = np.asarray(w, dtype=float)
    if kind == "square":  # problems.py:59
        return np.ones_like(w)
    if kind == "logistic":  # problems.py:84
        return expit(w) * expit(-w)
    if kind == "huber":  # problems.py:103-105
        return np.where(np.abs(w) <= 1.0, 2.0, 0.0)
    raise OracleDataError(kind)


def loss_conj(kind: str, y):
    y = np.asarray(y, dtype=float)
    if kind == "square":  # problems.py:60
        return 0.5 * y**2
    if kind == "logistic":  # problems.py:65-73
        inside = (y >= 0.0) & (y <= 1.0)
        yc = np.clip(y, 1e-12, 1.0 - 1e-12)
        ent = yc * np.log(yc) + (1.0 - yc) * np.log1p(-yc)
        return np.where((y == 0.0) | (y == 1.0), 0.0, np.where(inside, ent, np.inf))
    return None  # huber conj exists in the reference but the gap is only used when conj is set


def loss_has_conj(kind: str) -> bool:
    # problems.py:53-111: square/logistic/huber all carry a conjugate
    return kind in ("square", "logistic", "huber")


def huber_conj(y):  # problems.py:107-109
    y = np.asarray(y, dtype=float)
    return np.where(np.abs(y) <= 2.0, 0.25 * y**2, np.inf)


def _conj(kind, y):
    if kind == "huber":
        return huber_conj(y)
    return loss_conj(kind, y)


# --------------------------------------------------------------------------
# prox  (prox.py:38-48, 96-144)


def soft_threshold(v, kappa):  # prox.py:38-43
    if kappa < 0:
        raise OracleDataError("kappa")
    v = np.asarray(v, dtype=float)
    return np.sign(v) * np.maximum(np.abs(v) - kappa, 0.0)


def box_project(v, lo, hi):  # prox.py:46-48
    return np.clip(np.asarray(v, dtype=float), lo, hi)


def box_indicator(z, lo, hi, tol=1e-9):  # prox.py:138-144
    z = np.asarray(z, dtype=float)
    scale = 1.0 + np.max(np.abs(z), initial=0.0)
    if np.all(z >= lo - tol * scale) and np.all(z <= hi + tol * scale):
        return 0.0
    return np.inf


def box_support(y, lo, hi):  # prox.py:96-110
    y = np.asarray(y, dtype=float)
    pos, neg = y > 0, y < 0
    if np.any(pos & np.isinf(hi)) or np.any(neg & np.isinf(lo)):
        return np.inf
    total = 0.0
    total += np.sum(hi[pos] * y[pos])
    total += np.sum(lo[neg] * y[neg])
    return float(total)


def box_recession_distance(y, lo, hi):  # prox.py:113-135
    y = np.asarray(y, dtype=float)
    lf, uf = np.isfinite(lo), np.isfinite(hi)
    proj = y.copy()
    proj[lf & uf] = 0.0
    up = ~uf & lf
    proj[up] = np.maximum(y[up], 0.0)
    dn = ~lf & uf
    proj[dn] = np.minimum(y[dn], 0.0)
    return float(np.linalg.norm(y - proj))


# --------------------------------------------------------------------------
# Krylov  (krylov.py:35-112)


@dataclass
class CgOut:
    iterations: int
    final_relative_residual: float
    converged: bool


def pcg(matvec, b, x0=None, Minv=None, tol_rel=1e-8, max_iter=None):
    """krylov.py:35-95 -- warm-started PCG, recurrence residual with a true
    residual refresh every 50 iterations, SPD / finiteness checks."""
    b = np.asarray(b, dtype=float)
    n = b.size
    if max_iter is None:
        max_iter = 10 * n
    x = np.zeros(n) if x0 is None else np.asarray(x0, dtype=float).copy()
    b_norm = float(np.linalg.norm(b))
    denom = b_norm if b_norm > 0 else 1.0
    r = b - matvec(x)
    res = float(np.linalg.norm(r))
    if res <= tol_rel * denom:
        return x, CgOut(0, res / denom, True)
    z = Minv(r) if Minv is not None else r.copy()
    p = z.copy()
    rz = float(r @ z)
    k = 0
    for k in range(1, max_iter + 1):
        Ap = matvec(p)
        pAp = float(p @ Ap)
        if not np.isfinite(pAp):
            raise OracleNumerical("non-finite pAp")
        if pAp <= 0:
            raise OracleNotSPD(f"pAp={pAp}")
        alpha = rz / pAp
        x += alpha * p
        if k % 50 == 0:  # krylov.py:16, 80-83
            r = b - matvec(x)
        else:
            r -= alpha * Ap
        res = float(np.linalg.norm(r))
        if not np.isfinite(res):
            raise OracleNumerical("non-finite residual")
        if res <= tol_rel * denom:
            return x, CgOut(k, res / denom, True)
        z = Minv(r) if Minv is not None else r.copy()
        rz_new = float(r @ z)
        beta = rz_new / rz
        rz = rz_new
        p = z + beta * p
    return x, CgOut(k, res / denom, False)


def cg_tolerance(k, rp, rd, gamma=1.2):  # krylov.py:98-112
    if k < 1 or rp < 0 or rd < 0 or gamma <= 1:
        raise ValueError("cg_tolerance arguments")
    tol = min(np.sqrt(rp * rd), 1.0) / k**gamma
    return max(tol, 1e-12)


# --------------------------------------------------------------------------
# Nystrom sketch and preconditioner  (sketch.py:29-165)


def default_sketch_rank(n):  # sketch.py:29-31
    return max(1, min(50, math.ceil(n / 20)))


def sketch_width(n, r, oversample=None):  # sketch.py:93-95
    if oversample is None:
        oversample = 8 + r // 4
    return min(n, r + max(oversample, 0))


def raw_test_matrix(n, s, seed):
    """sketch.py:97-98 -- the raw Gaussian Omega before orthonormalisation.
    The GPU path receives exactly this array."""
    return np.random.default_rng(seed).standard_normal((n, s))


def nystrom_sketch(apply_cols: Callable, n: int, r: int, seed: int, oversample=None):
    """sketch.py:74-128.  ``apply_cols(V)`` returns the operator applied to
    every column of V (the reference applies column by column, sketch.py:69-71;
    per-column results are identical)."""
    if not 1 <= r <= n:
        raise OracleDataError("rank")
    s = sketch_width(n, r, oversample)
    Om = raw_test_matrix(n, s, seed)
    Om, _ = np.linalg.qr(Om, mode="reduced")
    Y = apply_cols(Om)
    trace_est = (n / s) * float(np.sum(Om * Y))
    shift = EPS * max(trace_est, 0.0)
    if shift == 0.0:
        shift = EPS
    Ys = Y + shift * Om
    core = Om.T @ Ys
    core = 0.5 * (core + core.T)
    try:
        L = np.linalg.cholesky(core)
        B = scipy.linalg.solve_triangular(L, Ys.T, lower=True).T
    except np.linalg.LinAlgError:
        w, V = np.linalg.eigh(core)
        scale = max(abs(w[-1]), shift)
        if w[0] < -1e-8 * scale:
            raise OracleDataError("operator is not positive semidefinite") from None
        keep = w > EPS * scale
        if not keep.any():
            return np.zeros((n, 0)), np.zeros(0)
        B = Ys @ (V[:, keep] / np.sqrt(w[keep]))
    U, sv, _ = np.linalg.svd(B, full_matrices=False)
    lam = np.maximum(sv**2 - shift, 0.0)
    return U[:, :r], lam[:r]


def precond_apply(U, lam, nu, v):  # sketch.py:143-151
    v = np.asarray(v, dtype=float)
    if U.shape[1] == 0:
        return v.copy()
    Utv = U.T @ v
    head = (lam[-1] + nu) * (Utv / (lam + nu))
    return U @ (head - Utv) + v


def dense_operator_columns(M):
    """Column-by-column apply of a dense matrix (operators.py:114-115 per column)."""
    return lambda V: np.column_stack([M @ V[:, j] for j in range(V.shape[1])])


# --------------------------------------------------------------------------
# problems  (problems.py:160-461)


@dataclass
class MLSpec:
    """problems.py:191-220 (dense A only)."""

    loss: str
    A: np.ndarray
    b: np.ndarray
    lambda1: float = 0.0
    lambda2: float = 0.0

    @property
    def n(self):
        return self.A.shape[1]


@dataclass
class QPSpec:
    """problems.py:160-188.  P and M are anything with ``@`` and ``.T``
    (ndarray, scipy sparse, ``DiagLowRank``); M = None is the identity."""

    P: object
    q: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    M: object = None

    @property
    def n(self):
        return self.P.shape[0]

    @property
    def m(self):
        return self.n if self.M is None else self.M.shape[0]


class DiagLowRank:
    """diag(d) + F F^T in factored form (operators.py:138-160)."""

    def __init__(self, d, F):
        self.d = np.asarray(d, dtype=float)
        self.F = np.asarray(F, dtype=float)
        self.shape = (self.d.size, self.d.size)

    def __matmul__(self, v):
        return self.d * v + self.F @ (self.F.T @ v)

    @property
    def T(self):
        return self


class StackOp:
    """[A_1; A_2; ...] (operators.py:163-191); parts with ``@`` and ``.T``."""

    def __init__(self, parts):
        self.parts = list(parts)
        self.off = np.cumsum([0] + [p.shape[0] for p in self.parts])
        self.shape = (int(self.off[-1]), self.parts[0].shape[1])

    def __matmul__(self, v):
        return np.concatenate([np.atleast_1d(p @ v) for p in self.parts])

    @property
    def T(self):
        outer = self

        class _Adj:
            shape = (outer.shape[1], outer.shape[0])

            def __matmul__(self, u):
                out = np.zeros(outer.shape[1])
                for p, lo, hi in zip(outer.parts, outer.off[:-1], outer.off[1:]):
                    out += p.T @ u[lo:hi]
                return out

        return _Adj()


class OnesRow:
    """v -> [sum v]; adjoint broadcasts (operators.py:194-203)."""

    def __init__(self, n):
        self.shape = (1, n)

    def __matmul__(self, v):
        return np.array([v.sum()])

    @property
    def T(self):
        n = self.shape[1]

        class _Adj:
            shape = (n, 1)

            def __matmul__(self, u):
                return np.full(n, u[0])

        return _Adj()


def estimate_extreme_eigs(matvec, n, iters, rng_seed):  # sketch.py:240-282
    if iters < 2:
        raise OracleDataError("iters >= 2")
    iters = min(iters, n)
    rng = np.random.default_rng(rng_seed)
    q = rng.standard_normal(n)
    q /= np.linalg.norm(q)
    Q = np.zeros((n, iters))
    alphas, betas = [], []
    Q[:, 0] = q
    scale = 0.0
    for j in range(iters):
        w = matvec(Q[:, j])
        alpha = float(Q[:, j] @ w)
        alphas.append(alpha)
        scale = max(scale, abs(alpha))
        w -= alpha * Q[:, j]
        if j > 0:
            w -= betas[-1] * Q[:, j - 1]
        for _ in range(2):
            w -= Q[:, : j + 1] @ (Q[:, : j + 1].T @ w)
        beta = float(np.linalg.norm(w))
        if j == iters - 1 or beta <= 1e-12 * max(scale, 1.0):
            break
        betas.append(beta)
        Q[:, j + 1] = w / beta
    T = np.diag(alphas)
    if betas:
        k = len(alphas)
        T += np.diag(betas[: k - 1], 1) + np.diag(betas[: k - 1], -1)
    ritz = np.linalg.eigvalsh(T)
    return float(ritz[-1]), float(ritz[0])


def estimate_error_norm(matvec, U, lam, n, iters, rng_seed):  # sketch.py:176-195
    rng = np.random.default_rng(rng_seed)
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    est = 0.0
    for _ in range(iters):
        w = matvec(v) - (U @ (lam * (U.T @ v)) if U.shape[1] else 0.0)
        est = float(np.linalg.norm(w))
        if est <= 0.0 or not np.isfinite(est):
            return max(est, 0.0)
        v = w / est
    return est


def adaptive_sketch(matvec, n, r0, r_max, nu, kappa_target, rng_seed, power_iters=10):  # sketch.py:204-237
    ranks = []
    r = r0
    while r < r_max:
        ranks.append(r)
        r *= 2
    ranks.append(r_max)
    seeds = np.random.SeedSequence(rng_seed).generate_state(2 * len(ranks))
    cols = lambda V: np.column_stack([matvec(V[:, j]) for j in range(V.shape[1])])
    out = None
    for i, rank in enumerate(ranks):
        U, lam = nystrom_sketch(cols, n, rank, int(seeds[2 * i]))
        out = (U, lam)
        err = estimate_error_norm(matvec, U, lam, n, power_iters, int(seeds[2 * i + 1]))
        tail = lam[-1] if lam.size else 0.0
        if 1.0 + (tail + err) / nu <= kappa_target:
            return out
    return out


def ml_residuals(p: MLSpec, x):  # problems.py:219-220
    return p.A @ x - p.b


def ml_smooth_value(p: MLSpec, x):  # problems.py:227-230
    r = ml_residuals(p, x)
    return float(np.sum(loss_value(p.loss, r)) + 0.5 * p.lambda2 * np.dot(x, x))


def ml_objective(p: MLSpec, x):  # problems.py:233-235
    return ml_smooth_value(p, x) + p.lambda1 * float(np.abs(x).sum())


def ml_gradient(p: MLSpec, x):  # problems.py:238-242
    return p.A.T @ loss_deriv(p.loss, ml_residuals(p, x)) + p.lambda2 * np.asarray(x, dtype=float)


def ml_weights(p: MLSpec, x):  # problems.py:260-261
    return np.asarray(loss_deriv2(p.loss, ml_residuals(p, x)), dtype=float)


def ml_hvp(p: MLSpec, w, v):  # problems.py:263-264
    return p.A.T @ (w * (p.A @ v)) + p.lambda2 * v


def ml_smooth_hvp(p: MLSpec, w, v):  # problems.py:270-271 (the sketch target)
    return p.A.T @ (w * (p.A @ v))


def ml_dual_point(p: MLSpec, x):  # problems.py:306-318
    nu = np.asarray(loss_deriv(p.loss, ml_residuals(p, x)), dtype=float)
    if p.lambda2 == 0.0:
        denom = float(np.max(np.abs(p.A.T @ nu), initial=0.0))
        if denom > p.lambda1:
            nu = nu * (p.lambda1 / denom)
    return nu


def ml_dual_value(p: MLSpec, nu):  # problems.py:321-332
    cv = _conj(p.loss, nu)
    if np.any(np.isinf(cv)):
        return -np.inf
    val = -float(np.sum(cv)) - float(p.b @ nu)
    if p.lambda2 > 0.0:
        excess = np.maximum(np.abs(p.A.T @ nu) - p.lambda1, 0.0)
        val -= float(np.sum(excess**2)) / (2.0 * p.lambda2)
    return val


def huber_subdiff_distance(p: MLSpec, x):  # problems.py:354-368
    w = ml_gradient(p, x)
    active = x != 0.0
    d2 = float(np.sum((w[active] + p.lambda1 * np.sign(x[active])) ** 2))
    d2 += float(np.sum(np.maximum(np.abs(w[~active]) - p.lambda1, 0.0) ** 2))
    return float(np.sqrt(d2))


def huber_subdiff_stop(tol=1e-4):  # problems.py:371-384 (on the sparse iterate z)
    return lambda p, z: huber_subdiff_distance(p, z) <= tol


def ml_dual_gap(p: MLSpec, x):  # problems.py:335-351
    nu = ml_dual_point(p, x)
    primal = ml_objective(p, x)
    dual = ml_dual_value(p, nu)
    if not np.isfinite(dual):
        return np.inf
    num = primal - dual
    denom = min(primal, abs(dual))
    if denom <= 1e-16:
        return 0.0 if abs(num) <= 1e-12 else np.inf
    return num / denom


# --------------------------------------------------------------------------
# solver  (admm.py:45-719, restricted to M = I, c = 0)


@dataclass
class Options:
    """admm.py:45-99 (the fields the in-scope path reads)."""

    sigma: float = 1e-6
    gamma: float = 1.2
    sketch_rank: Optional[int] = None
    resketch_every: int = 20
    norm_kind: str = "l2"
    eps_abs: float = 1e-4
    eps_rel: float = 1e-4
    eps_inf: float = 1e-8
    alpha: float = 1.6
    tau: float = 2.0
    mu: float = 10.0
    rho0: float = 1.0
    penalty_update_every: int = 25
    penalty_warmup: int = 100
    max_iter: int = 10000
    time_limit: Optional[float] = None
    use_preconditioner: bool = True
    exact_x_solve: bool = False
    use_dual_gap: Optional[bool] = None
    eps_dual_gap: float = 1e-4
    rng_seed: int = 0
    assume_full_rank: bool = False
    check_rank: bool = False
    custom_stop: Optional[Callable] = None  # (problem spec, z) -> bool, replaces the built-in test
    callback: Optional[Callable] = None  # callback(k) after every iteration (admm.py:610-611; bench timing)


@dataclass
class OracleResult:
    status: str
    x: np.ndarray
    z: np.ndarray
    u: np.ndarray
    objective: float
    iterations: int
    rp_norm: float
    rd_norm: float
    gap: Optional[float]
    cg_iters: list = field(default_factory=list)
    rho_hist: list = field(default_factory=list)
    gap_hist: list = field(default_factory=list)
    obj_hist: list = field(default_factory=list)
    rp_hist: list = field(default_factory=list)
    rd_hist: list = field(default_factory=list)
    penalty_events: list = field(default_factory=list)
    x_bar: Optional[np.ndarray] = None
    z_bar: Optional[np.ndarray] = None
    certificate: Optional[np.ndarray] = None
    n_sketches: int = 0
    total_s: float = 0.0
    setup_s: float = 0.0


def _norm(v, kind):  # admm.py:203-208
    if v.size == 0:
        return 0.0
    if kind == "linf":
        return float(np.max(np.abs(v)))
    return float(np.linalg.norm(v))


def solve(problem, opts: Optional[Options] = None) -> OracleResult:
    """admm.py:422-719 for ML problems (dense or sparse A) and box QPs with a
    general constraint map M."""
    t_start = time.perf_counter()
    opts = opts or Options()
    is_ml = isinstance(problem, MLSpec)
    n = problem.n
    kind = opts.norm_kind
    Mop = None if is_ml else problem.M
    identity_M = Mop is None
    m = n if identity_M else Mop.shape[0]
    M_apply = (lambda v: v) if identity_M else (lambda v: np.asarray(Mop @ v, dtype=float))
    M_adj = (lambda v: v) if identity_M else (lambda v: np.asarray(Mop.T @ v, dtype=float))

    # lowering (problems.py:387-450): f, grad, hess, g, prox with M = I, c = 0
    if is_ml:
        p = problem
        f = lambda x: ml_smooth_value(p, x)
        grad = lambda x: ml_gradient(p, x)
        g = lambda z: p.lambda1 * float(np.abs(z).sum())
        prox = lambda v, rho: soft_threshold(v, p.lambda1 / rho)
        const_hess = p.loss == "square"
        diag_shift = p.lambda2
        weights = ml_weights(p, np.zeros(n))  # MLHessian.__init__ update(0)
    else:
        qp = problem
        f = lambda x: 0.5 * float(x @ (qp.P @ x)) + float(qp.q @ x)
        grad = lambda x: qp.P @ x + qp.q
        g = lambda z: box_indicator(z, qp.lo, qp.hi)
        prox = lambda v, rho: box_project(v, qp.lo, qp.hi)
        const_hess = True
        diag_shift = 0.0
        weights = None

    def hess_apply(v):
        if is_ml:
            return ml_hvp(p, weights, v)
        return qp.P @ v

    def smooth_cols(V):  # sketch target, column by column (sketch.py:69-71)
        if is_ml:
            return np.column_stack([ml_smooth_hvp(p, weights, V[:, j]) for j in range(V.shape[1])])
        return np.column_stack([qp.P @ V[:, j] for j in range(V.shape[1])])

    x = np.zeros(n)
    z = np.zeros(m)
    u = np.zeros(m)
    rho = opts.rho0
    if is_ml:
        weights = ml_weights(p, x)  # admm.py:457
    Mx = M_apply(x).copy()
    x_bar_sum = np.zeros(n)
    z_bar_sum = np.zeros(m)
    bar_count = 0
    # offset policy (admm.py:462-474): ML lowerings and M = I QPs are full rank
    sigma_eff = opts.sigma
    if is_ml or identity_M or opts.assume_full_rank:
        sigma_eff = 0.0
    elif opts.check_rank:
        comp0 = lambda v: hess_apply(v) + rho * M_adj(M_apply(v))
        _, lam_min = estimate_extreme_eigs(comp0, n, min(max(2, n), 60), opts.rng_seed + 7)
        if lam_min > 1e-8:
            sigma_eff = 0.0

    use_gap = opts.use_dual_gap
    if use_gap is None:
        use_gap = is_ml and loss_has_conj(p.loss)
    if use_gap and not is_ml:
        raise OracleDataError("gap requires ML")

    r_sk = opts.sketch_rank or default_sketch_rank(n)
    r_sk = max(1, min(r_sk, n))
    nu_of = lambda rho_: rho_ + sigma_eff + diag_shift  # admm.py:490-491
    sketch = None
    pc_nu = None
    n_sk = 0
    last_sketch = 0
    rho_at_sketch = rho

    def build(seed):  # admm.py:493-507
        if identity_M:
            return nystrom_sketch(smooth_cols, n, r_sk, seed), nu_of(rho)
        rho_now = rho
        comp = lambda v: hess_apply(v) + rho_now * M_adj(M_apply(v))
        cols = lambda V: np.column_stack([comp(V[:, j]) for j in range(V.shape[1])])
        return nystrom_sketch(cols, n, r_sk, seed), max(sigma_eff, 1e-8)

    if opts.use_preconditioner:
        sketch, pc_nu = build(opts.rng_seed)
        rho_at_sketch = rho
        n_sk += 1

    def residuals():  # admm.py:215-224
        rp = Mx - z
        Mtu = M_adj(u)
        rd = grad(x) + rho * Mtu
        ps = max(_norm(Mx, kind), _norm(z, kind), _norm(np.zeros(m), kind))
        ds = _norm(rho * Mtu, kind)
        return rp, rd, _norm(rp, kind), _norm(rd, kind), ps, ds

    rp, rd, rpn, rdn, ps, ds = residuals()
    setup_s = time.perf_counter() - t_start

    res = OracleResult("iteration_limit", x, z, u, np.nan, 0, rpn, rdn, None)
    xw = deque(maxlen=26)
    uw = deque(maxlen=26)
    xw.append(x.copy())
    uw.append(u.copy())
    status = "iteration_limit"
    gap = None
    rho_frozen = False
    hits = 0
    best = np.inf
    trend = deque(maxlen=26)
    k = 0
    for k in range(1, opts.max_iter + 1):  # (k is state.k before the time check, admm.py:534-537)
        if opts.time_limit is not None and time.perf_counter() - t_start > opts.time_limit:
            status = "time_limit"
            break
        if not const_hess:
            weights = ml_weights(p, x)  # admm.py:539-540
        if sketch is not None:  # admm.py:545-551
            stale_hess = not const_hess and k - last_sketch >= opts.resketch_every
            stale_rho = not identity_M and rho != rho_at_sketch
            if stale_hess or stale_rho:
                sketch, pc_nu = build(opts.rng_seed + k)
                n_sk += 1
                last_sketch = k
                rho_at_sketch = rho
        tol = 1e-12 if opts.exact_x_solve else cg_tolerance(k, rpn, rdn, opts.gamma)

        # x_update (admm.py:243-275)
        shift = rho + sigma_eff
        if identity_M:
            matvec = lambda v: hess_apply(v) + shift * v
        else:
            matvec = lambda v, _r=rho: hess_apply(v) + _r * M_adj(M_apply(v)) + sigma_eff * v
        rhs = hess_apply(x) + sigma_eff * x - grad(x)
        target = z + 0.0 - u
        rhs = rhs + (rho * target if identity_M else rho * M_adj(target))
        Minv = (lambda v: precond_apply(sketch[0], sketch[1], pc_nu, v)) if sketch is not None else None
        x_new, cg = pcg(matvec, rhs, x0=x, Minv=Minv, tol_rel=tol, max_iter=10 * n)

        Mx_new = x_new if identity_M else M_apply(x_new)
        w = opts.alpha * Mx_new + (1.0 - opts.alpha) * (z + 0.0)  # admm.py:278-280
        x_prev, u_prev = x, u.copy()
        x = x_new
        Mx = Mx_new
        z_new = prox(w - 0.0 + u, rho)  # admm.py:283-296
        u = u + w - z_new - 0.0  # admm.py:299-300
        z = z_new
        if k >= 2:  # admm.py:580-583
            x_bar_sum += x
            z_bar_sum += z
            bar_count += 1
        rp, rd, rpn, rdn, ps, ds = residuals()
        objective = f(x) + g(z)
        gap = ml_dual_gap(p, z) if use_gap else None
        res.cg_iters.append(cg.iterations)
        res.rho_hist.append(rho)
        res.gap_hist.append(gap)
        res.obj_hist.append(objective)
        res.rp_hist.append(rpn)
        res.rd_hist.append(rdn)

        if opts.callback is not None:
            opts.callback(k)
        # check_termination (admm.py:227-240), or the custom rule (admm.py:613-616)
        if opts.custom_stop is not None:
            done = bool(opts.custom_stop(problem, z))
        elif gap is not None:
            done = gap <= opts.eps_dual_gap
        else:
            done = rpn <= np.sqrt(m) * opts.eps_abs + opts.eps_rel * ps and rdn <= np.sqrt(
                n
            ) * opts.eps_abs + opts.eps_rel * ds
        if done:
            status = "optimal"
            break

        xw.append(x.copy())
        uw.append(u.copy())
        if not is_ml and len(uw) == 26:  # admm.py:621-634
            dx = (xw[-1] - xw[0]) / 25
            du = (uw[-1] - uw[0]) / 25
            st, near = _infeasibility(dx, du, qp, opts, M_apply, M_adj)
            if near:
                rho_frozen = True
            if st is not None:
                status = st
                # admm.py:391, 405 (the certificate property prefers the primal one)
                res.certificate = rho * du if st.startswith("primal") else dx.copy()
                break

        # cycle guard (admm.py:643-675)
        best = min(best, max(rpn, rdn))
        trend.append(best)
        if len(xw) >= 4 and not rho_frozen and k <= 1000:
            xk = xw[-1]
            step = float(np.linalg.norm(xk - xw[-2]))
            locked = False
            if step > 1e-8 * max(1.0, float(np.linalg.norm(xk))):
                periods = range(2, min(len(xw) - 1, 10) + 1)
                rg = min(float(np.linalg.norm(xk - xw[-1 - q])) for q in periods)
                locked = rg <= 1e-3 * step
            hits = hits + 1 if locked else 0
            stagnant = len(trend) == trend.maxlen and trend[-1] >= 0.99 * trend[0]
            if hits >= 5 and stagnant:
                hits = 0
                trend.clear()
                rho, u, ev = _change_penalty(rho, u, rho * opts.tau, k)
                res.penalty_events.append(ev)
                if sketch is not None and identity_M:
                    pc_nu = nu_of(rho)
                xw.clear()
                uw.clear()
                xw.append(x.copy())
                uw.append(u.copy())

        # balanced-residual penalty rule (admm.py:677-698, 322-350)
        if (
            not rho_frozen
            and opts.penalty_update_every > 0
            and k >= opts.penalty_warmup
            and k % opts.penalty_update_every == 0
            and k <= 1000
        ):
            t_p = np.sqrt(rp.size) * opts.eps_abs + opts.eps_rel * ps
            t_d = np.sqrt(rd.size) * opts.eps_abs + opts.eps_rel * ds
            if t_p > 0 and t_d > 0:
                pm, dm = rpn / t_p, rdn / t_d
            else:
                pm, dm = rpn, rdn
            new = None
            if pm > opts.mu * dm:
                new = rho * opts.tau
            elif dm > opts.mu * pm:
                new = rho / opts.tau
            if new is not None:
                rho, u, ev = _change_penalty(rho, u, new, k)
                res.penalty_events.append(ev)
                if sketch is not None and identity_M:
                    pc_nu = nu_of(rho)
                xw.clear()
                uw.clear()
                xw.append(x.copy())
                uw.append(u.copy())

    res.status = status
    res.x, res.z, res.u = x, z, u
    res.objective = f(x) + g(z)
    res.iterations = k
    res.rp_norm, res.rd_norm = rpn, rdn
    res.gap = gap
    res.x_bar = x_bar_sum / bar_count if bar_count else None
    res.z_bar = z_bar_sum / bar_count if bar_count else None
    res.n_sketches = n_sk
    res.total_s = time.perf_counter() - t_start
    res.setup_s = setup_s
    return res


def _change_penalty(rho_old, u, rho_new, k):  # admm.py:303-319
    y_old = rho_old * u
    u = u * (rho_old / rho_new)
    y_new = rho_new * u
    denom = max(float(np.linalg.norm(y_old)), 1e-30)
    jump = float(np.linalg.norm(y_new - y_old)) / denom
    return rho_new, u, (k, rho_old, rho_new, jump)


def _infeasibility(dx, du, qp: QPSpec, opts: Options, M_apply=lambda v: v, M_adj=lambda v: v):  # admm.py:361-415
    eps = opts.eps_inf
    primal = dual = near_p = near_d = False
    dun = float(np.linalg.norm(du))
    if dun > 1e-14:
        t_map = float(np.linalg.norm(M_adj(du)))
        t_sup = box_support(du, qp.lo, qp.hi)
        primal = t_map < eps * dun and t_sup < eps * dun
        near_p = t_map < 10 * eps * dun and t_sup < 10 * eps * dun
    dxn = float(np.linalg.norm(dx))
    if dxn > 1e-14:
        s_obj = float(np.linalg.norm(qp.P @ dx))
        s_cone = box_recession_distance(M_apply(dx), qp.lo, qp.hi)
        s_lin = float(qp.q @ dx)
        dual = s_obj < eps * dxn and s_cone < eps * dxn and s_lin < eps * dxn
        near_d = s_obj < 10 * eps * dxn and s_cone < 10 * eps * dxn and s_lin < 10 * eps * dxn
    if primal and dual:
        st = "primal_and_dual_infeasible"
    elif primal:
        st = "primal_infeasible"
    elif dual:
        st = "dual_infeasible"
    else:
        st = None
    return st, near_p or near_d
