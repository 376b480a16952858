"""Problem interfaces of the hot path (``/root/reference/pkg/src/nysopt/problems.py``).

Same constructors and fields as the reference: ``MLProblem`` (square /
logistic / huber loss, l1 + l2 regularisation, problems.py:191-220),
``QPProblem`` (problems.py:160-188) and the convenience constructors
(problems.py:468-481).  Losses are identified by ``kind``; their derivatives
and conjugates are evaluated on the device by the K8-K12 kernels, so ``Loss``
carries the reference's flags rather than NumPy callables.

The ML oracles (objective, gradient, Hessian, dual point/value/gap) run on the
GPU through the C ABI; inside ``solve`` they are fused into the per-iteration
passes (admm.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from .errors import DataError
from .operators import (
    ConstantHessian,
    DenseOperator,
    HessianOperator,
    IdentityOperator,
    LinearOperator,
    MatrixFreeOperator,
    SparseOperator,
    as_operator,
    device_fn,
    like_input,
    to_device,
)
from .prox import Box, box_indicator, box_project, soft_threshold


def _loss_eval(kind: str, what: int) -> Callable:
    """Elementwise evaluation of a built-in loss on the device (nys_loss_eval_f64):
    NumPy (any shape, scalars) or device arrays in, the same kind out."""

    def fn(w):
        from .kernels import get_kernels

        shape = np.shape(w) if not isinstance(w, torch.Tensor) else tuple(w.shape)
        wt = to_device(np.asarray(w, dtype=float).reshape(-1) if not isinstance(w, torch.Tensor)
                       else w.reshape(-1)).contiguous()
        out = torch.empty_like(wt)
        if wt.numel():
            get_kernels().loss_eval(kind, what, wt, out)
        if isinstance(w, torch.Tensor):
            return out.reshape(shape)
        res = out.cpu().numpy().reshape(shape)
        return res if res.shape else float(res)

    return fn


@dataclass(frozen=True)
class Loss:
    """Scalar convex per-sample loss with its derivatives and optional conjugate
    (problems.py:35-50; the same fields in the same order).  ``value``,
    ``deriv``, ``deriv2`` and ``conj`` act elementwise; for the built-in kinds
    they default to the device evaluation of csrc/loss.cuh -- the expressions
    the fused kernels of ``solve`` use (``conj`` gives +inf outside its domain).
    ``solve`` itself selects its kernels by ``kind``."""

    kind: str
    value: Optional[Callable] = None
    deriv: Optional[Callable] = None
    deriv2: Optional[Callable] = None
    conj: Optional[Callable] = None
    deriv2_constant: bool = False

    def __post_init__(self):
        if self.kind in ("square", "logistic", "huber"):
            for what, name in enumerate(("value", "deriv", "deriv2", "conj")):
                if getattr(self, name) is None:
                    object.__setattr__(self, name, _loss_eval(self.kind, what))

    @property
    def has_conj(self) -> bool:
        # the conjugate's presence enables the duality-gap stopping rule (admm.py:476-478)
        return self.conj is not None


def square_loss() -> Loss:
    """l(w) = w^2/2, conjugate y^2/2 (problems.py:53-62)."""
    return Loss("square", deriv2_constant=True)


def logistic_loss() -> Loss:
    """l(w) = log(1 + e^w), conjugate the binary entropy (problems.py:76-86)."""
    return Loss("logistic")


def huber_loss() -> Loss:
    """w^2 on [-1, 1], 2|w| - 1 outside; conjugate y^2/4 on |y| <= 2 (problems.py:89-111)."""
    return Loss("huber")


def _loss_arg(loss: Loss):
    """What the row-wise kernels take: the kind of a built-in loss, else the Loss itself."""
    return loss.kind if loss.kind in ("square", "logistic", "huber") else loss


def builtin_loss(kind: str) -> Loss:
    factories = {"square": square_loss, "logistic": logistic_loss, "huber": huber_loss}
    if kind not in factories:
        raise DataError(f"unknown loss kind {kind!r}; expected one of {sorted(factories)}")
    return factories[kind]()


@dataclass
class QPProblem:
    """minimize (1/2) x'Px + q'x subject to l <= Mx <= u (problems.py:160-188)."""

    P: LinearOperator
    q: np.ndarray
    M: LinearOperator
    box: Box

    def __post_init__(self):
        self.P = as_operator(self.P)
        self.M = as_operator(self.M)
        self.q = np.asarray(self.q, dtype=float)
        if self.P.input_dim != self.P.output_dim:
            raise DataError("P must be square")
        if self.q.shape != (self.P.input_dim,):
            raise DataError("q must have length n")
        if self.M.input_dim != self.P.input_dim:
            raise DataError("M must map from dimension n")
        if self.box.dim != self.M.output_dim:
            raise DataError("box dimension must equal the number of constraint rows")

    @property
    def n(self) -> int:
        return self.P.input_dim

    @property
    def m(self) -> int:
        return self.M.output_dim


@dataclass
class MLProblem:
    """minimize sum_i l(a_i'x - b_i) + lambda1 ||x||_1 + (lambda2/2)||x||_2^2
    (problems.py:191-220)."""

    loss: Loss
    A: LinearOperator
    b: np.ndarray
    lambda1: float = 0.0
    lambda2: float = 0.0

    def __post_init__(self):
        self.A = as_operator(self.A)
        if isinstance(self.b, torch.Tensor):
            self.b = self.b.detach().cpu().numpy()
        self.b = np.asarray(self.b, dtype=float)
        if self.b.shape != (self.A.output_dim,):
            raise DataError("response vector length must equal the number of samples")
        if self.lambda1 < 0 or self.lambda2 < 0:
            raise DataError("regularization parameters must be nonnegative")
        if self.lambda1 == 0 and self.lambda2 == 0:
            raise DataError("at least one regularization parameter must be positive")

    @property
    def n(self) -> int:
        return self.A.input_dim

    @property
    def N(self) -> int:
        return self.A.output_dim

    def residuals(self, x):
        return like_input(self.A._apply_dev(to_device(x)) - to_device(self.b), x)


@dataclass
class GenericProblem:
    """Lowered form minimize f(x) + g(z) s.t. Mx - z = c (problems.py:125-157).

    On the B200 path the lowering keeps a back reference to the structured
    problem; arbitrary user callables (f, prox_g on NumPy) are outside the
    device hot path and are rejected by ``solve``."""

    n: int
    m: int
    # the reference's field order (problems.py:137-150).  The oracles of a lowered
    # ML / QP problem run on the device (NumPy or device arrays in, the same kind
    # out); the single-step API of admm.py (x_update, z_update, ...) uses them.
    f: Optional[Callable] = None
    grad_f: Optional[Callable] = None
    hess: Optional[HessianOperator] = None
    g: Optional[Callable] = None
    prox_g: Optional[Callable] = None
    M: Optional[LinearOperator] = None
    c: Optional[np.ndarray] = None
    is_quadratic: bool = False
    full_rank: bool = False
    prox_inexact: bool = False
    qp: Optional[QPProblem] = None
    ml: Optional[MLProblem] = None

    def __post_init__(self):
        # problems.py:152-158
        if self.M is None:
            self.M = IdentityOperator(self.n)
        self.c = np.zeros(self.m) if self.c is None else np.asarray(self.c, dtype=float)
        if self.M.input_dim != self.n or self.M.output_dim != self.m:
            raise DataError("constraint operator dimensions do not match (n, m)")
        if self.c.shape != (self.m,):
            raise DataError("offset c must have length m")
        if self.hess is not None and self.hess.input_dim != self.n:
            raise DataError("Hessian dimension must equal n")


def lasso_problem(A, b, lambda1: float) -> MLProblem:
    return MLProblem(square_loss(), A, b, lambda1=lambda1, lambda2=0.0)


def elastic_net_problem(A, b, lambda1: float, lambda2: float) -> MLProblem:
    return MLProblem(square_loss(), A, b, lambda1=lambda1, lambda2=lambda2)


def logistic_problem(A, b, lambda1: float, lambda2: float = 0.0) -> MLProblem:
    return MLProblem(logistic_loss(), A, b, lambda1=lambda1, lambda2=lambda2)


def huber_problem(A, b, lambda1: float) -> MLProblem:
    return MLProblem(huber_loss(), A, b, lambda1=lambda1, lambda2=0.0)


def lasso_as_qp(A, b, lambda1: float) -> QPProblem:
    """Block QP reformulation of the lasso with auxiliary magnitudes t
    (problems.py:484-502): variables (x, t), |x| <= t by two stacked identity
    blocks; P and the constraint matrix are kept sparse (CSR on the device)."""
    import scipy.sparse as sp

    A = np.asarray(A, dtype=float)
    b = np.asarray(b, dtype=float)
    n = A.shape[1]
    P = sp.bmat([[sp.csr_matrix(A.T @ A), None], [None, sp.csr_matrix((n, n))]])
    q = np.concatenate([-A.T @ b, lambda1 * np.ones(n)])
    eye = sp.eye(n)
    M = sp.bmat([[eye, eye], [eye, -eye]])
    lo = np.concatenate([np.zeros(n), np.full(n, -np.inf)])
    hi = np.concatenate([np.full(n, np.inf), np.zeros(n)])
    return QPProblem(SparseOperator(P.tocsr()), q, SparseOperator(M.tocsr()), Box(lo, hi))


def qp_lower(qp: QPProblem) -> GenericProblem:
    """problems.py:387-421 (full_rank iff M is the identity)."""
    P, q, box = qp.P, qp.q, qp.box

    @device_fn
    def f(x):
        xt = to_device(x)
        return 0.5 * float(torch.dot(xt, P._apply_dev(xt))) + float(torch.dot(to_device(q), xt))

    @device_fn
    def grad(x):
        xt = to_device(x)
        return like_input(P._apply_dev(xt) + to_device(q), x)

    return GenericProblem(n=qp.n, m=qp.m, f=f, grad_f=grad, hess=ConstantHessian(qp.P),
                          g=device_fn(lambda z: box_indicator(z, box)),
                          prox_g=device_fn(lambda v, rho, tol: box_project(v, box)),
                          M=qp.M, c=np.zeros(qp.m),
                          is_quadratic=True, full_rank=isinstance(qp.M, IdentityOperator), qp=qp)


def ml_lower(p: MLProblem) -> GenericProblem:
    """problems.py:424-450: M = I, c = 0, full rank."""
    return GenericProblem(n=p.n, m=p.n, f=device_fn(lambda x: ml_smooth_value(p, x)),
                          grad_f=device_fn(lambda x: ml_gradient(p, x)), hess=MLHessian(p),
                          g=device_fn(lambda z: p.lambda1 * float(to_device(z).abs().sum())),
                          prox_g=device_fn(lambda v, rho, tol: soft_threshold(v, p.lambda1 / rho)),
                          M=IdentityOperator(p.n), c=np.zeros(p.n),
                          is_quadratic=p.loss.deriv2_constant, full_rank=True, ml=p)


def lower(problem) -> GenericProblem:
    if isinstance(problem, GenericProblem):
        return problem
    if isinstance(problem, QPProblem):
        return qp_lower(problem)
    if isinstance(problem, MLProblem):
        return ml_lower(problem)
    raise DataError(f"cannot solve object of type {type(problem).__name__}")


# ---------------------------------------------------------------------------
# ML oracles on the device (problems.py:227-351).  Single-GPU helpers; the
# solver uses fused, sharded versions of the same kernels.


def _dense_A(p: MLProblem) -> Optional[torch.Tensor]:
    """The data matrix in HBM when A is dense (the GEMV/HVP kernels), else None."""
    return p.A.device_rows() if isinstance(p.A, DenseOperator) else None


def _a_rows(p: MLProblem, X: torch.Tensor) -> torch.Tensor:
    """A X[j] for the k rows of X: one multi-RHS GEMV for dense data, the
    operator's own kernel (CSR SpMV, ...) otherwise."""
    from .kernels import get_kernels

    kx = get_kernels()
    A = _dense_A(p)
    if A is not None:
        Y = kx.empty(X.shape[0], p.N)
        kx.gemv(A, X, Y)
        return Y
    return torch.stack([p.A._apply_dev(X[j].contiguous()) for j in range(X.shape[0])])


def _at_rows(p: MLProblem, T: torch.Tensor) -> torch.Tensor:
    """A^T T[j] for the k rows of T."""
    from .kernels import get_kernels

    kx = get_kernels()
    A = _dense_A(p)
    if A is not None:
        Y = kx.empty(T.shape[0], p.n)
        kx.gemvT(A, T, Y)
        return Y
    return torch.stack([p.A._apply_adjoint_dev(T[j].contiguous()) for j in range(T.shape[0])])


class _MLEval:
    """One pass A{x[,z]} -> row-wise loss epilogue -> A^T{...} on the device."""

    def __init__(self, p: MLProblem):
        from .kernels import get_kernels

        self.p = p
        self.kx = get_kernels()
        self.b = to_device(p.b)
        self.N, self.n = p.N, p.n

    def at(self, x, z=None):
        kx = self.kx
        X = torch.stack([to_device(x)] + ([to_device(z)] if z is not None else [])).contiguous()
        AX = _a_rows(self.p, X)
        tg, w, thx, tnu = (kx.empty(self.N) for _ in range(4))
        out = kx.zeros(8)
        kx.ml_rowwise(_loss_arg(self.p.loss), AX[0], AX[1] if z is not None else None, self.b, tg, w, thx,
                      tnu if z is not None else None, out)
        return AX, tg, w, thx, tnu, out


def ml_smooth_value(p: MLProblem, x) -> float:
    """sum_i l(a_i'x - b_i) + (lambda2/2)||x||^2 (problems.py:227-230)."""
    ev = _MLEval(p)
    _, _, _, _, _, out = ev.at(x)
    xt = to_device(x)
    return float(out[0]) + 0.5 * p.lambda2 * float(torch.dot(xt, xt))


def ml_objective(p: MLProblem, x) -> float:
    return ml_smooth_value(p, x) + p.lambda1 * float(to_device(x).abs().sum())


def ml_gradient(p: MLProblem, x):
    """A' l'(Ax - b) + lambda2 x (problems.py:238-242)."""
    ev = _MLEval(p)
    _, tg, _, _, _, _ = ev.at(x)
    g = _at_rows(p, tg.view(1, -1)).view(-1).contiguous()
    ev.kx.axpby(p.lambda2, to_device(x), 1.0, g)
    return like_input(g, x)


class MLHessian(HessianOperator):
    """A' diag(l''(Ax - b)) A + lambda2 I kept matrix-free (problems.py:245-273);
    the product is the fused HVP kernel K3."""

    def __init__(self, p: MLProblem, x=None):
        super().__init__(p.n)
        self.p = p
        self.diag_shift = p.lambda2
        self.is_constant = p.loss.deriv2_constant
        # nothing touches the device until the operator is used (ml_lower builds
        # one for every lowered problem; the engines have their own fused HVP)
        self._A = None
        self._w = None
        self._x0 = x
        self._started = False

    def _ensure(self) -> None:
        if not self._started:
            self.update(np.zeros(self.p.n) if self._x0 is None else self._x0)

    def update(self, x) -> None:
        if not self._started:
            self._started = True
            self._x0 = None
            self._A = _dense_A(self.p)
        if self.p.loss.kind == "square":
            self._w = None  # l'' == 1
            return
        ev = _MLEval(self.p)
        _, _, w, _, _, _ = ev.at(x)
        self._w = w

    @property
    def _weights(self):
        self._ensure()
        if self._w is None:
            return np.ones(self.p.N)
        return self._w.cpu().numpy()

    def _hvp(self, v, shift):
        from .kernels import get_kernels

        kx = get_kernels()
        self._ensure()
        y = kx.empty(self.input_dim)
        if self._A is not None:
            kx.hvp(self._A, self._w, v, shift, y, None, True)
            return y
        t = self.p.A._apply_dev(v)
        if self._w is not None:
            kx.vmul(1.0, self._w, t, 0.0, t)
        y = self.p.A._apply_adjoint_dev(t)
        if shift != 0.0:
            kx.axpby(shift, v, 1.0, y)
        return y

    def _apply_dev(self, v):
        return self._hvp(v, self.diag_shift)

    def _smooth_cols(self, V):
        from .kernels import get_kernels
        from .operators import adjoint_columns_dev

        kx = get_kernels()
        self._ensure()
        A = self._A
        if A is None:
            Z = self.p.A.apply_columns_dev(V.contiguous())
            if self._w is not None:
                kx.row_scale(Z, self._w)
            return adjoint_columns_dev(self.p.A, Z)
        N, n = A.shape
        s = V.shape[1]
        Z = kx.empty(N, s)
        kx.gemm(0, 0, N, s, n, 1.0, A, A.stride(0), V, V.stride(0), 0.0, Z, s)
        if self._w is not None:
            kx.row_scale(Z, self._w)
        Y = kx.empty(n, s)
        kx.gemm(1, 0, n, s, N, 1.0, A, A.stride(0), Z, s, 0.0, Y, s)
        return Y

    def smooth_part(self) -> LinearOperator:
        """A' diag(w) A, the sketching target (problems.py:266-273)."""

        @device_fn
        def mv(v):
            return self._hvp(to_device(v), 0.0)

        op = MatrixFreeOperator(self.input_dim, self.output_dim, mv, mv)
        op.apply_columns_dev = self._smooth_cols
        return op


def ml_hessian_operator(p: MLProblem, x) -> MLHessian:
    return MLHessian(p, x)


def ml_x_system(p: MLProblem, x, z, u, rho: float, hess: Optional[MLHessian] = None):
    """Matvec and right-hand side of the ML x-update (problems.py:280-303)."""
    if hess is None:
        hess = MLHessian(p, x)

    def matvec(v):
        vt = to_device(v)
        return like_input(hess._apply_dev(vt) + rho * vt, v)

    xt = to_device(x)
    rhs = hess._apply_dev(xt) - to_device(ml_gradient(p, xt)) + rho * (to_device(z) - to_device(u))
    return matvec, like_input(rhs, x)


def ml_dual_point(p: MLProblem, x):
    """nu = l'(Ax - b), scaled into ||A'nu||_inf <= lambda1 when lambda2 == 0
    (problems.py:306-318)."""
    ev = _MLEval(p)
    AX, tg, _, _, _, _ = ev.at(x)
    nu = tg
    if p.lambda2 == 0.0:
        at = _at_rows(p, nu.view(1, -1))
        denom = float(at.abs().max()) if at.numel() else 0.0
        if denom > p.lambda1:
            nu = nu * (p.lambda1 / denom)
    return like_input(nu, x)


def ml_dual_value(p: MLProblem, nu) -> float:
    """Dual objective at nu; -inf outside the conjugate's domain (problems.py:321-332)."""
    from .kernels import get_kernels

    kx = get_kernels()
    nut = to_device(nu)
    b = to_device(p.b)
    out = kx.zeros(4)
    kx.ml_conj_scaled(_loss_arg(p.loss), nut, 1.0, b, out)
    o = out.cpu().numpy()
    if o[1] > 0:
        return -np.inf
    val = -float(o[0]) - float(o[2])
    if p.lambda2 > 0.0:
        at = _at_rows(p, nut.view(1, -1))
        excess = torch.clamp(at.abs() - p.lambda1, min=0.0)
        val -= float(torch.sum(excess * excess)) / (2.0 * p.lambda2)
    return val


def ml_dual_gap(p: MLProblem, x) -> float:
    """(primal - dual) / min(primal, |dual|) (problems.py:335-351)."""
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


def huber_subdiff_distance(p: MLProblem, x) -> float:
    """l2 distance from 0 to the subdifferential of the huber-fit objective
    (problems.py:354-368): the gradient w = A' l'(Ax - b) + lambda2 x comes from
    the device passes; the support split is host arithmetic on n values."""
    if p.loss.kind != "huber":
        raise DataError("subdifferential stopping rule is defined for the huber loss")
    xh = x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x, dtype=float)
    w = ml_gradient(p, xh)
    w = w.detach().cpu().numpy() if isinstance(w, torch.Tensor) else np.asarray(w)
    active = xh != 0.0
    d2 = float(np.sum((w[active] + p.lambda1 * np.sign(xh[active])) ** 2))
    d2 += float(np.sum(np.maximum(np.abs(w[~active]) - p.lambda1, 0.0) ** 2))
    return float(np.sqrt(d2))


def huber_subdiff_stop(tol: float = 1e-4) -> Callable:
    """Termination rule on the sparse iterate z (problems.py:371-384)."""

    def stop(problem: GenericProblem, state) -> bool:
        if problem.ml is None:
            return False
        return huber_subdiff_distance(problem.ml, state.z) <= tol

    return stop

