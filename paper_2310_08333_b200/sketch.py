"""Randomized Nystrom sketch and preconditioner on the device
(``/root/reference/pkg/src/nysopt/sketch.py:29-165``).

Pipeline of ``sketch_device`` (K5):
  raw Omega = default_rng(seed).standard_normal((n, s))   -- host, the SAME
      array the reference draws (sketch.py:97-98), uploaded once;
  Q = CholeskyQR2(Omega)                                  -- same range as the
      reference's Householder Q (the sketch is basis-invariant);
  Y = target(Q) as GEMMs on the DMMA path (A^T(w o AQ) or P Q), all-reduced
      across row shards;
  shift / core / Cholesky (eigh fallback) / B / thin SVD / truncation
      -- nys_nystrom_core_f64, all on the GPU.
"""

from __future__ import annotations

import math
import time
from typing import Callable, Optional

import numpy as np
import torch

from .errors import DataError
from .operators import LinearOperator, like_input, to_device


def default_sketch_rank(n: int) -> int:
    """min(50, ceil(n/20)), at least 1 (sketch.py:29-31)."""
    return max(1, min(50, math.ceil(n / 20)))


def sketch_width(n: int, r: int, oversample: Optional[int] = None) -> int:
    """s = min(n, r + 8 + r//4) (sketch.py:93-95)."""
    if oversample is None:
        oversample = 8 + r // 4
    return min(n, r + max(oversample, 0))


def raw_test_matrix(n: int, s: int, seed: int) -> np.ndarray:
    """The reference's Gaussian test matrix before orthonormalisation."""
    return np.random.default_rng(seed).standard_normal((n, s))


def upload_pinned(a: np.ndarray, device=None) -> torch.Tensor:
    host = torch.from_numpy(np.ascontiguousarray(a))
    try:
        host = host.pin_memory()
    except RuntimeError:  # pragma: no cover - pinning can fail under memory pressure
        pass
    return host.to(device or torch.device("cuda", torch.cuda.current_device()), non_blocking=True)


def sketch_device(kx, apply_cols: Callable[[torch.Tensor], torch.Tensor], n: int, r: int, seed: int,
                  oversample: Optional[int] = None, omega: Optional[np.ndarray] = None,
                  reduce: Optional[Callable[[torch.Tensor], None]] = None):
    """nystrom_sketch (sketch.py:74-128) on the GPU; returns (U, lam) device
    tensors with U of shape n x rank (rank <= r; 0 for an empty sketch)."""
    if not 1 <= r <= n:
        raise DataError(f"sketch rank must satisfy 1 <= r <= {n}, got {r}")
    s = sketch_width(n, r, oversample)
    trace = _TRACE is not None
    t = [time.perf_counter()] if trace else None

    def mark():
        if trace:
            kx.sync()
            t.append(time.perf_counter())

    if omega is None and not trace and hasattr(kx, "gaussian_async") and reduce is None:
        # pipelined: no host synchronisation inside the sketch, one status read
        # at the end; a flagged failure (draw buffer short, singular Gram or core
        # pivot) re-runs the synchronous path from the same seed
        flags = torch.zeros(4, dtype=torch.int32, device=kx.device)
        Om = kx.empty(n, s)
        kx.gaussian_async(seed, Om, flags[0:1])
        Q = kx.empty(n, s)
        kx.orthonormalize_async(Om, Q, flags[1:3], r)
        Y = apply_cols(Q).contiguous()
        U = kx.empty(n, r)
        lam = kx.empty(r)
        kx.nystrom_core_async(Q, Y, U, lam, r, flags[3:4])
        if not bool(flags.any().item()):
            kx.d2h += 16
            return U, lam
    if omega is None:
        # the reference's default_rng(seed).standard_normal((n, s)), drawn on the GPU
        Om = kx.empty(n, s)
        kx.gaussian(seed, Om)
    else:
        Om = upload_pinned(omega, kx.device)
        kx.h2d += omega.nbytes
    mark()
    Q = kx.empty(n, s)
    kx.orthonormalize(Om, Q)
    mark()
    Y = apply_cols(Q).contiguous()
    if reduce is not None:
        reduce(Y)
    mark()
    U = kx.empty(n, r)
    lam = kx.empty(r)
    rr = kx.nystrom_core(Q, Y, U, lam, r)
    mark()
    if trace:
        d = np.diff(t) * 1e3
        _TRACE.append({"gauss_ms": d[0], "ortho_ms": d[1], "target_ms": d[2], "core_ms": d[3]})
    return U[:, :rr], lam[:rr]


class SketchLaunch:
    """A pipelined sketch enqueued on the stream with no host synchronisation:
    its status words are copied to pinned host memory behind an event, so the
    host can queue more work before it looks (`ok()` waits for the sketch only)."""

    def __init__(self, U, lam, flags_h, event, seed):
        self.U, self.lam, self.flags_h, self.event, self.seed = U, lam, flags_h, event, seed

    def ok(self) -> bool:
        self.event.synchronize()
        if _FORCE_FLAG and _FORCE_FLAG.pop():
            return False  # test hook: exercise the recovery path
        return not bool(self.flags_h.any())


# test hook: a list of booleans; each launched sketch's status check pops one and
# reports a failure when it is True (tests/test_gpu_solve.py)
_FORCE_FLAG: list = []


def sketch_device_launch(kx, apply_cols: Callable[[torch.Tensor], torch.Tensor], n: int, r: int, seed: int,
                         oversample: Optional[int] = None) -> Optional[SketchLaunch]:
    """The pipelined branch of ``sketch_device`` without its final status read
    (None where the pipelined path does not apply).  A flagged launch must be
    replaced by the synchronous ``sketch_device`` (same seed)."""
    if not (1 <= r <= n) or _TRACE is not None or not hasattr(kx, "gaussian_async"):
        return None
    s = sketch_width(n, r, oversample)
    flags = torch.zeros(4, dtype=torch.int32, device=kx.device)
    Om = kx.empty(n, s)
    kx.gaussian_async(seed, Om, flags[0:1])
    Q = kx.empty(n, s)
    kx.orthonormalize_async(Om, Q, flags[1:3], r)
    Y = apply_cols(Q).contiguous()
    U = kx.empty(n, r)
    lam = kx.empty(r)
    kx.nystrom_core_async(Q, Y, U, lam, r, flags[3:4])
    flags_h = torch.empty(4, dtype=torch.int32, pin_memory=True)
    flags_h.copy_(flags, non_blocking=True)
    kx.d2h += 16
    ev = torch.cuda.Event()
    ev.record(kx.stream)
    return SketchLaunch(U, lam, flags_h, ev, seed)


# development instrumentation: set to a list to collect per-stage sketch times
_TRACE: Optional[list] = None


class NystromSketch:
    """U diag(lambda_hat) U^T with orthonormal U (sketch.py:34-67).  Holds the
    factors in HBM; ``U`` / ``lambda_hat`` give NumPy copies like the reference."""

    def __init__(self, U, lambda_hat):
        self._n = int(U.shape[0])
        self._r = int(U.shape[1])
        self.U_dev = to_device(U) if self._r > 0 else None
        self.lam_dev = to_device(lambda_hat) if self._r > 0 else None
        self._U_host = None
        self._lam_host = None

    @property
    def U(self) -> np.ndarray:
        if self._U_host is None:
            self._U_host = np.zeros((self._n, 0)) if self._r == 0 else self.U_dev.cpu().numpy()
        return self._U_host

    @property
    def lambda_hat(self) -> np.ndarray:
        if self._lam_host is None:
            self._lam_host = np.zeros(0) if self._r == 0 else self.lam_dev.cpu().numpy()
        return self._lam_host

    @property
    def n(self) -> int:
        return self._n

    @property
    def rank(self) -> int:
        return self._r

    @classmethod
    def empty(cls, n: int) -> "NystromSketch":
        return cls(np.zeros((n, 0)), np.zeros(0))

    def approx_apply_dev(self, v: torch.Tensor) -> torch.Tensor:
        """U diag(lambda) U^T v (sketch.py:53-58): two skinny GEMVs + one scaling."""
        from .kernels import get_kernels

        kx = get_kernels()
        if self.rank == 0:
            return kx.zeros(self._n)
        h = kx.empty(1, self._r)
        kx.gemvT(self.U_dev, v.view(1, -1), h)  # U^T v
        kx.vmul(1.0, self.lam_dev, h.view(-1), 0.0, h.view(-1))
        y = kx.empty(1, self._n)
        kx.gemv(self.U_dev, h, y)
        return y.view(-1)

    def approx_apply(self, v):
        return like_input(self.approx_apply_dev(to_device(v)), v)

    def to_dense(self) -> np.ndarray:
        return (self.U * self.lambda_hat) @ self.U.T


def _operator_columns_dev(A: LinearOperator):
    return A.apply_columns_dev


def nystrom_sketch(A: LinearOperator, r: int, rng_seed: int, oversample: Optional[int] = None) -> NystromSketch:
    """Randomized Nystrom approximation of a symmetric PSD operator
    (sketch.py:74-128); deterministic for a fixed seed."""
    from .kernels import get_kernels

    n = A.input_dim
    if A.output_dim != n:
        raise DataError("nystrom_sketch requires a square operator")
    if not 1 <= r <= n:
        raise DataError(f"sketch rank must satisfy 1 <= r <= {n}, got {r}")
    U, lam = sketch_device(get_kernels(), _operator_columns_dev(A), n, r, rng_seed, oversample)
    if U.shape[1] == 0:
        return NystromSketch.empty(n)
    return NystromSketch(U, lam)


class NystromPreconditioner:
    """Factored inverse preconditioner for A + nu I (sketch.py:131-165):
    L^-1 = (lam_r + nu) U (diag(lam) + nu I)^-1 U^T + I - U U^T."""

    def __init__(self, sketch: NystromSketch, nu: float):
        if nu <= 0:
            raise DataError("preconditioner shift must be positive")
        self.sketch = sketch
        self.nu = float(nu)

    def apply_into(self, kx, v, out, rdot=None, rz=None) -> None:
        S = self.sketch
        if S.rank == 0:
            kx.precond_apply(None, None, self.nu, v, out, rdot, rz)
        else:
            kx.precond_apply(S.U_dev, S.lam_dev, self.nu, v, out, rdot, rz)

    def apply(self, v):
        from .kernels import get_kernels

        vt = to_device(v)
        out = torch.empty_like(vt)
        self.apply_into(get_kernels(), vt, out)
        return like_input(out, v)

    def update_shift(self, nu_new: float) -> None:
        if nu_new <= 0:
            raise DataError("preconditioner shift must be positive")
        self.nu = float(nu_new)

    def to_dense(self) -> np.ndarray:
        S = self.sketch
        n = S.n
        if S.rank == 0:
            return np.eye(n)
        inner = np.diag((S.lambda_hat[-1] + self.nu) / (S.lambda_hat + self.nu))
        return S.U @ inner @ S.U.T + np.eye(n) - S.U @ S.U.T


def precond_apply(P: NystromPreconditioner, v):
    return P.apply(v)


def update_shift(P: NystromPreconditioner, nu_new: float) -> None:
    P.update_shift(nu_new)


# ---------------------------------------------------------------------------
# Adaptive sizing and spectrum probes (sketch.py:176-306), on the device: every
# operator apply, norm and reorthogonalisation is a libnysgpu kernel; the host
# keeps the scalar recurrences (the reference's Python floats).


def _unit_gaussian(kx, n: int, seed: int) -> torch.Tensor:
    """default_rng(seed).standard_normal(n) drawn on the GPU, scaled to unit norm."""
    v = kx.empty(n)
    kx.gaussian(seed, v)
    st = kx.zeros(3)
    kx.vstats(v, None, st)
    nrm = math.sqrt(max(float(st[1]), 0.0))
    kx.axpby(0.0, v, 1.0 / nrm, v)
    return v


def estimate_error_norm(A: LinearOperator, S: NystromSketch, iters: int, rng_seed: int) -> float:
    """Power-method estimate of ||A - A_hat||_2 (sketch.py:176-195)."""
    from .kernels import get_kernels

    if iters < 1:
        raise DataError("estimate_error_norm requires iters >= 1")
    kx = get_kernels()
    n = A.input_dim
    v = _unit_gaussian(kx, n, rng_seed)
    est = 0.0
    st = kx.zeros(3)
    for _ in range(iters):
        w = A._apply_dev(v)
        kx.axpby(-1.0, S.approx_apply_dev(v), 1.0, w)
        kx.vstats(w, None, st)
        est = math.sqrt(max(float(st[1]), 0.0)) if math.isfinite(float(st[1])) else float(st[1])
        if est <= 0.0 or not np.isfinite(est):
            return max(est, 0.0)
        kx.axpby(0.0, w, 1.0 / est, w)
        v = w
    return est


def condition_bound(sketch: NystromSketch, err_norm: float, nu: float) -> float:
    """1 + (lam_r + ||E||) / nu, an upper bound on the preconditioned condition
    number (sketch.py:198-201)."""
    tail = float(sketch.lambda_hat[-1]) if sketch.rank > 0 else 0.0
    return 1.0 + (tail + err_norm) / nu


def adaptive_sketch(A: LinearOperator, r0: int, r_max: int, nu: float, kappa_target: float, rng_seed: int,
                    power_iters: int = 10) -> NystromSketch:
    """Doubling-rank sketch until the condition bound meets kappa_target
    (sketch.py:204-237); the seeds follow the reference's SeedSequence."""
    n = A.input_dim
    if not 1 <= r0 <= r_max <= n:
        raise DataError("adaptive_sketch requires 1 <= r0 <= r_max <= n")
    ranks = []
    r = r0
    while r < r_max:
        ranks.append(r)
        r *= 2
    ranks.append(r_max)
    seeds = np.random.SeedSequence(rng_seed).generate_state(2 * len(ranks))
    sketch = None
    for i, rank in enumerate(ranks):
        sketch = nystrom_sketch(A, rank, int(seeds[2 * i]))
        err = estimate_error_norm(A, sketch, power_iters, int(seeds[2 * i + 1]))
        if condition_bound(sketch, err, nu) <= kappa_target:
            return sketch
    return sketch


def estimate_extreme_eigs(A: LinearOperator, iters: int, rng_seed: int):
    """Extreme Ritz values (lambda_max, lambda_min) of a symmetric operator by
    Lanczos with full reorthogonalisation, twice (sketch.py:240-282).  The Lanczos
    basis lives in HBM as rows of Q; the projections Q w and Q^T h are GEMV
    kernels, the tridiagonal eigenvalues come from the device eigensolver."""
    from .kernels import get_kernels

    if iters < 2:
        raise DataError("estimate_extreme_eigs requires iters >= 2")
    kx = get_kernels()
    n = A.input_dim
    iters = min(iters, n)
    Q = kx.zeros(iters, n)
    Q[0].copy_(_unit_gaussian(kx, n, rng_seed))
    alphas: list = []
    betas: list = []
    scale = 0.0
    st = kx.zeros(4)
    for j in range(iters):
        qj = Q[j]
        w = A._apply_dev(qj).contiguous()
        kx.dot(qj, w, st[0:1])
        alpha = float(st[0])
        alphas.append(alpha)
        scale = max(scale, abs(alpha))
        kx.axpby(-alpha, qj, 1.0, w)
        if j > 0:
            kx.axpby(-betas[-1], Q[j - 1], 1.0, w)
        for _ in range(2):  # full reorthogonalisation, twice
            h = kx.empty(1, j + 1)
            kx.gemv(Q[:j + 1], w.view(1, -1), h)  # Q_j^T w  (Q stored by rows)
            c = kx.empty(1, n)
            kx.gemvT(Q[:j + 1], h, c)
            kx.axpby(-1.0, c.view(-1), 1.0, w)
        kx.vstats(w, None, st[1:4])
        beta = math.sqrt(max(float(st[2]), 0.0))
        if j == iters - 1 or beta <= 1e-12 * max(scale, 1.0):
            break
        betas.append(beta)
        kx.axpby(0.0, w, 1.0 / beta, w)
        Q[j + 1].copy_(w)
    k = len(alphas)
    if k == 1:
        return alphas[0], alphas[0]
    T = np.diag(alphas)
    T += np.diag(betas[:k - 1], 1) + np.diag(betas[:k - 1], -1)
    Td = to_device(T)
    V = kx.empty(k, k)
    lam = kx.empty(k)
    kx.syevj(Td, V, lam)  # descending
    ritz = lam.cpu().numpy()
    return float(ritz[0]), float(ritz[-1])


def diagonal_reduce(A: LinearOperator, d):
    """(D^{-1/2} A D^{-1/2}, d^{-1/2}) for the unit-shift form of (A + diag(d)) w = b
    (sketch.py:285-306)."""
    from .kernels import get_kernels
    from .operators import MatrixFreeOperator

    dh = np.asarray(d.detach().cpu().numpy() if isinstance(d, torch.Tensor) else d, dtype=float)
    if dh.size != A.input_dim:
        raise DataError("diagonal length must match the operator dimension")
    if np.any(dh <= 0):
        raise DataError("diagonal_reduce requires strictly positive d")
    s_dev = torch.rsqrt(to_device(dh))

    def matvec(v, _A=A, _s=s_dev):
        kx = get_kernels()
        t = kx.empty(_A.input_dim)
        kx.vmul(1.0, _s, to_device(v), 0.0, t)
        y = _A._apply_dev(t)
        kx.vmul(1.0, _s, y, 0.0, y)
        return y

    matvec.accepts_device = True  # operators.device_fn
    return MatrixFreeOperator(A.input_dim, A.input_dim, matvec, matvec), like_input(s_dev, d)
