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

    def approx_apply(self, v):
        vt = to_device(v)
        if self.rank == 0:
            return like_input(torch.zeros_like(vt), v)
        return like_input(self.U_dev @ (self.lam_dev * (self.U_dev.T @ vt)), v)

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
