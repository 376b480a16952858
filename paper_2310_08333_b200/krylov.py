"""Preconditioned conjugate gradient on the device
(``/root/reference/pkg/src/nysopt/krylov.py:35-112``).

The iteration runs entirely on the GPU: the matvec is the fused HVP (K3) or a
dense GEMV, the preconditioner is K6, the vector updates are the fused K7
kernels with device-resident alpha/beta.  The host reads back ONE 64-byte
scalar block per iteration to take the reference's exact stopping decision
(recurrence residual, true-residual refresh every 50, SPD and finiteness
checks), so iteration counts follow the reference step for step.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from . import _lib
from .errors import NotSPDError, NumericalError
from .operators import LinearOperator, like_input, to_device

TOL_FLOOR = 1e-12
_RESIDUAL_REFRESH = 50  # krylov.py:16


@dataclass
class CgReport:
    iterations: int
    final_relative_residual: float
    converged: bool


def cg_tolerance(k: int, rp_norm: float, rd_norm: float, gamma: float = 1.2) -> float:
    """min(sqrt(rp rd), 1) / k^gamma floored at 1e-12 (krylov.py:98-112)."""
    if k < 1:
        raise ValueError("iteration index must be >= 1")
    if rp_norm < 0 or rd_norm < 0:
        raise ValueError("residual norms must be nonnegative")
    if gamma <= 1:
        raise ValueError("gamma must exceed 1 for summability")
    tol = min(np.sqrt(rp_norm * rd_norm), 1.0) / k**gamma
    return max(tol, TOL_FLOOR)


class CgWork:
    """Device buffers of one PCG solve (reused across ADMM iterations)."""

    def __init__(self, kx, n: int, sc: Optional[torch.Tensor] = None):
        self.kx = kx
        self.n = n
        self.r = kx.empty(n)
        self.p = kx.empty(n)
        self.z = kx.empty(n)
        self.Ap = kx.empty(n)
        # slot 7 holds a kernel ticket: keep zero
        self.sc = kx.zeros(_lib.CG_NSLOTS) if sc is None else sc
        self.host = torch.zeros(_lib.CG_NSLOTS, dtype=torch.float64)
        if kx.device.type == "cuda":
            self.host = self.host.pin_memory()

    def slot(self, i: int) -> torch.Tensor:
        return self.sc[i:i + 1]

    def read(self) -> np.ndarray:
        self.host.copy_(self.sc, non_blocking=True)
        self.kx.d2h += self.host.numel() * 8
        self.kx.sync()
        return self.host.numpy()


MatvecInto = Callable[[torch.Tensor, torch.Tensor, Optional[torch.Tensor]], None]
PrecondInto = Callable[[torch.Tensor, torch.Tensor, Optional[torch.Tensor], Optional[torch.Tensor]], None]


def pcg_device(work: CgWork, matvec: MatvecInto, b: torch.Tensor, x: torch.Tensor,
               precond: Optional[PrecondInto], tol_rel: float, max_iter: int,
               started: bool = False) -> CgReport:
    """krylov.py:35-95 on device buffers; ``x`` is updated in place.

    ``matvec(v, out, dot)`` writes out = A v and, when ``dot`` is given, the
    device scalar v.out.  ``precond(v, out, rdot, rz)`` writes out = M^-1 v and
    rz = rdot.out.  With ``started`` the caller has already produced
    r = b - A x0 and the ||b||^2, ||r||^2 slots (the fused ADMM rhs kernel)."""
    kx = work.kx
    r, p, z, Ap, sc = work.r, work.p, work.z, work.Ap, work.sc
    if not started:
        matvec(x, Ap, None)
        kx.cg_start(b, Ap, r, sc)
    h = work.read()
    b_norm = math.sqrt(h[_lib.CG_B2])
    denom = b_norm if b_norm > 0 else 1.0
    res = math.sqrt(h[_lib.CG_RES2])
    if res <= tol_rel * denom:
        return CgReport(0, res / denom, True)

    def precondition():
        if precond is None:
            kx.precond_apply(None, None, 1.0, r, z, r, work.slot(_lib.CG_RZNEW))
        else:
            precond(r, z, r, work.slot(_lib.CG_RZNEW))

    precondition()
    kx.cg_dir(z, p, True, sc)
    k = 0
    for k in range(1, max_iter + 1):
        matvec(p, Ap, work.slot(_lib.CG_PAP))
        refresh = k % _RESIDUAL_REFRESH == 0
        kx.cg_step_xr(x, r, p, Ap, refresh, sc)
        if refresh:
            matvec(x, Ap, None)
            kx.cg_start(b, Ap, r, sc)
        h = work.read()
        flag = h[_lib.CG_FLAG]
        if flag == 1.0:
            raise NumericalError("non-finite value in conjugate gradient")
        if flag == 2.0:
            raise NotSPDError(f"nonpositive curvature p'Ap = {h[_lib.CG_PAP]:.3e}; operator is not SPD")
        res = math.sqrt(h[_lib.CG_RES2]) if h[_lib.CG_RES2] >= 0 else float("nan")
        if not math.isfinite(res):
            raise NumericalError("non-finite residual in conjugate gradient")
        if res <= tol_rel * denom:
            return CgReport(k, res / denom, True)
        precondition()
        kx.cg_dir(z, p, False, sc)
    return CgReport(k, res / denom, False)


def pcg_batched(work: CgWork, pb, max_iter: int, first_batch: int = 2, max_batch: int = 16) -> CgReport:
    """krylov.py:35-95 with the stop test on the device (nys_cg_iterate_f64).

    Launches batches of predicated iterations and reads the scalar block once
    per batch; the iteration sequence and the stopping decision are the
    reference's, only the number of host round trips changes.  The caller has
    set B2 / RES2 for r = b - A x0 (``started`` form of ``pcg_device``)."""
    kx = work.kx
    k = 1
    batch = max(1, first_batch)
    while True:
        kx.cg_iterate(pb, k, batch)
        h = work.read()
        done = int(h[_lib.CG_DONE])
        if done or k + batch > max_iter:
            break
        k += batch
        batch = min(max_batch, batch * 2)
    iters = int(h[_lib.CG_ITERS])
    resrel = float(h[_lib.CG_RESREL])
    if done == 2:
        raise NumericalError("non-finite value in conjugate gradient")
    if done == 3:
        raise NotSPDError(f"nonpositive curvature p'Ap = {h[_lib.CG_PAP]:.3e}; operator is not SPD")
    if done == 1:
        return CgReport(iters, resrel, True)
    return CgReport(iters if done == 4 else max_iter, resrel, False)


def _matvec_for(A, host_io: bool = False) -> MatvecInto:
    from .kernels import get_kernels

    kx = get_kernels()
    if isinstance(A, LinearOperator):
        from .operators import DenseOperator

        if isinstance(A, DenseOperator):
            M = A.device_rows()

            def mv(v, out, dot):
                kx.gemv(M, v.view(1, -1), out.view(1, -1))
                if dot is not None:
                    kx.shift_dot(v, 0.0, out, dot)

            return mv
        f = A._apply_dev
    elif host_io:
        # a caller working in NumPy hands in NumPy callables (krylov.py:35-44): its
        # own code runs on the host, the CG vectors and reductions stay on the device
        f = lambda v: to_device(np.asarray(A(v.cpu().numpy()), dtype=float))
    else:
        f = lambda v: to_device(A(v))

    def mv(v, out, dot):
        out.copy_(f(v))
        if dot is not None:
            kx.dot(v, out, dot)

    return mv


def _precond_for(Minv, host_io: bool = False) -> Optional[PrecondInto]:
    if Minv is None:
        return None
    from .kernels import get_kernels
    from .sketch import NystromPreconditioner

    kx = get_kernels()
    owner = getattr(Minv, "__self__", None)
    if isinstance(Minv, NystromPreconditioner) or isinstance(owner, NystromPreconditioner):
        pc = Minv if isinstance(Minv, NystromPreconditioner) else owner
        return lambda v, out, rdot, rz: pc.apply_into(kx, v, out, rdot, rz)

    def pre(v, out, rdot, rz):
        out.copy_(to_device(np.asarray(Minv(v.cpu().numpy()), dtype=float)) if host_io else to_device(Minv(v)))
        if rz is not None:
            kx.dot(rdot, out, rz)

    return pre


def pcg(A, b, x0=None, Minv=None, tol_rel: float = 1e-8, max_iter: Optional[int] = None):
    """Solve A x = b for SPD A (krylov.py:35-95).  ``A`` is a LinearOperator
    or a callable on CUDA tensors; ``Minv`` a NystromPreconditioner (or its
    ``apply``) or a callable.  NumPy ``b`` gives a NumPy solution."""
    from .kernels import get_kernels

    kx = get_kernels()
    bt = to_device(b)
    n = bt.numel()
    if max_iter is None:
        max_iter = 10 * n
    x = torch.zeros_like(bt) if x0 is None else to_device(x0).clone()
    work = CgWork(kx, n)
    host_io = not isinstance(b, torch.Tensor)
    rep = pcg_device(work, _matvec_for(A, host_io), bt, x, _precond_for(Minv, host_io), tol_rel, max_iter)
    return like_input(x, b), rep
