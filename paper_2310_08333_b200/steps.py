"""The reference's single-step API (``/root/reference/pkg/src/nysopt/admm.py:215-415``):
``compute_residuals``, ``check_termination``, ``x_update``,
``relaxed_constraint_point``, ``z_update``, ``u_update``, ``update_penalty``
and ``check_infeasibility`` -- same names, arguments and return types, so code
(and tests) written against ``nysopt.admm`` runs unchanged.

``solve`` does not call these: its engines run the same steps fused into a few
kernels per iteration (admm.py, general.py).  Here each step is its own call
on a host-side ``SolverState`` of NumPy arrays: the vectors go to the device,
the operator products, the PCG solve, the prox and the norms run there through
the C ABI, and the results come back as NumPy arrays.  There is no CPU path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from .admm import PenaltyEvent, Residuals, SolverOptions, SolverState, Status
from .krylov import CgReport, pcg
from .operators import IdentityOperator, to_device
from .problems import GenericProblem
from .prox import box_recession_distance, box_support
from .sketch import NystromPreconditioner


def _kx():
    from .kernels import get_kernels

    return get_kernels()


def _norm_dev(v: torch.Tensor, kind: str) -> float:
    """l2 or linf norm by the fixed-order reduction kernel of the general engine (nys_vstats_f64)."""
    if v.numel() == 0:
        return 0.0
    kx = _kx()
    out = kx.zeros(3)
    kx.vstats(v.contiguous(), None, out)  # [sum v, sum v^2, max |v|]
    h = out.cpu().numpy()
    return float(h[2]) if kind == "linf" else math.sqrt(max(float(h[1]), 0.0))


def _lin(a: float, x: torch.Tensor, b: float, y: torch.Tensor) -> torch.Tensor:
    """a x + b y as a fresh vector (nys_axpby_f64)."""
    out = y.clone()
    _kx().axpby(a, x.contiguous(), b, out)
    return out


def _np(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def compute_residuals(problem: GenericProblem, state: SolverState, options: SolverOptions) -> Residuals:
    """Primal residual Mx - z - c and dual residual grad f(x) + rho M'u (admm.py:215-224)."""
    x, z, u = to_device(state.x), to_device(state.z), to_device(state.u)
    c = to_device(problem.c)
    Mx = to_device(state.Mx) if state.Mx is not None else problem.M._apply_dev(x)
    rp = _lin(-1.0, c, 1.0, _lin(-1.0, z, 1.0, Mx))
    Mtu = problem.M._apply_adjoint_dev(u)
    rd = _lin(state.rho, Mtu, 1.0, to_device(problem.grad_f(state.x)))
    kind = options.norm_kind
    primal_scale = max(_norm_dev(Mx, kind), _norm_dev(z, kind), _norm_dev(c, kind))
    dual_scale = _norm_dev(_lin(state.rho, Mtu, 0.0, Mtu), kind)
    return Residuals(_np(rp), _np(rd), _norm_dev(rp, kind), _norm_dev(rd, kind), primal_scale, dual_scale,
                     size=int(rp.numel()))


def check_termination(res: Residuals, state: SolverState, options: SolverOptions,
                      gap: Optional[float] = None) -> bool:
    """Mixed absolute / relative residual test, or the duality-gap test (admm.py:227-240)."""
    if gap is not None:
        return gap <= options.eps_dual_gap
    m, n = np.size(state.z), np.size(state.x)
    primal_ok = res.rp_norm <= math.sqrt(m) * options.eps_abs + options.eps_rel * res.primal_scale
    dual_ok = res.rd_norm <= math.sqrt(n) * options.eps_abs + options.eps_rel * res.dual_scale
    return bool(primal_ok and dual_ok)


def x_update(problem: GenericProblem, state: SolverState, options: SolverOptions,
             preconditioner: Optional[NystromPreconditioner], tol: float,
             sigma_eff: float) -> tuple[np.ndarray, CgReport]:
    """The x-subproblem system solved by warm-started PCG on the device (admm.py:243-275):
    (H + rho M'M + sigma I) x = H x_k + sigma x_k - grad f(x_k) + rho M'(z + c - u)."""
    hess, M, rho = problem.hess, problem.M, state.rho
    identity_M = isinstance(M, IdentityOperator)
    shift = rho + sigma_eff

    def matvec(v):
        vt = to_device(v)
        if identity_M:
            return _lin(shift, vt, 1.0, hess._apply_dev(vt))
        y = _lin(rho, M._apply_adjoint_dev(M._apply_dev(vt)), 1.0, hess._apply_dev(vt))
        return _lin(sigma_eff, vt, 1.0, y)

    x = to_device(state.x)
    rhs = _lin(-1.0, to_device(problem.grad_f(state.x)), 1.0, _lin(sigma_eff, x, 1.0, hess._apply_dev(x)))
    target = _lin(-1.0, to_device(state.u), 1.0, _lin(1.0, to_device(problem.c), 1.0, to_device(state.z)))
    rhs = _lin(rho, target if identity_M else M._apply_adjoint_dev(target), 1.0, rhs)
    Minv = preconditioner.apply if preconditioner is not None else None
    x_new, rep = pcg(matvec, rhs, x0=x, Minv=Minv, tol_rel=tol, max_iter=10 * problem.n)
    return _np(to_device(x_new)), rep


def relaxed_constraint_point(Mx_new, state: SolverState, problem: GenericProblem, alpha: float) -> np.ndarray:
    """alpha Mx + (1 - alpha)(z + c) (admm.py:278-280)."""
    zc = _lin(1.0, to_device(problem.c), 1.0, to_device(state.z))
    return _np(_lin(alpha, to_device(Mx_new), 1.0 - alpha, zc))


def z_update(problem: GenericProblem, state: SolverState, options: SolverOptions, w) -> np.ndarray:
    """Proximal step at the over-relaxed point, tolerance tol0 / k^(2 gamma) (admm.py:283-296)."""
    prox_tol = options.prox_tol0 / max(state.k, 1) ** (2.0 * options.gamma)
    v = _lin(1.0, to_device(state.u), 1.0, _lin(-1.0, to_device(problem.c), 1.0, to_device(w)))
    vin = v if isinstance(state.u, torch.Tensor) else _np(v)  # the prox sees the caller's array kind
    return _np(to_device(problem.prox_g(vin, state.rho, max(prox_tol, 1e-15))))


def u_update(state: SolverState, w, z_new, problem: GenericProblem) -> np.ndarray:
    """u + w - z_new - c (admm.py:299-300)."""
    uw = _lin(1.0, to_device(w), 1.0, to_device(state.u))
    return _np(_lin(-1.0, to_device(problem.c), 1.0, _lin(-1.0, to_device(z_new), 1.0, uw)))


def _change_penalty(state: SolverState, rho_new: float, preconditioner: Optional[NystromPreconditioner] = None,
                    nu_of_rho: Optional[Callable[[float], float]] = None) -> PenaltyEvent:
    """New penalty with the scaled dual rescaled so that rho u is unchanged (admm.py:303-320)."""
    rho_old = state.rho
    kx = _kx()
    u_new = to_device(state.u).clone()
    out = kx.zeros(2)
    kx.scale_dual(u_new, rho_old, rho_new, out)  # u *= rho_old / rho_new; [||y_old||^2, ||y_new - y_old||^2]
    o = out.cpu().numpy()
    denom = max(math.sqrt(max(float(o[0]), 0.0)), 1e-30)
    jump = math.sqrt(max(float(o[1]), 0.0)) / denom
    if isinstance(state.u, np.ndarray):
        state.u[...] = _np(u_new)  # in place, as the reference's `state.u *= ...`
    else:
        state.u = u_new
    state.rho = rho_new
    if preconditioner is not None and nu_of_rho is not None:
        preconditioner.update_shift(nu_of_rho(rho_new))
    return PenaltyEvent(state.k, rho_old, rho_new, jump)


def update_penalty(state: SolverState, res: Residuals, options: SolverOptions,
                   preconditioner: Optional[NystromPreconditioner] = None,
                   nu_of_rho: Optional[Callable[[float], float]] = None) -> Optional[PenaltyEvent]:
    """Balanced-residual rule (admm.py:323-350): each residual is measured against
    its own termination threshold; tau up when the primal one dominates by mu,
    tau down in the mirror case, else no change (None)."""
    np_size = res.rp.size if res.rp is not None else res.size
    nd_size = res.rd.size if res.rd is not None else np.size(state.x)
    t_p = math.sqrt(np_size) * options.eps_abs + options.eps_rel * res.primal_scale
    t_d = math.sqrt(nd_size) * options.eps_abs + options.eps_rel * res.dual_scale
    if t_p > 0 and t_d > 0:
        p_meas, d_meas = res.rp_norm / t_p, res.rd_norm / t_d
    else:
        p_meas, d_meas = res.rp_norm, res.rd_norm
    if p_meas > options.mu * d_meas:
        rho_new = state.rho * options.tau
    elif d_meas > options.mu * p_meas:
        rho_new = state.rho / options.tau
    else:
        return None
    return _change_penalty(state, rho_new, preconditioner, nu_of_rho)


@dataclass
class InfeasibilityCheck:
    status: Optional[Status]
    certificate_primal: Optional[np.ndarray]
    certificate_dual: Optional[np.ndarray]
    near_trigger: bool


def check_infeasibility(delta_x, delta_u, problem: GenericProblem, options: SolverOptions,
                        rho: float) -> InfeasibilityCheck:
    """Approximate certificate tests on the iterate differences (admm.py:361-415);
    box-constrained QPs only.  Primal: M'du and the box support at du vanish
    relative to du.  Dual: P dx, the recession-cone distance of M dx vanish
    relative to dx and q'dx is (nearly) negative."""
    qp = problem.qp
    if qp is None:
        return InfeasibilityCheck(None, None, None, False)
    eps = options.eps_inf
    primal = dual = near_primal = near_dual = False
    cert_p = cert_d = None
    du, dx = to_device(delta_u), to_device(delta_x)

    du_norm = _norm_dev(du, "l2")
    if du_norm > 1e-14:
        t_map = _norm_dev(qp.M._apply_adjoint_dev(du), "l2")
        t_support = box_support(du, qp.box)
        primal = t_map < eps * du_norm and t_support < eps * du_norm
        near_primal = t_map < 10 * eps * du_norm and t_support < 10 * eps * du_norm
        if primal:
            cert_p = rho * _np(du)

    dx_norm = _norm_dev(dx, "l2")
    if dx_norm > 1e-14:
        s_obj = _norm_dev(qp.P._apply_dev(dx), "l2")
        s_cone = box_recession_distance(qp.M._apply_dev(dx), qp.box)
        lin = _kx().zeros(1)
        _kx().dot(to_device(qp.q).contiguous(), dx.contiguous(), lin)
        s_lin = float(lin)
        dual = s_obj < eps * dx_norm and s_cone < eps * dx_norm and s_lin < eps * dx_norm
        near_dual = s_obj < 10 * eps * dx_norm and s_cone < 10 * eps * dx_norm and s_lin < 10 * eps * dx_norm
        if dual:
            cert_d = _np(dx).copy()

    if primal and dual:
        status = Status.PRIMAL_AND_DUAL_INFEASIBLE
    elif primal:
        status = Status.PRIMAL_INFEASIBLE
    elif dual:
        status = Status.DUAL_INFEASIBLE
    else:
        status = None
    return InfeasibilityCheck(status, cert_p, cert_d, near_primal or near_dual)
