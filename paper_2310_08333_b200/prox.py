"""Proximal operators used by the hot path (``/root/reference/pkg/src/nysopt/prox.py``).

``soft_threshold`` (prox.py:38-43) and ``box_project`` (prox.py:46-48) run the
sm_100a elementwise kernels; inside ``solve`` they are fused into the single
ADMM elementwise kernel (K8).  ``Box`` keeps the reference's validation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import DataError
from .operators import like_input, to_device


@dataclass(frozen=True)
class Box:
    """Hyperrectangle [l, u]; entries of l may be -inf and of u +inf (prox.py:16-35)."""

    l: np.ndarray
    u: np.ndarray

    def __post_init__(self):
        l = np.asarray(self.l, dtype=float)
        u = np.asarray(self.u, dtype=float)
        if l.shape != u.shape:
            raise DataError("box bounds must have matching shapes")
        if np.any(l > u):
            raise DataError("box requires l <= u elementwise")
        object.__setattr__(self, "l", l)
        object.__setattr__(self, "u", u)

    @property
    def dim(self) -> int:
        return self.l.size


def soft_threshold(v, kappa: float):
    """Elementwise sign(v) * max(|v| - kappa, 0); kappa >= 0."""
    if kappa < 0:
        raise DataError("soft_threshold requires kappa >= 0")
    from .kernels import get_kernels

    vt = to_device(v)
    out = torch.empty_like(vt)
    get_kernels().soft_threshold(vt, kappa, out)
    return like_input(out, v)


def box_project(v, box: Box):
    """Clamp v into [l, u]."""
    from .kernels import get_kernels

    vt = to_device(v)
    out = torch.empty_like(vt)
    get_kernels().box_project(vt, to_device(box.l), to_device(box.u), out)
    return like_input(out, v)


def box_indicator(z, box: Box, tol: float = 1e-9) -> float:
    """0 if z lies in [l, u] within tol * (1 + max|z|), else +inf (prox.py:138-144)."""
    zt = to_device(z)
    scale = 1.0 + (float(zt.abs().max()) if zt.numel() else 0.0)
    lo, hi = to_device(box.l), to_device(box.u)
    ok = bool(torch.all(zt >= lo - tol * scale)) and bool(torch.all(zt <= hi + tol * scale))
    return 0.0 if ok else np.inf


def _numel(v) -> int:
    return int(v.numel()) if isinstance(v, torch.Tensor) else int(np.size(v))


def _box_cert(du, md, box: Box):
    """[sum_{y>0} u y, sum_{y<0} l y, #(inf x nonzero), ||md - cone(md)||^2] from
    the certificate kernel of the general engine (csrc/general.cu)."""
    from .kernels import get_kernels

    kx = get_kernels()
    out = kx.zeros(4)
    kx.box_cert(None if du is None else to_device(du).contiguous(), None if md is None else to_device(md).contiguous(),
                to_device(box.l), to_device(box.u), out)
    return out.cpu().numpy()


def box_support(y, box: Box) -> float:
    """Support function of [l, u]: sum_i u_i (y_i)_+ - l_i (-y_i)_+ (prox.py:96-110);
    a zero y_i contributes 0 whatever the bound, an infinite bound against a
    nonzero y_i of that sign makes the value +inf."""
    if _numel(y) == 0:
        return 0.0
    h = _box_cert(y, None, box)
    return float(np.inf) if h[2] > 0 else float((0.0 + h[0]) + h[1])


def box_recession_project(y, box: Box):
    """Coordinatewise projection onto the recession cone of [l, u] (prox.py:113-129):
    0 where both bounds are finite, y_+ / y_- where only one is, y where none."""
    yt = to_device(y)
    lo, hi = to_device(box.l), to_device(box.u)
    lf, uf = torch.isfinite(lo), torch.isfinite(hi)
    out = torch.where(lf & uf, torch.zeros_like(yt),
                      torch.where(lf, yt.clamp_min(0.0), torch.where(uf, yt.clamp_max(0.0), yt)))
    return like_input(out, y)


def box_recession_distance(y, box: Box) -> float:
    """l2 distance from y to the recession cone of [l, u] (prox.py:132-135)."""
    if _numel(y) == 0:
        return 0.0
    return float(np.sqrt(max(_box_cert(None, y, box)[3], 0.0)))


def simplex_project(v, tol: float = 1e-8):
    """Projection onto the probability simplex (prox.py:51-93): bisection on the
    threshold nu of sum (v - nu)_+ = 1 in [-max|v| - 1, max|v|], then the closed
    form for the active set the bisection identified when it is self-consistent.
    (Off the solver's hot path: the simplex prox belongs to the generic front
    end; elementwise device ops, the excess evaluated on the device.)"""
    if _numel(v) < 1:
        raise DataError("simplex_project requires a nonempty vector")
    if tol <= 0:
        raise DataError("simplex_project requires tol > 0")
    vt = to_device(v).to(torch.float64)
    if bool(torch.all(vt >= 0)) and abs(float(vt.sum()) - 1.0) <= tol:
        return like_input(vt.clone(), v)
    vmax = float(vt.abs().max())
    lo, hi = -vmax - 1.0, vmax
    nu = 0.5 * (lo + hi)
    for _ in range(200):
        nu = 0.5 * (lo + hi)
        e = float((vt - nu).clamp_min(0.0).sum()) - 1.0
        if abs(e) <= tol and hi - lo <= tol:
            break
        if e > 0:
            lo = nu
        else:
            hi = nu
    active = vt > nu
    na = int(active.sum())
    if na > 0:
        nu_exact = (float(vt[active].sum()) - 1.0) / na
        if bool(torch.all(vt[active] > nu_exact)) and bool(torch.all(vt[~active] <= nu_exact)):
            nu = nu_exact
    return like_input((vt - nu).clamp_min(0.0), v)


def simplex_indicator(z, tol: float = 1e-6) -> float:
    """0 if z is on the probability simplex within tol, else +inf (prox.py:147-152)."""
    zt = to_device(z)
    ok = bool(torch.all(zt >= -tol)) and abs(float(zt.sum()) - 1.0) <= tol
    return 0.0 if ok else float(np.inf)
