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
