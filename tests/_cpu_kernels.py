"""CPU test double of the kernel interface (paper_2310_08333_b200.kernels.Kernels).

TEST-ONLY.  It restates each C-ABI kernel with torch CPU ops so that the
host-side logic that does not depend on a GPU -- the row sharding, the
placement of the all-reduces, the packed scalar buffers, the ADMM control
flow -- can be exercised by multi-process gloo tests on a machine without a
GPU.  The product path never uses it (``solve`` defaults to the CUDA kernels
and fails loudly without them).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from paper_2310_08333_b200 import _lib

F64 = torch.float64


def _loss(kind, w):
    if kind == "square":
        return 0.5 * w * w, w.clone(), torch.ones_like(w)
    if kind == "logistic":
        ex = torch.sigmoid(w)
        return torch.logaddexp(torch.zeros_like(w), w), ex, ex * torch.sigmoid(-w)
    a = w.abs() <= 1.0
    return (torch.where(a, w * w, 2 * w.abs() - 1), torch.where(a, 2 * w, 2 * torch.sign(w)),
            torch.where(a, torch.full_like(w, 2.0), torch.zeros_like(w)))


def _conj(kind, y):
    if kind == "square":
        return 0.5 * y * y
    if kind == "logistic":
        inside = (y >= 0) & (y <= 1)
        yc = y.clamp(1e-12, 1 - 1e-12)
        ent = yc * torch.log(yc) + (1 - yc) * torch.log1p(-yc)
        out = torch.where(inside, ent, torch.full_like(y, math.inf))
        return torch.where((y == 0) | (y == 1), torch.zeros_like(y), out)
    return torch.where(y.abs() <= 2, 0.25 * y * y, torch.full_like(y, math.inf))


class CpuKernels:
    name = "cpu-double"

    def __init__(self):
        self.device = torch.device("cpu")
        self.launches = 0
        self.h2d = self.d2h = 0
        self.timed_name = None
        self.events = []

    def kernel_launches(self):
        return self.launches

    def empty(self, *shape):
        return torch.empty(*shape, dtype=F64)

    def zeros(self, *shape):
        return torch.zeros(*shape, dtype=F64)

    def sync(self):
        pass

    # K1-K3
    def gemv(self, A, X, Y):
        Y.copy_(X @ A.T)

    def gemvT(self, A, T, Y):
        Y.copy_(T @ A)

    def hvp(self, A, d, v, shift, y, pAp=None, finish=True):
        t = A @ v
        if d is not None:
            t = t * d
        y.copy_(A.T @ t)
        if finish:
            y.add_(shift * v)
            if pAp is not None:
                pAp.fill_(float(v @ y))

    def shift_dot(self, v, shift, y, dot=None):
        y.add_(shift * v)
        if dot is not None:
            dot.fill_(float(v @ y))

    def dot(self, a, b, out):
        out.fill_(float(a @ b))

    def precond_apply(self, U, lam, nu, v, z, rdot=None, rz=None):
        if U is None:
            z.copy_(v)
        else:
            h = U.T @ v
            head = (lam[-1] + nu) * (h / (lam + nu))
            z.copy_(U @ (head - h) + v)
        if rz is not None:
            rz.fill_(float(rdot @ z))

    # K7
    def cg_start(self, b, Ax, r, sc):
        r.copy_(b - Ax)
        sc[_lib.CG_B2] = float(b @ b)
        sc[_lib.CG_RES2] = float(r @ r)

    def cg_step_xr(self, x, r, p, Ap, refresh, sc):
        pAp, rz = float(sc[_lib.CG_PAP]), float(sc[_lib.CG_RZ])
        bad = not math.isfinite(pAp) or pAp <= 0
        sc[_lib.CG_FLAG] = 1.0 if not math.isfinite(pAp) else (2.0 if pAp <= 0 else 0.0)
        if bad:
            return
        alpha = rz / pAp
        sc[_lib.CG_ALPHA] = alpha
        x.add_(alpha * p)
        if not refresh:
            r.sub_(alpha * Ap)
            sc[_lib.CG_RES2] = float(r @ r)

    def cg_dir(self, z, p, first, sc):
        rz_new = float(sc[_lib.CG_RZNEW])
        if first:
            p.copy_(z)
        else:
            p.copy_(z + (rz_new / float(sc[_lib.CG_RZ])) * p)
        sc[_lib.CG_RZ] = rz_new

    # K8/K9
    def admm_rhs(self, hxA, gA, q, lambda2, sigma, rho, shift, x, z, u, rhs, r, sc):
        hx = hxA + lambda2 * x
        g = gA + lambda2 * x
        if q is not None:
            g = g + q
        b = hx + sigma * x - g + rho * (z - u)
        rhs.copy_(b)
        r.copy_(b - (hx + shift * x))
        sc[_lib.CG_B2] = float(b @ b)
        sc[_lib.CG_RES2] = float(r @ r)

    def admm_zu(self, x, z, u, alpha, prox_kind, kappa, lo, hi, xbar, zbar, accum):
        w = alpha * x + (1 - alpha) * z
        v = w + u
        if prox_kind == _lib.PROX_SOFT:
            zn = torch.sign(v) * torch.clamp(v.abs() - kappa, min=0.0)
        else:
            zn = torch.minimum(torch.maximum(v, lo), hi)
        u.copy_(u + w - zn)
        z.copy_(zn)
        if accum:
            xbar.add_(x)
            zbar.add_(zn)

    def admm_norms(self, x, z, u, gA, q, lambda2, rho, atnu, lambda1, lo, hi, out):
        rp = x - z
        g = gA + lambda2 * x
        if q is not None:
            g = g + q
        ru = rho * u
        rd = g + ru
        o = [0.0] * 16
        o[0], o[1] = float(rp @ rp), float(rp.abs().max())
        o[2], o[3] = float(rd @ rd), float(rd.abs().max())
        o[4], o[5] = float(x @ x), float(x.abs().max())
        o[6], o[7] = float(z @ z), float(z.abs().max())
        o[8], o[9] = float(ru @ ru), float(ru.abs().max())
        o[10] = float(z.abs().sum())
        o[11] = float(x @ gA)
        o[12] = float(q @ x) if q is not None else 0.0
        if atnu is not None:
            o[13] = float(atnu.abs().max())
            e = torch.clamp(atnu.abs() - lambda1, min=0.0)
            o[14] = float(e @ e)
        o[15] = max(0.0, float(torch.maximum(lo - z, z - hi).max())) if lo is not None else 0.0
        out.copy_(torch.tensor(o, dtype=F64))

    def ml_rowwise(self, loss, Ax, Az, b, tg, w, thx, tnu, out):
        o = [0.0] * 5
        if Ax is not None:
            val, d1, d2 = _loss(loss, Ax - b)
            o[0] = float(val.sum())
            if tg is not None:
                tg.copy_(d1)
            if w is not None:
                w.copy_(d2)
            if thx is not None:
                thx.copy_(d2 * Ax)
        if Az is not None:
            val, d1, _ = _loss(loss, Az - b)
            o[1] = float(val.sum())
            if tnu is not None:
                tnu.copy_(d1)
            cv = _conj(loss, d1)
            inf = torch.isinf(cv)
            o[2] = float(cv[~inf].sum())
            o[3] = float(inf.sum())
            o[4] = float(b @ d1)
        out[:5] = torch.tensor(o, dtype=F64)

    def ml_conj_scaled(self, loss, nu, c, b, out):
        y = nu * c
        cv = _conj(loss, y)
        inf = torch.isinf(cv)
        out.copy_(torch.tensor([float(cv[~inf].sum()), float(inf.sum()), float(b @ y)], dtype=F64))

    # K13/K14
    def window_norms(self, ring, cur, others, out):
        xc = ring[cur]
        vals = [float(xc @ xc)] + [float((xc - ring[o]) @ (xc - ring[o])) for o in others]
        out[: len(vals)] = torch.tensor(vals, dtype=F64)

    def scale_dual(self, u, rho_old, rho_new, out):
        yo = rho_old * u
        u.mul_(rho_old / rho_new)
        d = rho_new * u - yo
        out.copy_(torch.tensor([float(yo @ yo), float(d @ d)], dtype=F64))

    def qp_infeas(self, xa, xb, ua, ub, width, lo, hi, q, dx, out):
        d_x = (xa - xb) / width
        d_u = (ua - ub) / width
        dx.copy_(d_x)
        pos, neg = d_u > 0, d_u < 0
        ninf = float((pos & torch.isinf(hi)).sum() + (neg & torch.isinf(lo)).sum())
        sup = float((hi[pos & ~torch.isinf(hi)] * d_u[pos & ~torch.isinf(hi)]).sum()
                    + (lo[neg & ~torch.isinf(lo)] * d_u[neg & ~torch.isinf(lo)]).sum())
        lf, hf = torch.isfinite(lo), torch.isfinite(hi)
        proj = d_x.clone()
        proj[lf & hf] = 0.0
        proj[lf & ~hf] = torch.clamp(d_x[lf & ~hf], min=0.0)
        proj[~lf & hf] = torch.clamp(d_x[~lf & hf], max=0.0)
        e = d_x - proj
        out.copy_(torch.tensor([float(d_u @ d_u), sup, ninf, float(d_x @ d_x), float(e @ e),
                                float(q @ d_x) if q is not None else 0.0], dtype=F64))

    def row_scale(self, X, d):
        X.mul_(d[:, None])

    # K5
    def gemm(self, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, Cm, ldc):
        Am = A.reshape(-1)[: (K if ta else M) * lda].view(K if ta else M, lda)
        Am = Am[:, :M].T if ta else Am[:, :K]
        Bm = B.reshape(-1)[: (N if tb else K) * ldb].view(N if tb else K, ldb)
        Bm = Bm[:, :K].T if tb else Bm[:, :N]
        Cv = Cm.reshape(-1)[: M * ldc].view(M, ldc)[:, :N]
        Cv.copy_(alpha * (Am @ Bm) + (beta * Cv if beta != 0 else 0.0))

    def gaussian(self, seed, out):
        out.copy_(torch.from_numpy(np.random.default_rng(seed).standard_normal(tuple(out.shape))))

    def orthonormalize(self, Om, Q):
        Q.copy_(torch.linalg.qr(Om, mode="reduced")[0])

    def nystrom_core(self, Q, Y, U, lam, r):
        import scipy.linalg

        Qn, Yn = Q.numpy(), Y.numpy()
        n, s = Qn.shape
        eps = np.finfo(float).eps
        shift = eps * max((n / s) * float(np.sum(Qn * Yn)), 0.0) or eps
        Ys = Yn + shift * Qn
        core = Qn.T @ Ys
        core = 0.5 * (core + core.T)
        try:
            L = np.linalg.cholesky(core)
            B = scipy.linalg.solve_triangular(L, Ys.T, lower=True).T
        except np.linalg.LinAlgError:
            w, V = np.linalg.eigh(core)
            scale = max(abs(w[-1]), shift)
            if w[0] < -1e-8 * scale:
                from paper_2310_08333_b200.errors import DataError

                raise DataError("not PSD")
            keep = w > eps * scale
            if not keep.any():
                return 0
            B = Ys @ (V[:, keep] / np.sqrt(w[keep]))
        Us, sv, _ = np.linalg.svd(B, full_matrices=False)
        rr = min(r, Us.shape[1])
        U[:, :rr] = torch.from_numpy(Us[:, :rr].copy())
        lam[:rr] = torch.from_numpy(np.maximum(sv[:rr] ** 2 - shift, 0.0))
        return rr
