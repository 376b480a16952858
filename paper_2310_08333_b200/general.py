"""General-operator ADMM engine (``/root/reference/pkg/src/nysopt/admm.py:422-719``).

The dense engine (``admm.py``) is the hot path of BASELINE.json: dense ML data
or a dense QP with M = I, fused into a few kernels per iteration.  This engine
takes every other problem the reference accepts through its QP / ML front
ends:

  * ML problems whose data operator is sparse (``SparseOperator``: CSR SpMV on
    the device, the transpose built on the device) or any other device
    operator;
  * QPs with a general constraint map M (dense, sparse, diagonal, stacked,
    summing row, ...) and a structured or sparse objective matrix P
    (``DiagPlusLowRank``, ``DiagonalOperator``, ``SparseOperator``, ...);
  * the composite sketch target H + rho M^T M with the resketch after a
    penalty change (admm.py:499-505, 545-551), the eigenvalue probe of
    ``check_rank`` (admm.py:467-474) and the infeasibility tests with M != I
    (admm.py:361-415).

It follows the reference loop statement for statement with every vector in
HBM and every numeric step a libnysgpu kernel (``csrc/general.cu`` and the
shared vector kernels); the host only runs the scalar control flow on values
read back once per iteration (plus one scalar block per CG iteration, the
reference's stopping test).  There is no CPU fallback.
"""

from __future__ import annotations

import math
import time
from collections import deque
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import CapabilityError, DataError
from .krylov import CgReport, CgWork, cg_tolerance, pcg_device
from .operators import (IdentityOperator, LinearOperator, MatrixFreeOperator, SparseOperator, UserFn, adjoint_columns_dev,
                        device_fn,
                        to_device)
from .problems import GenericProblem
from .sketch import NystromPreconditioner, NystromSketch, default_sketch_rank, sketch_device

DELTA_WINDOW = 25  # admm.py:33
PENALTY_ADAPT_CUTOFF = 1000  # admm.py:29


class _Stats:
    """A device scalar block filled by reduction kernels and read with one copy."""

    def __init__(self, kx, n: int = 64):
        self.kx = kx
        self.dev = kx.zeros(n)
        self.host = torch.zeros(n, dtype=torch.float64).pin_memory()
        self.next = 0
        self.vals = None

    def slot(self, k: int) -> torch.Tensor:
        t = self.dev[self.next:self.next + k]
        self.next += k
        return t

    def read(self) -> np.ndarray:
        self.host.copy_(self.dev, non_blocking=True)
        self.kx.sync()
        self.vals = self.host.numpy().copy()
        self.next = 0
        return self.vals


def _norm(stats3: np.ndarray, kind: str) -> float:
    """admm.py:203-208 from vstats [sum, sum^2, max|.|]."""
    return float(stats3[2]) if kind == "linf" else math.sqrt(max(float(stats3[1]), 0.0))


class _MLPart:
    """ML pieces (problems.py:219-351) over an arbitrary data operator A."""

    def __init__(self, p, kx):
        self.p, self.kx = p, kx
        self.A: LinearOperator = p.A
        self.sparse = isinstance(p.A, SparseOperator)
        if self.sparse:
            self.fwd, self.bwd = p.A.device_csr(kx.device)
        self.N, self.n = p.N, p.n
        self.b = to_device(p.b, kx.device)
        # a built-in kind (the fused kernels) or the user's Loss object (its callables on the host)
        self.loss = p.loss.kind if p.loss.kind in _lib.LOSS else p.loss
        if not isinstance(self.loss, str) and not all(callable(getattr(p.loss, nm, None))
                                                      for nm in ("value", "deriv", "deriv2")):
            raise DataError(f"loss {p.loss.kind!r} is neither built in nor given with value / deriv / deriv2")
        self.l1, self.l2 = float(p.lambda1), float(p.lambda2)
        self.const = p.loss.deriv2_constant
        self.w = None  # l''(Ax - b) at the Hessian point; None == 1 (square loss)
        self.tg = kx.empty(self.N)
        self.wbuf = kx.empty(self.N)
        self.thx = kx.empty(self.N)
        self.tnu = kx.empty(self.N)
        self.rows_out = kx.zeros(8)

    # A v, A^T t (+ beta zin), in the operator's own kernels
    def a_fwd(self, v, dscale=None):
        kx = self.kx
        if self.sparse:
            y = kx.empty(self.N)
            kx.csr_spmv(self.fwd, v, y, dscale=dscale)
            return y
        y = self.A._apply_dev(v)
        if dscale is not None:
            kx.vmul(1.0, dscale, y, 0.0, y)
        return y

    def a_adj(self, t, beta=0.0, zin=None):
        kx = self.kx
        if self.sparse:
            y = kx.empty(self.n)
            kx.csr_spmv(self.bwd, t, y, beta=beta, zin=zin)
            return y
        y = self.A._apply_adjoint_dev(t)
        if beta != 0.0:
            kx.axpby(beta, zin, 1.0, y)
        return y

    def evaluate(self, x, out):
        """A x -> l'(Ax-b) (tg), l''(Ax-b) (wbuf), out[0] = sum l(Ax - b)."""
        ax = self.a_fwd(x)
        self.kx.ml_rowwise(self.loss, ax, None, self.b, self.tg, self.wbuf, self.thx, None, out)

    def update_hessian(self):
        """hess.update(x) (problems.py:260-261) from the last evaluate()."""
        if self.loss == "square":
            self.w = None
        else:
            if self.w is None:
                self.w = self.kx.empty(self.N)
            self.w.copy_(self.wbuf)

    def hess_apply(self, v):
        """A^T (w o A v) + lambda2 v (problems.py:263-264)."""
        return self.a_adj(self.a_fwd(v, self.w), self.l2, v) if self.l2 != 0.0 else self.a_adj(self.a_fwd(v, self.w))

    def smooth_cols(self, V):
        """A^T diag(w) A V, the sketch target (problems.py:266-273)."""
        kx = self.kx
        if self.sparse:
            Z = kx.empty(self.N, V.shape[1])
            kx.csr_spmm(self.fwd, V, Z, dscale=self.w)
            Y = kx.empty(self.n, V.shape[1])
            kx.csr_spmm(self.bwd, Z, Y)
            return Y
        Z = self.A.apply_columns_dev(V)
        if self.w is not None:
            kx.row_scale(Z, self.w)
        return adjoint_columns_dev(self.A, Z)

    def grad(self, x):
        """A^T l'(Ax - b) + lambda2 x from the last evaluate() (problems.py:238-242)."""
        return self.a_adj(self.tg, self.l2, x) if self.l2 != 0.0 else self.a_adj(self.tg)


class _GenericPart:
    """The oracles of a GenericProblem given as callables (problems.py:125-157):
    f, grad f, the Hessian operator, g and its (possibly inexact) prox.  NumPy
    callables, the reference's contract, get host copies; callables marked
    ``device_fn`` get the device tensors (operators.UserFn); everything around them -- the PCG solve, the
    sketch, residuals, windows, penalty logic -- is the engine's device path."""

    def __init__(self, gp: GenericProblem):
        missing = [nm for nm in ("f", "grad_f", "hess", "g", "prox_g") if getattr(gp, nm) is None]
        if missing:
            raise CapabilityError(f"generic problem without {', '.join(missing)}: nothing to solve")
        self.f, self.grad_f, self.g, self.prox_g = UserFn(gp.f), UserFn(gp.grad_f), UserFn(gp.g), UserFn(gp.prox_g)
        self.hess = gp.hess


class _GeneralEngine:
    def __init__(self, gp: GenericProblem, opts, kx):
        self.gp, self.opts, self.kx = gp, opts, kx
        self.n, self.m = gp.n, gp.m
        self.M: LinearOperator = gp.M
        self.identity_M = isinstance(gp.M, IdentityOperator)
        self.ml = _MLPart(gp.ml, kx) if gp.ml is not None else None
        self.gen = _GenericPart(gp) if gp.ml is None and gp.qp is None else None
        if self.gen is not None:
            self.P = self.gen.hess
            self.const_hess = bool(getattr(self.gen.hess, "is_constant", False)) or gp.is_quadratic
            self.diag_shift = float(getattr(self.gen.hess, "diag_shift", 0.0))
        elif self.ml is None:
            qp = gp.qp
            self.P = qp.P
            self.q = to_device(qp.q, kx.device)
            self.lo = to_device(qp.box.l, kx.device)
            self.hi = to_device(qp.box.u, kx.device)
            self.const_hess = True
            self.diag_shift = 0.0
        else:
            self.const_hess = self.ml.const
            self.diag_shift = self.ml.l2
        # the constraint offset of M x - z = c: zero for every lowered ML / QP problem
        self.c = to_device(gp.c, kx.device) if np.any(gp.c != 0.0) else None
        self.stats = _Stats(kx, 128)
        self._grad_x = None  # (x version, grad, f(x)) cache
        self._xver = 0

    # ------------------------------------------------------ problem pieces --
    def hess_apply(self, v):
        return self.ml.hess_apply(v) if self.ml else self.P._apply_dev(v)

    def M_apply(self, v):
        return v if self.identity_M else self.M._apply_dev(v)

    def M_adj(self, u):
        return u if self.identity_M else self.M._apply_adjoint_dev(u)

    def eval_at_x(self, x):
        """grad f(x) and the pieces of f(x), cached per iterate; for ML also the
        Hessian weights at x (admm.py:539-540)."""
        if self._grad_x is not None and self._grad_x[0] == self._xver:
            return self._grad_x[1], self._grad_x[2]
        kx = self.kx
        fout = self.stats.slot(8)
        if self.gen:
            g = self.gen.grad_f(x)
            fout.zero_()
            fout[0:1].fill_(self.gen.f.scalar(x))
        elif self.ml:
            self.ml.evaluate(x, fout)
            g = self.ml.grad(x)
            kx.dot(x, x, fout[5:6])
        else:
            px = self.P._apply_dev(x)
            g = px.clone()
            kx.axpby(1.0, self.q, 1.0, g)  # P x + q
            kx.dot(x, px, fout[0:1])
            kx.dot(self.q, x, fout[1:2])
        self._grad_x = (self._xver, g, fout)
        return g, fout

    def f_value(self, fout_h) -> float:
        if self.gen:
            return float(fout_h[0])
        if self.ml:
            return float(fout_h[0]) + 0.5 * self.ml.l2 * float(fout_h[5])  # problems.py:227-230
        return 0.5 * float(fout_h[0]) + float(fout_h[1])  # problems.py:396-397

    def g_launch(self, z):
        out = self.stats.slot(3)
        if self.gen:
            out.zero_()
            out[0:1].fill_(self.gen.g.scalar(z))
        elif self.ml:
            self.kx.absstats(z, self.ml.l1, out)
        else:
            self.kx.box_violation(z, self.lo, self.hi, out)
        return out

    def g_value(self, o) -> float:
        if self.gen:
            return float(o[0])
        if self.ml:
            return self.ml.l1 * float(o[0])
        scale = 1.0 + float(o[2])  # prox.py:138-144
        ok = o[0] <= 1e-9 * scale and o[1] <= 1e-9 * scale
        return 0.0 if ok else np.inf

    # ------------------------------------------------------------ the gap --
    def gap_at(self, z) -> float:
        """ml_dual_gap(p, z) (problems.py:335-351)."""
        ml, kx = self.ml, self.kx
        st = _Stats(kx, 16)
        ev = st.slot(8)
        az = ml.a_fwd(z)
        kx.ml_rowwise(ml.loss, az, None, ml.b, ml.tnu, None, None, None, ev)  # nu = l'(Az - b), sum l
        atnu = ml.a_adj(ml.tnu)
        ab = st.slot(3)
        kx.absstats(atnu, ml.l1, ab)
        zs = st.slot(3)
        kx.absstats(z, 0.0, zs)
        zz = st.slot(1)
        kx.dot(z, z, zz)
        h = st.read()
        primal = float(h[0]) + 0.5 * ml.l2 * float(h[14]) + ml.l1 * float(h[11])
        c = 1.0
        if ml.l2 == 0.0:
            denom = float(h[10])
            if denom > ml.l1:
                c = ml.l1 / denom
        co = kx.zeros(4)
        kx.ml_conj_scaled(ml.loss, ml.tnu, c, ml.b, co)
        o = co.cpu().numpy()
        if o[1] > 0:
            return np.inf
        dual = -float(o[0]) - float(o[2])
        if ml.l2 > 0.0:
            dual -= float(h[9]) / (2.0 * ml.l2)
        if not np.isfinite(dual):
            return np.inf
        num = primal - dual
        den = min(primal, abs(dual))
        if den <= 1e-16:
            return 0.0 if abs(num) <= 1e-12 else np.inf
        return num / den

    # --------------------------------------------------------- the sketch --
    def composite(self, v, rho):
        """v -> H v + rho M^T M v (admm.py:468-470, 499-505)."""
        y = self.hess_apply(v)
        self.kx.axpby(rho, self.M_adj(self.M_apply(v)), 1.0, y)
        return y

    def sketch_cols(self, rho):
        kx = self.kx
        if self.identity_M:
            if self.gen:
                return self.gen.hess.smooth_part().apply_columns_dev
            if self.ml:
                return self.ml.smooth_cols  # hess.smooth_part() (problems.py:266-273)
            return self.P.apply_columns_dev  # ConstantHessian: diag_shift == 0

        def cols(V):  # H V + rho M^T (M V)
            Y = self.P.apply_columns_dev(V) if self.ml is None else self.ml.smooth_cols(V)
            if self.ml is not None and self.ml.l2 != 0.0:
                kx.axpby(self.ml.l2, V.reshape(-1), 1.0, Y.view(-1))
            MtMV = adjoint_columns_dev(self.M, self.M.apply_columns_dev(V))
            kx.axpby(rho, MtMV.reshape(-1), 1.0, Y.view(-1))
            return Y

        return cols

    def build_preconditioner(self, seed, rho, sigma_eff, timings):
        t0 = time.perf_counter()
        U, lam = sketch_device(self.kx, self.sketch_cols(rho), self.n, self.r_sk, seed)
        S = NystromSketch.empty(self.n) if U.shape[1] == 0 else NystromSketch(U, lam)
        nu = (rho + sigma_eff + self.diag_shift) if self.identity_M else max(sigma_eff, 1e-8)
        timings.precond_s += time.perf_counter() - t0
        return NystromPreconditioner(S, nu)

    # -------------------------------------------------------------- solve --
    def run(self, x0, z0, u0, callback, t_start):
        from .admm import (IterationRecord, PenaltyEvent, Residuals, SolveResult, SolverState, Status,
                           Timings)
        from .sketch import estimate_extreme_eigs

        opts, kx, n, m = self.opts, self.kx, self.n, self.m

        def warm(v, dim, name):
            if v is None:
                return kx.zeros(dim)
            vt = to_device(v, kx.device)
            if vt.shape != (dim,):
                raise DataError(f"warm start {name} must have length {dim}, got shape {tuple(vt.shape)}")
            return vt.clone()

        x, z, u = warm(x0, n, "x0"), warm(z0, m, "z0"), warm(u0, m, "u0")
        rho = float(opts.rho0)
        xbar, zbar = kx.zeros(n), kx.zeros(m)
        bar_count = 0
        self._xver += 1
        g_x, _ = self.eval_at_x(x)
        if self.gen:
            self.gen.hess.update(x)
        if self.ml:
            self.ml.update_hessian()  # hess.update(x0) (admm.py:455)
        Mx = self.M_apply(x).clone()

        # offset policy (admm.py:462-474)
        sigma_eff = opts.sigma
        if self.gp.full_rank or opts.assume_full_rank:
            sigma_eff = 0.0
        elif opts.check_rank:
            rho_probe = rho
            probe = MatrixFreeOperator(n, n, device_fn(lambda v: self.composite(to_device(v), rho_probe)),
                                       device_fn(lambda v: self.composite(to_device(v), rho_probe)))
            _, lam_min = estimate_extreme_eigs(probe, min(max(2, n), 60), opts.rng_seed + 7)
            if lam_min > 1e-8:
                sigma_eff = 0.0

        use_gap = opts.use_dual_gap
        if use_gap is None:
            use_gap = self.ml is not None and self.gp.ml.loss.conj is not None
        if use_gap and self.ml is None:
            raise DataError("the duality-gap criterion requires an ML problem")

        timings = Timings()
        r_sk = opts.sketch_rank or default_sketch_rank(n)
        self.r_sk = max(1, min(r_sk, n))

        def nu_identity(r):
            return r + sigma_eff + self.diag_shift

        pc: Optional[NystromPreconditioner] = None
        last_sketch = 0
        rho_at_sketch = rho
        if opts.use_preconditioner:
            pc = self.build_preconditioner(opts.rng_seed, rho, sigma_eff, timings)
            rho_at_sketch = rho

        def residuals(x, z, u, Mx, rho):
            """compute_residuals (admm.py:215-224); launches only."""
            g, fout = self.eval_at_x(x)
            s_rp = self.stats.slot(3)
            if self.c is None:
                kx.vstats(Mx, z, s_rp)  # rp = Mx - z - c, c = 0
            else:
                zc = z.clone()
                kx.axpby(1.0, self.c, 1.0, zc)
                kx.vstats(Mx, zc, s_rp)
            s_mx = self.stats.slot(3)
            kx.vstats(Mx, None, s_mx)
            s_z = self.stats.slot(3)
            kx.vstats(z, None, s_z)
            s_d = self.stats.slot(4)
            kx.gdual(g, self.M_adj(u), rho, s_d)
            return (s_rp, s_mx, s_z, s_d, fout)

        def res_from(h, sl) -> Residuals:
            kind = opts.norm_kind
            o = self.stats.dev
            idx = [int(t.data_ptr() - o.data_ptr()) // 8 for t in sl[:4]]
            rp = _norm(h[idx[0]:idx[0] + 3], kind)
            nmx = _norm(h[idx[1]:idx[1] + 3], kind)
            nz = _norm(h[idx[2]:idx[2] + 3], kind)
            d = h[idx[3]:idx[3] + 4]
            if kind == "linf":
                rd, ds = float(d[2]), float(d[3])
            else:
                rd, ds = math.sqrt(max(d[0], 0.0)), math.sqrt(max(d[1], 0.0))
            return Residuals(None, None, rp, rd, max(nmx, nz, c_norm[kind]), ds, m)

        def offs(t):
            return int(t.data_ptr() - self.stats.dev.data_ptr()) // 8

        c_norm = {"l2": 0.0, "linf": 0.0}  # ||c|| in the primal scale (admm.py:222)
        if self.c is not None:
            c_norm = {"l2": float(np.linalg.norm(self.gp.c)), "linf": float(np.max(np.abs(self.gp.c)))}

        sl = residuals(x, z, u, Mx, rho)
        h = self.stats.read()
        res = res_from(h, sl)
        timings.setup_s = time.perf_counter() - t_start

        history, events = [], []
        iterates = [] if opts.record_iterates else None
        xw: deque = deque(maxlen=DELTA_WINDOW + 1)
        uw: deque = deque(maxlen=DELTA_WINDOW + 1)
        xw.append(x.clone())
        uw.append(u.clone())
        status = Status.ITERATION_LIMIT
        cert_p = cert_d = None
        gap = None
        rho_frozen = False
        cycle_hits = 0
        best_res = np.inf
        trend: deque = deque(maxlen=DELTA_WINDOW + 1)
        work = CgWork(kx, n)
        k_done = 0
        is_qp = self.gp.qp is not None
        lo = getattr(self, "lo", None)
        hi = getattr(self, "hi", None)

        def change_penalty(k, rho_old, rho_new):
            """admm.py:303-319 (the preconditioner shift only follows for M = I)."""
            out = kx.zeros(2)
            kx.scale_dual(u, rho_old, rho_new, out)
            o = out.cpu().numpy()
            denom = max(math.sqrt(max(o[0], 0.0)), 1e-30)
            jump = math.sqrt(max(o[1], 0.0)) / denom
            if pc is not None and self.identity_M:
                pc.update_shift(nu_identity(rho_new))
            return PenaltyEvent(k, rho_old, rho_new, jump)

        for k in range(1, opts.max_iter + 1):
            k_done = k
            if opts.time_limit is not None and time.perf_counter() - t_start > opts.time_limit:
                status = Status.TIME_LIMIT
                break
            if self.gen and not self.const_hess:
                self.gen.hess.update(x)  # admm.py:539-540
            if self.ml and not self.const_hess:
                self.eval_at_x(x)
                self.ml.update_hessian()
            if pc is not None:
                stale_hess = not self.const_hess and k - last_sketch >= opts.resketch_every
                stale_rho = not self.identity_M and rho != rho_at_sketch
                if stale_hess or stale_rho:
                    pc = self.build_preconditioner(opts.rng_seed + k, rho, sigma_eff, timings)
                    last_sketch = k
                    rho_at_sketch = rho
            tol = 1e-12 if opts.exact_x_solve else cg_tolerance(k, res.rp_norm, res.rd_norm, opts.gamma)

            # ---- x-update (admm.py:243-275)
            t0 = time.perf_counter()
            g_x, _ = self.eval_at_x(x)
            rhs = self.hess_apply(x)
            kx.axpby(sigma_eff, x, 1.0, rhs)
            kx.axpby(-1.0, g_x, 1.0, rhs)
            target = z.clone()
            kx.axpby(-1.0, u, 1.0, target)  # z + c - u
            if self.c is not None:
                kx.axpby(1.0, self.c, 1.0, target)
            kx.axpby(rho, target if self.identity_M else self.M_adj(target), 1.0, rhs)
            shift = rho + sigma_eff
            rho_now = rho

            def matvec(v, out, dot, _shift=shift, _rho=rho_now):
                y = self.hess_apply(v)
                if self.identity_M:
                    kx.axpby(_shift, v, 1.0, y)
                else:
                    kx.axpby(_rho, self.M_adj(self.M_apply(v)), 1.0, y)
                    kx.axpby(sigma_eff, v, 1.0, y)
                kx.copy(y, out)
                if dot is not None:
                    kx.dot(v, out, dot)

            precond = None
            if pc is not None:
                pcc = pc

                def precond(v, out, rdot, rz, _pc=pcc):
                    _pc.apply_into(kx, v, out, rdot, rz)

            x_new = x.clone()
            rep: CgReport = pcg_device(work, matvec, rhs, x_new, precond, tol, 10 * n)
            linsys_s = time.perf_counter() - t0
            timings.linsys_total_s += linsys_s

            Mx_new = x_new if self.identity_M else self.M_apply(x_new).clone()
            # ---- z/u (admm.py:278-300): w = alpha Mx + (1-alpha) z; z = prox(w + u); u += w - z
            t0 = time.perf_counter()
            x = x_new
            self._xver += 1
            Mx = Mx_new
            if self.gen:
                # w = alpha Mx + (1 - alpha) z; z = prox_g(w + u, rho, tol_k); u += w - z with
                # tol_k = prox_tol0 / k^(2 gamma) (admm.py:278-300)
                # (with an offset: w = alpha Mx + (1 - alpha)(z + c); z = prox_g(w - c + u); u += w - z - c)
                w = Mx.clone()
                kx.axpby(1.0 - opts.alpha, z, opts.alpha, w)
                if self.c is not None:
                    kx.axpby(1.0 - opts.alpha, self.c, 1.0, w)
                v = w.clone()
                kx.axpby(1.0, u, 1.0, v)
                if self.c is not None:
                    kx.axpby(-1.0, self.c, 1.0, v)
                prox_tol = opts.prox_tol0 / max(k, 1) ** (2.0 * opts.gamma)
                z = self.gen.prox_g(v, rho, max(prox_tol, 1e-15)).clone()
                kx.axpby(1.0, w, 1.0, u)
                kx.axpby(-1.0, z, 1.0, u)
                if self.c is not None:
                    kx.axpby(-1.0, self.c, 1.0, u)
            elif self.ml:
                kx.admm_zu(Mx, z, u, opts.alpha, _lib.PROX_SOFT, self.ml.l1 / rho, None, None, None, None, False)
            else:
                kx.admm_zu(Mx, z, u, opts.alpha, _lib.PROX_BOX, 0.0, lo, hi, None, None, False)
            prox_s = time.perf_counter() - t0
            timings.prox_total_s += prox_s
            if k >= 2:  # admm.py:580-583
                kx.axpby(1.0, x, 1.0, xbar)
                kx.axpby(1.0, z, 1.0, zbar)
                bar_count += 1

            sl = residuals(x, z, u, Mx, rho)
            gs = self.g_launch(z)
            h = self.stats.read()
            res = res_from(h, sl)
            objective = self.f_value(h[offs(sl[4]):]) + self.g_value(h[offs(gs):offs(gs) + 3])
            gap = self.gap_at(z) if use_gap else None
            avg_obj = None
            if opts.track_averaged_objective and bar_count > 0:
                avg_obj = self._averaged_objective(xbar, zbar, bar_count)
            history.append(IterationRecord(k=k, rp_norm=res.rp_norm, rd_norm=res.rd_norm, objective=objective,
                                           rho=rho, cg_iters=rep.iterations, cg_tol=tol, linsys_s=linsys_s,
                                           prox_s=prox_s, gap=gap, avg_objective=avg_obj))
            if iterates is not None:
                iterates.append((x.cpu().numpy(), z.cpu().numpy(), u.cpu().numpy()))
            if callback is not None:
                callback(k, res.rp_norm, res.rd_norm, objective, rho, rep.iterations)

            if opts.custom_stop is not None:
                if opts.custom_stop(self.gp, self._state(x, z, u, Mx, rho, k, xbar, zbar, bar_count)):
                    status = Status.OPTIMAL
                    break
            elif self._terminated(res, gap):
                status = Status.OPTIMAL
                break

            # ---- infeasibility on smoothed differences (admm.py:621-634)
            xw.append(x.clone())
            uw.append(u.clone())
            if is_qp and len(uw) == DELTA_WINDOW + 1:
                chk = self._infeasibility(xw, uw, rho)
                if chk[3]:
                    rho_frozen = True
                if chk[0] is not None:
                    status = Status(chk[0])
                    cert_p, cert_d = chk[1], chk[2]
                    break

            # ---- cycle guard (admm.py:636-675)
            best_res = min(best_res, max(res.rp_norm, res.rd_norm))
            trend.append(best_res)
            if len(xw) >= 4 and not rho_frozen and k <= PENALTY_ADAPT_CUTOFF:
                xk = xw[-1]
                st = _Stats(kx, 3 * 12)
                s_step = st.slot(3)
                kx.vstats(xk, xw[-2], s_step)
                s_x = st.slot(3)
                kx.vstats(xk, None, s_x)
                periods = list(range(2, min(len(xw) - 1, 10) + 1))
                s_p = []
                for p in periods:
                    sp = st.slot(3)
                    kx.vstats(xk, xw[-1 - p], sp)
                    s_p.append(sp)
                hh = st.read()
                step = math.sqrt(max(hh[1], 0.0))
                locked = False
                if step > 1e-8 * max(1.0, math.sqrt(max(hh[4], 0.0))):
                    return_gap = min(math.sqrt(max(hh[6 + 3 * j + 1], 0.0)) for j in range(len(periods)))
                    locked = return_gap <= 1e-3 * step
                cycle_hits = cycle_hits + 1 if locked else 0
                stagnant = len(trend) == trend.maxlen and trend[-1] >= 0.99 * trend[0]
                if cycle_hits >= 5 and stagnant:
                    cycle_hits = 0
                    trend.clear()
                    events.append(change_penalty(k, rho, rho * opts.tau))
                    rho = events[-1].rho_new
                    xw.clear()
                    uw.clear()
                    xw.append(x.clone())
                    uw.append(u.clone())

            # ---- balanced-residual penalty rule (admm.py:677-698, 322-350)
            if (not rho_frozen and opts.penalty_update_every > 0 and k >= opts.penalty_warmup
                    and k % opts.penalty_update_every == 0 and k <= PENALTY_ADAPT_CUTOFF):
                t_p = math.sqrt(m) * opts.eps_abs + opts.eps_rel * res.primal_scale
                t_d = math.sqrt(n) * opts.eps_abs + opts.eps_rel * res.dual_scale
                if t_p > 0 and t_d > 0:
                    p_meas, d_meas = res.rp_norm / t_p, res.rd_norm / t_d
                else:
                    p_meas, d_meas = res.rp_norm, res.rd_norm
                rho_new = None
                if p_meas > opts.mu * d_meas:
                    rho_new = rho * opts.tau
                elif d_meas > opts.mu * p_meas:
                    rho_new = rho / opts.tau
                if rho_new is not None:
                    events.append(change_penalty(k, rho, rho_new))
                    rho = rho_new
                    xw.clear()
                    uw.clear()
                    xw.append(x.clone())
                    uw.append(u.clone())

        timings.total_s = time.perf_counter() - t_start
        # final objective f(x) + g(z) (admm.py:706)
        self._grad_x = None
        _, fout = self.eval_at_x(x)
        gs = self.g_launch(z)
        h = self.stats.read()
        obj = self.f_value(h[offs(fout):]) + self.g_value(h[offs(gs):offs(gs) + 3])
        xbar_h = (xbar / bar_count).cpu().numpy() if bar_count else None
        zbar_h = (zbar / bar_count).cpu().numpy() if bar_count else None
        return SolveResult(status=status, x=x.cpu().numpy(), z=z.cpu().numpy(), u=u.cpu().numpy(), objective=obj,
                           iterations=k_done, rp_norm=res.rp_norm, rd_norm=res.rd_norm, history=history,
                           timings=timings, x_bar=xbar_h, z_bar=zbar_h, certificate_primal=cert_p,
                           certificate_dual=cert_d, penalty_events=events, iterates=iterates, gap=gap,
                           device_stats={"engine": "general", "kernel_launches": kx.kernel_launches()})

    # -------------------------------------------------------------- helpers --
    def _terminated(self, res, gap) -> bool:
        """check_termination (admm.py:227-240)."""
        if gap is not None:
            return gap <= self.opts.eps_dual_gap
        o = self.opts
        p_ok = res.rp_norm <= math.sqrt(self.m) * o.eps_abs + o.eps_rel * res.primal_scale
        d_ok = res.rd_norm <= math.sqrt(self.n) * o.eps_abs + o.eps_rel * res.dual_scale
        return bool(p_ok and d_ok)

    def _infeasibility(self, xw, uw, rho):
        """check_infeasibility (admm.py:361-415) with a general M."""
        kx, eps = self.kx, self.opts.eps_inf
        width = len(uw) - 1
        dx = xw[-1].clone()
        kx.axpby(-1.0, xw[0], 1.0, dx)
        kx.axpby(0.0, dx, 1.0 / width, dx)  # (x_last - x_first) / width
        du = uw[-1].clone()
        kx.axpby(-1.0, uw[0], 1.0, du)
        kx.axpby(0.0, du, 1.0 / width, du)
        st = _Stats(kx, 24)
        s_du = st.slot(3)
        kx.vstats(du, None, s_du)
        s_mtdu = st.slot(3)
        kx.vstats(self.M_adj(du), None, s_mtdu)
        s_dx = st.slot(3)
        kx.vstats(dx, None, s_dx)
        s_pdx = st.slot(3)
        kx.vstats(self.P._apply_dev(dx), None, s_pdx)
        s_box = st.slot(4)
        kx.box_cert(du, self.M_apply(dx), self.lo, self.hi, s_box)
        s_lin = st.slot(1)
        kx.dot(self.q, dx, s_lin)
        h = st.read()
        primal = dual = near_p = near_d = False
        cert_p = cert_d = None
        du_norm = math.sqrt(max(h[1], 0.0))
        if du_norm > 1e-14:
            t_map = math.sqrt(max(h[4], 0.0))
            t_sup = np.inf if h[14] > 0 else (0.0 + float(h[12])) + float(h[13])
            primal = t_map < eps * du_norm and t_sup < eps * du_norm
            near_p = t_map < 10 * eps * du_norm and t_sup < 10 * eps * du_norm
            if primal:
                cert_p = rho * du.cpu().numpy()
        dx_norm = math.sqrt(max(h[7], 0.0))
        if dx_norm > 1e-14:
            s_obj = math.sqrt(max(h[10], 0.0))
            s_cone = math.sqrt(max(h[15], 0.0))
            s_lin = float(h[16])
            dual = s_obj < eps * dx_norm and s_cone < eps * dx_norm and s_lin < eps * dx_norm
            near_d = s_obj < 10 * eps * dx_norm and s_cone < 10 * eps * dx_norm and s_lin < 10 * eps * dx_norm
            if dual:
                cert_d = dx.cpu().numpy()
        if primal and dual:
            status = "primal_and_dual_infeasible"
        elif primal:
            status = "primal_infeasible"
        elif dual:
            status = "dual_infeasible"
        else:
            status = None
        return status, cert_p, cert_d, near_p or near_d

    def _state(self, x, z, u, Mx, rho, k, xbar, zbar, bar_count):
        from .admm import SolverState

        return SolverState(x=x.cpu().numpy(), z=z.cpu().numpy(), u=u.cpu().numpy(), rho=rho, k=k,
                           Mx=Mx.cpu().numpy(), x_bar_sum=xbar.cpu().numpy(), z_bar_sum=zbar.cpu().numpy(),
                           bar_count=bar_count)

    def _averaged_objective(self, xbar, zbar, bar_count) -> float:
        """f(x_bar) + g(z_bar) (admm.py:589-591), on scratch buffers (the cached
        evaluation at x stays valid)."""
        kx = self.kx
        xb = xbar.clone()
        kx.axpby(0.0, xb, 1.0 / bar_count, xb)
        zb = zbar.clone()
        kx.axpby(0.0, zb, 1.0 / bar_count, zb)
        st = _Stats(kx, 16)
        fo = st.slot(8)
        if self.gen:
            return self.gen.f.scalar(xb) + self.gen.g.scalar(zb)
        if self.ml:
            kx.ml_rowwise(self.ml.loss, self.ml.a_fwd(xb), None, self.ml.b, None, None, None, None, fo)
            kx.dot(xb, xb, fo[5:6])
        else:
            kx.dot(xb, self.P._apply_dev(xb), fo[0:1])
            kx.dot(self.q, xb, fo[1:2])
        go = st.slot(3)
        if self.ml:
            kx.absstats(zb, self.ml.l1, go)
        else:
            kx.box_violation(zb, self.lo, self.hi, go)
        h = st.read()
        return self.f_value(h[0:8]) + self.g_value(h[8:11])
