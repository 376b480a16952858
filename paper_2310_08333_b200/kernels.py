"""Tensor-level wrappers of the C ABI (include/nysgpu.h).

``Kernels`` owns the stream and the workspaces of one solve and exposes every
kernel as a method over torch CUDA tensors (torch is only the device-buffer
allocator here).  The ADMM engine (``admm.py``) talks to nothing else, which
keeps the drop-in boundary in one place.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import check

F64 = torch.float64


def _p(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


class Kernels:
    """GPU implementation of the kernel interface used by the engine."""

    name = "cuda"

    def __init__(self, device: Optional[torch.device] = None):
        self.L = _lib.lib()
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.current_stream(self.device)
        self.sp = self.stream.cuda_stream
        self._ws: dict[str, torch.Tensor] = {}
        self.red = self.workspace("red", self.L.nys_reduce_workspace())
        self.launches = 0  # C-ABI calls (each launches >= 1 kernel)
        # instrumentation: CUDA-event timing of one kernel family, host<->device bytes
        self.timed_name: Optional[str] = None
        self.events: list = []
        self.h2d = 0
        self.d2h = 0

    def kernel_launches(self) -> int:
        """Kernels launched by libnysgpu so far (all instances in this process)."""
        return int(self.L.nys_launch_count())

    def _t0(self, name):
        if self.timed_name != name:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        return e

    def _t1(self, e) -> None:
        if e is not None:
            e2 = torch.cuda.Event(enable_timing=True)
            e2.record(self.stream)
            self.events.append((e, e2))

    def event_times_ms(self) -> list:
        self.sync()
        return [a.elapsed_time(b) for a, b in self.events]

    # ------------------------------------------------------------ memory --
    def workspace(self, name: str, nbytes: int) -> torch.Tensor:
        """Zero-filled device workspace (kernels keep tickets in it)."""
        nbytes = max(int(nbytes), 256)
        t = self._ws.get(name)
        if t is None or t.numel() < nbytes:
            t = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
            self._ws[name] = t
        return t

    def empty(self, *shape) -> torch.Tensor:
        return torch.empty(*shape, dtype=F64, device=self.device)

    def zeros(self, *shape) -> torch.Tensor:
        return torch.zeros(*shape, dtype=F64, device=self.device)

    def sync(self) -> None:
        self.stream.synchronize()

    # ------------------------------------------------------- K1/K2/K3 ----
    def gemv(self, A: torch.Tensor, X: torch.Tensor, Y: torch.Tensor) -> None:
        """Y[j] = A X[j] for the k rows of X (k <= 4)."""
        rows, n = A.shape
        k = X.shape[0]
        ws = self.workspace("gemv", self.L.nys_gemv_workspace(rows, n, k))
        self.launches += 1
        e = self._t0("gemv")
        check(self.L.nys_gemv_f64(A.data_ptr(), rows, n, A.stride(0), X.data_ptr(), X.stride(0), k,
                                  Y.data_ptr(), Y.stride(0), ws.data_ptr(), ws.numel(), self.sp), "gemv")
        self._t1(e)

    def gemvT(self, A: torch.Tensor, T: torch.Tensor, Y: torch.Tensor) -> None:
        """Y[j] = A^T T[j] for the k rows of T (k <= 4)."""
        rows, n = A.shape
        k = T.shape[0]
        ws = self.workspace("gemvT", self.L.nys_gemvT_workspace(rows, n, k))
        self.launches += 1
        e = self._t0("gemvT")
        check(self.L.nys_gemvT_f64(A.data_ptr(), rows, n, A.stride(0), T.data_ptr(), T.stride(0), k,
                                   Y.data_ptr(), Y.stride(0), ws.data_ptr(), ws.numel(), self.sp), "gemvT")
        self._t1(e)

    HVP_PLANS = {0: "gemv_n_kernel + gemv_t_kernel (two passes)", 1: "hvp_row_kernel",
                 2: "hvp_fused_kernel + gemv_t_reduce", 3: "hvp_cluster_kernel + gemv_t_reduce",
                 4: "hvp_strip_kernel"}

    def hvp_plan_name(self, rows: int, n: int) -> str:
        """The kernel(s) nys_hvp_f64 runs for a rows x n operand."""
        return self.HVP_PLANS.get(int(self.L.nys_hvp_plan(rows, n, n)), "hvp")

    def hvp(self, A, d, v, shift, y, pAp=None, finish=True) -> None:
        rows, n = A.shape
        ws = self.workspace("hvp", self.L.nys_hvp_workspace(rows, n))
        self.launches += 1
        e = self._t0("hvp")
        check(self.L.nys_hvp_f64(A.data_ptr(), rows, n, A.stride(0), _p(d), v.data_ptr(), float(shift),
                                 y.data_ptr(), _p(pAp), 1 if finish else 0, ws.data_ptr(), ws.numel(),
                                 self.sp), "hvp")
        self._t1(e)

    def shift_dot(self, v, shift, y, dot=None) -> None:
        self.launches += 1
        check(self.L.nys_shift_dot_f64(v.numel(), v.data_ptr(), float(shift), y.data_ptr(), _p(dot),
                                       self.red.data_ptr(), self.sp), "shift_dot")

    def dot(self, a, b, out) -> None:
        self.launches += 1
        check(self.L.nys_dot_f64(a.numel(), a.data_ptr(), b.data_ptr(), out.data_ptr(),
                                 self.red.data_ptr(), self.sp), "dot")

    # -------------------------------------------------------------- K6 ----
    def precond_apply(self, U, lam, nu, v, z, rdot=None, rz=None) -> None:
        n = v.numel()
        r = 0 if U is None else U.shape[1]
        ws = self.workspace("prec", self.L.nys_precond_workspace(n, r))
        self.launches += 1
        check(self.L.nys_precond_apply_f64(_p(U), n, r, U.stride(0) if r else 0, _p(lam), float(nu),
                                           v.data_ptr(), z.data_ptr(), _p(rdot), _p(rz), ws.data_ptr(),
                                           ws.numel(), self.sp), "precond")

    # -------------------------------------------------------------- K7 ----
    def cg_start(self, b, Ax, r, sc) -> None:
        self.launches += 1
        check(self.L.nys_cg_start_f64(b.numel(), b.data_ptr(), Ax.data_ptr(), r.data_ptr(), sc.data_ptr(),
                                      self.red.data_ptr(), self.sp), "cg_start")

    def cg_step_xr(self, x, r, p, Ap, refresh, sc) -> None:
        self.launches += 1
        check(self.L.nys_cg_step_xr_f64(x.numel(), x.data_ptr(), r.data_ptr(), p.data_ptr(), Ap.data_ptr(),
                                        1 if refresh else 0, sc.data_ptr(), self.red.data_ptr(), self.sp),
              "cg_step")

    def cg_problem(self, op_kind, A, d, shift, U, lam, nu, b, x, work, tol, max_iter):
        """Fill a ``nys_cg_problem`` for the batched CG driver (workspaces cached)."""
        rows, n = (A.shape[0], A.shape[1])
        r = 0 if U is None else U.shape[1]
        s_op, s_pc = C.c_size_t(0), C.c_size_t(0)
        # the preconditioner workspaces are sized for the largest supported rank so
        # that a descriptor built earlier never points at a reallocated buffer
        red_b = self.L.nys_cg_workspace(op_kind, rows, n, max(r, 512), C.byref(s_op), C.byref(s_pc))
        w_op = self.workspace("hvp" if op_kind == 0 else "densemv", s_op.value)
        w_pc = self.workspace("prec", s_pc.value)
        w_red = self.workspace("cgred", red_b)
        pb = _lib.CgProblem(
            op_kind=op_kind, A=A.data_ptr(), rows=rows, n=n, lda=A.stride(0), d=_p(d), shift=float(shift),
            U=_p(U), r=r, ldu=(U.stride(0) if r else 0), lam=_p(lam), nu=float(nu), b=b.data_ptr(),
            x=x.data_ptr(), res=work.r.data_ptr(), p=work.p.data_ptr(), z=work.z.data_ptr(),
            Ap=work.Ap.data_ptr(), sc=work.sc.data_ptr(), tol=float(tol), max_iter=int(max_iter),
            ws_op=w_op.data_ptr(), ws_op_bytes=w_op.numel(), ws_pc=w_pc.data_ptr(), ws_pc_bytes=w_pc.numel(),
            ws_red=w_red.data_ptr())
        if os.environ.get("NYS_CG_PERSIST", "1") != "0":
            w_cp = self.workspace("cgpersist", self.L.nys_cg_persist_workspace(n, 512))
            pb.ws_cp, pb.ws_cp_bytes = w_cp.data_ptr(), w_cp.numel()
        return pb

    # CUDA-event timing of the operator launches inside the batched CG driver
    def timing_enable(self, on: bool) -> None:
        self.L.nys_timing_enable(1 if on else 0)
        self._lib_timing = bool(on)

    def timing_commit(self, tag: int, last_real_k: int, units: int = 0) -> None:
        if getattr(self, "_lib_timing", False):
            check(self.L.nys_timing_commit(int(tag), int(last_real_k), int(units)), "timing_commit")

    def timing_read(self):
        tot, cnt = C.c_double(0.0), C.c_int64(0)
        self.L.nys_timing_read(C.byref(tot), C.byref(cnt))
        return float(tot.value), int(cnt.value)

    def admm_tail(self, t) -> None:
        self.launches += 1
        check(self.L.nys_admm_tail_f64(C.byref(t), self.sp), "admm_tail")

    def copy(self, src: torch.Tensor, dst: torch.Tensor) -> None:
        """dst[:] = src[:] (contiguous FP64, device or mapped pinned memory)."""
        self.launches += 1
        check(self.L.nys_copy_f64(src.data_ptr(), dst.data_ptr(), src.numel(), self.sp), "copy")

    def copy_to_pinned(self, src: torch.Tensor, dst: torch.Tensor) -> None:
        """Kernel copy of a small device vector into pinned host memory."""
        self.launches += 1
        check(self.L.nys_copy_f64(src.data_ptr(), dst.data_ptr(), src.numel(), self.sp), "copy")

    def readback(self, src: torch.Tensor, dst: torch.Tensor, gate_next: int, pred: int) -> None:
        """copy_to_pinned that also opens the next iteration's gate."""
        self.launches += 1
        check(self.L.nys_readback_f64(src.data_ptr(), dst.data_ptr(), src.numel(), gate_next, pred, self.sp),
              "readback")

    def admm_head(self, h) -> None:
        self.launches += 1
        check(self.L.nys_admm_head_f64(C.byref(h), self.sp), "admm_head")

    def admm_xupdate(self, h, pb, count: int) -> None:
        self.launches += 1
        check(self.L.nys_admm_xupdate_f64(C.byref(h), C.byref(pb), int(count), self.sp), "admm_xupdate")

    def cg_iterate(self, pb, k_first: int, count: int) -> None:
        self.launches += 1
        e = self._t0("cg")
        check(self.L.nys_cg_iterate_f64(C.byref(pb), int(k_first), int(count), self.sp), "cg_iterate")
        self._t1(e)

    def cg_dir(self, z, p, first, sc) -> None:
        self.launches += 1
        check(self.L.nys_cg_dir_f64(z.numel(), z.data_ptr(), p.data_ptr(), 1 if first else 0, sc.data_ptr(),
                                    self.sp), "cg_dir")

    # --------------------------------------------------------- K8/K9 ----
    def admm_rhs(self, hxA, gA, q, lambda2, sigma, rho, shift, x, z, u, rhs, r, sc) -> None:
        self.launches += 1
        check(self.L.nys_admm_rhs_f64(x.numel(), hxA.data_ptr(), gA.data_ptr(), _p(q), float(lambda2),
                                      float(sigma), float(rho), float(shift), x.data_ptr(), z.data_ptr(),
                                      u.data_ptr(), rhs.data_ptr(), r.data_ptr(), sc.data_ptr(),
                                      self.red.data_ptr(), self.sp), "admm_rhs")

    def admm_zu(self, x, z, u, alpha, prox_kind, kappa, lo, hi, xbar, zbar, accum) -> None:
        self.launches += 1
        check(self.L.nys_admm_zu_f64(x.numel(), x.data_ptr(), z.data_ptr(), u.data_ptr(), float(alpha),
                                     int(prox_kind), float(kappa), _p(lo), _p(hi), _p(xbar), _p(zbar),
                                     1 if accum else 0, self.sp), "admm_zu")

    def admm_norms(self, x, z, u, gA, q, lambda2, rho, atnu, lambda1, lo, hi, out) -> None:
        self.launches += 1
        check(self.L.nys_admm_norms_f64(x.numel(), x.data_ptr(), z.data_ptr(), u.data_ptr(), gA.data_ptr(),
                                        _p(q), float(lambda2), float(rho), _p(atnu), float(lambda1), _p(lo),
                                        _p(hi), out.data_ptr(), self.red.data_ptr(), self.sp), "admm_norms")

    def ml_rowwise(self, loss, Ax, Az, b, tg, w, thx, tnu, out) -> None:
        """Row-wise loss epilogue; ``loss`` is a built-in kind (the fused kernel) or a
        user-defined ``Loss`` (its NumPy callables, see ``_custom_rowwise``)."""
        if not isinstance(loss, str):
            return self._custom_rowwise(loss, Ax, Az, b, tg, w, thx, tnu, out)
        self.launches += 1
        check(self.L.nys_ml_rowwise_f64(b.numel(), _lib.LOSS[loss], _p(Ax), _p(Az), b.data_ptr(), _p(tg),
                                        _p(w), _p(thx), _p(tnu), out.data_ptr(), self.red.data_ptr(),
                                        self.sp), "ml_rowwise")

    def ml_conj_scaled(self, loss, nu, c, b, out) -> None:
        if not isinstance(loss, str):
            return self._custom_conj_scaled(loss, nu, c, b, out)
        self.launches += 1
        check(self.L.nys_ml_conj_scaled_f64(b.numel(), _lib.LOSS[loss], nu.data_ptr(), float(c), b.data_ptr(),
                                            out.data_ptr(), self.red.data_ptr(), self.sp), "conj_scaled")

    # user-defined losses (problems.py:35-50, "custom losses" of the reference's ML front
    # end): value / deriv / deriv2 / conj are the user's NumPy callables, so they -- and
    # only they -- run on the host, on copies of the N-vectors; same outputs as the kernels
    def _custom_rowwise(self, loss, Ax, Az, b, tg, w, thx, tnu, out) -> None:
        f64 = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.float64))  # noqa: E731
        put = lambda dst, a: dst.copy_(torch.from_numpy(f64(a)).to(dst.device))  # noqa: E731
        bh = b.cpu().numpy()
        s = np.zeros(5)
        if Ax is not None:
            ax = Ax.cpu().numpy()
            r1 = ax - bh
            s[0] = float(np.sum(loss.value(r1)))
            if tg is not None:
                put(tg, loss.deriv(r1))
            wi = f64(loss.deriv2(r1))
            if w is not None:
                put(w, wi)
            if thx is not None:
                put(thx, wi * ax)
        if Az is not None:
            r2 = Az.cpu().numpy() - bh
            s[1] = float(np.sum(loss.value(r2)))
            nu = f64(loss.deriv(r2))
            if tnu is not None:
                put(tnu, nu)
            if loss.conj is not None:
                cv = f64(loss.conj(nu))
                inf = np.isinf(cv)
                s[2], s[3] = float(cv[~inf].sum()), float(inf.sum())
            s[4] = float(bh @ nu)
        out[:5].copy_(torch.from_numpy(s).to(out.device))

    def _custom_conj_scaled(self, loss, nu, c, b, out) -> None:
        y = nu.cpu().numpy() * float(c)
        cv = np.asarray(loss.conj(y), dtype=np.float64)
        inf = np.isinf(cv)
        s = np.array([float(cv[~inf].sum()), float(inf.sum()), float(b.cpu().numpy() @ y)])
        out[:3].copy_(torch.from_numpy(s).to(out.device))

    # ------------------------------------------------------ K13/K14 ----
    def window_norms(self, ring, cur, others, out) -> None:
        arr = (C.c_int * max(1, len(others)))(*others)
        self.launches += 1
        check(self.L.nys_window_norms_f64(ring.shape[1], ring.data_ptr(), ring.stride(0), int(cur), arr,
                                          len(others), out.data_ptr(), self.red.data_ptr(), self.sp),
              "window_norms")

    def scale_dual(self, u, rho_old, rho_new, out) -> None:
        self.launches += 1
        check(self.L.nys_scale_dual_f64(u.numel(), u.data_ptr(), float(rho_old), float(rho_new),
                                        out.data_ptr(), self.red.data_ptr(), self.sp), "scale_dual")

    def qp_infeas(self, xa, xb, ua, ub, width, lo, hi, q, dx, out) -> None:
        self.launches += 1
        check(self.L.nys_qp_infeas_f64(xa.numel(), xa.data_ptr(), xb.data_ptr(), ua.data_ptr(), ub.data_ptr(),
                                       float(width), lo.data_ptr(), hi.data_ptr(), _p(q), dx.data_ptr(),
                                       out.data_ptr(), self.red.data_ptr(), self.sp), "qp_infeas")

    def axpby(self, a, x, b, y) -> None:
        self.launches += 1
        check(self.L.nys_axpby_f64(x.numel(), float(a), x.data_ptr(), float(b), y.data_ptr(), self.sp), "axpby")

    def loss_eval(self, loss: str, what: int, w, out) -> None:
        """out = loss value (0) / l' (1) / l'' (2) / conjugate (3) elementwise at w."""
        self.launches += 1
        check(self.L.nys_loss_eval_f64(_lib.LOSS[loss], int(what), w.numel(), w.data_ptr(), out.data_ptr(), self.sp),
              "loss_eval")

    def soft_threshold(self, v, kappa, out) -> None:
        self.launches += 1
        check(self.L.nys_soft_threshold_f64(v.numel(), v.data_ptr(), float(kappa), out.data_ptr(), self.sp),
              "soft_threshold")

    def box_project(self, v, lo, hi, out) -> None:
        self.launches += 1
        check(self.L.nys_box_project_f64(v.numel(), v.data_ptr(), lo.data_ptr(), hi.data_ptr(), out.data_ptr(),
                                         self.sp), "box_project")

    def row_scale(self, X, d) -> None:
        self.launches += 1
        check(self.L.nys_row_scale_f64(X.shape[0], X.shape[1], X.data_ptr(), X.stride(0), d.data_ptr(),
                                       self.sp), "row_scale")

    # -------------------------------------------------------------- K5 ----
    def gemm(self, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, Cm, ldc) -> None:
        ws = self.workspace("gemm", self.L.nys_gemm_workspace(M, N, K))
        self.launches += 1
        check(self.L.nys_gemm_f64(int(ta), int(tb), M, N, K, float(alpha), A.data_ptr(), lda, B.data_ptr(),
                                  ldb, float(beta), Cm.data_ptr(), ldc, ws.data_ptr(), ws.numel(), self.sp),
              "gemm")

    def gaussian(self, seed: int, out: torch.Tensor) -> None:
        """out <- np.random.default_rng(seed).standard_normal(out.shape), generated on the GPU."""
        import numpy as np

        st = np.random.PCG64(seed).state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        m64 = (1 << 64) - 1
        count = out.numel()
        ws = self.workspace("gauss", self.L.nys_gaussian_workspace(count))
        self.launches += 1
        check(self.L.nys_gaussian_f64(s >> 64, s & m64, inc >> 64, inc & m64, count, out.data_ptr(),
                                      ws.data_ptr(), ws.numel(), self.sp), "gaussian")

    def gaussian_stream(self, state: int, inc: int, out: torch.Tensor) -> int:
        """out <- the next out.numel() standard normals of the NumPy PCG64 stream at
        (state, inc); returns the 64-bit draws they consumed (the stream continues
        at state advanced by that many steps)."""
        m64 = (1 << 64) - 1
        count = out.numel()
        ws = self.workspace("gauss_stream", self.L.nys_gaussian_workspace(count))
        draws = C.c_int64(0)
        self.launches += 1
        check(self.L.nys_gaussian_draws_f64(state >> 64, state & m64, inc >> 64, inc & m64, count, out.data_ptr(),
                                            ws.data_ptr(), ws.numel(), C.byref(draws), self.sp), "gaussian")
        return int(draws.value)

    def orthonormalize(self, Om, Q) -> None:
        n, s = Om.shape
        ws = self.workspace("sketch", self.L.nys_orthonormalize_workspace(n, s))
        self.launches += 1
        check(self.L.nys_orthonormalize_f64(n, s, Om.data_ptr(), Q.data_ptr(), ws.data_ptr(), ws.numel(),
                                            self.sp), "orthonormalize")

    def nystrom_core(self, Q, Y, U, lam, r) -> int:
        n, s = Q.shape
        ws = self.workspace("sketch", max(self.L.nys_nystrom_workspace(n, s, r),
                                          self.L.nys_orthonormalize_workspace(n, s)))
        rr = C.c_int(0)
        self.launches += 1
        check(self.L.nys_nystrom_core_f64(n, s, r, Q.data_ptr(), Y.data_ptr(), U.data_ptr(), lam.data_ptr(),
                                          C.byref(rr), ws.data_ptr(), ws.numel(), self.sp), "nystrom")
        return int(rr.value)

    # asynchronous sketch stages: failures land in device status words
    def gaussian_async(self, seed: int, out: torch.Tensor, flag: torch.Tensor) -> None:
        import numpy as np

        st = np.random.PCG64(seed).state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        m64 = (1 << 64) - 1
        count = out.numel()
        ws = self.workspace("gauss", self.L.nys_gaussian_workspace(count))
        self.launches += 1
        check(self.L.nys_gaussian_async_f64(s >> 64, s & m64, inc >> 64, inc & m64, count, out.data_ptr(),
                                            flag.data_ptr(), ws.data_ptr(), ws.numel(), self.sp), "gaussian")

    def sketch_workspace(self, n: int, s: int, r: int) -> torch.Tensor:
        return self.workspace("sketch", max(self.L.nys_nystrom_workspace(n, s, r),
                                            self.L.nys_orthonormalize_workspace(n, s)))

    def orthonormalize_async(self, Om, Q, info: torch.Tensor, r: int) -> None:
        n, s = Om.shape
        ws = self.sketch_workspace(n, s, r)
        self.launches += 1
        check(self.L.nys_orthonormalize_async_f64(n, s, Om.data_ptr(), Q.data_ptr(), info.data_ptr(), ws.data_ptr(),
                                                  ws.numel(), self.sp), "orthonormalize")

    def nystrom_core_async(self, Q, Y, U, lam, r, info: torch.Tensor) -> None:
        n, s = Q.shape
        ws = self.sketch_workspace(n, s, r)
        self.launches += 1
        check(self.L.nys_nystrom_core_async_f64(n, s, r, Q.data_ptr(), Y.data_ptr(), U.data_ptr(), lam.data_ptr(),
                                                info.data_ptr(), ws.data_ptr(), ws.numel(), self.sp), "nystrom")

    def syevj(self, A, V, w) -> None:
        s = A.shape[0]
        ws = self.workspace("syevj", self.L.nys_syevj_workspace(s))
        self.launches += 1
        check(self.L.nys_syevj_f64(s, A.data_ptr(), V.data_ptr(), w.data_ptr(), ws.data_ptr(), ws.numel(),
                                   self.sp), "syevj")

    def ml_tail(self, loss, A, x, z, b, T, w, AT, rowsums, gb=None) -> None:
        """One-pass A{x,z} + loss epilogue + A^T{...} for wide rows (cluster tail);
        with gb = A^T b the square loss streams two products instead of three."""
        rows, n = A.shape
        ws = self.workspace("tail_gemvT", self.L.nys_tail_cluster_workspace(rows, n))
        self.launches += 1
        e = self._t0("ml_tail")
        if gb is None:
            check(self.L.nys_ml_tail_f64(A.data_ptr(), rows, n, A.stride(0), x.data_ptr(), _p(z), b.data_ptr(),
                                         _lib.LOSS[loss], T.data_ptr(), w.data_ptr(), AT.data_ptr(),
                                         rowsums.data_ptr(), ws.data_ptr(), ws.numel(), self.sp), "ml_tail")
        else:
            check(self.L.nys_ml_tail_gb_f64(A.data_ptr(), rows, n, A.stride(0), x.data_ptr(), _p(z), b.data_ptr(),
                                            _lib.LOSS[loss], gb.data_ptr(), T.data_ptr(), w.data_ptr(),
                                            AT.data_ptr(), rowsums.data_ptr(), ws.data_ptr(), ws.numel(), self.sp),
                  "ml_tail")
        self._t1(e)

    # ------------------------------------- sparse / general-operator engine --
    def csr_spmv(self, csr, x, y, alpha=1.0, dscale=None, beta=0.0, zin=None) -> None:
        """y = alpha * dscale o (A x) + beta * zin for a device CSR ``csr``."""
        self.launches += 1
        check(self.L.nys_csr_spmv_f64(csr.rows, csr.rowptr.data_ptr(), csr.col.data_ptr(), csr.val.data_ptr(),
                                      x.data_ptr(), float(alpha), _p(dscale), float(beta), _p(zin), y.data_ptr(),
                                      csr.group, self.sp), "csr_spmv")

    def csr_spmm(self, csr, X, Y, dscale=None) -> None:
        """Y = diag(dscale) A X (X: cols x s row-major)."""
        self.launches += 1
        check(self.L.nys_csr_spmm_f64(csr.rows, csr.rowptr.data_ptr(), csr.col.data_ptr(), csr.val.data_ptr(),
                                      X.data_ptr(), X.stride(0), X.shape[1], _p(dscale), Y.data_ptr(), Y.stride(0),
                                      self.sp), "csr_spmm")

    def csr_transpose(self, rows, cols, rowptr, col, val, trowptr, tcol, tval) -> None:
        ws = self.workspace("csrT", self.L.nys_csr_transpose_workspace(rows, cols))
        self.launches += 1
        check(self.L.nys_csr_transpose(rows, cols, rowptr.data_ptr(), col.data_ptr(), val.data_ptr(),
                                       trowptr.data_ptr(), tcol.data_ptr(), tval.data_ptr(), ws.data_ptr(),
                                       ws.numel(), self.sp), "csr_transpose")

    def vmul(self, a, d, x, b, y) -> None:
        """y = a (d o x) + b y."""
        self.launches += 1
        check(self.L.nys_vmul_f64(x.numel(), float(a), d.data_ptr(), x.data_ptr(), float(b), y.data_ptr(),
                                  self.sp), "vmul")

    def bcast(self, src, scale, y) -> None:
        self.launches += 1
        check(self.L.nys_bcast_f64(y.numel(), src.data_ptr(), float(scale), y.data_ptr(), self.sp), "bcast")

    def vstats(self, x, y, out) -> None:
        """out = [sum v, sum v^2, max|v|] of v = x - y (y may be None)."""
        self.launches += 1
        check(self.L.nys_vstats_f64(x.numel(), x.data_ptr(), _p(y), out.data_ptr(), self.red.data_ptr(),
                                    self.sp), "vstats")

    def absstats(self, v, lambda1, out) -> None:
        """out = [sum |v|, sum (|v| - lambda1)_+^2, max |v|]."""
        self.launches += 1
        check(self.L.nys_absstats_f64(v.numel(), v.data_ptr(), float(lambda1), out.data_ptr(), self.red.data_ptr(),
                                      self.sp), "absstats")

    def gdual(self, grad, mtu, rho, out) -> None:
        self.launches += 1
        check(self.L.nys_gdual_f64(grad.numel(), grad.data_ptr(), mtu.data_ptr(), float(rho), out.data_ptr(),
                                   self.red.data_ptr(), self.sp), "gdual")

    def box_cert(self, du, md, lo, hi, out) -> None:
        self.launches += 1
        check(self.L.nys_box_cert_f64(lo.numel(), _p(du), _p(md), lo.data_ptr(), hi.data_ptr(), out.data_ptr(),
                                      self.red.data_ptr(), self.sp), "box_cert")

    def box_violation(self, z, lo, hi, out) -> None:
        self.launches += 1
        check(self.L.nys_box_violation_f64(z.numel(), z.data_ptr(), lo.data_ptr(), hi.data_ptr(), out.data_ptr(),
                                           self.red.data_ptr(), self.sp), "box_violation")


_CACHE: dict = {}


def get_kernels() -> Kernels:
    """Kernels bound to the current device and torch stream (cached, so the
    operator-level API reuses its workspaces)."""
    _lib.lib()  # CapabilityError without the library or an sm_100 GPU (no CPU fallback)
    dev = torch.cuda.current_device()
    sp = torch.cuda.current_stream(dev).cuda_stream
    k = _CACHE.get((dev, sp))
    if k is None:
        k = Kernels(torch.device("cuda", dev))
        _CACHE[(dev, sp)] = k
    return k
