"""Inexact ADMM engine on the B200 (``/root/reference/pkg/src/nysopt/admm.py``).

Same public surface as the reference -- ``solve``, ``SolverOptions``,
``SolveResult``, ``IterationRecord``, ``PenaltyEvent``, ``Status``, ... --
and the same control flow line for line (CG tolerance schedule, gap / residual
termination, over-relaxation, windows, cycle guard, penalty adaptation, QP
infeasibility tests), so iteration counts follow the reference.  What changes
is where the arithmetic runs: all vectors live in HBM and every numeric step
is a sm_100a kernel behind the C ABI:

  per ADMM iteration (dense ML problem, M = I, c = 0)
    x-update   rhs + initial residual (fused K8) -> device PCG (K3 HVP, K6, K7)
    z/u        one fused over-relaxation/prox/dual kernel (K8)
    A-pass     one 2-RHS GEMV  A{x, z}                       (K1)
    epilogue   l'(Ax-b), w, w o Ax, nu = l'(Az-b) + sums       (K12)
    A^T-pass   one 3-RHS GEMV^T A^T{l', w o Ax, nu}            (K2)
    norms      residual norms / objective / gap pieces (K9)  -> one D2H

The reference spends 7 A-passes and 5 A^T-passes per iteration outside CG
(SURVEY.md §3.1); caching Ax, A^T l' and A^T(w o Ax) across iterations
brings that to one 2-RHS A-pass and one 3-RHS A^T-pass with identical
arithmetic meaning (differences are at the roundoff floor).

Row sharding (``torch.distributed`` initialised): each rank holds a row block
of A and b; the A^T-pass output and the row sums are all-reduced in one packed
buffer, HVP partials are all-reduced inside CG, the sketch Y is all-reduced.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
from collections import deque
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable, Optional

import numpy as np
import torch

from . import _lib
from .dist import Shard, current_shard
from .errors import CapabilityError, DataError, NotSPDError, NumericalError
from .krylov import CgReport, CgWork, cg_tolerance, pcg_batched, pcg_device
from .operators import DenseOperator, IdentityOperator, to_device
from .problems import GenericProblem, lower
from .sketch import (NystromPreconditioner, NystromSketch, default_sketch_rank, raw_test_matrix, sketch_device,
                     sketch_device_launch, sketch_width)

PENALTY_ADAPT_CUTOFF = 1000  # admm.py:29
DELTA_WINDOW = 25  # admm.py:33


class Status(str, Enum):
    OPTIMAL = "optimal"
    PRIMAL_INFEASIBLE = "primal_infeasible"
    DUAL_INFEASIBLE = "dual_infeasible"
    PRIMAL_AND_DUAL_INFEASIBLE = "primal_and_dual_infeasible"
    ITERATION_LIMIT = "iteration_limit"
    TIME_LIMIT = "time_limit"


@dataclass
class SolverOptions:
    """Tunable parameters (admm.py:45-99); same names, defaults and validation."""

    sigma: float = 1e-6
    gamma: float = 1.2
    sketch_rank: Optional[int] = None
    resketch_every: int = 20
    norm_kind: str = "l2"
    eps_abs: float = 1e-4
    eps_rel: float = 1e-4
    eps_inf: float = 1e-8
    alpha: float = 1.6
    tau: float = 2.0
    mu: float = 10.0
    rho0: float = 1.0
    penalty_update_every: int = 25
    penalty_warmup: int = 100
    max_iter: int = 10000
    time_limit: Optional[float] = None
    use_preconditioner: bool = True
    exact_x_solve: bool = False
    use_dual_gap: Optional[bool] = None
    eps_dual_gap: float = 1e-4
    rng_seed: int = 0
    assume_full_rank: bool = False
    check_rank: bool = False
    custom_stop: Optional[Callable] = None
    record_iterates: bool = False
    track_averaged_objective: bool = False
    prox_tol0: float = 1e-8

    def __post_init__(self):
        if self.sigma < 0:
            raise DataError("sigma must be nonnegative")
        if self.gamma <= 1:
            raise DataError("gamma must exceed 1")
        if not 0 < self.alpha < 2:
            raise DataError("over-relaxation alpha must lie in (0, 2)")
        if self.tau <= 1 or self.mu <= 1:
            raise DataError("penalty factors tau and mu must exceed 1")
        if self.rho0 <= 0:
            raise DataError("initial penalty must be positive")
        if self.norm_kind not in ("l2", "linf"):
            raise DataError("norm_kind must be 'l2' or 'linf'")


@dataclass
class SolverState:
    """Host snapshot of the iterate state (admm.py:101-127); filled for
    ``custom_stop`` callbacks and at the end of a solve."""

    x: np.ndarray
    z: np.ndarray
    u: np.ndarray
    rho: float
    k: int = 0
    x_prev: Optional[np.ndarray] = None
    u_prev: Optional[np.ndarray] = None
    Mx: Optional[np.ndarray] = None
    x_bar_sum: Optional[np.ndarray] = None
    z_bar_sum: Optional[np.ndarray] = None
    bar_count: int = 0

    @property
    def x_bar(self):
        return None if self.bar_count == 0 else self.x_bar_sum / self.bar_count

    @property
    def z_bar(self):
        return None if self.bar_count == 0 else self.z_bar_sum / self.bar_count


@dataclass
class Residuals:
    """admm.py:36-43 (same field order).  The engines fill the norms from their
    fused reductions and leave the vectors None; the single-step API
    (``compute_residuals``) returns them."""

    rp: Optional[np.ndarray]
    rd: Optional[np.ndarray]
    rp_norm: float
    rd_norm: float
    primal_scale: float
    dual_scale: float
    size: int = 0


@dataclass
class IterationRecord:
    k: int
    rp_norm: float
    rd_norm: float
    objective: float
    rho: float
    cg_iters: int
    cg_tol: float
    linsys_s: float
    prox_s: float
    gap: Optional[float] = None
    avg_objective: Optional[float] = None


@dataclass
class PenaltyEvent:
    k: int
    rho_old: float
    rho_new: float
    dual_jump_rel: float


@dataclass
class Timings:
    setup_s: float = 0.0
    precond_s: float = 0.0
    linsys_total_s: float = 0.0
    prox_total_s: float = 0.0
    total_s: float = 0.0


@dataclass
class SolveResult:
    status: Status
    x: np.ndarray
    z: np.ndarray
    u: np.ndarray
    objective: float
    iterations: int
    rp_norm: float
    rd_norm: float
    history: list
    timings: Timings
    x_bar: Optional[np.ndarray] = None
    z_bar: Optional[np.ndarray] = None
    certificate_primal: Optional[np.ndarray] = None
    certificate_dual: Optional[np.ndarray] = None
    penalty_events: list = field(default_factory=list)
    iterates: Optional[list] = None
    gap: Optional[float] = None
    device_stats: dict = field(default_factory=dict)

    @property
    def certificate(self):
        if self.status in (Status.PRIMAL_INFEASIBLE, Status.PRIMAL_AND_DUAL_INFEASIBLE):
            return self.certificate_primal
        if self.status == Status.DUAL_INFEASIBLE:
            return self.certificate_dual
        return None


# stats buffer layout (doubles)
_S_NORMS = 0  # 16 (nys_admm_norms_f64)
_S_WIN = 16  # 17 (window norms)
_S_INF = 33  # 6 (QP infeasibility pieces)
_S_PDX = 39  # 1 (||P dx||^2)
_S_CONJ = 40  # 3 (scaled conjugate sums)
_S_DUAL = 44  # 2 (penalty change)
_S_STOP = 46  # 1 (the device's termination decision, nys_admm_tail.stop_slot)
_S_LEN = 48
# device readback block: row sums (8) | CG scalars (16) | stats (_S_LEN)
_RB_LEN = 8 + 16 + _S_LEN


def _host_buffer(n, device):
    t = torch.zeros(n, dtype=torch.float64)
    return t.pin_memory() if device.type == "cuda" else t


@dataclass
class _Issued:
    """An ADMM iteration launched on the device (one-iteration-ahead pipeline)."""

    k: int
    par: int
    slot: int
    after: list
    batch: int
    tag: int
    shift: float
    exact: bool
    win_before: list
    reissue: Optional["_Issued"] = None
    polled: bool = False  # the readback block carries tag `tag` (no stream event to wait on)
    ring: bool = False    # iteration time from the per-iteration mark ring (no ev[0], ev[2])
    dev_stop: bool = False  # the tail ran the device stop test (it closes k+1's gate when it holds)


class _ParityWork:
    """CgWork view with the CG scalar block of one parity."""

    def __init__(self, cg: CgWork, sc: torch.Tensor):
        self.r, self.p, self.z, self.Ap, self.sc = cg.r, cg.p, cg.z, cg.Ap, sc


class _Engine:
    """Device-resident state and per-iteration kernel schedule of one solve."""

    def __init__(self, gp: GenericProblem, opts: SolverOptions, kx, shard: Optional[Shard]):
        self.kx = kx
        self.opts = opts
        self.gp = gp
        n = self.n = gp.n
        self.is_ml = gp.ml is not None
        self.t_events = None  # optional per-kernel CUDA-event timing (bench)
        if self.is_ml:
            p = gp.ml
            if not isinstance(p.A, DenseOperator):
                raise CapabilityError("the B200 path supports dense data matrices (DenseOperator) only")
            if p.loss.kind not in _lib.LOSS:
                raise CapabilityError(f"loss {p.loss.kind!r} is not implemented on the B200 path")
            self.shard = shard or current_shard(p.N)
            # b first: a host->device copy queued behind A's would wait for all of it
            self.b = to_device(p.b[self.shard.row_start:self.shard.row_stop], kx.device)
            # a pinned host matrix uploads in row chunks behind the setup (run())
            self.A = p.A.device_rows(self.shard, kx.device, overlap=True)
            self._a_chunks = p.A.take_pending(self.A)
            rows = self.rows = self.A.shape[0]
            self.loss = p.loss.kind
            self.l1, self.l2 = float(p.lambda1), float(p.lambda2)
            self.const_hess = p.loss.deriv2_constant
            self.diag_shift = self.l2
            # row-space buffers
            self.AXZ = kx.empty(2, rows)
            self.T = kx.empty(3, rows)  # l'(Ax-b), w o Ax, nu
            self.w = kx.empty(rows)
            # packed all-reduce buffer: A^T outputs (3 n) + row sums (8), then
            # the CG scalars and the stats so one D2H copy reads a whole iteration
            self.red = kx.zeros(3 * n + _RB_LEN)
            self.AT = self.red[:3 * n].view(3, n)  # gA, hxA, atnu
            self.rb_dev = self.red[3 * n:]
            # g_b = A^T b for the square loss: the one-pass tail then streams
            # A^T (A x) and A^T (A z) and subtracts it (nys_admm_tail.gb)
            # (row-sharded: this rank's A_loc^T b_loc, never all-reduced -- it is
            # subtracted from the rank's partial before the ranks' AT are summed)
            self.gb = kx.empty(n) if self.loss == "square" else None
            self._gb_ready = False
        else:
            qp = gp.qp
            if not isinstance(qp.P, DenseOperator):
                raise CapabilityError("the B200 path supports a dense QP matrix P only")
            if not isinstance(qp.M, IdentityOperator):
                raise CapabilityError("the B200 path supports QPs with M = I only")
            self.shard = Shard(0, 1, 0, n, n)  # P is replicated
            self.P = qp.P.device_rows(None, kx.device)
            self._a_chunks = None
            self.q = to_device(qp.q, kx.device)
            self.lo = to_device(qp.box.l, kx.device)
            self.hi = to_device(qp.box.u, kx.device)
            self.const_hess = True
            self.diag_shift = 0.0
            self.Px = kx.empty(1, n)
            self.dx = kx.empty(1, n)
            self.Pdx = kx.empty(1, n)
            self.rb_dev = kx.zeros(_RB_LEN)
        self.rowsums = self.rb_dev[:8]
        self.XZ = kx.zeros(2, n)  # x, z rows (one 2-RHS GEMV operand)
        self.x, self.z = self.XZ[0], self.XZ[1]
        self.u = kx.zeros(n)
        self.xbar = kx.zeros(n)
        self.zbar = kx.zeros(n)
        self.rhs = kx.empty(n)
        self.cg = CgWork(kx, n, self.rb_dev[8:8 + _lib.CG_NSLOTS])
        self.stats = self.rb_dev[8 + _lib.CG_NSLOTS:]
        self.rb_host = _host_buffer(_RB_LEN, kx.device)
        self.ring = kx.empty(DELTA_WINDOW + 2, n)
        self.uring = kx.empty(DELTA_WINDOW + 2, n) if not self.is_ml else None
        self.U = None
        self.lam = None
        self.pc_nu = 1.0
        self._last_cg = 8  # first x-update runs to the 1e-12 floor: start with a larger batch

    # ----------------------------------------------------------- passes --
    def evaluate(self, with_z: bool) -> None:
        """Data passes at the current (x, z): ML -> A{x,z}, loss epilogue,
        A^T{l', w o Ax, nu} (+ all-reduce); QP -> P x."""
        kx = self.kx
        if self.is_ml:
            k = 2 if with_z else 1
            kx.gemv(self.A, self.XZ[:k], self.AXZ[:k])
            kx.ml_rowwise(self.loss, self.AXZ[0], self.AXZ[1] if with_z else None, self.b,
                          self.T[0], self.w, self.T[1], self.T[2] if with_z else None, self.rowsums)
            kT = 3 if with_z else 2
            if self.gb is not None and not self._gb_ready and not with_z:
                # A^T b rides along as the third product of the setup pass
                self.T[2].copy_(self.b)
                kx.gemvT(self.A, self.T[:3], self.AT[:3])
                self.gb.copy_(self.AT[2])
                self._gb_ready = True
            else:
                kx.gemvT(self.A, self.T[:kT], self.AT[:kT])
                if self.gb is not None and not self._gb_ready:
                    kx.gemvT(self.A, self.b.view(1, -1), self.gb.view(1, -1))
                    self._gb_ready = True
            if self.shard.sharded:
                self.shard.allreduce(self.red[:3 * self.n + 8])
        else:
            kx.gemv(self.P, self.XZ[:1], self.Px)

    def norms(self, with_nu: bool) -> None:
        kx = self.kx
        if self.is_ml:
            kx.admm_norms(self.x, self.z, self.u, self.AT[0], None, self.l2, self.rho,
                          self.AT[2] if with_nu else None, self.l1, None, None, self.stats[_S_NORMS:_S_NORMS + 16])
        else:
            kx.admm_norms(self.x, self.z, self.u, self.Px[0], self.q, 0.0, self.rho, None, 0.0,
                          self.lo, self.hi, self.stats[_S_NORMS:_S_NORMS + 16])

    def read_stats(self) -> np.ndarray:
        """stats followed by the row sums (one D2H copy of the readback block)."""
        _, st = self._read_block()
        return st

    # ----------------------------------------------------------- matvec --
    def matvec(self, shift: float):
        kx = self.kx
        if self.is_ml:
            d = None if self.loss == "square" else self.w
            tot = self.diag_shift + shift
            if not self.shard.sharded:
                def mv(v, out, dot):
                    kx.hvp(self.A, d, v, tot, out, dot, True)
            else:
                def mv(v, out, dot):
                    kx.hvp(self.A, d, v, 0.0, out, None, False)
                    self.shard.allreduce(out)
                    kx.shift_dot(v, tot, out, dot)
        else:
            def mv(v, out, dot):
                kx.gemv(self.P, v.view(1, -1), out.view(1, -1))
                kx.shift_dot(v, shift, out, dot)
        return mv

    def precond(self):
        if self.U is None:
            return None
        kx = self.kx
        return lambda v, out, rdot, rz: kx.precond_apply(self.U, self.lam, self.pc_nu, v, out, rdot, rz)

    # ----------------------------------------------------------- sketch --
    def _sketch_target(self, chunks=None):
        """(cols, reduce): Y = H Q for the sketch target and the all-reduce of
        Y's row-shard partials (None unsharded).  ``chunks``: A is still being
        uploaded in row blocks [(r0, r1, event)]: Y = sum_c A_c^T (A_c Q), each
        block's GEMMs queued behind its copy (square loss: no row weights)."""
        kx = self.kx
        n = self.n
        if self.is_ml and chunks:
            A = self.A

            def cols(Q):
                rows = A.shape[0]
                s = Q.shape[1]
                Z = kx.empty(rows, s)
                Y = kx.empty(n, s)
                for c, (r0, r1, ev) in enumerate(chunks):
                    kx.stream.wait_event(ev)
                    kx.gemm(0, 0, r1 - r0, s, n, 1.0, A[r0:r1], A.stride(0), Q, s, 0.0, Z[r0:r1], s)
                    kx.gemm(1, 0, n, s, r1 - r0, 1.0, A[r0:r1], A.stride(0), Z[r0:r1], s, 0.0 if c == 0 else 1.0,
                            Y, s)
                return Y

            return cols, None
        if self.is_ml:
            A, w = self.A, (None if self.loss == "square" else self.w)

            def cols(Q):
                rows = A.shape[0]
                s = Q.shape[1]
                Z = kx.empty(rows, s)
                kx.gemm(0, 0, rows, s, n, 1.0, A, A.stride(0), Q, s, 0.0, Z, s)
                if w is not None:
                    kx.row_scale(Z, w)
                Y = kx.empty(n, s)
                kx.gemm(1, 0, n, s, rows, 1.0, A, A.stride(0), Z, s, 0.0, Y, s)
                return Y

            reduce = self.shard.allreduce if self.shard.sharded else None
        else:
            P = self.P

            def cols(Q):
                s = Q.shape[1]
                Y = kx.empty(n, s)
                kx.gemm(0, 0, n, s, n, 1.0, P, P.stride(0), Q, s, 0.0, Y, s)
                return Y

            reduce = None
        return cols, reduce

    def sketch(self, seed: int, omega: Optional[np.ndarray] = None, chunks=None) -> None:
        cols, reduce = self._sketch_target(chunks)
        U, lam = sketch_device(self.kx, cols, self.n, self.r_sk, seed, omega=omega, reduce=reduce)
        if U.shape[1] == 0:
            self.U, self.lam = None, None
        else:
            self.U, self.lam = U, lam
        self.n_sketches += 1

    def sketch_launch(self, seed: int):
        """Enqueue the sketch of iteration k (seed rng_seed + k) right behind
        iteration k-1 on the stream, before the host has read k-1: its input
        (the Hessian weights at k-1's iterate) is what k-1's tail leaves on the
        device.  None where only the synchronous sketch applies."""
        cols, reduce = self._sketch_target()
        if reduce is not None:
            return None
        return sketch_device_launch(self.kx, cols, self.n, self.r_sk, seed)

    def sketch_adopt(self, launch) -> None:
        self.U, self.lam = launch.U, launch.lam
        self.n_sketches += 1

    # ------------------------------------------------------------- run ---
    def run(self, x0, z0, u0, callback, t_start) -> SolveResult:
        opts, kx, n = self.opts, self.kx, self.n

        def warm(v, name, dst):
            if v is None:
                return
            vt = to_device(v, kx.device)
            if vt.shape != (n,):
                raise DataError(f"warm start {name} must have length {n}, got shape {tuple(vt.shape)}")
            dst.copy_(vt)

        warm(x0, "x0", self.x)
        warm(z0, "z0", self.z)
        warm(u0, "u0", self.u)
        self.rho = float(opts.rho0)
        self.n_sketches = 0

        # offset policy (admm.py:462-474): both in-scope lowerings are full rank
        sigma_eff = 0.0 if (self.gp.full_rank or opts.assume_full_rank) else opts.sigma
        use_gap = opts.use_dual_gap
        if use_gap is None:
            use_gap = self.is_ml and self.gp.ml.loss.has_conj
        if use_gap and not self.is_ml:
            raise DataError("the duality-gap criterion requires an ML problem")
        self.use_gap = use_gap
        # CUDA path: batched CG + predicated iteration tail (one host round trip
        # per ADMM iteration).  Row-sharded runs use it too: the drivers call the
        # all-reduce hook (nys_reduce_fn) between a rank's partials and their use,
        # so the exchange is enqueued on the stream like any kernel.
        self.fast = hasattr(kx, "admm_tail") and (
            not self.shard.sharded or os.environ.get("NYS_SHARD_FAST", "1") != "0")
        self.sigma_eff = sigma_eff
        if self.fast:
            self._make_tail()
        # one-iteration-ahead launches: iteration k+1 is queued before the host
        # has read k, whenever nothing that k's readback can trigger (penalty
        # change, cycle guard, resketch) changes k+1's launch parameters; a
        # stop at k rolls back k+1 from the snapshot its head kernel took
        lookahead = (self.fast and opts.custom_stop is None and not opts.record_iterates
                     and not opts.track_averaged_objective and os.environ.get("NYS_LOOKAHEAD", "1") != "0")
        pending: Optional[_Issued] = None
        # device-side termination (admm.py:227-240): the fused ML epilogue runs the
        # stop test itself and keeps the gate of an iteration launched ahead closed,
        # so a solve that stops at k never executes k+1 (no rollback)
        if lookahead and self.is_ml and not self.shard.sharded and _lib.dev_env("NYS_DEVICE_STOP", "1") != "0":
            for t in self._tails:
                t.stop_on, t.stop_gap = 1, 1 if self.use_gap else 0
                t.stop_linf = 1 if opts.norm_kind == "linf" else 0
                t.stop_slot = _S_STOP
                t.stop_eps_gap, t.stop_eps_abs, t.stop_eps_rel = opts.eps_dual_gap, opts.eps_abs, opts.eps_rel
                t.stop_sqrt_n = math.sqrt(n)

        timings = Timings()
        r_sk = opts.sketch_rank or default_sketch_rank(n)
        self.r_sk = max(1, min(r_sk, n))
        nu_identity = lambda rho: rho + sigma_eff + self.diag_shift  # admm.py:490-491

        # hess.update(x0) and the data passes at x0.  While A is still arriving
        # over PCIe (a pinned host matrix), a square-loss problem -- whose sketch
        # target A^T A does not depend on x0 -- sketches first, block by block
        # behind the copies; the data passes then wait for the whole matrix.
        chunks, self._a_chunks = self._a_chunks, None
        sketch_first = bool(chunks) and self.is_ml and self.loss == "square" and opts.use_preconditioner \
            and not self.shard.sharded

        def wait_all():
            for _, _, ev in chunks or ():
                kx.stream.wait_event(ev)

        if not sketch_first:
            wait_all()
            self.evaluate(with_z=False)
        last_sketch = 0
        have_pc = False
        if opts.use_preconditioner:
            t0 = time.perf_counter()
            self.sketch(opts.rng_seed, chunks=chunks if sketch_first else None)
            timings.precond_s += time.perf_counter() - t0
            self.pc_nu = nu_identity(self.rho)
            have_pc = True
        if sketch_first:
            wait_all()
            self.evaluate(with_z=False)
        self.norms(with_nu=False)
        st = self.read_stats()
        res = self._residuals(st)
        last_obj = self._objective(st)
        timings.setup_s = time.perf_counter() - t_start

        history: list[IterationRecord] = []
        events: list[PenaltyEvent] = []
        iterates = [] if opts.record_iterates else None
        win: deque = deque(maxlen=DELTA_WINDOW + 1)  # slots of (x, u) copies in the device rings
        self._win_append(win)
        status = Status.ITERATION_LIMIT
        cert_p = cert_d = None
        gap = None
        rho_frozen = False
        cycle_hits = 0
        best_res = np.inf
        trend: deque = deque(maxlen=DELTA_WINDOW + 1)
        bar_count = 0
        k_done = 0
        omega_next = None
        early = None  # sketch of the next iteration, enqueued behind the current one

        for k in range(1, opts.max_iter + 1):
            k_done = k  # the reference sets state.k = k before its time check (admm.py:534-537)
            if opts.time_limit is not None and time.perf_counter() - t_start > opts.time_limit:
                status = Status.TIME_LIMIT
                if pending is not None:
                    self._rollback()
                break
            # resketch on the cadence for iterate-dependent Hessians (admm.py:545-551)
            # (never due for an iteration launched ahead, by the lookahead rule)
            early_check = None
            if have_pc and not self.const_hess and k - last_sketch >= opts.resketch_every:
                t0 = time.perf_counter()
                if early is not None and early.seed == opts.rng_seed + k:
                    # enqueued behind iteration k-1 (see below); its status is read
                    # once iteration k is queued behind it
                    self.sketch_adopt(early)
                    early_check = early
                else:
                    self.sketch(opts.rng_seed + k)
                early = None
                timings.precond_s += time.perf_counter() - t0
                self.pc_nu = nu_identity(self.rho)
                last_sketch = k
            tol = 1e-12 if opts.exact_x_solve else cg_tolerance(k, res.rp_norm, res.rd_norm, opts.gamma)

            # x-update (admm.py:243-275): rhs and the initial residual r = b - A x0
            t0 = time.perf_counter()
            shift = self.rho + sigma_eff
            if self.fast:
                # head (rhs, device tolerance), CG batches with the device stop
                # test, predicated tail (z/u, data passes, norms, windows), readback
                it = pending if pending is not None else self._issue(k, shift, list(win), opts.exact_x_solve)
                pending = None
                if early_check is not None and not early_check.ok():
                    # the pipelined sketch flagged a failure (never expected for a
                    # Hessian + shift): undo iteration k, sketch synchronously
                    # (its fallbacks), and issue k again
                    self._rollback(resume=True, k=k - 1)
                    t0 = time.perf_counter()
                    self.sketch(opts.rng_seed + k)
                    timings.precond_s += time.perf_counter() - t0
                    it = self._issue(k, shift, list(win), opts.exact_x_solve)
                if lookahead and self._may_speculate(k, it, have_pc, last_sketch, rho_frozen, cycle_hits):
                    pending = self._issue(k + 1, shift, it.after, opts.exact_x_solve)
                elif (lookahead and have_pc and not self.const_hess and k + 1 <= opts.max_iter
                      and (k + 1) - last_sketch >= opts.resketch_every):
                    # the next iteration resketches: enqueue the sketch now, behind
                    # iteration k (wasted only if k terminates the solve)
                    t0 = time.perf_counter()
                    early = self.sketch_launch(opts.rng_seed + k + 1)
                    timings.precond_s += time.perf_counter() - t0
                rep, st, linsys_s, prox_s = self._retire(it, pending)
                if early is not None and self._cg_continued:
                    early = None  # k's CG needed more launches: the sketch saw a no-op tail
                if pending is not None and pending.reissue is not None:
                    pending = pending.reissue
                spec = it.slot
            else:
                if self.is_ml:
                    kx.admm_rhs(self.AT[1], self.AT[0], None, self.l2, sigma_eff, self.rho, shift,
                                self.x, self.z, self.u, self.rhs, self.cg.r, self.cg.sc)
                else:
                    kx.admm_rhs(self.Px[0], self.Px[0], self.q, 0.0, sigma_eff, self.rho, shift,
                                self.x, self.z, self.u, self.rhs, self.cg.r, self.cg.sc)
                rep = pcg_device(self.cg, self.matvec(shift), self.rhs, self.x, self.precond(), tol, 10 * n,
                                 started=True)
                linsys_s = time.perf_counter() - t0
                # z/u update (admm.py:562-576) + averaged sums (admm.py:580-583)
                t0 = time.perf_counter()
                if self.is_ml:
                    kx.admm_zu(self.x, self.z, self.u, opts.alpha, _lib.PROX_SOFT, self.l1 / self.rho, None, None,
                               self.xbar, self.zbar, k >= 2)
                else:
                    kx.admm_zu(self.x, self.z, self.u, opts.alpha, _lib.PROX_BOX, 0.0, self.lo, self.hi,
                               self.xbar, self.zbar, k >= 2)
                prox_s = time.perf_counter() - t0
                # data passes, norms, and (speculatively) the window reductions
                self.evaluate(with_z=use_gap)
                self.norms(with_nu=use_gap)
                spec = self._win_speculate(win)
                st = self.read_stats()
            self._last_cg = rep.iterations
            timings.linsys_total_s += linsys_s
            timings.prox_total_s += prox_s
            if k >= 2:
                bar_count += 1
            res = self._residuals(st)
            objective = self._objective(st)
            last_obj = objective
            gap = self._gap(st) if use_gap else None

            avg_obj = None
            if opts.track_averaged_objective and bar_count > 0:
                avg_obj = self._averaged_objective(bar_count)

            history.append(IterationRecord(k, res.rp_norm, res.rd_norm, objective, self.rho, rep.iterations,
                                           tol, linsys_s, prox_s, gap, avg_obj))
            if iterates is not None:
                iterates.append((self.x.cpu().numpy(), self.z.cpu().numpy(), self.u.cpu().numpy()))
            if callback is not None:
                callback(k, res.rp_norm, res.rd_norm, objective, self.rho, rep.iterations)

            if opts.custom_stop is not None:
                if opts.custom_stop(self.gp, self._snapshot(k, bar_count)):
                    status = Status.OPTIMAL
                    break
            elif self._terminated(res, gap):
                status = Status.OPTIMAL
                if pending is not None:
                    if it.dev_stop and st[_S_STOP] == 1.0:
                        pending = None  # the device kept k+1's gate closed: k+1 did nothing
                    else:
                        self._rollback()
                break
            if self.fast and it.dev_stop and st[_S_STOP] == 1.0:
                # the device stopped where the host continues (not expected: the same
                # operations on the same values): open k+1's gate, launch it again
                if _lib.dev_env("NYS_STOP_DEBUG", None):
                    print(f"device/host stop mismatch at k={k}: gap={gap} res={res}", flush=True)
                self.gates[(k + 1) % 2] = 1.0
                if pending is not None:
                    pending = self._issue(pending.k, pending.shift, pending.win_before, pending.exact)

            # windows (admm.py:621-634): commit the speculative append
            self._win_commit(win, spec)
            if not self.is_ml and len(win) == DELTA_WINDOW + 1:
                st_inf, near, cp, cd = self._infeasibility(st, win)
                if near:
                    rho_frozen = True
                if st_inf is not None:
                    status, cert_p, cert_d = st_inf, cp, cd
                    if pending is not None:
                        self._rollback()
                    break

            # cycle guard (admm.py:643-675)
            best_res = min(best_res, max(res.rp_norm, res.rd_norm))
            trend.append(best_res)
            if len(win) >= 4 and not rho_frozen and k <= PENALTY_ADAPT_CUTOFF:
                step = math.sqrt(max(st[_S_WIN + 1], 0.0))
                xk_norm = math.sqrt(max(st[_S_WIN], 0.0))
                locked = False
                if step > 1e-8 * max(1.0, xk_norm):
                    nper = min(len(win) - 1, 10) - 1
                    rg = min(math.sqrt(max(st[_S_WIN + 2 + j], 0.0)) for j in range(nper))
                    locked = rg <= 1e-3 * step
                cycle_hits = cycle_hits + 1 if locked else 0
                stagnant = len(trend) == trend.maxlen and trend[-1] >= 0.99 * trend[0]
                if cycle_hits >= 5 and stagnant:
                    if pending is not None:  # not expected under the lookahead rule
                        self._rollback(resume=True, k=k)
                        pending = None
                    cycle_hits = 0
                    trend.clear()
                    events.append(self._change_penalty(k, self.rho * opts.tau, have_pc, nu_identity))
                    win.clear()
                    self._win_append(win)

            # balanced-residual penalty rule (admm.py:677-698)
            if (not rho_frozen and opts.penalty_update_every > 0 and k >= opts.penalty_warmup
                    and k % opts.penalty_update_every == 0 and k <= PENALTY_ADAPT_CUTOFF):
                t_p = math.sqrt(n) * opts.eps_abs + opts.eps_rel * res.primal_scale
                t_d = math.sqrt(n) * opts.eps_abs + opts.eps_rel * res.dual_scale
                if t_p > 0 and t_d > 0:
                    pm, dm = res.rp_norm / t_p, res.rd_norm / t_d
                else:
                    pm, dm = res.rp_norm, res.rd_norm
                new = None
                if pm > opts.mu * dm:
                    new = self.rho * opts.tau
                elif dm > opts.mu * pm:
                    new = self.rho / opts.tau
                if new is not None:
                    if pending is not None:  # not expected under the lookahead rule
                        self._rollback(resume=True, k=k)
                        pending = None
                    events.append(self._change_penalty(k, new, have_pc, nu_identity))
                    win.clear()
                    self._win_append(win)

        x = self.x.cpu().numpy()
        z = self.z.cpu().numpy()
        u = self.u.cpu().numpy()
        x_bar = z_bar = None
        if bar_count > 0:
            x_bar = self.xbar.cpu().numpy() / bar_count
            z_bar = self.zbar.cpu().numpy() / bar_count
        kx.d2h += 5 * n * 8
        timings.total_s = time.perf_counter() - t_start
        return SolveResult(
            status=status, x=x, z=z, u=u, objective=last_obj, iterations=k_done,
            rp_norm=res.rp_norm, rd_norm=res.rd_norm, history=history, timings=timings,
            x_bar=x_bar, z_bar=z_bar, certificate_primal=cert_p, certificate_dual=cert_d,
            penalty_events=events, iterates=iterates, gap=gap,
            device_stats={"kernel_launches": kx.launches, "sketches": self.n_sketches,
                          "world": self.shard.world, "pipelined": bool(self.fast)},
        )

    # ------------------------------------------------------ host maths ----
    def _residuals(self, st) -> Residuals:
        """admm.py:215-224 from the fused norms (M = I, c = 0)."""
        s = st[_S_NORMS:]
        if self.opts.norm_kind == "linf":
            rp, rd, nx, nz, nru = s[1], s[3], s[5], s[7], s[9]
        else:
            rp, rd, nx, nz, nru = (math.sqrt(max(s[i], 0.0)) for i in (0, 2, 4, 6, 8))
        return Residuals(None, None, rp, rd, max(nx, nz, 0.0), nru, self.n)

    def _objective(self, st) -> float:
        s = st[_S_NORMS:]
        if self.is_ml:
            f = float(st[_S_LEN + 0]) + 0.5 * self.l2 * s[4]  # problems.py:227-230
            return f + self.l1 * s[10]  # g(z) = lambda1 ||z||_1
        f = 0.5 * s[11] + s[12]  # problems.py:396-397
        scale = 1.0 + s[7]
        g = 0.0 if s[15] <= 1e-9 * scale else np.inf  # prox.py:138-144
        return f + g

    def _gap(self, st) -> float:
        """ml_dual_gap at z (problems.py:306-351) from the fused sums."""
        s = st[_S_NORMS:]
        rs = st[_S_LEN:]
        primal = float(rs[1]) + 0.5 * self.l2 * s[6] + self.l1 * s[10]
        conj_sum, n_inf, b_nu = float(rs[2]), float(rs[3]), float(rs[4])
        if self.l2 == 0.0:
            denom = s[13]  # ||A' nu||_inf
            if denom > self.l1:
                c = self.l1 / denom
                if self.loss in ("square", "huber"):
                    # degree-2 homogeneous conjugates inside their domain
                    conj_sum, b_nu = conj_sum * c * c, b_nu * c
                elif self.fast and self._tails[0].conj_out:
                    o = st[_S_CONJ:_S_CONJ + 3]  # computed by the tail with the same c
                else:
                    out = self.stats[_S_CONJ:_S_CONJ + 3]
                    self.kx.ml_conj_scaled(self.loss, self.T[2], c, self.b, out)
                    if self.shard.sharded:
                        self.shard.allreduce(out)
                    o = out.cpu().numpy()
                if self.loss not in ("square", "huber"):
                    conj_sum, n_inf, b_nu = float(o[0]), float(o[1]), float(o[2])
        if n_inf > 0:
            return np.inf
        dual = -conj_sum - b_nu
        if self.l2 > 0.0:
            dual -= float(s[14]) / (2.0 * self.l2)
        if not np.isfinite(dual):
            return np.inf
        num = primal - dual
        denom = min(primal, abs(dual))
        if denom <= 1e-16:
            return 0.0 if abs(num) <= 1e-12 else np.inf
        return num / denom

    def _terminated(self, res: Residuals, gap) -> bool:
        """admm.py:227-240."""
        if gap is not None:
            return gap <= self.opts.eps_dual_gap
        o = self.opts
        p_ok = res.rp_norm <= math.sqrt(self.n) * o.eps_abs + o.eps_rel * res.primal_scale
        d_ok = res.rd_norm <= math.sqrt(self.n) * o.eps_abs + o.eps_rel * res.dual_scale
        return bool(p_ok and d_ok)

    def _change_penalty(self, k, rho_new, have_pc, nu_identity) -> PenaltyEvent:
        """admm.py:303-319: rescale u so rho u is unchanged; shift the preconditioner."""
        rho_old = self.rho
        out = self.stats[_S_DUAL:_S_DUAL + 2]
        self.kx.scale_dual(self.u, rho_old, rho_new, out)
        o = out.cpu().numpy()
        self.rho = rho_new
        denom = max(math.sqrt(max(o[0], 0.0)), 1e-30)
        jump = math.sqrt(max(o[1], 0.0)) / denom
        if have_pc:
            self.pc_nu = nu_identity(rho_new)
        return PenaltyEvent(k, rho_old, rho_new, jump)

    # ---------------------------------------------------------- windows --
    def _free_slot(self, win) -> int:
        used = set(win)
        return next(i for i in range(self.ring.shape[0]) if i not in used)

    def _win_append(self, win) -> None:
        slot = self._free_slot(win)
        self.ring[slot].copy_(self.x)
        if self.uring is not None:
            self.uring[slot].copy_(self.u)
        win.append(slot)

    def _win_speculate(self, win):
        """Copy the new (x, u) into a free ring slot and launch the window
        reductions for the deque state after the append, so that one readback
        serves the stats, the cycle guard and the QP infeasibility test."""
        slot = self._free_slot(win)
        self.ring[slot].copy_(self.x)
        if self.uring is not None:
            self.uring[slot].copy_(self.u)
        after = list(win) + [slot]
        if len(after) > DELTA_WINDOW + 1:
            after = after[1:]
        if len(after) >= 4:
            nper = min(len(after) - 1, 10) - 1
            others = [after[-2]] + [after[-1 - p] for p in range(2, 2 + nper)]
            self.kx.window_norms(self.ring, slot, others, self.stats[_S_WIN:_S_WIN + 17])
        if not self.is_ml and len(after) == DELTA_WINDOW + 1:
            first, last = after[0], after[-1]
            self.kx.qp_infeas(self.ring[last], self.ring[first], self.uring[last], self.uring[first],
                              float(DELTA_WINDOW), self.lo, self.hi, self.q, self.dx[0],
                              self.stats[_S_INF:_S_INF + 6])
            self.kx.gemv(self.P, self.dx, self.Pdx)
            self.kx.dot(self.Pdx[0], self.Pdx[0], self.stats[_S_PDX:_S_PDX + 1])
        return slot

    def _win_commit(self, win, slot) -> None:
        win.append(slot)

    # ------------------------------------------------ fused iteration ----
    def _make_tail(self):
        """Device state of the one-iteration-ahead pipeline.

        Iteration k uses the parity p = k % 2 copies of: the readback block
        (row sums | CG scalars | stats), the CG problem descriptor, the tail
        descriptor, the gate g[p] ("may run": opened by the tail of k-1) and
        the CG tolerance slot.  The host can therefore launch k+1 before it
        has read k (admm.py:520-700 stay on the host, one iteration behind).
        The workspaces have their own keys so they are never reallocated
        under the descriptors."""
        kx, L, n = self.kx, self.kx.L, self.n
        self.rbs = kx.zeros(2, _RB_LEN)
        self.rbs_host = [_host_buffer(_RB_LEN + 1, kx.device) for _ in range(2)]  # + completion tag
        # pinned host memory is device-addressable under UVA: a kernel writes the
        # readback block straight into it (no copy engine in the pipeline)
        self._kernel_readback = (hasattr(kx, "readback") and kx.device.type == "cuda"
                                 and _lib.dev_env("NYS_KERNEL_READBACK", "1") != "0")
        self.gates = kx.zeros(2)
        self.gates[1] = 1.0  # iteration 1 (parity 1) may run
        self.tols = kx.zeros(2)
        # row order of the last pass over A of iteration parity p (L2 reuse)
        self.orders = kx.zeros(2)
        self.snap = kx.zeros(5, n)
        self._done_ev = [torch.cuda.Event() for _ in range(2)]
        self._ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(2)]
        # 1: events around the x-update and the tail; 2: only around the whole
        # iteration (no event between the two kernel groups); 0: none
        # 0 (default): no stream events inside the iteration chain (each costs a
        # launch gap: measured 2585 vs 2557 iters/s on config 2); the history's
        # linsys_s is then the host wall time between retired iterations, as the
        # reference's per-iteration timings are wall times
        self._iter_events = int(_lib.dev_env("NYS_ITER_EVENTS", "0"))
        self._t_retire = None
        self._fuse_readback = _lib.dev_env("NYS_FUSE_READBACK", "1") != "0"
        # with the fused readback the host polls the block's completion tag, so no
        # stream event sits between an iteration's last kernel and the next x-update
        self._poll = self._fuse_readback and _lib.dev_env("NYS_POLL_READBACK", "1") != "0"
        self._ev_ring = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        self._seq = 0
        ptr = lambda x: x.data_ptr() if x is not None else None
        self._reduce_fn = None
        if self.shard.sharded:
            # the all-reduce hook of the C drivers: buffers are recognised by address
            self._reduce_views = {}

            def _reduce(buf, count, user, stream):
                base = self._reduce_views[buf]
                self.shard.allreduce(base.view(-1)[:count])

            self._reduce_fn = _lib.REDUCE_FN(_reduce)  # kept alive with the engine
            for v in (self.AT if self.is_ml else None, self.cg.Ap):
                if v is not None:
                    self._reduce_views[v.data_ptr()] = v
        self._tails, self._pbs, self._heads = [], [], []
        for par in range(2):
            blk = self.rbs[par]
            st = blk[8 + _lib.CG_NSLOTS:]
            sc = blk[8:8 + _lib.CG_NSLOTS]
            t = _lib.AdmmTail()
            t.n = n
            t.XZ = self.XZ.data_ptr()
            t.u, t.xbar, t.zbar = self.u.data_ptr(), self.xbar.data_ptr(), self.zbar.data_ptr()
            t.alpha = float(self.opts.alpha)
            t.norms = st.data_ptr()
            t.ring, t.ring_ld = self.ring.data_ptr(), self.ring.stride(0)
            t.uring = ptr(self.uring)
            t.wnorms = st[_S_WIN:].data_ptr()
            t.infeas = st[_S_INF:].data_ptr()
            t.pdx2 = st[_S_PDX:].data_ptr()
            t.width = float(DELTA_WINDOW)
            t.pred = sc[_lib.CG_RUNNING:].data_ptr()
            t.order = self.orders[par:].data_ptr()
            # the gate of k+1 opens after k's tail: in the readback kernel when
            # there is one, else at the end of the tail
            t.gate_next = None if self._kernel_readback else self.gates[1 - par:].data_ptr()
            if self.is_ml:
                rows = self.rows
                t.kind, t.loss, t.rows = 0, _lib.LOSS[self.loss], rows
                t.A, t.lda, t.b = self.A.data_ptr(), self.A.stride(0), self.b.data_ptr()
                t.lambda1, t.lambda2 = self.l1, self.l2
                t.with_z = 1 if self.use_gap else 0
                t.AXZ, t.T, t.w, t.AT = self.AXZ.data_ptr(), self.T.data_ptr(), self.w.data_ptr(), self.AT.data_ptr()
                t.rowsums = blk.data_ptr()
                if self.gb is not None and self.use_gap:
                    t.gb = self.gb.data_ptr()
                if self.use_gap and self.l2 == 0.0 and self.loss not in ("square", "huber"):
                    t.conj_out = st[_S_CONJ:].data_ptr()
                wg = kx.workspace("tail_gemv", L.nys_gemv_workspace(rows, n, 2))
                wt = kx.workspace("tail_gemvT", max(L.nys_gemvT_workspace(rows, n, 3),
                                                    L.nys_tail_cluster_workspace(rows, n)))
            else:
                t.kind, t.rows = 1, n
                t.A, t.lda = self.P.data_ptr(), self.P.stride(0)
                t.lo, t.hi, t.q = self.lo.data_ptr(), self.hi.data_ptr(), self.q.data_ptr()
                t.AT = self.Px.data_ptr()
                t.dx, t.Pdx = self.dx.data_ptr(), self.Pdx.data_ptr()
                wg = kx.workspace("tail_gemv", L.nys_gemv_workspace(n, n, 1))
                wt = kx.workspace("tail_gemvT", 256)
            wr = kx.workspace("tail_red", L.nys_reduce_workspace())
            if self._reduce_fn is not None:
                t.reduce = C.cast(self._reduce_fn, C.c_void_p)
                self._reduce_views[blk.data_ptr()] = blk
                if t.conj_out:
                    self._reduce_views[st[_S_CONJ:].data_ptr()] = st[_S_CONJ:]
            t.ws_gemv, t.ws_gemv_bytes = wg.data_ptr(), wg.numel()
            t.ws_gemvT, t.ws_gemvT_bytes = wt.data_ptr(), wt.numel()
            t.ws_red = wr.data_ptr()
            self._tails.append(t)

            h = _lib.AdmmHead()
            h.n = n
            if self.is_ml:
                h.hxA, h.gA, h.q, h.lambda2 = self.AT[1].data_ptr(), self.AT[0].data_ptr(), None, self.l2
            else:
                h.hxA = h.gA = self.Px[0].data_ptr()
                h.q, h.lambda2 = self.q.data_ptr(), 0.0
            h.x, h.z, h.u = self.x.data_ptr(), self.z.data_ptr(), self.u.data_ptr()
            h.xbar, h.zbar = self.xbar.data_ptr(), self.zbar.data_ptr()
            h.rhs, h.r, h.sc = self.rhs.data_ptr(), self.cg.r.data_ptr(), sc.data_ptr()
            h.snap = self.snap.data_ptr()
            h.gate, h.gate_next = self.gates[par:].data_ptr(), self.gates[1 - par:].data_ptr()
            h.norm_kind = 1 if self.opts.norm_kind == "linf" else 0
            h.tol_out = self.tols[par:].data_ptr()
            h.ws_red = kx.red.data_ptr()
            h.zu = C.addressof(t)  # the persistent x-update may run the tail's z/u step
            self._heads.append(h)
            self._pbs.append(None)

    def _cg_problem(self, par, shift):
        """The parity-par CG descriptor for the current operator shift and
        preconditioner (rebuilt only when those change)."""
        key = (shift, self.pc_nu, None if self.U is None else self.U.data_ptr(), self.n_sketches)
        pb = self._pbs[par]
        if pb is None or pb._key != key:
            kx, n = self.kx, self.n
            work = _ParityWork(self.cg, self.rbs[par][8:8 + _lib.CG_NSLOTS])
            if self.is_ml:
                pb = kx.cg_problem(0, self.A, None if self.loss == "square" else self.w, self.diag_shift + shift,
                                   self.U, self.lam, self.pc_nu, self.rhs, self.x, work, 1e-12, 10 * n)
            else:
                pb = kx.cg_problem(1, self.P, None, shift, self.U, self.lam, self.pc_nu, self.rhs, self.x, work,
                                   1e-12, 10 * n)
            pb.gate = self.gates[par:].data_ptr()
            pb.tol_dev = self.tols[par:].data_ptr()
            if self._reduce_fn is not None:
                pb.reduce = C.cast(self._reduce_fn, C.c_void_p)
                self._reduce_views[pb.Ap] = self.cg.Ap
            pb.order_in = self.orders[1 - par:].data_ptr()
            pb.order_out = self.orders[par:].data_ptr()
            pb._key = key
            self._pbs[par] = pb
        return pb

    def _issue(self, k, shift, win_before, exact):
        """Launch iteration k (head, batched CG, predicated tail, readback);
        `win_before` is the window as it will be before k's append."""
        kx, par = self.kx, k % 2
        h, t = self._heads[par], self._tails[par]
        h.rho, h.shift = float(self.rho), float(shift)
        # the previous iteration's norms (the setup pass for k = 1)
        h.prev = (self.stats if k == 1 else self.rbs[1 - par][8 + _lib.CG_NSLOTS:]).data_ptr()
        h.sigma = float(self.sigma_eff)
        if exact:
            h.tol_fixed, h.kpow = 1e-12, 1.0
        else:
            h.tol_fixed, h.kpow = 0.0, float(k ** self.opts.gamma)
        pb = self._cg_problem(par, shift)
        self._seq += 1
        pb.timing_tag = self._seq
        slot = self._free_slot(win_before)
        after = list(win_before) + [slot]
        if len(after) > DELTA_WINDOW + 1:
            after = after[1:]
        t.accum = 1 if k >= 2 else 0
        t.rho = float(self.rho)
        t.kappa = float(self.l1 / self.rho) if self.is_ml else 0.0
        t.slot = slot
        if len(after) >= 4:
            nper = min(len(after) - 1, 10) - 1
            others = [after[-2]] + [after[-1 - p] for p in range(2, 2 + nper)]
        else:
            others = []
        t.nothers = len(others)
        for j, o in enumerate(others):
            t.others[j] = o
        t.qp_infeas = 1 if (not self.is_ml and len(after) == DELTA_WINDOW + 1) else 0
        if t.qp_infeas:
            t.inf_first, t.inf_last = after[0], after[-1]
        batch = min(16, max(2, self._last_cg + 1))
        ev = self._ev[par]
        fused = self._kernel_readback and self._fuse_readback
        poll = fused and self._poll
        if self._iter_events and not poll:
            ev[0].record(kx.stream)
        kx.admm_xupdate(h, pb, batch)  # head + PCG (one persistent kernel when it fits)
        if self._iter_events == 1:
            ev[1].record(kx.stream)
            if poll:
                self._ev_ring[k % 4].record(kx.stream)
        if fused:
            # the tail's last kernel copies the block into mapped host memory itself
            t.rb_src, t.rb_dst = self.rbs[par].data_ptr(), self.rbs_host[par].data_ptr()
            t.rb_n, t.rb_gate = self.rbs[par].numel(), self.gates[1 - par:].data_ptr()
            t.rb_tag = float(self._seq) if poll else 0.0
        kx.admm_tail(t)
        if self._iter_events and not poll:
            ev[2].record(kx.stream)
        polled = False
        if t.rb_done:
            self.kx.d2h += _RB_LEN * 8
            if poll:
                polled = True
            else:
                self._done_ev[par].record(self.kx.stream)
        else:
            self._readback(par)
        return _Issued(k, par, slot, after, batch, self._seq, shift, exact, list(win_before), polled=polled,
                       ring=poll, dev_stop=bool(t.stop_ran))

    def _read_block(self):
        """The setup / per-step readback block in one D2H copy; returns
        (sc, stats + row sums)."""
        rb, C = self.rb_host, _lib.CG_NSLOTS
        rb.copy_(self.rb_dev, non_blocking=True)
        self.kx.d2h += _RB_LEN * 8
        self.kx.sync()
        h = rb.numpy().copy()
        return h[8:8 + C], np.concatenate([h[8 + C:], h[:8]])

    def _readback(self, par):
        if self._kernel_readback:
            t = self._tails[par]
            # a tail that ran the device stop test already opened (or kept closed)
            # the next gate: the extra copy must not reopen it
            gate = None if t.stop_ran else self.gates[1 - par:].data_ptr()
            self.kx.readback(self.rbs[par], self.rbs_host[par], gate, t.pred)
        else:
            self.rbs_host[par][:_RB_LEN].copy_(self.rbs[par], non_blocking=True)
        self.kx.d2h += _RB_LEN * 8
        self._done_ev[par].record(self.kx.stream)

    def _read(self, par, tag=None):
        if tag is None:
            self._done_ev[par].synchronize()
        else:
            # spin on the completion tag the tail's last kernel stores after the block
            buf = self.rbs_host[par].numpy()
            spins = 0
            while buf[_RB_LEN] != tag:
                spins += 1
                if spins % 4096 == 0:
                    time.sleep(0)
                    if spins % (4096 * 64) == 0:
                        self.kx.sync()  # surfaces a device error; the tag must be there after it
                        if buf[_RB_LEN] != tag:
                            raise NumericalError("readback block of the iteration never arrived")
        h = self.rbs_host[par].numpy()[:_RB_LEN].copy()
        C = _lib.CG_NSLOTS
        return h[8:8 + C], np.concatenate([h[8 + C:], h[:8]])

    def _retire(self, it, nxt):
        """Wait for iteration `it`, finish its CG if the batch was short (and
        re-launch the speculated successor, whose closed gate made it a
        no-op), and return (CgReport, stats, linsys_s, prox_s)."""
        kx, par = self.kx, it.par
        sc, st = self._read(par, float(it.tag) if it.polled else None)
        ev = self._ev[par]
        now = time.perf_counter()
        if it.ring:
            # no events around the x-update and the tail: the whole iteration, from
            # the ring of per-iteration marks between the two kernel groups, else
            # the host wall time since the previous retired iteration
            if self._iter_events == 1:
                lin_ms = (self._ev_ring[(it.k - 1) % 4].elapsed_time(self._ev_ring[it.k % 4])
                          if it.k > 1 else 0.0)
            else:
                lin_ms = 1e3 * (now - self._t_retire) if self._t_retire is not None else 0.0
            tail_ms = 0.0
        elif self._iter_events == 1:
            lin_ms, tail_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
        elif self._iter_events == 2:
            lin_ms, tail_ms = ev[0].elapsed_time(ev[2]), 0.0
        else:
            lin_ms = 1e3 * (now - self._t_retire) if self._t_retire is not None else 0.0
            tail_ms = 0.0
        self._t_retire = now
        k_last, batch = it.batch, it.batch
        self._cg_continued = False
        max_iter = 10 * self.n
        done = int(sc[_lib.CG_DONE])
        while done == 0 and k_last < max_iter:
            batch = min(16, 2 * batch)
            pb = self._pbs[par]
            ev[0].record(kx.stream)
            kx.cg_iterate(pb, k_last + 1, batch)
            ev[1].record(kx.stream)
            kx.admm_tail(self._tails[par])
            ev[2].record(kx.stream)
            self._readback(par)
            k_last += batch
            sc, st = self._read(par)
            lin_ms += ev[0].elapsed_time(ev[1])
            tail_ms += ev[1].elapsed_time(ev[2])
            done = int(sc[_lib.CG_DONE])
            self._cg_continued = True
        if hasattr(kx, "timing_commit"):
            kx.timing_commit(it.tag, int(sc[_lib.CG_ITERS]) if done else k_last, int(sc[_lib.CG_NHVP]))
        if nxt is not None and k_last > it.batch:
            # the successor ran with a closed gate: launch it again
            if hasattr(kx, "timing_commit"):
                kx.timing_commit(nxt.tag, 0)
            nxt.reissue = self._issue(nxt.k, nxt.shift, nxt.win_before, nxt.exact)
        if done == 2:
            raise NumericalError("non-finite value in conjugate gradient")
        if done == 3:
            raise NotSPDError(f"nonpositive curvature p'Ap = {sc[_lib.CG_PAP]:.3e}; operator is not SPD")
        iters = int(sc[_lib.CG_ITERS])
        rep = CgReport(iters, float(sc[_lib.CG_RESREL]), done == 1)
        return rep, st, lin_ms / 1e3, tail_ms / 1e3

    def _rollback(self, resume: bool = False, k: int = 0):
        """Undo a speculated iteration: restore (x, z, u, xbar, zbar) from the
        snapshot its head took.  With resume, also redo the data passes at the
        restored point (the speculated tail overwrote them) and reset the gates
        so that iteration k+1 can be launched again."""
        self.kx.sync()
        self.x.copy_(self.snap[0])
        self.z.copy_(self.snap[1])
        self.u.copy_(self.snap[2])
        self.xbar.copy_(self.snap[3])
        self.zbar.copy_(self.snap[4])
        if resume:
            self.evaluate(with_z=self.use_gap)
            self.gates[(k + 1) % 2] = 1.0
            self.gates[k % 2] = 0.0

    def _may_speculate(self, k, it, have_pc, last_sketch, rho_frozen, cycle_hits) -> bool:
        """May iteration k+1 be launched before k is read?  Only if no outcome
        of k can change k+1's launch: no resketch due at k+1, no penalty check
        at k (admm.py:677-698), no possible cycle-guard trigger at k
        (admm.py:643-675: needs 5 consecutive hits), k+1 within max_iter."""
        o = self.opts
        if k + 1 > o.max_iter:
            return False
        if have_pc and not self.const_hess and (k + 1) - last_sketch >= o.resketch_every:
            return False
        if (not rho_frozen and o.penalty_update_every > 0 and k >= o.penalty_warmup
                and k % o.penalty_update_every == 0 and k <= PENALTY_ADAPT_CUTOFF):
            return False
        if len(it.after) >= 4 and not rho_frozen and k <= PENALTY_ADAPT_CUTOFF and cycle_hits >= 4:
            return False
        return True

    def _infeasibility(self, st, win):
        """admm.py:361-415 with M = I from the speculative reductions."""
        eps = self.opts.eps_inf
        s = st[_S_INF:]
        primal = dual = near_p = near_d = False
        cp = cd = None
        du = math.sqrt(max(s[0], 0.0))
        if du > 1e-14:
            t_map = du
            t_sup = np.inf if s[2] > 0 else float(s[1])
            primal = t_map < eps * du and t_sup < eps * du
            near_p = t_map < 10 * eps * du and t_sup < 10 * eps * du
            if primal:
                last, first = win[-1], win[0]
                cp = self.rho * ((self.uring[last] - self.uring[first]) / DELTA_WINDOW).cpu().numpy()
        dxn = math.sqrt(max(s[3], 0.0))
        if dxn > 1e-14:
            s_obj = math.sqrt(max(st[_S_PDX], 0.0))
            s_cone = math.sqrt(max(s[4], 0.0))
            s_lin = float(s[5])
            dual = s_obj < eps * dxn and s_cone < eps * dxn and s_lin < eps * dxn
            near_d = s_obj < 10 * eps * dxn and s_cone < 10 * eps * dxn and s_lin < 10 * eps * dxn
            if dual:
                # from the ring slots of k's window (never written by a speculated
                # k+1), not from the shared dx buffer k+1's tail may already reuse
                last, first = win[-1], win[0]
                cd = ((self.ring[last] - self.ring[first]) / DELTA_WINDOW).cpu().numpy()
        if primal and dual:
            status = Status.PRIMAL_AND_DUAL_INFEASIBLE
        elif primal:
            status = Status.PRIMAL_INFEASIBLE
        elif dual:
            status = Status.DUAL_INFEASIBLE
        else:
            status = None
        return status, near_p or near_d, cp, cd

    # ------------------------------------------------------------ misc ----
    def _snapshot(self, k, bar_count) -> SolverState:
        x = self.x.cpu().numpy()
        return SolverState(x=x, z=self.z.cpu().numpy(), u=self.u.cpu().numpy(), rho=self.rho, k=k, Mx=x,
                           x_bar_sum=self.xbar.cpu().numpy(), z_bar_sum=self.zbar.cpu().numpy(),
                           bar_count=bar_count)

    def _averaged_objective(self, bar_count) -> float:
        """f(x_bar) + g(z_bar) (admm.py:589-591): extra data pass, only when asked."""
        kx = self.kx
        xb = self.xbar / bar_count
        zb = self.zbar / bar_count
        if self.is_ml:
            XB = xb.view(1, -1).contiguous()
            ab = kx.empty(1, self.rows)
            kx.gemv(self.A, XB, ab)
            out = kx.zeros(8)
            kx.ml_rowwise(self.loss, ab[0], None, self.b, None, None, None, None, out)
            if self.shard.sharded:
                self.shard.allreduce(out)
            f = float(out[0]) + 0.5 * self.l2 * float(torch.dot(xb, xb))
            return f + self.l1 * float(zb.abs().sum())
        pxb = kx.empty(1, self.n)
        kx.gemv(self.P, xb.view(1, -1).contiguous(), pxb)
        f = 0.5 * float(torch.dot(xb, pxb[0])) + float(torch.dot(self.q, xb))
        scale = 1.0 + float(zb.abs().max())
        ok = bool(torch.all(zb >= self.lo - 1e-9 * scale)) and bool(torch.all(zb <= self.hi + 1e-9 * scale))
        return f + (0.0 if ok else np.inf)


def solve(problem, options: Optional[SolverOptions] = None, x0=None, z0=None, u0=None,
          callback: Optional[Callable] = None, kernels=None, shard: Optional[Shard] = None) -> SolveResult:
    """Run the splitting method on a QP or ML problem (admm.py:422-719).

    Drop-in for ``nysopt.solve``; the extra keyword arguments are for the
    harness (an explicit kernel backend / shard, used by the multi-rank tests)."""
    t_start = time.perf_counter()
    options = options or SolverOptions()
    gp = lower(problem)
    if kernels is None:
        from .kernels import get_kernels

        kernels = get_kernels()
    if not _dense_path(gp):
        # sparse data, structured P, general constraint maps: the general-operator
        # engine (general.py), same control flow, one device pass per operator
        if shard is not None and shard.sharded:
            raise CapabilityError("row sharding covers dense data matrices only")
        from .general import _GeneralEngine

        return _GeneralEngine(gp, options, kernels).run(x0, z0, u0, callback, t_start)
    eng = _Engine(gp, options, kernels, shard)
    return eng.run(x0, z0, u0, callback, t_start)


def _dense_path(gp: GenericProblem) -> bool:
    """Problems the fused dense engine takes: dense ML data, or a dense QP
    matrix with M = I (BASELINE.json's configs)."""
    if gp.ml is not None:
        return isinstance(gp.ml.A, DenseOperator) and gp.ml.loss.kind in _lib.LOSS
    if gp.qp is None:
        return False  # oracles given as callables (GenericProblem): the general engine
    return isinstance(gp.qp.P, DenseOperator) and isinstance(gp.qp.M, IdentityOperator)


# the reference's single-step API (admm.py:215-415) and the names its admm module
# re-exports; imported last: steps.py needs the classes above
from .krylov import pcg  # noqa: E402,F401
from .operators import MatrixFreeOperator  # noqa: E402,F401
from .problems import ml_dual_gap  # noqa: E402,F401
from .prox import box_recession_distance, box_support  # noqa: E402,F401
from .sketch import estimate_extreme_eigs, nystrom_sketch  # noqa: E402,F401
from .steps import (  # noqa: E402,F401
    InfeasibilityCheck,
    check_infeasibility,
    check_termination,
    compute_residuals,
    relaxed_constraint_point,
    u_update,
    update_penalty,
    x_update,
    z_update,
)
