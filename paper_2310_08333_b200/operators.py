"""Device-backed linear operators with the reference's operator contract
(``/root/reference/pkg/src/nysopt/operators.py:20-319``).

``apply(v, out=None)`` / ``apply_adjoint(u, out=None)`` accept NumPy arrays
(returned as NumPy, like the reference) or torch CUDA tensors (returned on the
device).  The dense operator runs the sm_100a GEMV kernels (K1/K2) through the
C ABI; there is no CPU fallback.

Dense operators run the GEMV kernels of the hot path (SURVEY.md §8(a)
R6-R8).  The structured and sparse operators of operators.py:89-228 (CSR data,
diagonal, diagonal-plus-low-rank, vertical stacks, the summing row,
function-defined Hessians) run the general-operator kernels
(``csrc/general.cu``); ``solve`` routes problems that use them to the
general-operator engine (``general.py``).
"""

from __future__ import annotations

import os
from typing import Callable, Optional

import numpy as np
import torch

from . import _lib
from .dist import Shard, current_shard
from .errors import CapabilityError, DimensionMismatchError

F64 = torch.float64


def _kx():
    from .kernels import get_kernels

    return get_kernels()


def to_device(v, device=None) -> torch.Tensor:
    """Contiguous FP64 CUDA tensor view/copy of ``v``."""
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    if isinstance(v, torch.Tensor):
        return v.to(device=device, dtype=F64).contiguous()
    a = np.ascontiguousarray(np.asarray(v, dtype=float))
    return torch.from_numpy(a).to(device)


def like_input(t: torch.Tensor, ref):
    """Return ``t`` in the container type of ``ref`` (NumPy in, NumPy out)."""
    if isinstance(ref, torch.Tensor):
        return t
    return t.cpu().numpy()


def device_fn(fn: Callable) -> Callable:
    """Mark a callable as taking and returning CUDA tensors (see ``UserFn``)."""
    fn.accepts_device = True
    return fn


class UserFn:
    """A callable supplied through the reference's API (a matrix-free operator's
    matvec, a Hessian-vector product, f / grad f / prox of a GenericProblem).
    The reference's contract is NumPy in, NumPy out, so that is what an unmarked
    callable gets: host copies of the device vectors, its result sent straight
    back.  The user's code is then the only thing that runs on the host.
    Callables marked with ``device_fn`` (this package's own lowered oracles, or
    device-aware user code) get the CUDA tensors themselves."""

    def __init__(self, fn: Callable):
        self.fn = fn
        self.host = not getattr(fn, "accepts_device", False)

    @staticmethod
    def _to_host(a):
        return a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a

    def raw(self, *args):
        if self.host:
            return self.fn(*[self._to_host(a) for a in args])
        return self.fn(*args)

    def __call__(self, *args) -> torch.Tensor:
        out = self.raw(*args)
        return to_device(out if isinstance(out, torch.Tensor) else np.asarray(out, dtype=float))

    def scalar(self, *args) -> float:
        return float(self.raw(*args))


class LinearOperator:
    """A map v -> Av with known dimensions and an optional adjoint
    (operators.py:20-73)."""

    def __init__(self, input_dim: int, output_dim: int):
        if input_dim < 1 or output_dim < 1:
            raise DimensionMismatchError("operator dimensions must be positive")
        self.input_dim = int(input_dim)
        self.output_dim = int(output_dim)

    @property
    def has_adjoint(self) -> bool:
        return type(self)._apply_adjoint_dev is not LinearOperator._apply_adjoint_dev

    def apply(self, v, out=None):
        vt = to_device(v)
        if vt.shape != (self.input_dim,):
            raise DimensionMismatchError(
                f"apply expected vector of length {self.input_dim}, got shape {tuple(vt.shape)}"
            )
        res = self._apply_dev(vt)
        return _write_out(res, v, out)

    def apply_adjoint(self, u, out=None):
        if not self.has_adjoint:
            raise CapabilityError(f"{type(self).__name__} does not support an adjoint")
        ut = to_device(u)
        if ut.shape != (self.output_dim,):
            raise DimensionMismatchError(
                f"apply_adjoint expected vector of length {self.output_dim}, got shape {tuple(ut.shape)}"
            )
        res = self._apply_adjoint_dev(ut)
        return _write_out(res, u, out)

    # device implementations: CUDA tensor in, fresh CUDA tensor out
    def _apply_dev(self, v: torch.Tensor) -> torch.Tensor:
        raise NotImplementedError

    def _apply_adjoint_dev(self, u: torch.Tensor) -> torch.Tensor:
        raise NotImplementedError

    def apply_columns_dev(self, V: torch.Tensor) -> torch.Tensor:
        """Apply to every column of the row-major n x s matrix V; column-by-column
        by default (sketch.py:69-71), overridden with GEMMs where possible."""
        cols = [self._apply_dev(V[:, j].contiguous()) for j in range(V.shape[1])]
        return torch.stack(cols, dim=1).contiguous()

    def to_dense(self) -> np.ndarray:
        cols = np.eye(self.input_dim)
        return np.column_stack([self.apply(cols[:, j]) for j in range(self.input_dim)])


def _write_out(res: torch.Tensor, ref, out):
    if out is None:
        return like_input(res, ref)
    if isinstance(out, torch.Tensor):
        out.copy_(res)
    else:
        np.copyto(out, res.cpu().numpy())
    return out


class IdentityOperator(LinearOperator):
    """Identity map (operators.py:76-86)."""

    def __init__(self, dim: int):
        super().__init__(dim, dim)

    def _apply_dev(self, v):
        return v.clone()

    def _apply_adjoint_dev(self, u):
        return u.clone()

    def apply_columns_dev(self, V):
        return V.clone()

    def apply_adjoint_columns_dev(self, U):
        return U.clone()


class DenseOperator(LinearOperator):
    """Operator backed by a dense 2-d array (operators.py:104-118).

    ``a`` may be a NumPy array (uploaded to HBM on first use and cached) or a
    CUDA tensor already resident in HBM.  Under ``torch.distributed`` each
    rank uploads only its row shard.
    """

    def __init__(self, a):
        self._host_t = None
        if isinstance(a, torch.Tensor):
            if a.ndim != 2:
                raise DimensionMismatchError("dense operator requires a 2-d array")
            self._dev_full = a.to(dtype=F64).contiguous() if a.is_cuda else None
            self.a = a if not a.is_cuda else None
            if self.a is not None:
                if a.dtype == F64 and a.is_contiguous():
                    self._host_t = a  # pinned host data can be uploaded in overlapped chunks
                self.a = self.a.numpy()
        else:
            arr = np.asarray(a, dtype=float)
            if arr.ndim != 2:
                raise DimensionMismatchError("dense operator requires a 2-d array")
            self.a = arr
            self._dev_full = None
        shape = (self._dev_full.shape if self._dev_full is not None else self.a.shape)
        super().__init__(shape[1], shape[0])
        self._shards: dict = {}
        self._pending: dict = {}
        self._local = None  # (row_start, row_stop) when only a row block is resident
        self._host_local = None

    @classmethod
    def from_local_rows(cls, a_local: torch.Tensor, rows_global: int, row_start: int) -> "DenseOperator":
        """A rows_global x n operator of which this process holds only rows
        [row_start, row_start + a_local.shape[0]) in HBM (config 5: every rank
        generates its own row blocks, BASELINE.json configs[4]).  The solve's
        shard must be exactly that row range."""
        if isinstance(a_local, np.ndarray):
            a_local = torch.from_numpy(np.ascontiguousarray(a_local, dtype=float))
        if not (isinstance(a_local, torch.Tensor) and a_local.ndim == 2):
            raise DimensionMismatchError("local rows must be a 2-d array")
        op = cls.__new__(cls)
        op.a = None
        op._dev_full = None
        LinearOperator.__init__(op, a_local.shape[1], rows_global)
        op._shards = {}
        op._pending = {}
        op._host_t = None
        op._local = (row_start, row_start + a_local.shape[0])
        op._host_local = None
        if a_local.is_cuda:
            op._shards[(row_start, row_start + a_local.shape[0], str(a_local.device))] = a_local.contiguous()
        else:
            # host rows (pinned for the bench's end-to-end leg): uploaded by the
            # first device_rows() call of the solve, like a full host matrix
            op._host_local = a_local.to(dtype=F64).contiguous()
        return op

    # -- device data ---------------------------------------------------------
    UPLOAD_CHUNKS = 8

    def _pinned_rows(self, shard: Shard) -> Optional[torch.Tensor]:
        """A pinned host tensor view of the shard's rows, when the host copy is pinned."""
        host = getattr(self, "_host_t", None)
        if host is None or not host.is_pinned():
            return None
        return host[shard.row_start:shard.row_stop]

    def device_rows(self, shard: Optional[Shard] = None, device=None, overlap: bool = False) -> torch.Tensor:
        """The (row-shard of the) matrix in HBM, uploaded once.

        ``overlap``: a pinned host matrix is copied in row chunks on a side
        stream and the tensor is returned at once; the caller takes the chunk
        events with ``take_pending`` and makes its stream wait on each chunk
        before touching those rows (the solve overlaps the upload with its
        setup sketch).  Without it every pending chunk is waited for."""
        if shard is None:
            shard = Shard(0, 1, 0, self.output_dim, self.output_dim)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        key = (shard.row_start, shard.row_stop, str(device))
        t = self._shards.get(key)
        if t is not None and not overlap:
            self._wait_pending(t)
        if overlap and _lib.dev_env("NYS_UPLOAD_OVERLAP", "1") == "0":
            overlap = False
        if t is None and overlap and self._dev_full is None and self._local is None:
            src = self._pinned_rows(shard)
            if src is not None:
                t = torch.empty(tuple(src.shape), dtype=F64, device=device)
                self._pending[t.data_ptr()] = _chunked_upload(src, t, self.UPLOAD_CHUNKS)
                self._shards[key] = t
        if t is None and self._local is not None and getattr(self, "_host_local", None) is not None \
                and (shard.row_start, shard.row_stop) == self._local:
            t = self._host_local.to(device, non_blocking=self._host_local.is_pinned())
            self._shards[key] = t
        if t is None and self._local is not None:
            raise DimensionMismatchError(f"rows {self._local} are resident here, the solve's shard is "
                                         f"[{shard.row_start}, {shard.row_stop})")
        if t is None:
            if self._dev_full is not None:
                t = self._dev_full[shard.row_start:shard.row_stop].to(device)
            else:
                blk = np.ascontiguousarray(self.a[shard.row_start:shard.row_stop])
                t = torch.from_numpy(blk).to(device)
            self._shards[key] = t
        return t

    def take_pending(self, t: torch.Tensor):
        """[(row0, row1, event)] of an overlapped upload into ``t`` (None when
        complete); the caller now owns the waits."""
        return self._pending.pop(t.data_ptr(), None)

    def _wait_pending(self, t: torch.Tensor) -> None:
        chunks = self._pending.pop(t.data_ptr(), None)
        if chunks:
            cur = torch.cuda.current_stream(t.device)
            for _, _, ev in chunks:
                cur.wait_event(ev)

    def release(self) -> None:
        """Drop cached device copies (the host array is kept)."""
        self._shards.clear()
        self._pending.clear()

    # -- apply -------------------------------------------------------------------
    def _apply_dev(self, v):
        kx = _kx()
        A = self.device_rows()
        y = kx.empty(1, self.output_dim)
        kx.gemv(A, v.view(1, -1), y)
        return y.view(-1)

    def _apply_adjoint_dev(self, u):
        kx = _kx()
        A = self.device_rows()
        y = kx.empty(1, self.input_dim)
        kx.gemvT(A, u.view(1, -1), y)
        return y.view(-1)

    def apply_columns_dev(self, V):
        kx = _kx()
        A = self.device_rows()
        rows, n = A.shape
        s = V.shape[1]
        Y = kx.empty(rows, s)
        kx.gemm(0, 0, rows, s, n, 1.0, A, A.stride(0), V, V.stride(0), 0.0, Y, s)
        return Y


_UPLOAD_STREAMS: dict = {}


def _chunked_upload(src: torch.Tensor, dst: torch.Tensor, chunks: int):
    """Copy pinned host rows into ``dst`` in ``chunks`` row blocks on a side
    stream; returns [(row0, row1, event)] (PCIe runs while the caller computes)."""
    dev = dst.device
    us = _UPLOAD_STREAMS.get(dev)
    if us is None:
        us = torch.cuda.Stream(dev)
        _UPLOAD_STREAMS[dev] = us
    # dst's memory may have just been freed on the current stream; the current
    # stream in turn waits on every chunk event before using (or freeing) dst,
    # so the allocator's stream-ordered reuse stays safe without record_stream
    us.wait_stream(torch.cuda.current_stream(dev))
    rows = dst.shape[0]
    step = -(-rows // max(1, chunks))
    out = []
    with torch.cuda.stream(us):
        for r0 in range(0, rows, step):
            r1 = min(rows, r0 + step)
            dst[r0:r1].copy_(src[r0:r1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(us)
            out.append((r0, r1, ev, src))
    return [(r0, r1, ev) for r0, r1, ev, _ in out]


class DeviceCSR:
    """A CSR matrix resident in HBM: int64 row pointer, int32 columns, FP64 values,
    and the lanes-per-row group the SpMV kernel uses for it."""

    def __init__(self, rows: int, cols: int, rowptr: torch.Tensor, col: torch.Tensor, val: torch.Tensor):
        self.rows, self.cols = int(rows), int(cols)
        self.rowptr, self.col, self.val = rowptr, col, val
        nnz = int(val.numel())
        mean = nnz / max(self.rows, 1)
        g = 1
        while g < 32 and g < mean:
            g *= 2
        self.group = g

    @classmethod
    def upload(cls, a, device) -> "DeviceCSR":
        rowptr = torch.from_numpy(np.ascontiguousarray(a.indptr, dtype=np.int64)).to(device)
        col = torch.from_numpy(np.ascontiguousarray(a.indices, dtype=np.int32)).to(device)
        val = torch.from_numpy(np.ascontiguousarray(a.data, dtype=np.float64)).to(device)
        if val.numel() == 0:  # keep valid pointers for an all-zero matrix
            col = torch.zeros(1, dtype=torch.int32, device=device)
            val = torch.zeros(1, dtype=torch.float64, device=device)
        return cls(a.shape[0], a.shape[1], rowptr, col, val)

    def transpose(self, kx) -> "DeviceCSR":
        """CSR of the transpose, built on the device (deterministic counting transpose)."""
        dev = self.rowptr.device
        nnz = int(self.rowptr[-1])
        trowptr = torch.empty(self.cols + 1, dtype=torch.int64, device=dev)
        tcol = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        tval = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
        if nnz == 0:  # all-zero matrix: valid pointers, nothing to place
            trowptr.zero_()
            tcol.zero_()
            tval.zero_()
        else:
            kx.csr_transpose(self.rows, self.cols, self.rowptr, self.col, self.val, trowptr, tcol, tval)
        return DeviceCSR(self.cols, self.rows, trowptr, tcol, tval)


class SparseOperator(LinearOperator):
    """Operator backed by a scipy sparse matrix stored as CSR (operators.py:121-135).

    The CSR arrays are uploaded to HBM on first use together with the CSR of the
    transpose (built on the device), so ``apply`` (``a @ v``) and
    ``apply_adjoint`` (``a.T @ u``) are both row-parallel SpMV kernels."""

    def __init__(self, a):
        import scipy.sparse as sp

        if not sp.issparse(a):
            raise DimensionMismatchError("SparseOperator requires a scipy sparse matrix")
        a = a.tocsr()
        if not a.has_canonical_format:
            a = a.copy()
            a.sum_duplicates()  # the device transpose needs distinct columns per row
        super().__init__(a.shape[1], a.shape[0])
        self.a = a
        self._dev: dict = {}

    def device_csr(self, device=None):
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        key = str(device)
        pair = self._dev.get(key)
        if pair is None:
            kx = _kx()
            fwd = DeviceCSR.upload(self.a, device)
            pair = (fwd, fwd.transpose(kx))
            self._dev[key] = pair
        return pair

    def release(self) -> None:
        self._dev.clear()

    def _apply_dev(self, v):
        kx = _kx()
        fwd, _ = self.device_csr()
        y = kx.empty(self.output_dim)
        kx.csr_spmv(fwd, v, y)
        return y

    def _apply_adjoint_dev(self, u):
        kx = _kx()
        _, bwd = self.device_csr()
        y = kx.empty(self.input_dim)
        kx.csr_spmv(bwd, u, y)
        return y

    def apply_columns_dev(self, V):
        kx = _kx()
        fwd, _ = self.device_csr()
        Y = kx.empty(self.output_dim, V.shape[1])
        kx.csr_spmm(fwd, V.contiguous(), Y)
        return Y

    def apply_adjoint_columns_dev(self, U):
        kx = _kx()
        _, bwd = self.device_csr()
        Y = kx.empty(self.input_dim, U.shape[1])
        kx.csr_spmm(bwd, U.contiguous(), Y)
        return Y


class DiagonalOperator(LinearOperator):
    """Multiplication by diag(d) (operators.py:89-101)."""

    def __init__(self, d):
        d = np.asarray(d.detach().cpu().numpy() if isinstance(d, torch.Tensor) else d, dtype=float)
        super().__init__(d.size, d.size)
        self.d = d
        self._dd = None

    def _ddev(self):
        if self._dd is None:
            self._dd = to_device(self.d)
        return self._dd

    def _apply_dev(self, v):
        kx = _kx()
        y = kx.empty(self.output_dim)
        kx.vmul(1.0, self._ddev(), v, 0.0, y)
        return y

    def _apply_adjoint_dev(self, u):
        return self._apply_dev(u)

    def apply_columns_dev(self, V):
        Y = V.contiguous().clone()
        _kx().row_scale(Y, self._ddev())
        return Y

    def apply_adjoint_columns_dev(self, U):
        return self.apply_columns_dev(U)


class DiagPlusLowRank(LinearOperator):
    """Symmetric diag(d) + F F^T kept in factored form (operators.py:138-160):
    apply = d o v + F (F^T v), two skinny GEMVs and one elementwise pass."""

    def __init__(self, d, F):
        d = np.asarray(d, dtype=float)
        F = np.asarray(F, dtype=float)
        if F.ndim != 2 or F.shape[0] != d.size:
            raise DimensionMismatchError("factor F must be n-by-k with n = len(d)")
        super().__init__(d.size, d.size)
        self.d = d
        self.F = F
        self._dev = None

    def _devs(self):
        if self._dev is None:
            self._dev = (to_device(self.d), to_device(np.ascontiguousarray(self.F)))
        return self._dev

    def _apply_dev(self, v):
        kx = _kx()
        d, F = self._devs()
        t = kx.empty(1, F.shape[1])
        kx.gemvT(F, v.view(1, -1), t)  # F^T v
        y = kx.empty(1, self.output_dim)
        kx.gemv(F, t, y)  # F (F^T v)
        y = y.view(-1)
        kx.vmul(1.0, d, v, 1.0, y)  # d o v + F (F^T v)
        return y

    def _apply_adjoint_dev(self, u):
        return self._apply_dev(u)

    def apply_columns_dev(self, V):
        kx = _kx()
        d, F = self._devs()
        n, k = F.shape
        s = V.shape[1]
        V = V.contiguous()
        T = kx.empty(k, s)
        kx.gemm(1, 0, k, s, n, 1.0, F, F.stride(0), V, V.stride(0), 0.0, T, s)
        Y = V.clone()
        kx.row_scale(Y, d)
        kx.gemm(0, 0, n, s, k, 1.0, F, F.stride(0), T, s, 1.0, Y, s)
        return Y

    def apply_adjoint_columns_dev(self, U):
        return self.apply_columns_dev(U)


class StackedOperator(LinearOperator):
    """Vertical concatenation [A_1; A_2; ...] on a common domain
    (operators.py:163-191); the adjoint sums the part adjoints."""

    def __init__(self, ops):
        ops = list(ops)
        if not ops:
            raise DimensionMismatchError("stack_vertical requires at least one operator")
        n = ops[0].input_dim
        for op in ops:
            if op.input_dim != n:
                raise DimensionMismatchError("stacked operators must share input_dim")
        super().__init__(n, sum(op.output_dim for op in ops))
        self.ops = ops
        self._offsets = np.cumsum([0] + [op.output_dim for op in ops])

    @property
    def has_adjoint(self) -> bool:
        return all(op.has_adjoint for op in self.ops)

    def _apply_dev(self, v):
        kx = _kx()
        y = kx.empty(self.output_dim)
        for op, lo, hi in zip(self.ops, self._offsets[:-1], self._offsets[1:]):
            kx.copy(op._apply_dev(v), y[lo:hi])
        return y

    def _apply_adjoint_dev(self, u):
        kx = _kx()
        out = kx.zeros(self.input_dim)
        for op, lo, hi in zip(self.ops, self._offsets[:-1], self._offsets[1:]):
            kx.axpby(1.0, op._apply_adjoint_dev(u[lo:hi].contiguous()), 1.0, out)
        return out

    def apply_columns_dev(self, V):
        return torch.cat([op.apply_columns_dev(V) for op in self.ops], dim=0).contiguous()

    def apply_adjoint_columns_dev(self, U):
        kx = _kx()
        out = kx.zeros(self.input_dim, U.shape[1])
        flat = out.view(-1)
        for op, lo, hi in zip(self.ops, self._offsets[:-1], self._offsets[1:]):
            kx.axpby(1.0, adjoint_columns_dev(op, U[lo:hi].contiguous()).reshape(-1), 1.0, flat)
        return out


class OnesRowOperator(LinearOperator):
    """The 1-by-n summing map v -> (sum v); adjoint broadcasts a scalar
    (operators.py:194-203)."""

    def __init__(self, dim: int):
        super().__init__(dim, 1)

    def _apply_dev(self, v):
        out = _kx().empty(3)
        _kx().vstats(v, None, out)
        return out[:1]

    def _apply_adjoint_dev(self, u):
        y = _kx().empty(self.input_dim)
        _kx().bcast(u, 1.0, y)
        return y

    def apply_columns_dev(self, V):
        kx = _kx()
        n, s = V.shape
        ones = torch.ones(1, n, dtype=F64, device=V.device)
        Y = kx.empty(1, s)
        kx.gemm(0, 0, 1, s, n, 1.0, ones, n, V.contiguous(), s, 0.0, Y, s)
        return Y

    def apply_adjoint_columns_dev(self, U):
        kx = _kx()
        s = U.shape[1]
        ones = torch.ones(self.input_dim, 1, dtype=F64, device=U.device)
        Y = kx.empty(self.input_dim, s)
        kx.gemm(0, 0, self.input_dim, s, 1, 1.0, ones, 1, U.contiguous(), s, 0.0, Y, s)
        return Y


def adjoint_columns_dev(op: LinearOperator, U: torch.Tensor) -> torch.Tensor:
    """op^T applied to every column of the row-major m x s matrix U."""
    f = getattr(op, "apply_adjoint_columns_dev", None)
    if f is not None:
        return f(U)
    cols = [op._apply_adjoint_dev(U[:, j].contiguous()) for j in range(U.shape[1])]
    return torch.stack(cols, dim=1).contiguous()


class MatrixFreeOperator(LinearOperator):
    """Operator defined by callables (operators.py:206-228): ``matvec`` and
    ``rmatvec`` on CUDA tensors, or NumPy-only callables as the reference takes
    them (``UserFn``)."""

    def __init__(self, input_dim: int, output_dim: int, matvec: Callable, rmatvec: Optional[Callable] = None):
        super().__init__(input_dim, output_dim)
        self._matvec = UserFn(matvec)
        self._rmatvec = UserFn(rmatvec) if rmatvec is not None else None

    @property
    def has_adjoint(self) -> bool:
        return self._rmatvec is not None

    def _apply_dev(self, v):
        return self._matvec(v)

    def _apply_adjoint_dev(self, u):
        return self._rmatvec(u)


class HessianOperator(LinearOperator):
    """Curvature of the smooth objective at the current iterate
    (operators.py:231-264)."""

    is_constant: bool = True
    diag_shift: float = 0.0

    def __init__(self, dim: int):
        super().__init__(dim, dim)

    def update(self, x) -> None:
        pass

    def smooth_part(self) -> LinearOperator:
        if self.diag_shift == 0.0:
            return self
        shift = self.diag_shift
        return MatrixFreeOperator(
            self.input_dim, self.output_dim,
            device_fn(lambda v: self._apply_dev(to_device(v)) - shift * to_device(v)),
            device_fn(lambda u: self._apply_dev(to_device(u)) - shift * to_device(u)),
        )

    def _apply_adjoint_dev(self, u):
        return self._apply_dev(u)


class FunctionHessian(HessianOperator):
    """Hessian-vector product supplied as a callable ``hvp(x, v)`` (on CUDA
    tensors, or NumPy-only as the reference takes it: ``UserFn``;
    operators.py:280-297); ``update`` stores the evaluation point."""

    is_constant = False

    def __init__(self, dim: int, hvp: Callable, x0=None):
        super().__init__(dim)
        self._hvp = UserFn(hvp)
        self._x = None if x0 is None else x0  # moved to the device at first use

    def update(self, x) -> None:
        self._x = to_device(x).clone()

    def _apply_dev(self, v):
        if not isinstance(self._x, torch.Tensor):
            self._x = torch.zeros_like(v) if self._x is None else to_device(self._x)
        return self._hvp(self._x, v)


class ConstantHessian(HessianOperator):
    """Hessian that never changes (quadratic objectives), operators.py:267-277."""

    def __init__(self, op: LinearOperator):
        if op.input_dim != op.output_dim:
            raise DimensionMismatchError("a Hessian must be square")
        super().__init__(op.input_dim)
        self.op = op

    def _apply_dev(self, v):
        return self.op._apply_dev(v)

    def apply_columns_dev(self, V):
        return self.op.apply_columns_dev(V)


def as_operator(a) -> LinearOperator:
    """Coerce an ndarray / CUDA tensor / scipy sparse matrix / operator into a
    LinearOperator (operators.py:300-309)."""
    if isinstance(a, LinearOperator):
        return a
    import scipy.sparse as sp

    if sp.issparse(a):
        return SparseOperator(a)
    if isinstance(a, torch.Tensor):
        return DenseOperator(a)
    arr = np.asarray(a, dtype=float)
    if arr.ndim != 2:
        raise DimensionMismatchError("expected a 2-d matrix or a LinearOperator")
    return DenseOperator(arr)


def stack_vertical(ops) -> "StackedOperator":
    """Vertically stack operators sharing a common input dimension (operators.py:312-314)."""
    return StackedOperator(ops)


def update_hessian(op: HessianOperator, x) -> None:
    op.update(x)
