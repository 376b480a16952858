"""Device-backed linear operators with the reference's operator contract
(``/root/reference/pkg/src/nysopt/operators.py:20-319``).

``apply(v, out=None)`` / ``apply_adjoint(u, out=None)`` accept NumPy arrays
(returned as NumPy, like the reference) or torch CUDA tensors (returned on the
device).  The dense operator runs the sm_100a GEMV kernels (K1/K2) through the
C ABI; there is no CPU fallback.

In scope: Identity, Dense, MatrixFree, the Hessian
contract and ConstantHessian.  Structured/sparse operators (operators.py:89-228)
are outside the north-star path and raise ``CapabilityError`` if handed to
``solve``.
"""

from __future__ import annotations

from typing import Callable, Optional

import numpy as np
import torch

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


class DenseOperator(LinearOperator):
    """Operator backed by a dense 2-d array (operators.py:104-118).

    ``a`` may be a NumPy array (uploaded to HBM on first use and cached) or a
    CUDA tensor already resident in HBM.  Under ``torch.distributed`` each
    rank uploads only its row shard.
    """

    def __init__(self, a):
        if isinstance(a, torch.Tensor):
            if a.ndim != 2:
                raise DimensionMismatchError("dense operator requires a 2-d array")
            self._dev_full = a.to(dtype=F64).contiguous() if a.is_cuda else None
            self.a = a if not a.is_cuda else None
            if self.a is not None:
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
    def device_rows(self, shard: Optional[Shard] = None, device=None) -> torch.Tensor:
        """The (row-shard of the) matrix in HBM, uploaded once."""
        if shard is None:
            shard = Shard(0, 1, 0, self.output_dim, self.output_dim)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        key = (shard.row_start, shard.row_stop, str(device))
        t = self._shards.get(key)
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

    def release(self) -> None:
        """Drop cached device copies (the host array is kept)."""
        self._shards.clear()

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


class MatrixFreeOperator(LinearOperator):
    """Operator defined by device callables (operators.py:206-228): ``matvec``
    and ``rmatvec`` take and return CUDA tensors."""

    def __init__(self, input_dim: int, output_dim: int, matvec: Callable, rmatvec: Optional[Callable] = None):
        super().__init__(input_dim, output_dim)
        self._matvec = matvec
        self._rmatvec = rmatvec

    @property
    def has_adjoint(self) -> bool:
        return self._rmatvec is not None

    def _apply_dev(self, v):
        return to_device(self._matvec(v))

    def _apply_adjoint_dev(self, u):
        return to_device(self._rmatvec(u))


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
            lambda v: self._apply_dev(to_device(v)) - shift * to_device(v),
            lambda u: self._apply_dev(to_device(u)) - shift * to_device(u),
        )

    def _apply_adjoint_dev(self, u):
        return self._apply_dev(u)


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
    """Coerce an ndarray / CUDA tensor / operator into a LinearOperator
    (operators.py:300-309).  Sparse input is outside the dense hot path."""
    if isinstance(a, LinearOperator):
        return a
    try:
        import scipy.sparse as sp

        if sp.issparse(a):
            raise CapabilityError("sparse operators are not implemented on the B200 path (dense only)")
    except ImportError:  # pragma: no cover
        pass
    if isinstance(a, torch.Tensor):
        return DenseOperator(a)
    arr = np.asarray(a, dtype=float)
    if arr.ndim != 2:
        raise DimensionMismatchError("expected a 2-d matrix or a LinearOperator")
    return DenseOperator(arr)


def update_hessian(op: HessianOperator, x) -> None:
    op.update(x)
