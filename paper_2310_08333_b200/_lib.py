"""ctypes binding of libnysgpu.so (the C ABI declared in include/nysgpu.h).

The product path has NO CPU fallback: ``lib()`` raises ``CapabilityError`` when
the library is missing or no sm_100 device is visible, and every kernel
status code is turned into the reference's exception classes
(``/root/reference/pkg/src/nysopt/errors.py:4-29``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import CapabilityError, DataError, DimensionMismatchError, NotSPDError, NumericalError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnysgpu.so")

NYS_OK = 0
NYS_ERR_ARG = 1
NYS_ERR_CUDA = 2
NYS_ERR_NOT_SPD = 3
NYS_ERR_NONFINITE = 4
NYS_ERR_NOT_PSD = 5
NYS_ERR_UNSUPPORTED = 6
NYS_ERR_WORKSPACE = 7
NYS_ERR_NO_DEVICE = 8

def dev_env(name, default=None):
    """Development switch ``name`` (an ``NYS_*`` A/B variable of DESIGN.md §5):
    honoured only when ``NYS_DEV_SWITCHES=1`` is set as well; otherwise the
    default (the measured-best choice) applies and the environment is ignored."""
    if os.environ.get("NYS_DEV_SWITCHES") == "1":
        return os.environ.get(name, default)
    return default


LOSS = {"square": 0, "logistic": 1, "huber": 2}
PROX_SOFT, PROX_BOX = 0, 1

# CG scalar slots (nys_cg_slot)
CG_RZ, CG_PAP, CG_ALPHA, CG_RES2, CG_RZNEW, CG_B2, CG_FLAG = 0, 1, 2, 3, 4, 5, 6
CG_TICKET, CG_DONE, CG_ITERS, CG_RESREL, CG_RUNNING, CG_NSLOTS = 7, 8, 9, 10, 11, 16
CG_NHVP = 12
CG_SKIPPED = 5  # sc[CG_DONE] of a solve whose gate was closed
NORMS_NOUT = 16
ROWS_NOUT = 5

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int
F64 = C.c_double
SZ = C.c_size_t


class CgProblem(C.Structure):
    """Mirror of ``nys_cg_problem`` (include/nysgpu.h)."""

    _fields_ = [
        ("op_kind", C.c_int), ("A", P), ("rows", I64), ("n", I64), ("lda", I64), ("d", P),
        ("shift", F64), ("U", P), ("r", C.c_int), ("ldu", I64), ("lam", P), ("nu", F64),
        ("b", P), ("x", P), ("res", P), ("p", P), ("z", P), ("Ap", P), ("sc", P),
        ("tol", F64), ("max_iter", I64), ("ws_op", P), ("ws_op_bytes", SZ), ("ws_pc", P),
        ("ws_pc_bytes", SZ), ("ws_red", P), ("gate", P), ("tol_dev", P), ("timing_tag", I64),
        ("ws_cp", P), ("ws_cp_bytes", SZ), ("order_in", P), ("order_out", P),
        ("reduce", P), ("reduce_user", P),
    ]

class AdmmTail(C.Structure):
    """Mirror of ``nys_admm_tail`` (include/nysgpu.h)."""

    _fields_ = [
        ("kind", C.c_int), ("loss", C.c_int), ("n", I64), ("rows", I64), ("A", P), ("lda", I64), ("b", P),
        ("XZ", P), ("u", P), ("xbar", P), ("zbar", P), ("accum", C.c_int),
        ("alpha", F64), ("kappa", F64), ("lo", P), ("hi", P), ("q", P),
        ("lambda1", F64), ("lambda2", F64), ("rho", F64), ("with_z", C.c_int),
        ("AXZ", P), ("T", P), ("w", P), ("AT", P), ("rowsums", P), ("norms", P),
        ("ring", P), ("uring", P), ("ring_ld", I64), ("slot", C.c_int),
        ("nothers", C.c_int), ("others", C.c_int * 16), ("wnorms", P),
        ("qp_infeas", C.c_int), ("inf_first", C.c_int), ("inf_last", C.c_int), ("width", F64),
        ("dx", P), ("Pdx", P), ("infeas", P), ("pdx2", P),
        ("ws_gemv", P), ("ws_gemv_bytes", SZ), ("ws_gemvT", P), ("ws_gemvT_bytes", SZ), ("ws_red", P),
        ("pred", P), ("gate_next", P), ("conj_out", P), ("order", P), ("zu_done", C.c_int),
        ("reduce", P), ("reduce_user", P),
        ("rb_src", P), ("rb_dst", P), ("rb_n", I64), ("rb_gate", P), ("rb_tag", F64), ("rb_done", C.c_int),
        ("stop_on", C.c_int), ("stop_gap", C.c_int), ("stop_linf", C.c_int), ("stop_slot", C.c_int),
        ("stop_ran", C.c_int),
        ("stop_eps_gap", F64), ("stop_eps_abs", F64), ("stop_eps_rel", F64), ("stop_sqrt_n", F64),
        ("gb", P),
    ]

# nys_reduce_fn (include/nysgpu.h): the host-side all-reduce hook of the sharded drivers
REDUCE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)


class AdmmHead(C.Structure):
    """Mirror of ``nys_admm_head`` (include/nysgpu.h)."""

    _fields_ = [
        ("n", I64), ("hxA", P), ("gA", P), ("q", P), ("lambda2", F64), ("sigma", F64), ("rho", F64),
        ("shift", F64), ("x", P), ("z", P), ("u", P), ("xbar", P), ("zbar", P), ("rhs", P), ("r", P),
        ("sc", P), ("snap", P), ("gate", P), ("gate_next", P), ("prev", P), ("norm_kind", C.c_int),
        ("kpow", F64), ("tol_fixed", F64), ("tol_out", P), ("ws_red", P), ("zu", P),
    ]


# name: (restype, argtypes)
SIGNATURES = {
    "nys_admm_tail_f64": (I32, [C.POINTER(AdmmTail), P]),
    "nys_admm_head_f64": (I32, [C.POINTER(AdmmHead), P]),
    "nys_admm_xupdate_f64": (I32, [C.POINTER(AdmmHead), C.POINTER(CgProblem), I32, P]),
    "nys_abi_version": (I32, []),
    "nys_copy_f64": (I32, [P, P, I64, P]),
    "nys_readback_f64": (I32, [P, P, I64, P, P, P]),
    "nys_status_string": (C.c_char_p, [I32]),
    "nys_device_check": (I32, []),
    "nys_launch_count": (C.c_ulonglong, []),
    "nys_reduce_workspace": (SZ, []),
    "nys_gemv_workspace": (SZ, [I64, I64, I32]),
    "nys_gemv_f64": (I32, [P, I64, I64, I64, P, I64, I32, P, I64, P, SZ, P]),
    "nys_gemvT_workspace": (SZ, [I64, I64, I32]),
    "nys_gemvT_f64": (I32, [P, I64, I64, I64, P, I64, I32, P, I64, P, SZ, P]),
    "nys_hvp_workspace": (SZ, [I64, I64]),
    "nys_hvp_f64": (I32, [P, I64, I64, I64, P, P, F64, P, P, I32, P, SZ, P]),
    "nys_hvp_plan": (I32, [I64, I64, I64]),
    "nys_shift_dot_f64": (I32, [I64, P, F64, P, P, P, P]),
    "nys_dot_f64": (I32, [I64, P, P, P, P, P]),
    "nys_precond_workspace": (SZ, [I64, I32]),
    "nys_precond_apply_f64": (I32, [P, I64, I32, I64, P, F64, P, P, P, P, P, SZ, P]),
    "nys_cg_start_f64": (I32, [I64, P, P, P, P, P, P]),
    "nys_cg_step_xr_f64": (I32, [I64, P, P, P, P, I32, P, P, P]),
    "nys_cg_dir_f64": (I32, [I64, P, P, I32, P, P]),
    "nys_cg_workspace": (SZ, [I32, I64, I64, I32, C.POINTER(SZ), C.POINTER(SZ)]),
    "nys_cg_iterate_f64": (I32, [C.POINTER(CgProblem), I64, I32, P]),
    "nys_timing_enable": (I32, [I32]),
    "nys_timing_commit": (I32, [I64, I64, I64]),
    "nys_cg_persist_workspace": (SZ, [I64, I32]),
    "nys_timing_read": (I32, [C.POINTER(F64), C.POINTER(I64)]),
    "nys_admm_rhs_f64": (I32, [I64, P, P, P, F64, F64, F64, F64, P, P, P, P, P, P, P, P]),
    "nys_admm_zu_f64": (I32, [I64, P, P, P, F64, I32, F64, P, P, P, P, I32, P]),
    "nys_admm_norms_f64": (I32, [I64, P, P, P, P, P, F64, F64, P, F64, P, P, P, P, P]),
    "nys_ml_rowwise_f64": (I32, [I64, I32, P, P, P, P, P, P, P, P, P, P]),
    "nys_ml_conj_scaled_f64": (I32, [I64, I32, P, F64, P, P, P, P]),
    "nys_window_norms_f64": (I32, [I64, P, I64, I32, C.POINTER(C.c_int), I32, P, P, P]),
    "nys_scale_dual_f64": (I32, [I64, P, F64, F64, P, P, P]),
    "nys_qp_infeas_f64": (I32, [I64, P, P, P, P, F64, P, P, P, P, P, P, P]),
    "nys_axpby_f64": (I32, [I64, F64, P, F64, P, P]),
    "nys_soft_threshold_f64": (I32, [I64, P, F64, P, P]),
    "nys_loss_eval_f64": (I32, [I32, I32, I64, P, P, P]),
    "nys_box_project_f64": (I32, [I64, P, P, P, P, P]),
    "nys_row_scale_f64": (I32, [I64, I64, P, I64, P, P]),
    "nys_gemm_workspace": (SZ, [I64, I64, I64]),
    "nys_gemm_tile": (I32, [I32]),
    "nys_gemm_f64": (I32, [I32, I32, I64, I64, I64, F64, P, I64, P, I64, F64, P, I64, P, SZ, P]),
    "nys_gaussian_workspace": (SZ, [I64]),
    "nys_gaussian_async_f64": (I32, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, I64, P, P, P, SZ, P]),
    "nys_orthonormalize_async_f64": (I32, [I64, I32, P, P, P, P, SZ, P]),
    "nys_nystrom_core_async_f64": (I32, [I64, I32, I32, P, P, P, P, P, P, SZ, P]),
    "nys_gaussian_f64": (I32, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, I64, P, P, SZ, P]),
    "nys_gaussian_draws_f64": (I32, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, I64, P, P, SZ, P, P]),
    "nys_orthonormalize_workspace": (SZ, [I64, I32]),
    "nys_orthonormalize_f64": (I32, [I64, I32, P, P, P, SZ, P]),
    "nys_nystrom_workspace": (SZ, [I64, I32, I32]),
    "nys_nystrom_core_f64": (I32, [I64, I32, I32, P, P, P, P, C.POINTER(C.c_int), P, SZ, P]),
    "nys_syevj_workspace": (SZ, [I32]),
    "nys_syevj_f64": (I32, [I32, P, P, P, P, SZ, P]),
    "nys_tail_cluster_workspace": (SZ, [I64, I64]),
    "nys_ml_tail_f64": (I32, [P, I64, I64, I64, P, P, P, I32, P, P, P, P, P, SZ, P]),
    "nys_ml_tail_gb_f64": (I32, [P, I64, I64, I64, P, P, P, I32, P, P, P, P, P, P, SZ, P]),
    "nys_csr_spmv_f64": (I32, [I64, P, P, P, P, F64, P, F64, P, P, I32, P]),
    "nys_csr_spmm_f64": (I32, [I64, P, P, P, P, I64, I32, P, P, I64, P]),
    "nys_csr_transpose_workspace": (SZ, [I64, I64]),
    "nys_csr_transpose": (I32, [I64, I64, P, P, P, P, P, P, P, SZ, P]),
    "nys_vmul_f64": (I32, [I64, F64, P, P, F64, P, P]),
    "nys_bcast_f64": (I32, [I64, P, F64, P, P]),
    "nys_vstats_f64": (I32, [I64, P, P, P, P, P]),
    "nys_gdual_f64": (I32, [I64, P, P, F64, P, P, P]),
    "nys_absstats_f64": (I32, [I64, P, F64, P, P, P]),
    "nys_box_cert_f64": (I32, [I64, P, P, P, P, P, P, P]),
    "nys_box_violation_f64": (I32, [I64, P, P, P, P, P, P]),
}

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """dlopen the library and bind every declared symbol (no device needed)."""
    if not os.path.exists(path):
        raise CapabilityError(
            f"libnysgpu.so not found at {path}; build it with `python -m paper_2310_08333_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib() -> C.CDLL:
    """The loaded library, after checking that an sm_100 GPU is present."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                import torch

                if not torch.cuda.is_available():
                    raise CapabilityError("no CUDA device: the B200 path has no CPU fallback")
                l = load_library()
                if l.nys_abi_version() != 1:
                    raise CapabilityError("libnysgpu ABI version mismatch")
                torch.cuda.init()
                if l.nys_device_check() != NYS_OK:
                    raise CapabilityError("libnysgpu requires an sm_100 (B200) device")
                _lib = l
    return _lib


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI status to the reference exception hierarchy."""
    if rc == NYS_OK:
        return
    msg = f"{what}: {lib().nys_status_string(rc).decode()}" if _lib is not None else what
    if rc == NYS_ERR_ARG:
        raise DimensionMismatchError(msg)
    if rc == NYS_ERR_NOT_SPD:
        raise NotSPDError(msg)
    if rc == NYS_ERR_NONFINITE:
        raise NumericalError(msg)
    if rc == NYS_ERR_NOT_PSD:
        raise DataError("operator is not positive semidefinite (negative pivot in sketch core)")
    if rc in (NYS_ERR_UNSUPPORTED, NYS_ERR_NO_DEVICE):
        raise CapabilityError(msg)
    raise NumericalError(f"CUDA failure in {what} (status {rc})")
