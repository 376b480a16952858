"""The C-ABI library loads on a machine without a GPU and exports exactly the
entry points include/nysgpu.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nysgpu.h")
LIB = os.path.join(ROOT, "paper_2310_08333_b200", "libnysgpu.so")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(nys_[A-Za-z0-9_]+)\s*\(", src))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2310_08333_b200.build import build

        build()
    from paper_2310_08333_b200 import _lib

    return _lib.load_library()


def test_header_declares_the_hot_path():
    fns = header_functions()
    for required in ("nys_gemv_f64", "nys_gemvT_f64", "nys_hvp_f64", "nys_precond_apply_f64",
                     "nys_cg_step_xr_f64", "nys_admm_zu_f64", "nys_admm_norms_f64", "nys_gemm_f64",
                     "nys_nystrom_core_f64", "nys_gaussian_f64", "nys_syevj_f64"):
        assert required in fns


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = header_functions() - exported
    assert not missing, missing
    for name in header_functions():
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)


def test_ctypes_bindings_cover_the_header():
    from paper_2310_08333_b200 import _lib

    assert set(_lib.SIGNATURES) == header_functions()


def test_host_only_queries(lib):
    assert lib.nys_abi_version() == 1
    assert lib.nys_status_string(5) == b"operator is not positive semidefinite"
    assert lib.nys_reduce_workspace() > 0
    assert lib.nys_hvp_workspace(5000, 10000) >= 5000 * 8
    assert lib.nys_gemm_workspace(133, 133, 10000) > 0
    assert lib.nys_gaussian_workspace(1_330_000) > 2 * 8 * 1_330_000
    assert lib.nys_syevj_workspace(383) > 0


def test_sm100a_code_in_the_library():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_product_path_fails_loudly_without_gpu():
    import numpy as np
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2310_08333_b200 as nys

    with pytest.raises(nys.CapabilityError):
        nys.solve(nys.lasso_problem(np.eye(4), np.ones(4), 0.1))
