"""The drop-in boundary by name: every public name the reference package defines
in the modules of the hot path (``nysopt/__init__.py:12-95`` and the modules its
own test-suite imports from) exists here under the same module path.  The name
lists were read off the reference (``dir()`` of each module, its own definitions
and the re-exports its tests use); nothing here needs a GPU -- importing must
work without one."""

import importlib
import inspect

import pytest

PKG = "paper_2310_08333_b200"

NAMES = {
    "": ["Box", "CapabilityError", "CgReport", "ConstantHessian", "DataError", "DenseOperator", "DiagPlusLowRank",
         "DiagonalOperator", "DimensionMismatchError", "FunctionHessian", "GenericProblem", "HessianOperator",
         "IdentityOperator", "InputError", "IterationRecord", "LinearOperator", "Loss", "MLProblem",
         "MatrixFreeOperator", "NotSPDError", "NumericalError", "NysoptError", "NystromPreconditioner",
         "NystromSketch", "OnesRowOperator", "PenaltyEvent", "QPProblem", "SolveResult", "SolverOptions",
         "SolverState", "SparseOperator", "StackedOperator", "Status", "adaptive_sketch", "as_operator",
         "box_project", "box_recession_distance", "box_support", "builtin_loss", "cg_tolerance", "condition_bound",
         "default_sketch_rank", "diagonal_reduce", "elastic_net_problem", "estimate_error_norm",
         "estimate_extreme_eigs", "huber_loss", "huber_problem", "huber_subdiff_distance", "huber_subdiff_stop",
         "lasso_as_qp", "lasso_problem", "logistic_loss", "logistic_problem", "lower", "ml_dual_gap",
         "ml_dual_point", "ml_dual_value", "ml_gradient", "ml_hessian_operator", "ml_objective", "ml_smooth_value",
         "ml_x_system", "nystrom_sketch", "pcg", "precond_apply", "qp_lower", "simplex_project", "soft_threshold",
         "solve", "square_loss", "stack_vertical", "update_hessian", "update_shift"],
    ".admm": ["InfeasibilityCheck", "IterationRecord", "PenaltyEvent", "Residuals", "SolveResult", "SolverOptions",
              "SolverState", "Status", "Timings", "check_infeasibility", "check_termination", "compute_residuals",
              "relaxed_constraint_point", "solve", "u_update", "update_penalty", "x_update", "z_update",
              "box_recession_distance", "box_support", "cg_tolerance", "estimate_extreme_eigs", "ml_dual_gap",
              "nystrom_sketch", "pcg", "MatrixFreeOperator"],
    ".problems": ["GenericProblem", "Loss", "MLHessian", "MLProblem", "QPProblem", "SparseOperator", "box_indicator",
                  "box_project", "builtin_loss", "elastic_net_problem", "huber_loss", "huber_problem",
                  "huber_subdiff_distance", "huber_subdiff_stop", "lasso_as_qp", "lasso_problem", "logistic_loss",
                  "logistic_problem", "lower", "ml_dual_gap", "ml_dual_point", "ml_dual_value", "ml_gradient",
                  "ml_hessian_operator", "ml_lower", "ml_objective", "ml_smooth_value", "ml_x_system", "qp_lower",
                  "soft_threshold", "square_loss"],
    ".operators": ["ConstantHessian", "DenseOperator", "DiagPlusLowRank", "DiagonalOperator", "FunctionHessian",
                   "HessianOperator", "IdentityOperator", "LinearOperator", "MatrixFreeOperator", "OnesRowOperator",
                   "SparseOperator", "StackedOperator", "as_operator", "stack_vertical", "update_hessian"],
    ".krylov": ["CgReport", "cg_tolerance", "pcg", "TOL_FLOOR"],
    ".sketch": ["NystromPreconditioner", "NystromSketch", "adaptive_sketch", "condition_bound",
                "default_sketch_rank", "diagonal_reduce", "estimate_error_norm", "estimate_extreme_eigs",
                "nystrom_sketch", "precond_apply", "update_shift"],
    ".prox": ["Box", "box_indicator", "box_project", "box_recession_distance", "box_recession_project",
              "box_support", "simplex_indicator", "simplex_project", "soft_threshold"],
    ".errors": ["CapabilityError", "DataError", "DimensionMismatchError", "InputError", "NotSPDError",
                "NumericalError", "NysoptError"],
    ".bench": ["BenchConfig", "CSV_HEADER", "RunRecord", "build_problem", "gen_bounded_ls", "gen_huber_data",
               "gen_logistic_data", "gen_portfolio_data", "gen_regression_data", "portfolio_equivalent_qp",
               "portfolio_generic_problem", "portfolio_operator_qp", "read_libsvm", "read_qp_files", "run_bench",
               "write_libsvm"],
    ".bench.records": ["BenchConfig", "RunRecord", "CSV_HEADER"],
    ".bench.datagen": ["gen_bounded_ls", "gen_huber_data", "gen_logistic_data", "gen_portfolio_data",
                       "gen_regression_data", "portfolio_equivalent_qp", "portfolio_generic_problem",
                       "portfolio_operator_qp"],
    ".bench.runner": ["build_problem", "record_from_result", "run_bench", "solve", "write_record", "SolverOptions",
                      "SolveResult"],
    ".bench.io": ["read_libsvm", "read_qp_files", "write_libsvm"],
    ".cli": ["main"],
}


@pytest.mark.parametrize("sub", sorted(NAMES))
def test_reference_names_exist(sub):
    mod = importlib.import_module(PKG + sub)
    missing = [nm for nm in NAMES[sub] if not hasattr(mod, nm)]
    assert not missing, f"{PKG}{sub} lacks {missing}"


def test_dataclass_field_order_matches_reference():
    """Positional construction as in the reference: GenericProblem
    (problems.py:137-150), Loss (problems.py:45-50), Residuals (admm.py:36-43),
    InfeasibilityCheck (admm.py:353-358)."""
    import dataclasses

    import paper_2310_08333_b200 as nys
    from paper_2310_08333_b200 import admm

    fields = lambda c: [f.name for f in dataclasses.fields(c)]  # noqa: E731
    assert fields(nys.GenericProblem)[:14] == ["n", "m", "f", "grad_f", "hess", "g", "prox_g", "M", "c", "is_quadratic",
                                               "full_rank", "prox_inexact", "qp", "ml"]
    assert fields(nys.Loss) == ["kind", "value", "deriv", "deriv2", "conj", "deriv2_constant"]
    assert fields(admm.Residuals)[:6] == ["rp", "rd", "rp_norm", "rd_norm", "primal_scale", "dual_scale"]
    assert fields(admm.InfeasibilityCheck) == ["status", "certificate_primal", "certificate_dual", "near_trigger"]


def test_step_signatures_match_reference():
    """Argument names and order of the single-step API (admm.py:215-415)."""
    from paper_2310_08333_b200 import admm

    want = {
        "compute_residuals": ["problem", "state", "options"],
        "check_termination": ["res", "state", "options", "gap"],
        "x_update": ["problem", "state", "options", "preconditioner", "tol", "sigma_eff"],
        "relaxed_constraint_point": ["Mx_new", "state", "problem", "alpha"],
        "z_update": ["problem", "state", "options", "w"],
        "u_update": ["state", "w", "z_new", "problem"],
        "update_penalty": ["state", "res", "options", "preconditioner", "nu_of_rho"],
        "check_infeasibility": ["delta_x", "delta_u", "problem", "options", "rho"],
    }
    for name, args in want.items():
        assert list(inspect.signature(getattr(admm, name)).parameters) == args, name


def test_lowered_problem_carries_oracles():
    """ml_lower / qp_lower fill f, grad_f, hess, g, prox_g (problems.py:387-450) without touching a device."""
    import numpy as np

    import paper_2310_08333_b200 as nys

    g = nys.lower(nys.lasso_problem(np.eye(3), np.ones(3), 0.1))
    assert all(getattr(g, nm) is not None for nm in ("f", "grad_f", "hess", "g", "prox_g"))
    assert g.full_rank and g.is_quadratic and g.ml is not None
    q = nys.qp_lower(nys.QPProblem(np.eye(2), np.zeros(2), nys.IdentityOperator(2), nys.Box(np.zeros(2), np.ones(2))))
    assert all(getattr(q, nm) is not None for nm in ("f", "grad_f", "hess", "g", "prox_g")) and q.qp is not None
    with pytest.raises(nys.DataError):
        nys.GenericProblem(n=3, m=2, M=nys.IdentityOperator(3), c=np.zeros(2))
