"""Host-side logic of the drop-in API that runs without a GPU: option
validation, tolerance schedule, sketch sizing, problem validation, error
classes, the config generators and the GPU Gaussian stream's host restatement."""

import numpy as np
import pytest

import paper_2310_08333_b200 as nys
from paper_2310_08333_b200 import datagen
from paper_2310_08333_b200.sketch import raw_test_matrix, sketch_width


def test_cg_tolerance_known_answers():
    # krylov.py:98-112, test_krylov.py:118-122
    assert nys.cg_tolerance(2, 0.01, 0.01) == pytest.approx(0.004353, abs=1e-6)
    assert nys.cg_tolerance(1, 0.0, 1.0) == 1e-12
    assert nys.cg_tolerance(1, 4.0, 4.0) == 1.0
    for bad in ((0, 1.0, 1.0), (1, -1.0, 1.0)):
        with pytest.raises(ValueError):
            nys.cg_tolerance(*bad)
    with pytest.raises(ValueError):
        nys.cg_tolerance(1, 1.0, 1.0, gamma=1.0)


def test_default_sketch_rank_and_width():
    assert nys.default_sketch_rank(10) == 1
    assert nys.default_sketch_rank(200) == 10
    assert nys.default_sketch_rank(5000) == 50
    # s = min(n, r + 8 + r//4): 70/133/133/258/383 for the five configs
    assert [sketch_width(10**6, r) for r in (50, 100, 100, 200, 300)] == [70, 133, 133, 258, 383]
    assert sketch_width(4, 2) == 4


def test_solver_options_validation():
    nys.SolverOptions()
    for kw in (dict(sigma=-1), dict(gamma=1.0), dict(alpha=2.0), dict(alpha=0.0), dict(tau=1.0),
               dict(mu=0.5), dict(rho0=0.0), dict(norm_kind="l1")):
        with pytest.raises(nys.DataError):
            nys.SolverOptions(**kw)


def test_problem_validation():
    A = np.ones((3, 2))
    with pytest.raises(nys.DataError):
        nys.MLProblem(nys.square_loss(), A, np.ones(2), 0.1, 0.0)
    with pytest.raises(nys.DataError):
        nys.MLProblem(nys.square_loss(), A, np.ones(3), 0.0, 0.0)
    with pytest.raises(nys.DataError):
        nys.MLProblem(nys.square_loss(), A, np.ones(3), -1.0, 0.0)
    with pytest.raises(nys.DataError):
        nys.builtin_loss("hinge")
    with pytest.raises(nys.DataError):
        nys.Box(np.ones(2), np.zeros(2))
    with pytest.raises(nys.DimensionMismatchError):
        nys.DenseOperator(np.ones(3))
    p = nys.lasso_problem(A, np.ones(3), 0.5)
    assert (p.n, p.N) == (2, 3) and p.loss.deriv2_constant
    q = nys.QPProblem(np.eye(2), np.zeros(2), nys.IdentityOperator(2), nys.Box(np.zeros(2), np.ones(2)))
    assert nys.lower(q).full_rank and nys.lower(p).full_rank


def test_error_hierarchy_matches_reference():
    # errors.py:4-29
    assert issubclass(nys.NotSPDError, nys.NumericalError)
    assert issubclass(nys.NumericalError, ArithmeticError)
    assert issubclass(nys.DataError, ValueError)
    assert issubclass(nys.CapabilityError, TypeError)
    assert issubclass(nys.DimensionMismatchError, ValueError)
    for e in (nys.DataError, nys.CapabilityError, nys.NumericalError, nys.InputError):
        assert issubclass(e, nys.NysoptError)


def test_raw_test_matrix_is_the_reference_stream():
    # sketch.py:97-98: default_rng(seed).standard_normal((n, s))
    np.testing.assert_array_equal(raw_test_matrix(50, 7, 3), np.random.default_rng(3).standard_normal((50, 7)))


def test_ziggurat_restatement_matches_numpy():
    """The GPU Gaussian kernel restates PCG64 + NumPy's ziggurat; the build-time
    self-check (same algorithm in Python) must reproduce NumPy exactly."""
    from paper_2310_08333_b200.gen_tables import _check, extract_tables

    ki, wi, fi = extract_tables()
    assert ki.shape == wi.shape == fi.shape == (256,)
    _check(ki, wi, fi, seed=2024, count=3000)


def test_config_generators_shapes_and_determinism():
    d = datagen.make_config(1, scale=0.1)
    assert d.A.shape == (100, 200) and d.b.shape == (100,) and d.kind == "lasso"
    d2 = datagen.make_config(1, scale=0.1)
    np.testing.assert_array_equal(d.A, d2.A)
    assert d.lambda1 == pytest.approx(0.1 * np.max(np.abs(d.A.T @ d.b)))
    g = datagen.make_config(2, scale=0.05)
    assert g.loss == "logistic" and g.lambda2 == 1e-3 and np.all(g.b == 0)
    np.testing.assert_allclose(np.linalg.norm(g.A, axis=0), 1.0)
    q = datagen.make_config(3, scale=0.02)
    np.testing.assert_allclose(q.P, q.P.T)
    assert q.lo.min() == 0.0 and q.hi.max() == 1.0
    blk, noise = datagen.cfg5_block(3, rows_per_block=4, n=10)
    assert blk.shape == (4, 10) and noise.shape == (4,)
