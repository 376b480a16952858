"""Pin the CPU oracle (oracle/port.py) against the reference's own outputs.

The fixtures in tests/golden were produced by running the reference package
(tests/golden/make_golden.py).  The oracle restates the reference arithmetic
in the same operation order, so on the same inputs it must reproduce the
reference trajectory exactly (same iteration and CG counts) and the iterates
to roundoff."""

import numpy as np
import pytest

from conftest import load_golden
import cases

from oracle import port

FAST = [k for k in cases.SOLVE_CASES if not k.startswith("cfg")] + ["cfg1"] + list(cases.GENERAL_CASES)


def oracle_problem(spec):
    if "lasso_qp" in spec:  # problems.py:484-502 in the port's own types
        import scipy.sparse as sp

        A, b, lam = spec["lasso_qp"]
        n = A.shape[1]
        P = sp.bmat([[sp.csr_matrix(A.T @ A), None], [None, sp.csr_matrix((n, n))]]).tocsr()
        q = np.concatenate([-A.T @ b, lam * np.ones(n)])
        eye = sp.eye(n)
        M = sp.bmat([[eye, eye], [eye, -eye]]).tocsr()
        lo = np.concatenate([np.zeros(n), np.full(n, -np.inf)])
        hi = np.concatenate([np.full(n, np.inf), np.zeros(n)])
        return port.QPSpec(P, q, lo, hi, M)
    if "P" in spec:
        def op(a, n):
            if isinstance(a, dict) and "dplr" in a:
                return port.DiagLowRank(*a["dplr"])
            if isinstance(a, dict) and "diag" in a:
                return port.DiagLowRank(a["diag"], np.zeros((a["diag"].size, 0)))
            if isinstance(a, dict) and "stack" in a:
                return port.StackOp([port.OnesRow(n) if t == "ones" else np.eye(n) for t in a["stack"]])
            return a

        P = op(spec["P"], None)
        M = spec.get("M")
        return port.QPSpec(P, spec["q"], spec["lo"], spec["hi"], None if M is None else op(M, P.shape[0]))
    return port.MLSpec(spec["loss"], spec["A"], spec["b"], spec["lambda1"], spec["lambda2"])


def oracle_options(name):
    o, tol = cases.split_stop(cases.options_for(name))
    if tol is not None:
        o["custom_stop"] = port.huber_subdiff_stop(tol)
    return port.Options(**o)


@pytest.mark.parametrize("name", FAST)
def test_oracle_matches_reference_solve(name):
    gold = load_golden(f"solve_{name}.npz")
    spec = cases.ALL_CASES[name][0]()
    res = port.solve(oracle_problem(spec), oracle_options(name))
    assert res.status == str(gold["status"])
    assert res.iterations == int(gold["iterations"])
    np.testing.assert_array_equal(np.array(res.cg_iters), gold["cg_iters"])
    np.testing.assert_allclose(res.rho_hist, gold["rho"], rtol=0, atol=0)
    assert abs(res.objective - float(gold["objective"])) <= 1e-12 * abs(float(gold["objective"]))
    np.testing.assert_allclose(res.x, gold["x"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(res.z, gold["z"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(res.u, gold["u"], rtol=1e-9, atol=1e-12)
    if gold["x_bar"].size:
        np.testing.assert_allclose(res.x_bar, gold["x_bar"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(res.z_bar, gold["z_bar"], rtol=1e-9, atol=1e-12)
    # penalty events: same iterations and penalties exactly, jumps to roundoff
    ev = np.array(res.penalty_events, dtype=float).reshape(-1, 4)
    pe = gold["penalty_events"]
    assert ev.shape == pe.shape, (ev, pe)
    np.testing.assert_array_equal(ev[:, :3], pe[:, :3])
    np.testing.assert_allclose(ev[:, 3], pe[:, 3], rtol=0, atol=1e-12)
    if "certificate" in gold and gold["certificate"].size:
        np.testing.assert_allclose(res.certificate, gold["certificate"], rtol=1e-9, atol=1e-12)
    else:
        assert res.certificate is None


def test_oracle_kernels_match_reference():
    gold = load_golden("kernels_ml.npz")
    A, b, x, v = cases.hvp_case()
    for loss in ("square", "logistic", "huber"):
        for lam2 in (0.0, 0.3):
            key = f"{loss}_{lam2}"
            p = port.MLSpec(loss, A, b, 0.7, lam2)
            w = port.ml_weights(p, x)
            np.testing.assert_allclose(port.ml_hvp(p, w, v), gold[f"hvp_{key}"], rtol=1e-13, atol=1e-13)
            np.testing.assert_allclose(port.ml_gradient(p, x), gold[f"grad_{key}"], rtol=1e-13, atol=1e-13)
            assert port.ml_objective(p, x) == pytest.approx(float(gold[f"obj_{key}"]), rel=1e-14)
            g = float(gold[f"gap_{key}"])
            got = port.ml_dual_gap(p, x)
            if np.isfinite(g):
                assert got == pytest.approx(g, rel=1e-12)
            else:
                assert not np.isfinite(got)


def test_oracle_sketch_and_precond_match_reference():
    gold = load_golden("kernels_sketch.npz")
    M, r, seed = cases.sketch_case()
    U, lam = port.nystrom_sketch(port.dense_operator_columns(M), M.shape[0], r, seed)
    np.testing.assert_allclose(lam, gold["lam"], rtol=1e-13)
    np.testing.assert_allclose(np.abs(U.T @ gold["U"]), np.eye(r), atol=1e-10)
    PV = np.column_stack([port.precond_apply(U, lam, 0.5, gold["V"][:, j]) for j in range(5)])
    np.testing.assert_allclose(PV, gold["PV"], rtol=1e-12, atol=1e-12)


def test_oracle_pcg_matches_reference():
    gold = load_golden("kernels_pcg.npz")
    H, b, x0 = cases.pcg_case()
    x1, rep1 = port.pcg(lambda v: H @ v, b, x0=x0, tol_rel=1e-10)
    assert rep1.iterations == int(gold["it_plain"])
    np.testing.assert_allclose(x1, gold["x_plain"], rtol=1e-12, atol=1e-14)
    U, lam = port.nystrom_sketch(port.dense_operator_columns(H - 0.7 * np.eye(H.shape[0])), H.shape[0], 6, 4)
    x2, rep2 = port.pcg(lambda v: H @ v, b, x0=x0, Minv=lambda v: port.precond_apply(U, lam, 0.7, v), tol_rel=1e-10)
    assert rep2.iterations == int(gold["it_prec"])
    np.testing.assert_allclose(x2, gold["x_prec"], rtol=1e-12, atol=1e-14)


def test_oracle_known_answers():
    # krylov.py KAT (test_krylov.py:118-122)
    assert port.cg_tolerance(2, 0.01, 0.01) == pytest.approx(0.004353, abs=1e-6)
    assert port.cg_tolerance(1, 0.0, 5.0) == 1e-12
    # precond diag(2,1), nu=1 (test_sketch.py:100-104)
    U, lam = port.nystrom_sketch(port.dense_operator_columns(np.diag([2.0, 1.0])), 2, 2, 0)
    np.testing.assert_allclose(port.precond_apply(U, lam, 1.0, np.ones(2)), [2 / 3, 1.0], atol=1e-7)
    # soft threshold examples (test_prox.py:19-23 style)
    np.testing.assert_allclose(port.soft_threshold(np.array([3.0, -0.5, 1.0, -2.0]), 1.0), [2.0, 0.0, 0.0, -1.0])
    with pytest.raises(port.OracleDataError):
        port.nystrom_sketch(port.dense_operator_columns(np.diag([1.0, -1.0, 0.5])), 3, 3, 0)


def test_oracle_spectrum_probes_match_reference():
    """Lanczos extreme eigenvalues, power-method error norm and the adaptive
    rank schedule (sketch.py:176-282)."""
    gold = load_golden("kernels_spectrum.npz")
    A = gold["A"]
    n = A.shape[0]
    hi, lo = port.estimate_extreme_eigs(lambda v: A @ v, n, 30, 4)
    assert hi == pytest.approx(float(gold["eig_hi"]), rel=1e-12)
    assert lo == pytest.approx(float(gold["eig_lo"]), rel=1e-9)
    hi2, lo2 = port.estimate_extreme_eigs(lambda v: v.copy(), 10, 10, 0)
    assert (hi2, lo2) == pytest.approx((float(gold["eye_hi"]), float(gold["eye_lo"])), rel=1e-14)
    U, lam = port.nystrom_sketch(port.dense_operator_columns(A), n, 6, 8)
    err = port.estimate_error_norm(lambda v: A @ v, U, lam, n, 20, 9)
    assert err == pytest.approx(float(gold["err6"]), rel=1e-12)
    for key, tgt in (("10", 10.0), ("30", 30.0), ("100", 100.0), ("1000", 1e3), ("inf", np.inf)):
        U, lam = port.adaptive_sketch(lambda v: A @ v, n, 2, 32, 0.5, tgt, 3)
        assert lam.size == int(gold[f"adapt_rank_{key}"])
        np.testing.assert_allclose(lam, gold[f"adapt_lam_{key}"], rtol=1e-12)


def test_oracle_sparse_apply_matches_reference():
    gold = load_golden("kernels_sparse.npz")
    A = cases._sparse_ml("square", 300, 200, 51)["A"]
    np.testing.assert_allclose(A @ gold["v"], gold["Av"], rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(A.T @ gold["t"], gold["Atv"], rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("i", range(cases.FUZZ_COUNT - cases.FUZZ_MEDIUM))
def test_oracle_matches_reference_on_randomised_problems(i):
    """The oracle against the reference's outputs on the 36 small randomised problems of the
    differential test (cases.fuzz_case; solve_fuzz.npz made by make_golden.py): every front end
    incl. a general M, random options; same status, iteration count, total CG count and number
    of penalty events exactly, iterates to 1e-9."""
    gold = load_golden("solve_fuzz.npz")
    spec, o = cases.fuzz_case(i)
    res = port.solve(oracle_problem(spec), port.Options(**o))
    meta = gold[f"c{i}_meta"]
    assert res.status == str(gold[f"c{i}_status"])
    assert res.iterations == int(meta[0])
    assert int(sum(res.cg_iters)) == int(meta[4])
    assert len(res.penalty_events) == int(meta[5])
    np.testing.assert_allclose(res.x, gold[f"c{i}_x"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(res.z, gold[f"c{i}_z"], rtol=1e-9, atol=1e-12)
