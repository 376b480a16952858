"""The reference's single-step API, loss callables, box / simplex helpers and
generic-problem front end (admm.py:215-415, problems.py:35-157, prox.py:51-152)
on the B200, against NumPy restatements of the same formulas (the reference's
own tests for these, ``tests/test_admm.py`` / ``test_problems.py`` /
``test_prox.py``, check the same identities)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nys():
    import paper_2310_08333_b200 as nys

    return nys


def _qp(nys, rng, n=12):
    B = rng.standard_normal((n, n))
    P = B @ B.T + 0.5 * np.eye(n)
    q = rng.standard_normal(n)
    return nys.QPProblem(P, q, nys.IdentityOperator(n), nys.Box(-np.ones(n), np.ones(n))), P, q


def _state(nys, gp, rng, rho=0.7):
    from paper_2310_08333_b200.admm import SolverState

    st = SolverState(x=rng.standard_normal(gp.n), z=rng.standard_normal(gp.m), u=rng.standard_normal(gp.m), rho=rho,
                     x_bar_sum=np.zeros(gp.n), z_bar_sum=np.zeros(gp.m))
    st.k = 3
    return st


def test_compute_residuals_and_termination(nys, rng):
    from paper_2310_08333_b200.admm import check_termination, compute_residuals

    qp, P, q = _qp(nys, rng)
    gp = nys.qp_lower(qp)
    st = _state(nys, gp, rng)
    for kind in ("l2", "linf"):
        opts = nys.SolverOptions(norm_kind=kind)
        res = compute_residuals(gp, st, opts)
        rp, rd = st.x - st.z, P @ st.x + q + st.rho * st.u
        nrm = (lambda v: np.max(np.abs(v))) if kind == "linf" else np.linalg.norm
        np.testing.assert_allclose(res.rp, rp, atol=1e-13)
        np.testing.assert_allclose(res.rd, rd, atol=1e-12)
        assert res.rp_norm == pytest.approx(nrm(rp), rel=1e-13)
        assert res.rd_norm == pytest.approx(nrm(rd), rel=1e-13)
        assert res.primal_scale == pytest.approx(max(nrm(st.x), nrm(st.z)), rel=1e-13)
        assert res.dual_scale == pytest.approx(nrm(st.rho * st.u), rel=1e-13)
        assert not check_termination(res, st, opts)
        assert check_termination(res, st, opts, gap=0.0)
    st.z = st.x.copy()
    st.u = -(P @ st.x + q) / st.rho
    assert check_termination(compute_residuals(gp, st, nys.SolverOptions()), st, nys.SolverOptions())


def test_x_update_solves_the_subproblem_system(nys, rng):
    """(P + (rho + sigma) I) x+ = sigma x - q + rho (z - u) for a QP with M = I (admm.py:243-275)."""
    from paper_2310_08333_b200.admm import x_update

    qp, P, q = _qp(nys, rng, n=30)
    gp = nys.qp_lower(qp)
    st = _state(nys, gp, rng, rho=1.3)
    sigma = 1e-3
    S = nys.nystrom_sketch(gp.hess.smooth_part(), 8, rng_seed=1)
    for pc in (None, nys.NystromPreconditioner(S, st.rho + sigma)):
        x_new, rep = x_update(gp, st, nys.SolverOptions(), pc, 1e-12, sigma)
        ref = np.linalg.solve(P + (st.rho + sigma) * np.eye(gp.n), sigma * st.x - q + st.rho * (st.z - st.u))
        assert rep.converged and isinstance(x_new, np.ndarray)
        np.testing.assert_allclose(x_new, ref, rtol=1e-9, atol=1e-10)


def test_x_update_general_constraint_map(nys, rng):
    from paper_2310_08333_b200.admm import x_update

    n, m = 10, 14
    B = rng.standard_normal((n, n))
    P, M = B @ B.T + np.eye(n), rng.standard_normal((m, n))
    q = rng.standard_normal(n)
    gp = nys.qp_lower(nys.QPProblem(P, q, M, nys.Box(-np.ones(m), np.ones(m))))
    st = _state(nys, gp, rng, rho=0.4)
    x_new, rep = x_update(gp, st, nys.SolverOptions(), None, 1e-12, 1e-6)
    ref = np.linalg.solve(P + 0.4 * M.T @ M + 1e-6 * np.eye(n), 1e-6 * st.x - q + 0.4 * M.T @ (st.z - st.u))
    np.testing.assert_allclose(x_new, ref, rtol=1e-8, atol=1e-9)


def test_relax_prox_dual_steps(nys, rng):
    from paper_2310_08333_b200.admm import relaxed_constraint_point, u_update, z_update

    A, b = rng.standard_normal((20, 9)), rng.standard_normal(20)
    gp = nys.lower(nys.lasso_problem(A, b, 0.3))
    st = _state(nys, gp, rng, rho=2.0)
    Mx = rng.standard_normal(9)
    w = relaxed_constraint_point(Mx, st, gp, 1.6)
    np.testing.assert_allclose(w, 1.6 * Mx - 0.6 * st.z, atol=1e-14)
    z_new = z_update(gp, st, nys.SolverOptions(), w)
    v = w + st.u
    np.testing.assert_allclose(z_new, np.sign(v) * np.maximum(np.abs(v) - 0.15, 0.0), atol=1e-14)
    np.testing.assert_allclose(u_update(st, w, z_new, gp), st.u + w - z_new, atol=1e-14)


def test_update_penalty_keeps_the_unscaled_dual(nys, rng):
    from paper_2310_08333_b200.admm import Residuals, update_penalty

    qp, _, _ = _qp(nys, rng)
    gp = nys.qp_lower(qp)
    st = _state(nys, gp, rng, rho=1.0)
    y = st.rho * st.u.copy()
    opts = nys.SolverOptions()
    big_p = Residuals(np.ones(12), np.ones(12), 100.0, 1e-3, 1.0, 1.0)
    ev = update_penalty(st, big_p, opts)
    assert ev is not None and st.rho == pytest.approx(opts.tau) and ev.rho_old == 1.0 and ev.k == st.k
    np.testing.assert_allclose(st.rho * st.u, y, rtol=1e-14)
    ev = update_penalty(st, Residuals(np.ones(12), np.ones(12), 1e-3, 100.0, 1.0, 1.0), opts)
    assert st.rho == pytest.approx(1.0)
    assert update_penalty(st, Residuals(np.ones(12), np.ones(12), 1.0, 1.0, 1.0, 1.0), opts) is None


def test_check_infeasibility_certificates(nys):
    """Dual: P = 0, q = -1, box [0, inf) recedes along dx = 1 (tests/test_admm.py:391-401);
    primal: du with M'du = 0 and a negative support value."""
    from paper_2310_08333_b200.admm import check_infeasibility

    n = 4
    qp = nys.QPProblem(np.zeros((n, n)), -np.ones(n), nys.IdentityOperator(n), nys.Box(np.zeros(n), np.full(n, np.inf)))
    gp, opts = nys.qp_lower(qp), nys.SolverOptions()
    chk = check_infeasibility(np.ones(n), np.zeros(n), gp, opts, 1.0)
    assert chk.status == nys.Status.DUAL_INFEASIBLE and np.allclose(chk.certificate_dual, 1.0)
    assert check_infeasibility(-np.ones(n), np.zeros(n), gp, opts, 1.0).status is None
    M = np.array([[1.0], [-1.0]])  # x <= -1 and -x <= -1: empty
    qp2 = nys.QPProblem(np.eye(1), np.zeros(1), M, nys.Box(np.full(2, -np.inf), -np.ones(2)))
    chk2 = check_infeasibility(np.zeros(1), np.ones(2), nys.qp_lower(qp2), opts, 2.0)
    assert chk2.status == nys.Status.PRIMAL_INFEASIBLE and np.allclose(chk2.certificate_primal, 2.0)
    ml = nys.lower(nys.lasso_problem(np.eye(2), np.ones(2), 0.1))
    assert check_infeasibility(np.ones(2), np.ones(2), ml, opts, 1.0).status is None


@pytest.mark.parametrize("kind", ["square", "logistic", "huber"])
def test_loss_callables_match_formulas(nys, kind, rng):
    """value / deriv / deriv2 / conj of problems.py:53-111, scalars and arrays, incl. Fenchel-Young equality."""
    loss = nys.builtin_loss(kind)
    w = np.concatenate([rng.standard_normal(50) * 3, [0.0, 1.0, -1.0, 40.0, -40.0]])
    expit = lambda t: 1.0 / (1.0 + np.exp(-t))  # noqa: E731
    if kind == "square":
        val, d1, d2 = 0.5 * w * w, w, np.ones_like(w)
    elif kind == "logistic":
        val, d1, d2 = np.logaddexp(0.0, w), expit(w), expit(w) * expit(-w)
    else:
        val = np.where(np.abs(w) <= 1, w * w, 2 * np.abs(w) - 1)
        d1, d2 = np.where(np.abs(w) <= 1, 2 * w, 2 * np.sign(w)), np.where(np.abs(w) <= 1, 2.0, 0.0)
    np.testing.assert_allclose(loss.value(w), val, rtol=1e-14, atol=1e-300)
    np.testing.assert_allclose(loss.deriv(w), d1, rtol=1e-14, atol=1e-300)
    np.testing.assert_allclose(loss.deriv2(w), d2, rtol=1e-13, atol=1e-300)
    assert isinstance(loss.value(0.5), float) and loss.value(w.reshape(5, 11)).shape == (5, 11)
    wi = w[np.abs(w) < 5]
    y = np.asarray(loss.deriv(wi))
    np.testing.assert_allclose(np.asarray(loss.value(wi)) + np.asarray(loss.conj(y)), wi * y, rtol=1e-9, atol=1e-9)
    outside = {"square": None, "logistic": np.array([-0.1, 1.1]), "huber": np.array([-2.5, 2.5])}[kind]
    if outside is not None:
        assert np.all(np.isinf(loss.conj(outside)))
    if kind == "logistic":
        assert np.all(np.asarray(loss.conj(np.array([0.0, 1.0]))) == 0.0)


def test_box_support_and_recession(nys, rng):
    box = nys.Box(np.array([-1.0, 0.0, -np.inf, -np.inf, 2.0]), np.array([1.0, np.inf, 3.0, np.inf, 2.0]))
    y = np.array([2.0, -1.0, 0.5, 0.0, -3.0])
    assert nys.box_support(y, box) == pytest.approx(2.0 * 1.0 + 0.0 + 3.0 * 0.5 + 0.0 + 2.0 * -3.0)
    assert nys.box_support(np.array([0.0, 1.0, 0.0, 0.0, 0.0]), box) == np.inf
    assert nys.box_support(np.zeros(5), box) == 0.0
    from paper_2310_08333_b200.prox import box_recession_project

    d = np.array([0.7, -2.0, 4.0, -5.0, 1.0])
    np.testing.assert_allclose(box_recession_project(d, box), [0.0, 0.0, 0.0, -5.0, 0.0])
    assert nys.box_recession_distance(d, box) == pytest.approx(np.sqrt(0.49 + 4.0 + 16.0 + 1.0))


def _simplex_sorted(v):
    u = np.sort(v)[::-1]
    css = np.cumsum(u) - 1.0
    k = np.nonzero(u - css / np.arange(1, v.size + 1) > 0)[0][-1]
    return np.maximum(v - css[k] / (k + 1.0), 0.0)


def test_simplex_project_matches_sort_oracle(nys, rng):
    from paper_2310_08333_b200.prox import simplex_indicator

    for n in (1, 2, 17, 300):
        v = rng.standard_normal(n) * 2
        z = nys.simplex_project(v)
        np.testing.assert_allclose(z, _simplex_sorted(v), atol=1e-12)
        assert simplex_indicator(z) == 0.0
    on = np.array([0.25, 0.75, 0.0])
    np.testing.assert_array_equal(nys.simplex_project(on), on)
    assert simplex_indicator(np.array([0.5, 0.6])) == np.inf
    with pytest.raises(nys.DataError):
        nys.simplex_project(np.array([]))


def test_pcg_takes_numpy_callables(nys, rng):
    """krylov.py:35-44: a NumPy caller hands in NumPy matvec / preconditioner callables."""
    B = rng.standard_normal((8, 8))
    A = B @ B.T + np.eye(8)
    b = rng.standard_normal(8)
    x, rep = nys.pcg(lambda v: A @ v, b, Minv=lambda r: r / np.diag(A), tol_rel=1e-12)
    assert rep.converged and np.allclose(A @ x, b, atol=1e-9)
    with pytest.raises(nys.NumericalError):
        nys.pcg(lambda v: np.full_like(v, np.nan), np.ones(3), tol_rel=1e-10)


def test_generic_problem_with_numpy_callables_agrees_with_lasso(nys, rng):
    """A lasso handed over as f / grad f / Hessian-vector product / prox callables on NumPy
    arrays (tests/test_acceptance.py:73-105) reaches the structured problem's solution; the prox
    tolerance schedule tol0 / k^(2 gamma) is what the prox sees (tests/test_admm.py:283-311)."""
    A, b = rng.standard_normal((60, 25)), rng.standard_normal(60)
    lam = 0.1 * np.max(np.abs(A.T @ b))
    seen = []

    def prox(v, rho, tol):
        seen.append(tol)
        return np.sign(v) * np.maximum(np.abs(v) - lam / rho, 0.0)

    gen = nys.GenericProblem(n=25, m=25, f=lambda x: 0.5 * np.linalg.norm(A @ x - b) ** 2,
                             grad_f=lambda x: A.T @ (A @ x - b), hess=nys.FunctionHessian(25, lambda x, v: A.T @ (A @ v)),
                             g=lambda z: lam * np.abs(z).sum(), prox_g=prox, M=nys.IdentityOperator(25), c=np.zeros(25),
                             full_rank=True, prox_inexact=True)
    r_gen = nys.solve(gen, nys.SolverOptions(eps_abs=1e-7, eps_rel=1e-7, max_iter=5000, rng_seed=0, prox_tol0=1e-8))
    r_ml = nys.solve(nys.lasso_problem(A, b, lam), nys.SolverOptions(eps_dual_gap=1e-9, max_iter=5000, rng_seed=0))
    assert r_gen.status == r_ml.status == nys.Status.OPTIMAL
    np.testing.assert_allclose(r_gen.z, r_ml.z, atol=1e-5)
    assert len(seen) == r_gen.iterations and seen[3] == pytest.approx(1e-8 / 4 ** 2.4)
    assert all(b2 <= a2 for a2, b2 in zip(seen, seen[1:]))


def test_portfolio_three_formulations_agree(nys):
    """bench/datagen.py:148-214: the lifted QP, the operator QP and the simplex-prox
    splitting of one portfolio problem have the same optimum (tests/test_bench.py)."""
    from paper_2310_08333_b200 import bench

    d, F, mu, gamma = bench.gen_portfolio_data(2, 0)
    n = d.size
    opts = nys.SolverOptions(eps_abs=1e-6, eps_rel=1e-6, max_iter=20000, rng_seed=0)
    r_qp = nys.solve(bench.portfolio_equivalent_qp(d, F, mu, gamma), opts)
    r_op = nys.solve(bench.portfolio_operator_qp(d, F, mu, gamma), opts)
    r_gen = nys.solve(bench.portfolio_generic_problem(d, F, mu, gamma), opts)
    assert r_qp.status == r_op.status == r_gen.status == nys.Status.OPTIMAL
    obj = lambda x: 0.5 * gamma * (x @ (d * x) + np.sum((F.T @ x) ** 2)) - mu @ x  # noqa: E731
    vals = [obj(r_qp.x[:n]), obj(r_op.x), obj(r_gen.z)]
    assert max(vals) - min(vals) <= 1e-3 * max(1.0, abs(min(vals)))


def test_steps_match_reference_golden(nys):
    """Every single-step function on a general-M QP and a logistic problem against the
    REFERENCE's outputs on the same seeded inputs (tests/golden/kernels_steps.npz,
    written by make_golden.run_steps from the nysopt package itself)."""
    import cases
    from conftest import load_golden
    from paper_2310_08333_b200.admm import (SolverState, check_infeasibility, check_termination, compute_residuals,
                                            relaxed_constraint_point, u_update, update_penalty, x_update, z_update)

    gold = load_golden("kernels_steps.npz")
    inp = cases.steps_inputs()
    qp = nys.QPProblem(inp["P"], inp["q"], inp["M"], nys.Box(inp["lo"], inp["hi"]))
    ml = nys.logistic_problem(inp["A"], inp["b"], 0.2, 0.05)
    for tag, gp, z, u in (("qp", nys.qp_lower(qp), inp["z_qp"], inp["u_qp"]),
                          ("ml", nys.lower(ml), inp["z_ml"], inp["u_ml"])):
        st = SolverState(x=inp["x"].copy(), z=z.copy(), u=u.copy(), rho=0.8, x_bar_sum=np.zeros(gp.n),
                         z_bar_sum=np.zeros(gp.m))
        st.k = 4
        gp.hess.update(st.x)
        for kind in ("l2", "linf"):
            opts = nys.SolverOptions(norm_kind=kind)
            res = compute_residuals(gp, st, opts)
            got = [res.rp_norm, res.rd_norm, res.primal_scale, res.dual_scale]
            np.testing.assert_allclose(got, gold[f"{tag}_{kind}_res"], rtol=1e-12)
            assert int(check_termination(res, st, opts)) == int(gold[f"{tag}_{kind}_term"])
            if kind == "l2":
                np.testing.assert_allclose(res.rp, gold[f"{tag}_rp"], rtol=1e-12, atol=1e-13)
                np.testing.assert_allclose(res.rd, gold[f"{tag}_rd"], rtol=1e-12, atol=1e-12)
        opts = nys.SolverOptions()
        x_new, rep = x_update(gp, st, opts, None, 1e-11, 1e-4)
        np.testing.assert_allclose(x_new, gold[f"{tag}_xnew"], rtol=1e-8, atol=1e-10)
        assert abs(rep.iterations - int(gold[f"{tag}_cg_iters"])) <= 1
        w = relaxed_constraint_point(gp.M.apply(gold[f"{tag}_xnew"]), st, gp, opts.alpha)
        np.testing.assert_allclose(w, gold[f"{tag}_w"], rtol=1e-12, atol=1e-13)
        z_new = z_update(gp, st, opts, w)
        np.testing.assert_allclose(z_new, gold[f"{tag}_znew"], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(u_update(st, w, z_new, gp), gold[f"{tag}_unew"], rtol=1e-12, atol=1e-13)
        ev = update_penalty(st, compute_residuals(gp, st, opts), nys.SolverOptions(mu=1.05))
        pen = gold[f"{tag}_pen"]
        assert ev is not None and [ev.rho_old, ev.rho_new] == [pen[0], pen[1]] and abs(ev.dual_jump_rel - pen[2]) < 1e-12
        np.testing.assert_allclose(st.u, gold[f"{tag}_u_after_pen"], rtol=1e-13)
    chk = check_infeasibility(inp["x"], inp["u_qp"], nys.qp_lower(qp), nys.SolverOptions(eps_inf=10.0), 0.8)
    assert (chk.status.value if chk.status else "none") == str(gold["inf_status"])
    assert int(chk.near_trigger) == int(gold["inf_near"])


def test_custom_loss_oracles(nys, rng):
    """A user-defined Loss (problems.py:35-50) through the ML oracles: objective, gradient,
    Hessian-vector product and dual value against NumPy."""
    import cases

    loss = cases.pseudo_huber(nys)
    A, b = rng.standard_normal((40, 15)), rng.standard_normal(40)
    p = nys.MLProblem(loss, A, b, 0.2, 0.05)
    x, v = rng.standard_normal(15), rng.standard_normal(15)
    r = A @ x - b
    assert nys.ml_smooth_value(p, x) == pytest.approx(np.sum(np.sqrt(1 + r * r) - 1) + 0.025 * x @ x, rel=1e-12)
    assert nys.ml_objective(p, x) == pytest.approx(nys.ml_smooth_value(p, x) + 0.2 * np.abs(x).sum(), rel=1e-12)
    np.testing.assert_allclose(nys.ml_gradient(p, x), A.T @ (r / np.sqrt(1 + r * r)) + 0.05 * x, rtol=1e-12)
    H = nys.ml_hessian_operator(p, x)
    np.testing.assert_allclose(H.apply(v), A.T @ ((1 + r * r) ** -1.5 * (A @ v)) + 0.05 * v, rtol=1e-11)
    nu = nys.ml_dual_point(p, x)
    at = A.T @ nu
    want = -np.sum(1 - np.sqrt(1 - nu * nu)) - b @ nu - np.sum(np.maximum(np.abs(at) - 0.2, 0) ** 2) / (2 * 0.05)
    assert nys.ml_dual_value(p, nu) == pytest.approx(want, rel=1e-11)
    assert nys.ml_dual_gap(p, x) >= -1e-12
