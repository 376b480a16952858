"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the development container (the only place ``/root/reference`` exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py          # default cases
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py --big    # + config 4 (~10 min)

It imports ``nysopt`` from ``/root/reference/pkg/src`` (read-only, no install),
feeds it the seeded inputs of ``tests/golden/cases.py`` and stores only the
outputs as compressed ``.npz`` files next to this script.  Nothing on the GPU
box reads ``/root/reference``: the tests there use these committed fixtures.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import nysopt  # noqa: E402  (the reference)
from nysopt import (  # noqa: E402
    Box,
    DenseOperator,
    IdentityOperator,
    MLProblem,
    NystromPreconditioner,
    QPProblem,
    SolverOptions,
    builtin_loss,
    nystrom_sketch,
    pcg,
)
from nysopt.problems import MLHessian, ml_dual_gap, ml_gradient, ml_objective  # noqa: E402

import cases  # noqa: E402


def ref_problem(spec):
    return cases.build_problem(spec, nysopt)


def make_inputs():
    """Inputs made by the reference's own generators (stored, not re-derived)."""
    from nysopt.bench import gen_huber_data

    from nysopt.bench import gen_portfolio_data

    d, F, mu, gamma = gen_portfolio_data(2, 5)  # n = 200 assets, k = 2 factors
    np.savez_compressed(os.path.join(HERE, "input_portfolio.npz"), d=d, F=F, mu=mu, gamma=np.float64(gamma))
    for name, (n, seed) in (("huber_cycle_a", (100, 2)), ("huber_cycle_b", (60, 0))):
        A, b, lam1 = gen_huber_data(n, seed)  # tests/test_admm.py:577-589
        np.savez_compressed(os.path.join(HERE, f"input_{name}.npz"), loss=np.array("huber"), A=A, b=b,
                            lambda1=np.float64(lam1), lambda2=np.float64(0.0))


def run_solve(name):
    spec = cases.ALL_CASES[name][0]()
    o, stop_tol = cases.split_stop(cases.options_for(name))
    if stop_tol is not None:
        o["custom_stop"] = nysopt.huber_subdiff_stop(stop_tol)
    opts = SolverOptions(**o)
    t0 = time.perf_counter()
    res = nysopt.solve(ref_problem(spec), opts)
    dt = time.perf_counter() - t0
    hist = res.history
    out = dict(
        x=res.x,
        z=res.z,
        u=res.u,
        objective=np.float64(res.objective),
        iterations=np.int64(res.iterations),
        status=np.array(res.status.value),
        rp_norm=np.float64(res.rp_norm),
        rd_norm=np.float64(res.rd_norm),
        gap=np.float64(np.nan if res.gap is None else res.gap),
        cg_iters=np.array([h.cg_iters for h in hist], dtype=np.int64),
        cg_tol=np.array([h.cg_tol for h in hist]),
        rho=np.array([h.rho for h in hist]),
        obj_hist=np.array([h.objective for h in hist]),
        rp_hist=np.array([h.rp_norm for h in hist]),
        rd_hist=np.array([h.rd_norm for h in hist]),
        gap_hist=np.array([np.nan if h.gap is None else h.gap for h in hist]),
        penalty_events=np.array([[e.k, e.rho_old, e.rho_new, e.dual_jump_rel] for e in res.penalty_events]).reshape(-1, 4),
        certificate=res.certificate if res.certificate is not None else np.zeros(0),
        n_history=np.int64(len(hist)),
        x_bar=res.x_bar if res.x_bar is not None else np.zeros(0),
        z_bar=res.z_bar if res.z_bar is not None else np.zeros(0),
        ref_total_s=np.float64(dt),
        ref_setup_s=np.float64(res.timings.setup_s),
        ref_precond_s=np.float64(res.timings.precond_s),
        ref_linsys_s=np.float64(res.timings.linsys_total_s),
    )
    if "A" in spec and "generic" not in spec:
        p = ref_problem(spec)
        out["ml_objective_z"] = np.float64(ml_objective(p, res.z))
    np.savez_compressed(os.path.join(HERE, f"solve_{name}.npz"), **out)
    print(f"{name}: iters={res.iterations} status={res.status.value} obj={res.objective:.12e} "
          f"cg={int(out['cg_iters'].sum())} t={dt:.2f}s", flush=True)


def run_kernels():
    # fused HVP / gradient / gap at a logistic point (problems.py:238-351)
    A, b, x, v = cases.hvp_case()
    out = {}
    for loss in ("square", "logistic", "huber"):
        for lam2 in (0.0, 0.3):
            p = MLProblem(builtin_loss(loss), A, b, 0.7, lam2)
            H = MLHessian(p, x)
            key = f"{loss}_{lam2}"
            out[f"hvp_{key}"] = H.apply(v)
            out[f"w_{key}"] = H._weights
            out[f"grad_{key}"] = ml_gradient(p, x)
            out[f"obj_{key}"] = np.float64(ml_objective(p, x))
            out[f"gap_{key}"] = np.float64(ml_dual_gap(p, x))
    np.savez_compressed(os.path.join(HERE, "kernels_ml.npz"), **out)

    # Nystrom sketch + preconditioner (sketch.py:74-151)
    M, r, seed = cases.sketch_case()
    S = nystrom_sketch(DenseOperator(M), r, rng_seed=seed)
    pc = NystromPreconditioner(S, nu=0.5)
    rng = np.random.default_rng(9)
    V = rng.standard_normal((M.shape[0], 5))
    PV = np.column_stack([pc.apply(V[:, j]) for j in range(5)])
    np.savez_compressed(os.path.join(HERE, "kernels_sketch.npz"), U=S.U, lam=S.lambda_hat, V=V, PV=PV)

    # PCG with and without the preconditioner (krylov.py:35-95)
    H, bb, x0 = cases.pcg_case()
    S2 = nystrom_sketch(DenseOperator(H - 0.7 * np.eye(H.shape[0])), 6, rng_seed=4)
    pc2 = NystromPreconditioner(S2, nu=0.7)
    x1, rep1 = pcg(DenseOperator(H), bb, x0=x0, tol_rel=1e-10)
    x2, rep2 = pcg(DenseOperator(H), bb, x0=x0, Minv=pc2.apply, tol_rel=1e-10)
    np.savez_compressed(
        os.path.join(HERE, "kernels_pcg.npz"),
        x_plain=x1, it_plain=np.int64(rep1.iterations), x_prec=x2, it_prec=np.int64(rep2.iterations),
    )
    # spectrum probes and adaptive sizing (sketch.py:176-282)
    from nysopt import adaptive_sketch, condition_bound, estimate_error_norm, estimate_extreme_eigs

    out = {}
    rng = np.random.default_rng(404)
    Apsd = cases.random_psd(50, rng, decay=np.logspace(2, -2, 50))
    hi, lo = estimate_extreme_eigs(DenseOperator(Apsd), iters=30, rng_seed=4)
    out["eig_hi"], out["eig_lo"] = np.float64(hi), np.float64(lo)
    hi2, lo2 = estimate_extreme_eigs(DenseOperator(np.eye(10)), iters=10, rng_seed=0)  # breakdown
    out["eye_hi"], out["eye_lo"] = np.float64(hi2), np.float64(lo2)
    S = nystrom_sketch(DenseOperator(Apsd), 6, rng_seed=8)
    out["err6"] = np.float64(estimate_error_norm(DenseOperator(Apsd), S, 20, rng_seed=9))
    out["cond6"] = np.float64(condition_bound(S, float(out["err6"]), 0.5))
    for tgt in (10.0, 30.0, 100.0, 1e3, np.inf):
        Sa = adaptive_sketch(DenseOperator(Apsd), r0=2, r_max=32, nu=0.5, kappa_target=tgt, rng_seed=3)
        key = "inf" if not np.isfinite(tgt) else f"{tgt:g}"
        out[f"adapt_rank_{key}"] = np.int64(Sa.rank)
        out[f"adapt_lam_{key}"] = Sa.lambda_hat
    out["A"] = Apsd
    np.savez_compressed(os.path.join(HERE, "kernels_spectrum.npz"), **out)

    # sparse operator applies (operators.py:121-135) on the ragged CSR data
    d = cases._sparse_ml("square", 300, 200, 51)
    A = nysopt.SparseOperator(d["A"])
    v = np.random.default_rng(5).standard_normal(200)
    t = np.random.default_rng(6).standard_normal(300)
    np.savez_compressed(os.path.join(HERE, "kernels_sparse.npz"), v=v, t=t, Av=A.apply(v), Atv=A.apply_adjoint(t))
    print("kernel fixtures written", flush=True)


def run_bench_goldens():
    """The reference's benchmark generators and runner (bench/datagen.py,
    bench/runner.py): generator outputs and run records of small configs."""
    from nysopt.bench import (BenchConfig, gen_bounded_ls, gen_huber_data, gen_logistic_data, gen_portfolio_data,
                              gen_regression_data, run_bench)

    out = {}
    out["reg_A"], out["reg_b"] = gen_regression_data(20, 10, 1)
    out["hub_A"], out["hub_b"], lam = gen_huber_data(20, 3)
    out["hub_lam"] = np.float64(lam)
    out["pf_d"], out["pf_F"], out["pf_mu"], g = gen_portfolio_data(1, 2)
    out["log_A"], lam = gen_logistic_data(20, 10, 4)
    out["log_lam"] = np.float64(lam)
    qp = gen_bounded_ls(20, 5)
    out["bls_P"], out["bls_q"] = qp.P.a, qp.q
    runs = [("lasso", dict(n=60)), ("elastic_net", dict(n=50)), ("logistic", dict(n=40)), ("huber", dict(n=60)),
            ("bounded_ls", dict(n=80)), ("portfolio", dict(k=1, portfolio_path="qp")),
            ("portfolio", dict(k=1, portfolio_path="operators")), ("lasso", dict(n=40, norm="linf", tol=1e-6))]
    for i, (prob, kw) in enumerate(runs):
        rec = run_bench(BenchConfig(problem=prob, seed=3, **kw))
        out[f"run{i}_status"] = np.array(rec.status)
        out[f"run{i}_iters"] = np.int64(rec.iters)
        out[f"run{i}_objective"] = np.float64(rec.objective)
        out[f"run{i}_n"] = np.int64(rec.n)
        print(f"bench run {prob} {kw}: {rec.status} {rec.iters} {rec.objective:.10e}", flush=True)
    np.savez_compressed(os.path.join(HERE, "bench_runs.npz"), **out)


def run_steps():
    """The reference's single-step API (admm.py:215-415) on a general-M QP and a
    logistic problem: residuals, x-update (plain and Nystrom-preconditioned),
    relax / prox / dual steps, the penalty rule and the infeasibility tests."""
    from nysopt.admm import (SolverState, check_infeasibility, check_termination, compute_residuals,
                             relaxed_constraint_point, u_update, update_penalty, x_update, z_update)
    from nysopt import logistic_problem, lower, qp_lower

    inp = cases.steps_inputs()
    out = {}
    qp = QPProblem(inp["P"], inp["q"], inp["M"], Box(inp["lo"], inp["hi"]))
    ml = logistic_problem(inp["A"], inp["b"], 0.2, 0.05)
    for tag, gp, z, u in (("qp", qp_lower(qp), inp["z_qp"], inp["u_qp"]), ("ml", lower(ml), inp["z_ml"], inp["u_ml"])):
        st = SolverState(x=inp["x"].copy(), z=z.copy(), u=u.copy(), rho=0.8, x_bar_sum=np.zeros(gp.n),
                         z_bar_sum=np.zeros(gp.m))
        st.k = 4
        gp.hess.update(st.x)
        for kind in ("l2", "linf"):
            opts = SolverOptions(norm_kind=kind)
            res = compute_residuals(gp, st, opts)
            out[f"{tag}_{kind}_res"] = np.array([res.rp_norm, res.rd_norm, res.primal_scale, res.dual_scale])
            out[f"{tag}_{kind}_term"] = np.int64(check_termination(res, st, opts))
            if kind == "l2":
                out[f"{tag}_rp"], out[f"{tag}_rd"] = res.rp, res.rd
        opts = SolverOptions()
        x_new, rep = x_update(gp, st, opts, None, 1e-11, 1e-4)
        out[f"{tag}_xnew"], out[f"{tag}_cg_iters"] = x_new, np.int64(rep.iterations)
        Mx_new = gp.M.apply(x_new)
        w = relaxed_constraint_point(Mx_new, st, gp, opts.alpha)
        z_new = z_update(gp, st, opts, w)
        out[f"{tag}_w"], out[f"{tag}_znew"], out[f"{tag}_unew"] = w, z_new, u_update(st, w, z_new, gp)
        res = compute_residuals(gp, st, opts)
        ev = update_penalty(st, res, SolverOptions(mu=1.05))
        out[f"{tag}_pen"] = np.array([np.nan] * 3 if ev is None else [ev.rho_old, ev.rho_new, ev.dual_jump_rel])
        out[f"{tag}_u_after_pen"] = st.u.copy()
    gpq = qp_lower(qp)
    dx, du = inp["x"], inp["u_qp"]
    chk = check_infeasibility(dx, du, gpq, SolverOptions(eps_inf=10.0), 0.8)
    out["inf_status"] = np.array(str(chk.status.value if chk.status else "none"))
    out["inf_near"] = np.int64(chk.near_trigger)
    np.savez_compressed(os.path.join(HERE, "kernels_steps.npz"), **out)
    print("steps:", {k: (v.shape if hasattr(v, "shape") and v.shape else v) for k, v in out.items()
                     if k.endswith(("iters", "pen", "status"))}, flush=True)


def run_fuzz():
    """The reference on the randomised small problems of cases.fuzz_case."""
    out = {}
    for i in range(cases.FUZZ_COUNT):
        spec, o = cases.fuzz_case(i)
        res = nysopt.solve(ref_problem(spec), SolverOptions(**o))
        out[f"c{i}_x"], out[f"c{i}_z"] = res.x, res.z
        out[f"c{i}_meta"] = np.array([res.iterations, res.objective, res.rp_norm, res.rd_norm,
                                      sum(h.cg_iters for h in res.history), len(res.penalty_events)])
        out[f"c{i}_status"] = np.array(res.status.value)
        print(f"fuzz {i}: {res.status.value} iters={res.iterations} obj={res.objective:.8e} "
              f"events={len(res.penalty_events)}", flush=True)
    np.savez_compressed(os.path.join(HERE, "solve_fuzz.npz"), **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also run config 4 (~10 min)")
    ap.add_argument("--only", nargs="*", default=None)
    args = ap.parse_args()
    names = args.only if args.only else (list(cases.DEFAULT_SOLVES) + list(cases.GENERAL_CASES) + list(cases.GENERIC_CASES)
                                         + (["cfg4"] if args.big else []))
    make_inputs()
    if not args.only:
        run_kernels()
        run_bench_goldens()
        run_steps()
        run_fuzz()
    for name in names:
        run_solve(name)


if __name__ == "__main__":
    main()
