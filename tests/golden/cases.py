"""Seeded inputs for the golden parity cases.

Inputs are regenerated from seeds (NumPy PCG64 is bit-reproducible across
machines with the same NumPy), so the committed fixtures hold only the
reference's OUTPUTS.  ``make_golden.py`` feeds these inputs to the reference
package; the tests feed the same inputs to the oracle and to the GPU path.
"""

from __future__ import annotations

import numpy as np

from paper_2310_08333_b200 import datagen


def random_psd(n, rng, rank=None, decay=None):
    """Symmetric PSD matrix with a controlled spectrum (same construction as the
    reference test oracle ``tests/_oracles.py:152-161``)."""
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    if decay is not None:
        lam = np.asarray(decay, dtype=float)
    elif rank is not None:
        lam = np.concatenate([rng.uniform(0.5, 2.0, size=rank), np.zeros(n - rank)])
    else:
        lam = rng.uniform(0.1, 2.0, size=n)
    return (Q * lam) @ Q.T


# ---- solve cases: name -> dict(kind, builder) --------------------------------


def _ml_small(kind, N, n, seed, lam2=0.0, lam_frac=0.1):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((N, n)) / np.sqrt(N)
    xt = np.zeros(n)
    sup = rng.choice(n, size=max(1, n // 10), replace=False)
    xt[sup] = rng.standard_normal(sup.size)
    if kind == "logistic":
        y = np.where(rng.random(N) < 1.0 / (1.0 + np.exp(-(A @ xt) * 3.0)), 1.0, -1.0)
        A = -y[:, None] * A
        b = np.zeros(N)
        lam1 = lam_frac * float(np.max(np.abs(A.T @ np.ones(N)))) / 2.0
    else:
        b = A @ xt + 0.05 * rng.standard_normal(N)
        if kind == "huber":
            idx = rng.choice(N, size=max(1, N // 20), replace=False)
            b[idx] += 5.0
        lam1 = lam_frac * float(np.max(np.abs(A.T @ b)))
    return dict(loss=kind, A=A, b=b, lambda1=lam1, lambda2=lam2)


def _qp_small(N, n, seed):
    A, b, P, q = datagen.boxqp_data(N, n, seed)
    return dict(P=P, q=q, lo=np.zeros(n), hi=np.ones(n))


def _cfg(c):
    d = datagen.make_config(c)
    if d.kind == "boxqp":
        return dict(P=d.P, q=d.q, lo=d.lo, hi=d.hi)
    return dict(loss=d.loss, A=d.A, b=d.b, lambda1=d.lambda1, lambda2=d.lambda2)


def _cfg5_shard(j=0):
    """Config 5's row block j (12500 x 200000, 20 GB): exactly the rows one GPU
    holds in the 8-GPU run, solved as a standalone LASSO with its own lambda
    (0.1 ||A_j' b_j||_inf) - the per-GPU size of config 5 at a size the CPU
    reference finishes in ~15 min."""
    Ab, noise = datagen.cfg5_block(j)
    b = Ab @ datagen.cfg5_truth() + noise
    lam = 0.1 * float(np.max(np.abs(Ab.T @ b)))
    return dict(loss="square", A=Ab, b=b, lambda1=lam, lambda2=0.0)


def _from_inputs(name):
    """Inputs produced by a reference generator (``make_golden.py`` stores them
    next to the outputs: ``input_<name>.npz``), e.g. the robust-regression data
    of the reference's cycle-guard test (``tests/test_admm.py:577-589``)."""
    import os

    d = dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), f"input_{name}.npz")))
    if "P" in d:
        return dict(P=d["P"], q=d["q"], lo=d["lo"], hi=d["hi"])
    return dict(loss=str(d["loss"]), A=d["A"], b=d["b"], lambda1=float(d["lambda1"]), lambda2=float(d["lambda2"]))


def _qp_unbounded(n=10, seed=9):
    """P = 0, q < 0, box [0, inf): dual infeasible (tests/test_admm.py:391-401,
    with M = I as the identity operator)."""
    rng = np.random.default_rng(seed)
    q = -np.abs(rng.standard_normal(n))
    return dict(P=np.zeros((n, n)), q=q, lo=np.zeros(n), hi=np.full(n, np.inf))


# ---- general-operator cases (sparse data, structured P, general M) ----------


def _sparse(N, n, seed, density):
    """Seeded CSR data with ragged rows, one empty row and one empty column."""
    import scipy.sparse as sp

    rng = np.random.default_rng(seed)
    mask = rng.random((N, n)) < density
    vals = rng.standard_normal((N, n)) / np.sqrt(N * density)
    D = np.where(mask, vals, 0.0)
    D[7, :] = 0.0
    D[:, 3] = 0.0
    return sp.csr_matrix(D)


def _sparse_ml(kind, N, n, seed, density=0.05, lam2=0.0, lam_frac=0.1):
    A = _sparse(N, n, seed, density)
    rng = np.random.default_rng(seed + 1000)
    xt = np.zeros(n)
    sup = rng.choice(n, size=max(1, n // 10), replace=False)
    xt[sup] = rng.standard_normal(sup.size)
    if kind == "logistic":
        y = np.where(rng.random(N) < 1.0 / (1.0 + np.exp(-(A @ xt) * 3.0)), 1.0, -1.0)
        A = A.multiply(-y[:, None]).tocsr()
        b = np.zeros(N)
        lam1 = lam_frac * float(np.max(np.abs(A.T @ np.ones(N)))) / 2.0
    else:
        b = A @ xt + 0.05 * rng.standard_normal(N)
        lam1 = lam_frac * float(np.max(np.abs(A.T @ b)))
    return dict(loss=kind, A=A, b=b, lambda1=lam1, lambda2=lam2)


def _lasso_qp(N=60, n=30, seed=31):
    """lasso_as_qp inputs (problems.py:484-502): the QP itself is built by each
    consumer's own lasso_as_qp (sparse P and a sparse 2x2-block M)."""
    d = _ml_small("square", N, n, seed)
    return dict(lasso_qp=(d["A"], d["b"], d["lambda1"]))


def _portfolio(path):
    """Portfolio allocation on the reference generator's data (stored inputs):
    path "operators" = diag-plus-low-rank P and the stacked [1'; I] map
    (datagen.py:180-193); "qp" = the lifted QP with a sparse M (datagen.py:148-177)."""
    import os

    import scipy.sparse as sp

    f = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "input_portfolio.npz"))
    d, F, mu, gamma = f["d"], f["F"], f["mu"], float(f["gamma"])
    n, k = F.shape
    if path == "operators":
        return dict(P={"dplr": (gamma * d, np.sqrt(gamma) * F)}, q=-mu, M={"stack": ["ones", "eye"]},
                    lo=np.concatenate([[1.0], np.zeros(n)]), hi=np.concatenate([[1.0], np.full(n, np.inf)]))
    P = {"diag": np.concatenate([gamma * d, gamma * np.ones(k)])}
    M = sp.bmat([[sp.csr_matrix(F.T), -sp.eye(k)], [sp.csr_matrix(np.ones((1, n))), None],
                 [sp.eye(n), None]]).tocsr()
    return dict(P=P, q=np.concatenate([-mu, np.zeros(k)]), M=M,
                lo=np.concatenate([np.zeros(k), [1.0], np.zeros(n)]),
                hi=np.concatenate([np.zeros(k), [1.0], np.full(n, np.inf)]))


def _qp_primal_infeasible(n=20, m=60, seed=4):
    """Contradictory parallel rows planted in a random sparse-pattern dense M
    (the construction of tests/test_admm.py:365-388)."""
    rng = np.random.default_rng(seed)
    Pt = rng.random((n, n))
    P = Pt.T @ Pt
    q = rng.random(n)
    M = rng.standard_normal((m, n)) * (rng.random((m, n)) < 0.3)
    hi = 3 + rng.standard_normal(m)
    lo = -3 + rng.standard_normal(m)
    lo, hi = np.minimum(lo, hi), np.maximum(lo, hi)
    j = m // 2
    M[j] = M[j + 1]
    lo[j] = hi[j + 1] + 10 * rng.random()
    hi[j] = lo[j] + 0.5
    return dict(P=P, q=q, M=M, lo=lo, hi=hi)


def _qp_check_rank(seed=12345):
    """PD P (6x6) with a dense 8x6 M (tests/test_admm.py:605-615 shapes)."""
    rng = np.random.default_rng(seed)
    P = rng.standard_normal((6, 6))
    P = P @ P.T + 0.5 * np.eye(6)
    M = rng.standard_normal((8, 6))
    return dict(P=P, q=rng.standard_normal(6), M=M, lo=-np.ones(8), hi=np.ones(8))


def _qp_dense_M(n=40, m=60, seed=41):
    """Rank-deficient P (rank n/2) with a tall dense M: sigma_eff = sigma."""
    rng = np.random.default_rng(seed)
    P = random_psd(n, rng, rank=n // 2)
    M = rng.standard_normal((m, n)) / np.sqrt(n)
    return dict(P=P, q=rng.standard_normal(n), M=M, lo=-np.ones(m), hi=np.ones(m))


def _generic(kind, seed, offset=False):
    """Problems handed over as callables (problems.py:125-157): "lasso" = a lasso through
    f / grad f / Hessian-vector product / soft-threshold prox on NumPy arrays, optionally
    with a nonzero constraint offset c (x - z = c); "portfolio" = the simplex-prox
    splitting of the stored portfolio data (bench/datagen.py:184-214)."""
    if kind == "portfolio":
        import os

        f = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "input_portfolio.npz"))
        return dict(generic="portfolio", d=f["d"], F=f["F"], mu=f["mu"], gamma=float(f["gamma"]))
    g = np.random.default_rng(seed)
    N, n = 80, 40
    A = g.standard_normal((N, n)) / np.sqrt(N)
    xs = np.where(g.random(n) < 0.2, g.standard_normal(n), 0.0)
    b = A @ xs + 0.01 * g.standard_normal(N)
    lam = 0.1 * float(np.max(np.abs(A.T @ b)))
    c = 0.05 * g.standard_normal(n) if offset else np.zeros(n)
    return dict(generic="lasso", A=A, b=b, lam=lam, c=c)


def pseudo_huber(ns):
    """A user-defined loss (problems.py:35-50): l(w) = sqrt(1 + w^2) - 1 with its derivatives and
    its conjugate 1 - sqrt(1 - y^2) on |y| <= 1 (+inf outside)."""
    def conj(y):
        y = np.asarray(y, dtype=float)
        inside = np.abs(y) <= 1.0
        return np.where(inside, 1.0 - np.sqrt(np.clip(1.0 - y * y, 0.0, None)), np.inf)

    return ns.Loss(kind="pseudo_huber", value=lambda w: np.sqrt(1.0 + np.asarray(w, dtype=float) ** 2) - 1.0,
                   deriv=lambda w: np.asarray(w, dtype=float) / np.sqrt(1.0 + np.asarray(w, dtype=float) ** 2),
                   deriv2=lambda w: (1.0 + np.asarray(w, dtype=float) ** 2) ** -1.5, conj=conj)


def build_generic(spec, ns):
    if spec["generic"] == "portfolio":
        import importlib

        bench = importlib.import_module(ns.__name__ + ".bench")
        return bench.portfolio_generic_problem(spec["d"], spec["F"], spec["mu"], spec["gamma"])
    A, b, lam, c = spec["A"], spec["b"], spec["lam"], spec["c"]
    n = A.shape[1]
    return ns.GenericProblem(
        n=n, m=n, f=lambda x: 0.5 * float(np.linalg.norm(A @ x - b) ** 2), grad_f=lambda x: A.T @ (A @ x - b),
        hess=ns.FunctionHessian(n, lambda x, v: A.T @ (A @ v)), g=lambda z: lam * float(np.abs(z).sum()),
        prox_g=lambda v, rho, tol: np.sign(v) * np.maximum(np.abs(v) - lam / rho, 0.0),
        M=ns.IdentityOperator(n), c=c, full_rank=True)


def build_problem(spec, ns):
    """Problem of a case spec in the namespace ``ns`` (the reference package or
    this repo's: both export the same constructors)."""
    if "generic" in spec:
        return build_generic(spec, ns)
    if spec.get("loss") == "pseudo_huber":
        return ns.MLProblem(pseudo_huber(ns), spec["A"], spec["b"], spec["lambda1"], spec["lambda2"])
    if "lasso_qp" in spec:
        return ns.lasso_as_qp(*spec["lasso_qp"])
    if "P" not in spec:
        return ns.MLProblem(ns.builtin_loss(spec["loss"]), spec["A"], spec["b"], spec["lambda1"], spec["lambda2"])
    import scipy.sparse as sp

    def op(a, n):
        if isinstance(a, dict) and "dplr" in a:
            return ns.DiagPlusLowRank(*a["dplr"])
        if isinstance(a, dict) and "diag" in a:
            return ns.DiagonalOperator(a["diag"])
        if isinstance(a, dict) and "stack" in a:
            parts = [ns.OnesRowOperator(n) if t == "ones" else ns.IdentityOperator(n) for t in a["stack"]]
            return ns.stack_vertical(parts)
        if sp.issparse(a):
            return ns.SparseOperator(a)
        return ns.DenseOperator(a)

    P = op(spec["P"], None)
    n = P.input_dim
    M = ns.IdentityOperator(n) if spec.get("M") is None else op(spec["M"], n)
    return ns.QPProblem(P, spec["q"], M, ns.Box(spec["lo"], spec["hi"]))


GENERAL_CASES = {
    "sparse_lasso": (lambda: _sparse_ml("square", 300, 200, 51), dict(sketch_rank=10, rng_seed=51)),
    "sparse_logistic": (lambda: _sparse_ml("logistic", 400, 150, 52, density=0.08, lam2=1e-3),
                        dict(sketch_rank=10, rng_seed=52)),
    "sparse_enet_rho": (lambda: _sparse_ml("square", 250, 120, 53, density=0.1, lam2=0.05),
                        dict(sketch_rank=8, rng_seed=53, rho0=0.02, penalty_warmup=5, penalty_update_every=5)),
    "lasso_as_qp": (lambda: _lasso_qp(), dict(sketch_rank=10, rng_seed=31, max_iter=3000)),
    "lasso_as_qp_rho": (lambda: _lasso_qp(), dict(sketch_rank=10, rng_seed=31, max_iter=3000, rho0=10.0,
                                                  penalty_warmup=5, penalty_update_every=5)),
    "portfolio_ops": (lambda: _portfolio("operators"), dict(rng_seed=5, max_iter=3000)),
    "portfolio_qp": (lambda: _portfolio("qp"), dict(rng_seed=5, max_iter=3000)),
    "qp_primal_infeas_M": (lambda: _qp_primal_infeasible(), dict(max_iter=4000, eps_inf=1e-4)),
    "qp_check_rank": (lambda: _qp_check_rank(), dict(check_rank=True, max_iter=300, rng_seed=2)),
    "qp_assume_rank": (lambda: _qp_check_rank(), dict(assume_full_rank=True, max_iter=300, rng_seed=2)),
    "qp_dense_M": (lambda: _qp_dense_M(), dict(sketch_rank=8, rng_seed=41, max_iter=3000)),
}

# problems given as callables (the reference's generic front end); pinned to the
# reference's outputs directly (the CPU oracle covers the ML / QP forms only)
GENERIC_CASES = {
    "generic_lasso": (lambda: _generic("lasso", 61), dict(sketch_rank=8, rng_seed=61, max_iter=3000)),
    "generic_offset": (lambda: _generic("lasso", 62, offset=True),
                       dict(sketch_rank=8, rng_seed=62, max_iter=3000, rho0=5.0, penalty_warmup=5,
                            penalty_update_every=5)),
    "generic_portfolio": (lambda: _generic("portfolio", 0), dict(rng_seed=5, max_iter=3000)),
    # a user-defined loss through the ML front end (gap stop via its conjugate; resketches every 20)
    "custom_loss": (lambda: {**_ml_small("square", 150, 60, 71, lam2=1e-3, lam_frac=0.1), "loss": "pseudo_huber"},
                    dict(sketch_rank=8, rng_seed=71, max_iter=3000, eps_dual_gap=1e-10)),
}


# penalty adaptation from the first iterations (admm.py:677-698): rho0 far from
# balance makes the balanced-residual rule fire every 5 iterations
_PEN = dict(penalty_warmup=5, penalty_update_every=5)

# name: (problem builder, options dict)
SOLVE_CASES = {
    "lasso_small": (lambda: _ml_small("square", 120, 200, 11), dict(sketch_rank=10, rng_seed=11)),
    "lasso_tall": (lambda: _ml_small("square", 300, 80, 12), dict(sketch_rank=8, rng_seed=12)),
    "enet_small": (lambda: _ml_small("square", 150, 120, 13, lam2=0.05), dict(sketch_rank=12, rng_seed=13)),
    "logistic_small": (lambda: _ml_small("logistic", 300, 150, 14, lam2=1e-3, lam_frac=0.1), dict(sketch_rank=10, rng_seed=14)),
    "logistic_l1only": (lambda: _ml_small("logistic", 200, 100, 15, lam2=0.0, lam_frac=0.2), dict(sketch_rank=8, rng_seed=15)),
    "huber_small": (lambda: _ml_small("huber", 200, 100, 16), dict(sketch_rank=8, rng_seed=16)),
    "lasso_noprec": (lambda: _ml_small("square", 120, 200, 17), dict(use_preconditioner=False, rng_seed=17)),
    "lasso_linf": (lambda: _ml_small("square", 120, 200, 18), dict(sketch_rank=10, rng_seed=18, norm_kind="linf", use_dual_gap=False)),
    "lasso_exact": (lambda: _ml_small("square", 100, 150, 19), dict(sketch_rank=10, rng_seed=19, exact_x_solve=True)),
    "boxqp_small": (lambda: _qp_small(400, 200, 20), dict(sketch_rank=20, rng_seed=20)),
    # wide rows (n > 12800: the cluster HVP), also solved row-sharded (tests/test_gpu_sharded.py)
    "lasso_wide": (lambda: _ml_small("square", 400, 20000, 61), dict(sketch_rank=20, rng_seed=61)),
    # --- adaptive control flow: penalty changes, cycle guard, certificates, time limit
    "lasso_rho_hi": (lambda: _ml_small("square", 120, 200, 11), dict(sketch_rank=10, rng_seed=11, rho0=100.0, **_PEN)),
    "lasso_rho_lo": (lambda: _ml_small("square", 120, 200, 11), dict(sketch_rank=10, rng_seed=11, rho0=0.01, **_PEN)),
    "logistic_rho_hi": (lambda: _ml_small("logistic", 300, 150, 14, lam2=1e-3, lam_frac=0.1),
                        dict(sketch_rank=10, rng_seed=14, rho0=100.0, **_PEN)),
    "logistic_rho_lo": (lambda: _ml_small("logistic", 300, 150, 14, lam2=1e-3, lam_frac=0.1),
                        dict(sketch_rank=10, rng_seed=14, rho0=0.01, **_PEN)),
    "boxqp_rho": (lambda: _qp_small(400, 200, 20), dict(sketch_rank=20, rng_seed=20, rho0=50.0, **_PEN)),
    "huber_cycle_a": (lambda: _from_inputs("huber_cycle_a"),
                      dict(huber_stop=1e-4, max_iter=8000, use_dual_gap=False)),
    "huber_cycle_b": (lambda: _from_inputs("huber_cycle_b"),
                      dict(huber_stop=1e-4, max_iter=8000, use_dual_gap=False)),
    "qp_unbounded": (lambda: _qp_unbounded(), dict(max_iter=4000)),
    "lasso_time0": (lambda: _ml_small("square", 120, 200, 11), dict(sketch_rank=10, rng_seed=11, time_limit=0.0)),
    "cfg1": (lambda: _cfg(1), dict(sketch_rank=50, rng_seed=0)),
    "cfg3": (lambda: _cfg(3), dict(sketch_rank=100, rng_seed=2)),
    "cfg2": (lambda: _cfg(2), dict(sketch_rank=100, rng_seed=1)),
    "cfg4": (lambda: _cfg(4), dict(sketch_rank=200, rng_seed=3)),
    "cfg5_shard": (lambda: _cfg5_shard(0), dict(sketch_rank=300, rng_seed=4)),
}

ALL_CASES = {**SOLVE_CASES, **GENERAL_CASES, **GENERIC_CASES}

# tolerances of the configs: eps_abs = eps_rel = eps_dual_gap = 1e-4 (BASELINE.json)
BASE_OPTIONS = dict(eps_abs=1e-4, eps_rel=1e-4, eps_dual_gap=1e-4)

# cases the default generator run produces (cfg4 / cfg5_shard need 10-20 min of CPU: --only)
DEFAULT_SOLVES = [k for k in SOLVE_CASES if k not in ("cfg4", "cfg5_shard")]


def options_for(name):
    """Options of a case; a ``huber_stop`` entry stands for
    ``custom_stop=huber_subdiff_stop(tol)`` (see ``split_stop``)."""
    opts = dict(BASE_OPTIONS)
    opts.update(ALL_CASES[name][1])
    return opts


def split_stop(opts):
    """(options without ``huber_stop``, its tolerance or None): each consumer
    builds the custom stop from its own package's ``huber_subdiff_stop``."""
    opts = dict(opts)
    return opts, opts.pop("huber_stop", None)


# ---- kernel-level cases -------------------------------------------------------


def hvp_case(seed=101, N=70, n=45):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((N, n))
    b = rng.standard_normal(N)
    x = rng.standard_normal(n) * 0.3
    v = rng.standard_normal(n)
    return A, b, x, v


def sketch_case(seed=202, n=40, r=8):
    rng = np.random.default_rng(seed)
    return random_psd(n, rng, decay=np.logspace(1, -3, n)), r, 7


def pcg_case(seed=303, n=30):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((2 * n, n))
    H = A.T @ A + 0.7 * np.eye(n)
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n) * 0.1
    return H, b, x0


def steps_inputs(seed=77):
    """Seeded inputs of the single-step fixtures (shared with tests/test_gpu_steps.py)."""
    g = np.random.default_rng(seed)
    n, m, N = 14, 19, 30
    B = g.standard_normal((n, n))
    inp = dict(P=B @ B.T + 0.3 * np.eye(n), q=g.standard_normal(n), M=g.standard_normal((m, n)),
               lo=-np.abs(g.standard_normal(m)), hi=np.abs(g.standard_normal(m)),
               A=g.standard_normal((N, n)), b=np.sign(g.standard_normal(N)),
               x=g.standard_normal(n), z_qp=g.standard_normal(m), u_qp=g.standard_normal(m),
               z_ml=g.standard_normal(n), u_ml=g.standard_normal(n), Mx_new=g.standard_normal(m))
    inp["hi"][:3] = np.inf
    inp["lo"][2:5] = -np.inf
    return inp


# ---------------------------------------------------------------------------
# Randomised small problems (differential test against the reference): shapes
# from 1 x 1 up, odd sizes, N < n and N > n, every front end and a spread of
# options; FUZZ_COUNT specs, each a pure function of its index.
FUZZ_COUNT = 48


FUZZ_MEDIUM = 12  # the last FUZZ_MEDIUM cases: dense ML / box-QP shapes in the hundreds to thousands
# (persistent and batched PCG plans, even and odd widths, rows below and above the SM count)


def fuzz_case(i):
    g = np.random.default_rng(9000 + i)
    kind = ["lasso", "enet", "logistic", "boxqp", "qp_M"][i % 5]
    N, n = int(g.integers(1, 61)), int(g.integers(1, 41))
    if i >= FUZZ_COUNT - FUZZ_MEDIUM:
        kind = ["lasso", "enet", "logistic", "boxqp"][i % 4]
        N, n = int(g.integers(60, 1500)), int(g.integers(60, 2500))
        if kind == "boxqp":
            n = int(g.integers(150, 900))
    opts = dict(alpha=float(g.choice([1.0, 1.5, 1.8])), rho0=float(g.choice([0.1, 1.0, 10.0])),
                norm_kind=str(g.choice(["l2", "linf"])), use_preconditioner=bool(g.random() < 0.8),
                sketch_rank=int(g.choice([1, 3, 8])), penalty_update_every=int(g.choice([0, 5, 25])),
                penalty_warmup=int(g.choice([5, 50])), rng_seed=int(g.integers(0, 1000)), max_iter=400,
                eps_abs=1e-5, eps_rel=1e-5, eps_dual_gap=1e-5)
    if kind in ("lasso", "enet", "logistic"):
        A = g.standard_normal((N, n)) / np.sqrt(max(N, 1))
        if kind == "logistic":
            A = -np.sign(g.standard_normal(N))[:, None] * A
            b = np.zeros(N)
            lam1 = 0.1 * float(np.max(np.abs(A.T @ np.ones(N)))) / 2.0
        else:
            b = g.standard_normal(N)
            lam1 = 0.1 * float(np.max(np.abs(A.T @ b)))
        lam2 = 0.0 if kind == "lasso" else float(g.choice([1e-3, 0.1]))
        if g.random() < 0.3:
            opts["use_dual_gap"] = False
        spec = dict(loss="logistic" if kind == "logistic" else "square", A=A, b=b, lambda1=lam1, lambda2=lam2)
    else:
        B = g.standard_normal((n, max(1, n // 2)))
        P = B @ B.T + float(g.choice([0.0, 0.1])) * np.eye(n)
        q = g.standard_normal(n)
        if kind == "boxqp":
            spec = dict(P=P, q=q, lo=-np.abs(g.standard_normal(n)), hi=np.abs(g.standard_normal(n)))
        else:
            m = int(g.integers(1, 31))
            M = g.standard_normal((m, n))
            lo, hi = -np.abs(g.standard_normal(m)) - 0.1, np.abs(g.standard_normal(m)) + 0.1
            lo[g.random(m) < 0.2] = -np.inf
            hi[g.random(m) < 0.2] = np.inf
            spec = dict(P=P, q=q, M=M, lo=lo, hi=hi)
    return spec, opts
