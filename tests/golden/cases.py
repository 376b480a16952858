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

# tolerances of the configs: eps_abs = eps_rel = eps_dual_gap = 1e-4 (BASELINE.json)
BASE_OPTIONS = dict(eps_abs=1e-4, eps_rel=1e-4, eps_dual_gap=1e-4)

# cases the default generator run produces (cfg4 / cfg5_shard need 10-20 min of CPU: --only)
DEFAULT_SOLVES = [k for k in SOLVE_CASES if k not in ("cfg4", "cfg5_shard")]


def options_for(name):
    """Options of a case; a ``huber_stop`` entry stands for
    ``custom_stop=huber_subdiff_stop(tol)`` (see ``split_stop``)."""
    opts = dict(BASE_OPTIONS)
    opts.update(SOLVE_CASES[name][1])
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
