import sys, numpy as np
which = sys.argv[1]
if which == 'ref':
    sys.path.insert(0,'/root/reference/pkg/src')
    import nysopt as N
else:
    sys.path.insert(0,'/root/repo' if len(sys.argv)<3 else sys.argv[2])
    import paper_2310_08333_b200 as N
n, rank, nu = 500, 20, 1e-2
lam = 1e4 * (np.arange(1, n + 1, dtype=float) ** -2)
for seed in range(4):
    g = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(g.standard_normal((n, n)))
    A_base = (Q * lam) @ Q.T
    H = A_base + nu * np.eye(n)
    b = g.standard_normal(n)
    H_op = N.DenseOperator(H)
    _, plain = N.pcg(H_op, b, tol_rel=1e-8, max_iter=10 * n)
    sk = N.nystrom_sketch(N.DenseOperator(A_base), rank, rng_seed=seed)
    P = N.NystromPreconditioner(sk, nu)
    _, pre = N.pcg(H_op, b, Minv=P.apply, tol_rel=1e-8, max_iter=10 * n)
    lamh = np.asarray(sk.lambda_hat if isinstance(sk.lambda_hat, np.ndarray) else sk.lambda_hat.cpu().numpy())
    print(seed, plain.iterations, pre.iterations, 'rank', len(lamh), 'lam head', lamh[:3], 'tail', lamh[-3:], 'resid', plain.final_residual if hasattr(plain,'final_residual') else None)
