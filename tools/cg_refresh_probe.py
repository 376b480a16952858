"""Probe: PCG across the residual refresh (k = 50) on the lasso_rho_lo system
(A^T A + 0.01 I, Nystrom rank 10).  Prints the residual per iteration for the
batched device CG, the persistent kernel, and NumPy with the same U, lambda."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cases  # noqa: E402
import paper_2310_08333_b200 as nys  # noqa: E402
from paper_2310_08333_b200 import _lib  # noqa: E402
from paper_2310_08333_b200.kernels import get_kernels  # noqa: E402
from paper_2310_08333_b200.krylov import CgWork  # noqa: E402

spec = cases.SOLVE_CASES["lasso_rho_lo"][0]()
A, b = spec["A"], spec["b"]
N, n = A.shape
shift = 0.01
kx = get_kernels()
Ad = torch.from_numpy(A).cuda()
H = nys.MLHessian(nys.lasso_problem(A, b, 0.1))
S = nys.nystrom_sketch(H.smooth_part(), 10, 11)
U, lam = S.U, S.lambda_hat
rhs_h = A.T @ b
bn = np.linalg.norm(rhs_h)


def pre(v):
    h = U.T @ v
    return (lam[-1] + shift) * (U @ (h / (lam + shift))) + v - U @ h


x = np.zeros(n); r = rhs_h.copy(); z = pre(r); p = z.copy(); rz = r @ z
ref = []
for k in range(1, 200):
    Ap = A.T @ (A @ p) + shift * p
    a = rz / (p @ Ap); x += a * p
    r = rhs_h - (A.T @ (A @ x) + shift * x) if k % 50 == 0 else r - a * Ap
    ref.append(np.linalg.norm(r) / bn)
    if ref[-1] <= 1e-12:
        break
    z = pre(r); rzn = r @ z; p = z + rzn / rz * p; rz = rzn
print("numpy iters", len(ref))

for persist in (False, True):
    os.environ["NYS_CG_PERSIST"] = "1" if persist else "0"
    work = CgWork(kx, n)
    rhs = torch.from_numpy(rhs_h).cuda()
    xd = torch.zeros(n, dtype=torch.float64, device="cuda")
    pb = kx.cg_problem(0, Ad, None, shift, S.U_dev, S.lam_dev, shift, rhs, xd, work, 1e-12, 10 * n)
    kx.hvp(Ad, None, xd, shift, work.Ap)
    kx.cg_start(rhs, work.Ap, work.r, work.sc)
    res = []
    if persist:
        kx.cg_iterate(pb, 1, 1)
        h = work.read()
        print("persist done", h[_lib.CG_DONE], "iters", h[_lib.CG_ITERS], "resrel", h[_lib.CG_RESREL])
        continue
    for k in range(1, 120):
        kx.cg_iterate(pb, k, 1)
        h = work.read()
        res.append(np.sqrt(h[_lib.CG_RES2]) / bn)
        if h[_lib.CG_DONE]:
            break
    print("batched done", h[_lib.CG_DONE], "iters", len(res))
    for k in (45, 48, 49, 50, 51, 52, 55, 60, 70):
        if k <= len(res) and k <= len(ref):
            print(f"  k={k} gpu {res[k-1]:.6e} numpy {ref[k-1]:.6e}")
    # true residual at the end
    xh = xd.cpu().numpy()
    print("  true rel residual gpu x", np.linalg.norm(rhs_h - A.T @ (A @ xh) - shift * xh) / bn)
