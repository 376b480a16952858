"""Small runs of the newer kernels for compute-sanitizer (memcheck / racecheck):
the wide-row cluster HVP, the strip HVP, the chained Gaussian stream, the
persistent PCG on an ML problem and on a box QP, the fused readback.

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cases  # noqa: E402
import paper_2310_08333_b200 as nys  # noqa: E402
from paper_2310_08333_b200 import devgen  # noqa: E402
from paper_2310_08333_b200.kernels import get_kernels  # noqa: E402

kx = get_kernels()
g = np.random.default_rng(0)
for rows, n in ((7, 20000), (40, 30002)):
    A = torch.from_numpy(g.standard_normal((rows, n))).cuda()
    d = torch.from_numpy(g.uniform(0.1, 1.0, rows)).cuda()
    v = torch.from_numpy(g.standard_normal(n)).cuda()
    y = kx.empty(n)
    pAp = kx.zeros(1)
    kx.hvp(A, d, v, 0.5, y, pAp, True)
    ref = A.T @ (d * (A @ v)) + 0.5 * v
    print("hvp", rows, n, float((y - ref).abs().max()))
out = kx.empty(3, 777)
devgen.cfg5_block_into(kx, 2, out, 3, 777, piece=500)
print("devgen ok")
for name in ("logistic_small", "boxqp_small"):
    spec = cases.SOLVE_CASES[name][0]()
    if "P" in spec:
        n = spec["P"].shape[0]
        prob = nys.QPProblem(nys.DenseOperator(spec["P"]), spec["q"], nys.IdentityOperator(n),
                             nys.Box(spec["lo"], spec["hi"]))
    else:
        prob = nys.MLProblem(nys.builtin_loss(spec["loss"]), spec["A"], spec["b"], spec["lambda1"], spec["lambda2"])
    res = nys.solve(prob, nys.SolverOptions(**cases.options_for(name)))
    print(name, res.status.value, res.iterations)
torch.cuda.synchronize()
print("done")
