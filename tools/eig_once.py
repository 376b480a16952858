"""One call of the small eigensolver (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2310_08333_b200.kernels import get_kernels  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 133
kx = get_kernels()
g = np.random.default_rng(0)
M = g.standard_normal((s, s))
M = M @ M.T + s * np.eye(s)
V = kx.empty(s, s)
w = kx.empty(s)
kx.syevj(torch.from_numpy(M).cuda(), V, w)
torch.cuda.synchronize()
err = np.abs(M @ V.cpu().numpy() - V.cpu().numpy() * w.cpu().numpy()).max()
print("residual", err)
