"""orthonormalize() of an n x s Gaussian, a few times (for ncu captures of
the Gram GEMM and the fused Cholesky-inverse kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2310_08333_b200.kernels import get_kernels  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
s = int(sys.argv[2]) if len(sys.argv) > 2 else 133
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
kx = get_kernels()
Om = torch.from_numpy(np.random.default_rng(0).standard_normal((n, s))).cuda()
Q = kx.empty(n, s)
for _ in range(reps):
    kx.orthonormalize(Om, Q)
torch.cuda.synchronize()
Qn = Q.cpu().numpy()
print("orth err", np.abs(Qn.T @ Qn - np.eye(s)).max())
