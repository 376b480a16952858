"""A few HVP launches on a config-sized A (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2310_08333_b200.kernels import get_kernels  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
kx = get_kernels()
A = kx.empty(rows, n)
A.normal_()
v = kx.empty(n)
v.normal_()
d = kx.empty(rows)
d.uniform_()
y = kx.empty(n)
pAp = kx.zeros(1)
for _ in range(reps):
    kx.hvp(A, d, v, 1.0, y, pAp, True)
torch.cuda.synchronize()
print("ok", float(pAp))
