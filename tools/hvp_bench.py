"""CUDA-event timing of back-to-back HVP launches (K3) on a config-sized A.

    python tools/hvp_bench.py [rows n reps [nod]]     (nod: unit row weights, d = NULL)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2310_08333_b200.kernels import get_kernels  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
nod = len(sys.argv) > 4 and sys.argv[4] == "nod"
kx = get_kernels()
A = kx.empty(rows, n)
A.normal_()
v = kx.empty(n)
v.normal_()
d = None if nod else kx.empty(rows).uniform_()
y = kx.empty(n)
pAp = kx.zeros(1)
for _ in range(5):
    kx.hvp(A, d, v, 1.0, y, pAp, True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(kx.stream)
for _ in range(reps):
    kx.hvp(A, d, v, 1.0, y, pAp, True)
e1.record(kx.stream)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
gb = (8 * rows * n + 8 * (2 * n + rows)) / (us * 1e-6) / 1e9
print(f"hvp {rows}x{n}{' d=NULL' if nod else ''}: {us:.1f} us/launch, {gb:.0f} GB/s algorithmic")
