"""CUDA-event timing of the ADMM tail's data passes on a wide-row A: the
one-pass cluster tail (nys_ml_tail_f64) against gemv_n(k=2) + row-wise epilogue
+ gemv_t(k=3).   python tools/tail_bench.py [rows n reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2310_08333_b200.kernels import get_kernels  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
LOSS = sys.argv[4] if len(sys.argv) > 4 else "logistic"
ZDENS = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0  # density of z (the prox output is sparse)
kx = get_kernels()
A = kx.empty(rows, n).normal_()
XZ = kx.empty(2, n).normal_()
if ZDENS < 1.0:
    XZ[1].mul_((torch.rand(n, device=XZ.device) < ZDENS).double())
b = kx.empty(rows).normal_()
T = kx.empty(3, rows)
w = kx.empty(rows)
AT = kx.empty(3, n)
rs = kx.zeros(8)
AXZ = kx.empty(2, rows)


gb = kx.empty(n).normal_()


def fused():
    kx.ml_tail(LOSS, A, XZ[0], XZ[1], b, T, w, AT, rs)


def fused_gb():
    kx.ml_tail(LOSS, A, XZ[0], XZ[1], b, T, w, AT, rs, gb=gb)


def split():
    kx.gemv(A, XZ, AXZ)
    kx.ml_rowwise(LOSS, AXZ[0], AXZ[1], b, T[0], w, T[1], T[2], rs)
    kx.gemvT(A, T, AT)


for name, f in (("cluster tail", fused), ("cluster tail with g_b", fused_gb), ("gemv_n + rowwise + gemv_t", split)):
    try:
        for _ in range(3):
            f()
    except Exception as e:  # no plan for this variant at this width
        print(f"{name} {rows}x{n}: {type(e).__name__}")
        continue
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(kx.stream)
    for _ in range(reps):
        f()
    e1.record(kx.stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print(f"{name} {rows}x{n} z density {ZDENS}: {us:.1f} us, {8 * rows * n / (us * 1e-6) / 1e9:.0f} GB/s of A per pass")
