"""FP64 yardstick for the sketch GEMMs' roofline: cuBLAS DGEMM (torch.matmul, float64)
on 8192^3 (best of 5, CUDA events) and on the config-2 sketch shapes.

    python tools/fp64_peak.py
"""
import torch

def tflops(m, n, k, reps=5):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return 2.0 * m * n * k / best / 1e12

print(f"cuBLAS DGEMM 8192^3: {tflops(8192, 8192, 8192):.1f} TF/s")
print(f"cuBLAS DGEMM 5000 x 133 x 10000 (A Q): {tflops(5000, 133, 10000):.1f} TF/s")
print(f"cuBLAS DGEMM 10000 x 133 x 5000 (A^T Z): {tflops(10000, 133, 5000):.1f} TF/s")
