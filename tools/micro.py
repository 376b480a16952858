"""Micro-benchmarks of individual C-ABI calls (development tool).

    python tools/micro.py
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def timeit(fn, reps=10, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def main():
    from paper_2310_08333_b200.kernels import get_kernels

    kx = get_kernels()
    out = {}
    g = np.random.default_rng(0)
    for s in (133, 258, 383):
        M = g.standard_normal((s, s))
        M = M @ M.T + s * np.eye(s)
        Md = torch.from_numpy(M).cuda()
        V = kx.empty(s, s)
        w = kx.empty(s)
        out[f"syevj_{s}_ms"] = timeit(lambda: kx.syevj(Md.clone(), V, w), reps=3, warm=1)
        n = {133: 10000, 258: 100000, 383: 200000}[s]
        Om = kx.empty(n, s)
        kx.gaussian(1, Om)
        Q = kx.empty(n, s)
        out[f"ortho_{n}x{s}_ms"] = timeit(lambda: kx.orthonormalize(Om, Q), reps=3, warm=1)
        Y = kx.empty(n, s)
        Y.copy_(Q * 2.0)
        U = kx.empty(n, s)
        lam = kx.empty(s)
        out[f"core_{n}x{s}_ms"] = timeit(lambda: kx.nystrom_core(Q, Y.clone(), U, lam, s - 30), reps=3, warm=1)
        out[f"gauss_{n}x{s}_ms"] = timeit(lambda: kx.gaussian(3, Om), reps=3, warm=1)
    # GEMM rates
    for (M_, N_, K_) in ((5000, 133, 10000), (10000, 133, 5000), (20000, 258, 100000)):
        A = kx.empty(M_, K_)
        A.normal_()
        B = kx.empty(K_, N_)
        B.normal_()
        C = kx.empty(M_, N_)
        ms = timeit(lambda: kx.gemm(0, 0, M_, N_, K_, 1.0, A, K_, B, N_, 0.0, C, N_), reps=3, warm=1)
        out[f"gemm_nn_{M_}x{N_}x{K_}_TFLOPs"] = 2 * M_ * N_ * K_ / ms / 1e9
        At = kx.empty(K_, M_)
        At.normal_()
        ms = timeit(lambda: kx.gemm(1, 0, M_, N_, K_, 1.0, At, M_, B, N_, 0.0, C, N_), reps=3, warm=1)
        out[f"gemm_tn_{M_}x{N_}x{K_}_TFLOPs"] = 2 * M_ * N_ * K_ / ms / 1e9
        del A, At, B, C
    # cuBLAS DGEMM yardstick (comparison only, not on the product path)
    A = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    ms = timeit(lambda: A @ A, reps=3, warm=1)
    out["cublas_dgemm_8192_TFLOPs"] = 2 * 8192**3 / ms / 1e9
    C = kx.empty(8192, 8192)
    ms = timeit(lambda: kx.gemm(0, 0, 8192, 8192, 8192, 1.0, A, 8192, A, 8192, 0.0, C, 8192), reps=3, warm=1)
    out["nys_dgemm_8192_TFLOPs"] = 2 * 8192**3 / ms / 1e9
    # GEMV rates (read bandwidth)
    for rows, n in ((5000, 10000), (20000, 100000)):
        A = kx.empty(rows, n)
        A.normal_()
        for k in (1, 2, 3):
            X = kx.empty(k, n)
            X.normal_()
            Y = kx.empty(k, rows)
            ms = timeit(lambda: kx.gemv(A, X, Y), reps=10)
            out[f"gemv_k{k}_{rows}x{n}_GBs"] = 8 * rows * n / ms / 1e6
            T = kx.empty(k, rows)
            T.normal_()
            Z = kx.empty(k, n)
            ms = timeit(lambda: kx.gemvT(A, T, Z), reps=10)
            out[f"gemvT_k{k}_{rows}x{n}_GBs"] = 8 * rows * n / ms / 1e6
        v = kx.empty(n)
        v.normal_()
        y = kx.empty(n)
        ms = timeit(lambda: kx.hvp(A, None, v, 1.0, y, None, True), reps=10)
        out[f"hvp_{rows}x{n}_algGBs"] = 8 * rows * n / ms / 1e6
        del A
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
