"""CUDA-event timing of the sketch's two large GEMMs (A Q and A^T Z) per CTA
tile shape of nys_gemm_f64 (nys_gemm_tile forces a shape; -1 = the planner).
    python tools/gemm_bench.py [rows n s]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2310_08333_b200.kernels import get_kernels  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
s = int(sys.argv[3]) if len(sys.argv) > 3 else 258
kx = get_kernels()
A = kx.empty(rows, n).normal_()
Q = kx.empty(n, s).normal_()
Y = kx.empty(rows, s)
Z = kx.empty(n, s)
nshapes = kx.L.nys_gemm_tile(-1)
for name, call, flop in (
        ("A Q", lambda: kx.gemm(0, 0, rows, s, n, 1.0, A, n, Q, s, 0.0, Y, s), 2.0 * rows * n * s),
        ("A^T Z", lambda: kx.gemm(1, 0, n, s, rows, 1.0, A, n, Y, s, 0.0, Z, s), 2.0 * rows * n * s)):
    for shape in list(range(nshapes)) + [-1]:
        kx.L.nys_gemm_tile(shape)
        call()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        reps = 3
        e0.record(kx.stream)
        for _ in range(reps):
            call()
        e1.record(kx.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"{name} {rows}x{n} s={s} shape {shape:2d}: {ms:9.3f} ms  {flop / ms / 1e9:6.2f} TF/s", flush=True)
kx.L.nys_gemm_tile(-1)

if os.environ.get("GEMM_CLOCKS"):
    # SM clock / power while the A Q product runs back to back (is the DMMA stream power-limited?)
    import subprocess
    import threading
    import time

    samples, stop = [], threading.Event()

    def poll():
        while not stop.is_set():
            out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                                  "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True).stdout
            samples.append(out.strip())
            time.sleep(0.2)

    th = threading.Thread(target=poll)
    th.start()
    t0 = time.time()
    while time.time() - t0 < 4.0:
        for _ in range(5):
            kx.gemm(0, 0, rows, s, n, 1.0, A, n, Q, s, 0.0, Y, s)
        torch.cuda.synchronize()
    stop.set()
    th.join()
    print("clocks.sm, power.draw, throttle mask while A Q runs:", samples[3:-1:3])
