"""Where the host spends one solve: time inside _read (spin-waiting for the
GPU's readback block), inside _issue (building + launching an iteration) and
the rest (development tool).  python tools/spin_prof.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_08333_b200 as nys  # noqa: E402
from paper_2310_08333_b200 import admm  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
d, opts = bench.build_problem(cfg)
A = torch.from_numpy(d.P if d.kind == "boxqp" else d.A).cuda()
prob = bench.make_gpu_problem(d, A)
acc = {"_read": 0.0, "_issue": 0.0, "sketch": 0.0, "_make_tail": 0.0, "__init__": 0.0, "evaluate": 0.0,
       "read_stats": 0.0}
for name in list(acc):
    f = getattr(admm._Engine, name)

    def wrap(*a, _f=f, _n=name, **k):
        t = time.perf_counter()
        try:
            return _f(*a, **k)
        finally:
            acc[_n] += time.perf_counter() - t
    setattr(admm._Engine, name, wrap)
for _ in range(3):
    nys.solve(prob, opts)
torch.cuda.synchronize()
for k in acc:
    acc[k] = 0.0
R = 20
t0 = time.perf_counter()
for _ in range(R):
    r = nys.solve(prob, opts)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / R
print(f"config {cfg}: {r.iterations} iterations, wall {wall * 1e3:.3f} ms/solve, setup {r.timings.setup_s * 1e3:.3f} ms")
for k, v in acc.items():
    print(f"  {k:12s} {v / R * 1e3:8.3f} ms/solve  {v / R / r.iterations * 1e6:8.1f} us/iter")
