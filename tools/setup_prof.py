"""Host-side cost of the setup of one solve, by function (cProfile, cumulative;
20 solves of the same problem; development tool).

    python tools/setup_prof.py [config]
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_08333_b200 as nys  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
d, opts = bench.build_problem(cfg)
A = torch.from_numpy(d.P if d.kind == "boxqp" else d.A).cuda()
prob = bench.make_gpu_problem(d, A)
for _ in range(3):
    nys.solve(prob, opts)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    r = nys.solve(prob, opts)
torch.cuda.synchronize()
print(f"wall per solve {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms, setup_s {r.timings.setup_s * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    nys.solve(prob, opts)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(60)
st.sort_stats("tottime").print_stats(30)
