"""A short config solve (max_iter iterations, after one warm-up), for ncu captures
of the per-iteration kernels.

    python tools/solve_short.py [config] [max_iter]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_08333_b200 as nys  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
d, opts = bench.build_problem(cfg)
opts.max_iter = iters
A = torch.from_numpy(d.P if d.kind == "boxqp" else d.A).cuda()
prob = bench.make_gpu_problem(d, A)
nys.solve(prob, opts)
torch.cuda.synchronize()
r = nys.solve(prob, opts)
torch.cuda.synchronize()
print("ok", r.iterations)
