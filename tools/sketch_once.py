"""One Nystrom sketch of the config-2 Hessian (setup of a 1-iteration solve),
after a warm-up solve; for ncu launch lists of the sketch kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_08333_b200 as nys  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
d, opts = bench.build_problem(cfg)
opts.max_iter = 1
A = torch.from_numpy(d.P if d.kind == "boxqp" else d.A).cuda()
prob = bench.make_gpu_problem(d, A)
nys.solve(prob, opts)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("sketch")
nys.solve(prob, opts)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok")
