"""cProfile of the host side of one solve (development tool)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_08333_b200 as nys  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
d, opts = bench.build_problem(cfg)
A = torch.from_numpy(d.P if d.kind == "boxqp" else d.A).cuda()
prob = bench.make_gpu_problem(d, A)
nys.solve(prob, opts)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
nys.solve(prob, opts)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(45)
