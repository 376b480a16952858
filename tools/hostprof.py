"""Host-side time split of one solve: wall time, time blocked in stream syncs,
time inside the C-ABI launch calls (development tool).

    python tools/hostprof.py [config]
"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_08333_b200 as nys  # noqa: E402
from paper_2310_08333_b200.kernels import get_kernels  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
d, opts = bench.build_problem(cfg)
A = torch.from_numpy(d.P if d.kind == "boxqp" else d.A).cuda()
prob = bench.make_gpu_problem(d, A)
kx = get_kernels()
nys.solve(prob, opts)
torch.cuda.synchronize()

acc = collections.defaultdict(float)
cnt = collections.Counter()


def wrap(name):
    f = getattr(kx, name)

    def g(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        acc[name] += time.perf_counter() - t0
        cnt[name] += 1
        return r

    setattr(kx, name, g)


for nm in ("sync", "cg_iterate", "admm_tail", "admm_rhs", "cg_problem", "gemm", "gaussian", "nystrom_core",
           "orthonormalize", "row_scale", "gemv", "gemvT"):
    if hasattr(kx, nm):
        wrap(nm)
orig_item = torch.Tensor.cpu
t0 = time.perf_counter()
r = nys.solve(prob, opts)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"config {cfg}: iterations {r.iterations} wall {wall * 1e3:.1f} ms "
      f"({wall * 1e6 / r.iterations:.0f} us/iter)")
tot = 0.0
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    tot += v if k != "sync" else 0
    print(f"  {k:16s} {cnt[k]:6d} calls {v * 1e3:8.2f} ms  {v * 1e6 / max(cnt[k], 1):7.1f} us/call")
print(f"  host outside syncs: {(wall - acc['sync']) * 1e3:.1f} ms ({(wall - acc['sync']) * 1e6 / r.iterations:.0f} us/iter); "
      f"inside launch wrappers {tot * 1e3:.1f} ms")
