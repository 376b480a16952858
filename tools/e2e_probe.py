"""Where the config-4 end-to-end solve's time goes: upload alone, solve from
HBM, solve from pinned host memory with and without the overlapped upload."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_08333_b200 as nys  # noqa: E402

d, opts, A_dev = bench.build_cfg4_device(1, 0, True)
host = d.A_host
print("host pinned:", host.is_pinned(), tuple(host.shape))


def timed(f, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
    return min(out), r


dst = torch.empty_like(A_dev)
print("upload alone: %.3f s" % timed(lambda: dst.copy_(host, non_blocking=True))[0])
del dst
t, r = timed(lambda: nys.solve(bench.make_gpu_problem(d, A_dev), opts))
print("solve from HBM: %.3f s (setup %.3f, iters %d)" % (t, r.timings.setup_s, r.iterations))
for ov in ("1", "0"):
    os.environ["NYS_UPLOAD_OVERLAP"] = ov
    t, r = timed(lambda: nys.solve(bench.make_gpu_problem(d, host), opts))
    print("solve from pinned host, overlap=%s: %.3f s (setup %.3f, precond %.3f)" % (ov, t, r.timings.setup_s,
                                                                                   r.timings.precond_s))
from paper_2310_08333_b200 import operators as _ops  # noqa: E402

print("upload streams used:", list(_ops._UPLOAD_STREAMS))
os.environ["NYS_UPLOAD_OVERLAP"] = "1"
p = bench.make_gpu_problem(d, host)
op = p.A
t = op.device_rows(None, None, overlap=True)
ch = op.take_pending(t)
print("chunks:", None if ch is None else [(a, b) for a, b, _ in ch])
torch.cuda.synchronize()
# GPU timeline of the overlapped setup: events at each chunk and around the sketch GEMMs
import paper_2310_08333_b200.admm as admm  # noqa: E402
from paper_2310_08333_b200.kernels import get_kernels  # noqa: E402

kx = get_kernels()
t0 = time.perf_counter()
r = nys.solve(bench.make_gpu_problem(d, host), nys.SolverOptions(**{**opts.__dict__, "max_iter": 1}))
torch.cuda.synchronize()
print("one-iteration solve from pinned host: %.3f s (setup %.3f, precond %.3f)" % (time.perf_counter() - t0,
                                                                                   r.timings.setup_s,
                                                                                   r.timings.precond_s))
