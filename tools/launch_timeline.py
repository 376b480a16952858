"""Per-kernel launch-call vs GPU start/end times for one solve (torch.profiler
chrome trace, development tool): shows whether the GPU waits on the host.
    python tools/launch_timeline.py [config] > out.txt"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2310_08333_b200 as nys  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
d, opts = bench.build_problem(cfg)
A = torch.from_numpy(d.P if d.kind == "boxqp" else d.A).cuda()
prob = bench.make_gpu_problem(d, A)
for _ in range(3):
    nys.solve(prob, opts)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    nys.solve(prob, opts)
    torch.cuda.synchronize()
path = "/tmp/lt_trace.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
runtime = {e["args"]["correlation"]: e for e in ev if e.get("cat") == "cuda_runtime" and "correlation" in e.get("args", {})}
kern = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
kern.sort(key=lambda e: e["ts"])
t0 = kern[0]["ts"]
prev_end = None
for e in kern:
    c = e["args"].get("correlation")
    r = runtime.get(c)
    call = r["ts"] - t0 if r else float("nan")
    callend = r["ts"] + r["dur"] - t0 if r else float("nan")
    s = e["ts"] - t0
    gap = s - prev_end if prev_end is not None else 0.0
    print(f"{s:9.1f} +{gap:6.1f} dur {e['dur']:7.1f}  call {call:9.1f}-{callend:9.1f} ({r['name'][:28] if r else '?':28s}) {e['name'][:60]}")
    prev_end = s + e["dur"]
