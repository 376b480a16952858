"""Phase / kernel-family breakdown of one solve (development tool).

    python tools/profile_solve.py --config 2 [--families hvp,gemv,gemvT]

Prints SolveResult.timings, the CG/ADMM counts and, per kernel family, the
CUDA-event time summed over the solve (each family is timed in its own run so
the events of one do not perturb another).
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--families", default="hvp,gemv,gemvT")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    import bench
    import paper_2310_08333_b200 as nys
    from paper_2310_08333_b200.kernels import get_kernels

    d, opts = bench.build_problem(args.config)
    A = torch.from_numpy(d.P if d.kind == "boxqp" else d.A).cuda()
    prob = bench.make_gpu_problem(d, A)
    kx = get_kernels()
    res = nys.solve(prob, opts)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.reps):
        res = nys.solve(prob, opts)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / args.reps
    out = {"wall_s": wall, "iterations": res.iterations, "cg_total": int(sum(h.cg_iters for h in res.history)),
           "timings": res.timings.__dict__, "launch_calls": res.device_stats}
    from paper_2310_08333_b200 import sketch as sk

    sk._TRACE = []
    nys.solve(prob, opts)
    tr = sk._TRACE
    sk._TRACE = None
    out["sketch_stages_ms_avg"] = {k: float(np.mean([x[k] for x in tr])) for k in tr[0]}
    for fam in args.families.split(","):
        kx.timed_name = fam
        kx.events = []
        nys.solve(prob, opts)
        ts = kx.event_times_ms()
        kx.timed_name = None
        out[f"fam_{fam}"] = {"count": len(ts), "total_ms": sum(ts), "avg_us": 1e3 * sum(ts) / max(1, len(ts))}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
