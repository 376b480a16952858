"""GPU timeline of one solve via torch.profiler (CUPTI): kernel time by name,
GPU busy fraction, idle gaps (development tool).

    python tools/trace_solve.py --config 2 [--json out.json]
"""

import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--json", default=None)
    ap.add_argument("--seq", type=int, default=-1, help="print the kernel sequence after the Nth cg_persist launch")
    args = ap.parse_args()
    import bench
    import paper_2310_08333_b200 as nys

    if args.config == 4:
        d, opts, A = bench.build_cfg4_device(1, 0, False)
    elif args.config == 5:
        d, opts, A = bench.build_cfg5(1, 0)
    else:
        d, opts = bench.build_problem(args.config)
        A = torch.from_numpy(d.P if d.kind == "boxqp" else d.A).cuda()
    prob = bench.make_gpu_problem(d, A)
    nys.solve(prob, opts)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        res = nys.solve(prob, opts)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.device_time_total > 0]
    # kernel intervals (us)
    ivs = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
    by = collections.defaultdict(lambda: [0, 0.0])
    for s, t, nm in ivs:
        by[nm][0] += 1
        by[nm][1] += t - s
    busy = 0.0
    cur_s, cur_t, cur_nm = None, None, None
    gaps = []
    ctx = collections.defaultdict(lambda: [0, 0.0])  # (before -> after) gap context
    for s, t, nm in ivs:
        if cur_t is None or s > cur_t:
            if cur_t is not None:
                busy += cur_t - cur_s
                gaps.append(s - cur_t)
                if s - cur_t > 5:
                    key = cur_nm.split("(")[0][-40:] + " -> " + nm.split("(")[0][-40:]
                    ctx[key][0] += 1
                    ctx[key][1] += s - cur_t
            cur_s, cur_t = s, t
        else:
            cur_t = max(cur_t, t)
        cur_nm = nm
    if cur_t is not None:
        busy += cur_t - cur_s
    span = ivs[-1][1] - ivs[0][0] if ivs else 0.0
    top = sorted(by.items(), key=lambda kv: -kv[1][1])[:25]
    out = {
        "iterations": res.iterations, "span_ms": span / 1e3, "gpu_busy_ms": busy / 1e3,
        "gpu_busy_frac": busy / span if span else 0.0, "kernels": len(ivs),
        "idle_gaps_ms_total": sum(gaps) / 1e3, "gaps_over_20us": sum(1 for g in gaps if g > 20),
        "top": [{"name": nm[:90], "count": c, "total_ms": tot / 1e3, "avg_us": tot / c} for nm, (c, tot) in top],
        "gap_contexts": [{"between": k, "count": c, "total_ms": tot / 1e3}
                         for k, (c, tot) in sorted(ctx.items(), key=lambda kv: -kv[1][1])[:20]],
    }
    if args.seq >= 0:
        starts = [i for i, (_, _, nm) in enumerate(ivs) if "cg_persist" in nm]
        if len(starts) > args.seq + 1:
            a, b = starts[args.seq], starts[args.seq + 1]
            t0 = ivs[a][0]
            prev = t0
            for s, t, nm in ivs[a:b + 1]:
                print(f"seq {s - t0:9.1f} +{s - prev:6.1f} {t - s:8.1f} us  {nm.split('(')[0][-60:]}")
                prev = t
    print(json.dumps(out, indent=1))
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
