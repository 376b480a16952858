"""Benchmark of the B200 inexact-ADMM hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Workload (N=1): BASELINE.json configs[1] = config 2, dense elastic-net
logistic regression, A 5000 x 10000 FP64 (400 MB, larger than the 126 MB L2,
so no L2 flush is needed between steps), Nystrom rank 100, tolerances 1e-4.
A step is one complete ``solve`` to tolerance (358 ADMM iterations, 18
Nystrom sketches).  ``value`` = ADMM iterations/s over the timed steps with A
already resident in HBM; ``e2e`` = the same metric through the public API with
A in pinned host memory, uploaded inside every step, results read back.
N > 1 (torchrun): A is row-sharded over the ranks with NCCL all-reduces of the
A^T partials (strong scaling: total work fixed).

``--impl reference`` times the reference algorithm on the host CPU (the
pinned NumPy oracle, oracle/port.py -- the Python reference cannot travel to
the GPU box) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CPU_SAMPLE_ITERS = 60  # 3 sketches per 60 iterations, the full solve's sketch density


def _env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 8:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def build_problem(cfg: int, A_op=None):
    import paper_2310_08333_b200 as nys
    from paper_2310_08333_b200 import datagen

    d = datagen.make_config(cfg)
    opts = nys.SolverOptions(sketch_rank=d.rank, rng_seed=d.seed, eps_abs=1e-4, eps_rel=1e-4, eps_dual_gap=1e-4)
    return d, opts


class Cfg5Data:
    """Config 5 (BASELINE.json configs[4]): generated in HBM per rank
    (paper_2310_08333_b200/devgen.py), never on the host."""

    cfg, kind, loss, rank, seed = 5, "lasso", "square", 300, 4

    def __init__(self, N, n, lam, b):
        self.N, self.n, self.lambda1, self.lambda2, self.b = N, n, lam, 0.0, b
        self.A = None


def build_cfg5(world, rank):
    """This rank's row blocks of config 5 generated on its GPU; lambda =
    0.1 ||A^T b||_inf with one n-vector all-reduce (SURVEY.md 8(e) setup)."""
    import torch

    import paper_2310_08333_b200 as nys
    from paper_2310_08333_b200 import datagen, devgen
    from paper_2310_08333_b200.kernels import get_kernels

    kx = get_kernels()
    nb = datagen.CFG5_BLOCKS
    if nb % world:
        raise SystemExit(f"config 5 shards whole 12500-row blocks: world size must divide {nb}")
    blocks = range(rank * nb // world, (rank + 1) * nb // world)
    A_loc, b_loc, _ = devgen.cfg5_device(kx, blocks)
    N, n = devgen.CFG5_ROWS, devgen.CFG5_N
    atb = kx.empty(1, n)
    kx.gemvT(A_loc, b_loc.view(1, -1).contiguous(), atb)
    b_parts = [torch.empty_like(b_loc) for _ in range(world)]
    if world > 1:
        torch.distributed.all_reduce(atb)
        torch.distributed.all_gather(b_parts, b_loc)
    else:
        b_parts = [b_loc]
    lam = 0.1 * float(atb.abs().max())
    b = torch.cat(b_parts).cpu().numpy()
    d = Cfg5Data(N, n, lam, b)
    row0 = blocks[0] * devgen.CFG5_BLOCK_ROWS
    op = nys.DenseOperator(A_loc) if world == 1 else nys.DenseOperator.from_local_rows(A_loc, N, row0)
    prob = nys.MLProblem(nys.builtin_loss("square"), op, b, lam, 0.0)
    opts = nys.SolverOptions(sketch_rank=d.rank, rng_seed=d.seed, eps_abs=1e-4, eps_rel=1e-4, eps_dual_gap=1e-4)
    return d, opts, A_loc, prob


def make_gpu_problem(d, A):
    import paper_2310_08333_b200 as nys

    if d.kind == "boxqp":
        n = d.P.shape[0]
        return nys.QPProblem(nys.DenseOperator(A), d.q, nys.IdentityOperator(n), nys.Box(d.lo, d.hi))
    return nys.MLProblem(nys.builtin_loss(d.loss), nys.DenseOperator(A), d.b, d.lambda1, d.lambda2)


def cpu_reference_rate(d, opts_gpu, max_iter, reps=1):
    """The reference algorithm on the host (oracle port) over a bounded sample."""
    from oracle import port

    if d.kind == "boxqp":
        prob = port.QPSpec(d.P, d.q, d.lo, d.hi)
    else:
        prob = port.MLSpec(d.loss, d.A, d.b, d.lambda1, d.lambda2)
    o = port.Options(sketch_rank=opts_gpu.sketch_rank, rng_seed=opts_gpu.rng_seed, eps_abs=1e-4, eps_rel=1e-4,
                     eps_dual_gap=1e-4, max_iter=max_iter)
    times, iters = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = port.solve(prob, o)
        times.append(time.perf_counter() - t0)
        iters.append(r.iterations)
    return times, iters


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        return max((i.get("num_threads", 1) for i in info if i.get("user_api") == "blas"), default=os.cpu_count())
    except Exception:
        return os.cpu_count()


def run_reference(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return
    d, opts = build_problem(args.config)
    sample = min(CPU_SAMPLE_ITERS, 10**9)
    cpu_reference_rate(d, opts, sample, reps=max(0, min(args.warmup, 1)))  # warm caches / BLAS threads
    times, iters = cpu_reference_rate(d, opts, sample, reps=args.steps)
    tot_t, tot_i = sum(times), sum(iters)
    value = tot_i / tot_t
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": "ADMM iters/s", "value": value, "unit": "iters/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(args, d, world),
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": cores, "kind": "port",
                         "sample": f"first {sample} ADMM iterations of config {args.config} per step "
                                   f"(3 Nystrom sketches, same density as the full solve), NumPy/OpenBLAS"},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(args, d, world):
    if d.A is None:  # config 5: device-generated
        N, n = d.N, d.n
    else:
        n = d.P.shape[0] if d.kind == "boxqp" else d.A.shape[1]
        N = d.A.shape[0]
    return {"workload": f"config {args.config}: {d.kind} {N}x{n} FP64, rank {d.rank}, tol 1e-4, solve to tolerance",
            "config_index": args.config, "rows": N, "features": n, "sketch_rank": d.rank,
            "parallelism": f"row-shard x{world}" if world > 1 else "single GPU",
            "l2_policy": "A (%.0f MB) larger than the 126 MB L2; no flush" % (8 * N * n / 1e6)}


def run_ours(args):
    import torch

    rank, world, local = _env_rank()
    if world > 1:
        local = local % max(1, torch.cuda.device_count())  # (ranks sharing a GPU: gloo test mode)
        torch.cuda.set_device(local)
        # NCCL over NVLink; NYS_DIST_BACKEND=gloo lets several ranks share one GPU
        # to exercise this multi-rank code path (host-staged collectives, not a measurement)
        torch.distributed.init_process_group(os.environ.get("NYS_DIST_BACKEND", "nccl"))
    else:
        torch.cuda.set_device(0)
    import paper_2310_08333_b200 as nys
    from paper_2310_08333_b200.kernels import get_kernels

    kx = get_kernels()
    if args.config == 5:
        # 160 GB: generated in HBM per rank (each rank holds only its row blocks)
        d, opts, A_dev, prob = build_cfg5(world, rank)
        host_A = None
        args.no_e2e = args.no_cpu = True
    else:
        d, opts = build_problem(args.config)
        host_A = d.P if d.kind == "boxqp" else d.A
        # A resident in HBM for the kernel-side metric (each rank: its row shard inside solve)
        A_dev = torch.from_numpy(host_A).cuda()
        prob = make_gpu_problem(d, A_dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def maxred(x):
        if world > 1:
            t = torch.tensor([x], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            return float(t)
        return x

    for _ in range(args.warmup):
        res = nys.solve(prob, opts)
    # timed region: whole solves, no instrumentation
    launches0 = kx.kernel_launches()
    iters = 0
    barrier()
    st = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(st)
        for _ in range(args.steps):
            res = nys.solve(prob, opts)
            iters += res.iterations
        e1.record(st)
        barrier()
    el_ms = maxred(e0.elapsed_time(e1))
    launches = kx.kernel_launches() - launches0
    value = iters / (el_ms / 1e3)
    tts = el_ms / 1e3 / args.steps

    # one extra, instrumented solve: every x-update PCG launch is bracketed by
    # CUDA events on the solve's stream.  With the persistent solver
    # (csrc/cg_persist.cu) one launch is a whole CG solve and counts its
    # operator applications; otherwise each HVP launch is bracketed alone
    # (predicated no-op launches excluded).  Its duration gives the share.
    kx.timing_enable(True)
    barrier()
    i0 = torch.cuda.Event(enable_timing=True)
    i1 = torch.cuda.Event(enable_timing=True)
    i0.record(st)
    nys.solve(prob, opts)
    i1.record(st)
    barrier()
    inst_ms = i0.elapsed_time(i1)
    k_total_ms, k_count = kx.timing_read()
    kx.timing_enable(False)

    # roofline of the dominant kernel: algorithmic bytes per operator application
    # (8 N n + 8 (2n + N)) x applications / measured time
    n = A_dev.shape[1]
    if args.config == 5:
        rows_loc = A_dev.shape[0]
    else:
        rows_loc = d.A.shape[0] // world if d.kind != "boxqp" else n
    alg_bytes = 8 * rows_loc * n + 8 * (2 * n + rows_loc)
    peak, peak_kind = _peaks()
    persistent = os.environ.get("NYS_CG_PERSIST", "1") != "0" and n <= 13312 and (d.kind == "boxqp" or world == 1)
    kname = "cg_persist_kernel" if persistent else "hvp"
    roof = None
    traffic_db = {}
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic_db = json.load(open(tf))
        except Exception:
            traffic_db = {}
    if k_count:
        avg_ms = k_total_ms / k_count
        achieved = alg_bytes / (avg_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic_db.get(f"cfg{args.config}_{kname}") if world == 1 else None,
                "alg_bytes_per_unit": alg_bytes, "unit_of_work": "one Hessian application (HVP) of the PCG, "
                "incl. the CG vector phases when the persistent solver runs", "ms_per_unit": avg_ms,
                "units_timed": k_count, "share_of_step": k_total_ms / inst_ms,
                "timing": "CUDA events around every PCG launch of one extra instrumented solve (not the timed steps)"}
    # the HVP kernel alone (K3, csrc/hvp.cu), back to back on the same A and row weights
    hvp_alone = None
    if d.kind != "boxqp" and world == 1 and args.config != 5:
        v = torch.randn(n, dtype=torch.float64, device=A_dev.device)
        y = torch.empty_like(v)
        dw = torch.rand(A_dev.shape[0], dtype=torch.float64, device=A_dev.device)
        pap = torch.zeros(1, dtype=torch.float64, device=A_dev.device)
        for _ in range(3):
            kx.hvp(A_dev, dw, v, 1.0, y, pap, True)
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        reps = 20
        h0.record(st)
        for _ in range(reps):
            kx.hvp(A_dev, dw, v, 1.0, y, pap, True)
        h1.record(st)
        torch.cuda.synchronize()
        hms = h0.elapsed_time(h1) / reps
        ha = alg_bytes / (hms / 1e3) / 1e9
        hvp_alone = {"kernel": "hvp_row_kernel", "achieved": ha, "peak": peak, "unit": "GB/s", "frac": ha / peak,
                     "ms_per_launch": hms, "traffic": traffic_db.get(f"cfg{args.config}_hvp"),
                     "timing": f"CUDA events around {reps} back-to-back launches"}

    # e2e: public API with host buffers (pinned), upload + readback inside each step
    e2e = None
    if not args.no_e2e:
        pinned = torch.from_numpy(host_A).pin_memory()
        host_view = pinned.numpy()
        kx.h2d = kx.d2h = 0
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        e_iters = 0
        t0.record(st)
        for _ in range(max(1, args.steps)):
            p2 = make_gpu_problem(d, host_view)
            r2 = nys.solve(p2, opts)
            e_iters += r2.iterations
        t1.record(st)
        barrier()
        e_ms = maxred(t0.elapsed_time(t1))
        steps_e = max(1, args.steps)
        a_bytes = host_A.nbytes // world
        b_bytes = 0 if d.kind == "boxqp" else d.b.nbytes // world
        e2e = {"value": e_iters / (e_ms / 1e3), "unit": "iters/s",
               "h2d_bytes_per_step": int(a_bytes + b_bytes + kx.h2d / steps_e),
               "d2h_bytes_per_step": int(kx.d2h / steps_e), "time_to_tolerance_s": e_ms / 1e3 / steps_e}

    if args.config == 5:
        e2e = {"unavailable": "config 5 is generated in HBM per rank (160 GB); there is no host copy to upload"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        times, its = cpu_reference_rate(d, opts, CPU_SAMPLE_ITERS, reps=1)
        cpu = {"value": its[0] / times[0], "unit": "iters/s", "cores": blas_threads(), "kind": "port",
               "sample": f"first {CPU_SAMPLE_ITERS} ADMM iterations of config {args.config} (oracle port, "
                         f"NumPy/OpenBLAS, {times[0]:.1f} s)"}

    if rank == 0:
        line = {
            "metric": "ADMM iters/s", "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_block(args, d, world), time_to_tolerance_s=tts, iterations=res.iterations,
                           status=res.status.value, objective=res.objective, sketches=res.device_stats.get("sketches")),
            "roofline": roof, "hvp_alone": hvp_alone, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
