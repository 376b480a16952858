"""Benchmark of the B200 inexact-ADMM hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Workload (default): BASELINE.json configs[3] = config 4, the configuration the
metric is quoted on "at 1/2/4/8 B200": dense LASSO, A 20000 x 100000 FP64
(16 GB, far larger than the 126 MB L2, so no L2 flush is needed between
steps), Nystrom rank 200, tolerances 1e-4, 57 ADMM iterations to tolerance.
A step is one complete ``solve`` to tolerance.  ``value`` = ADMM
iterations/s = iterations / (total - setup) over the timed
solves with A already resident in HBM; ``result.time_to_tolerance_s`` is the
whole solve.  ``e2e`` = the same solves through the public API with A in
pinned host memory, uploaded inside every step, iterates read back
(iterations over the whole wall time, setup and upload included).
N > 1: ``--gpus N`` self-launches N ranks through torch.distributed.run when
WORLD_SIZE is unset; A is row-sharded with NCCL all-reduces of the A^T
partials (strong scaling: total work fixed).  Config 5 (160 GB) shards whole
12500-row blocks, each rank generating its own in HBM.

``--impl reference`` times the reference on the host CPU: the unmodified
``nysopt`` package from ``baseline/_ref`` (kind "reference") when it is
installed there, else the pinned NumPy oracle port (kind "port"), with all
host threads, one setup then W untimed + K timed ADMM iterations of the same
config (iterations / (time - setup), the BASELINE.md §2 metric).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_CONFIG = 4
CPU_SAMPLE = (2, 6)  # our line's cpu_baseline: setup + 2 untimed + 6 timed iterations


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


def build_problem(cfg: int):
    """Host inputs of config ``cfg`` (datagen recipe) and its options."""
    import paper_2310_08333_b200 as nys
    from paper_2310_08333_b200 import datagen

    d = datagen.make_config(cfg)
    return d, options_for(d)


def options_for(d, max_iter=None, **kw):
    import paper_2310_08333_b200 as nys

    o = dict(sketch_rank=d.rank, rng_seed=d.seed, eps_abs=1e-4, eps_rel=1e-4, eps_dual_gap=1e-4)
    if max_iter is not None:
        o["max_iter"] = max_iter
    o.update(kw)
    return nys.SolverOptions(**o)


class DevData:
    """Inputs generated in HBM (configs 4 and 5): A is only on the device
    (and, where a host copy is needed, in pinned host memory)."""

    def __init__(self, cfg, kind, loss, N, n, rank, seed, lam, b):
        self.cfg, self.kind, self.loss, self.N, self.n, self.rank, self.seed = cfg, kind, loss, N, n, rank, seed
        self.lambda1, self.lambda2, self.b = lam, 0.0, b
        self.A = None
        self.P = None


def build_cfg4_device(world, rank, need_host):
    """Config 4 with A generated in HBM (devgen.lasso_device, bit-for-bit the
    host recipe's A); every rank generates the whole stream, computes the same
    b and lambda, and keeps its own rows.  With ``need_host`` (one rank: the
    e2e leg and the CPU baseline) A is copied to pinned host memory and b and
    lambda come from it with NumPy, exactly as datagen.make_config(4)."""
    import paper_2310_08333_b200 as nys
    from paper_2310_08333_b200 import datagen, devgen
    from paper_2310_08333_b200.dist import row_range
    from paper_2310_08333_b200.kernels import get_kernels

    kx = get_kernels()
    c = datagen.CONFIGS[4]
    N, n = c["N"], c["n"]
    r0, r1 = row_range(N, rank, world)
    A, b, lam, _, A_host = devgen.lasso_device(kx, N, n, c["seed"], c["nnz_frac"], rows=(r0, r1),
                                               host_b=need_host)
    d = DevData(4, "lasso", "square", N, n, c["rank"], c["seed"], lam, b)
    d.A_host = A_host  # pinned (need_host) or None
    d.row0 = r0
    return d, options_for(d), A


def build_cfg5(world, rank):
    """This rank's row blocks of config 5 generated on its GPU; lambda =
    0.1 ||A^T b||_inf with one n-vector all-reduce (SURVEY.md 8(e) setup)."""
    import torch

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
    c = datagen.CONFIGS[5]
    d = DevData(5, "lasso", "square", N, n, c["rank"], c["seed"], lam, b)
    d.A_host = None
    d.row0 = blocks[0] * devgen.CFG5_BLOCK_ROWS
    return d, options_for(d), A_loc


def make_gpu_problem(d, A, world=1):
    """The public-API problem; ``A`` is the device matrix (or, for DevData,
    this rank's rows: device or pinned host)."""
    import paper_2310_08333_b200 as nys

    if d.kind == "boxqp":
        n = d.P.shape[0]
        return nys.QPProblem(nys.DenseOperator(A), d.q, nys.IdentityOperator(n), nys.Box(d.lo, d.hi))
    if isinstance(d, DevData) and world > 1:
        op = nys.DenseOperator.from_local_rows(A, d.N, d.row0)
    else:
        op = nys.DenseOperator(A)
    return nys.MLProblem(nys.builtin_loss(d.loss), op, d.b, d.lambda1, d.lambda2)


# ------------------------------------------------------------------ CPU arm --


def _ref_nysopt():
    """The unmodified reference package from baseline/_ref, or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "nysopt")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import nysopt  # noqa: F401

        return nysopt
    except Exception:
        return None


def cpu_sample(d, W, K, A_host=None, prefer_reference=True):
    """Host-CPU timing of the reference algorithm on config ``d``: one setup,
    then W untimed and K timed ADMM iterations (one solve with max_iter = W + K,
    per-iteration marks from its callback).  Returns a dict with the rate
    iterations / (time after setup), the setup time and what ran."""
    A = A_host if A_host is not None else d.A
    # all host threads for the BLAS, whatever a launcher set (torchrun exports
    # OMP_NUM_THREADS=1 to every rank)
    try:
        from threadpoolctl import threadpool_limits

        _limits = threadpool_limits(limits=os.cpu_count(), user_api="blas")
        from threadpoolctl import threadpool_info

        threads = max([i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"] or [1])
    except Exception:  # pragma: no cover - threadpoolctl missing
        _limits, threads = None, None
    mod = _ref_nysopt() if prefer_reference else None
    marks = []
    cb = lambda *a: marks.append(time.perf_counter())
    if mod is not None:
        kind = "reference"
        if d.kind == "boxqp":
            prob = mod.QPProblem(mod.DenseOperator(d.P), d.q, mod.IdentityOperator(d.P.shape[0]), mod.Box(d.lo, d.hi))
        else:
            prob = mod.MLProblem(mod.builtin_loss(d.loss), A, d.b, d.lambda1, d.lambda2)
        opts = mod.SolverOptions(sketch_rank=d.rank, rng_seed=d.seed, eps_abs=1e-4, eps_rel=1e-4,
                                 eps_dual_gap=1e-4, max_iter=W + K)
        t0 = time.perf_counter()
        res = mod.solve(prob, opts, callback=cb)
        setup = res.timings.setup_s
        its = res.iterations
    else:
        from oracle import port

        kind = "port"
        if d.kind == "boxqp":
            prob = port.QPSpec(d.P, d.q, d.lo, d.hi)
        else:
            prob = port.MLSpec(d.loss, A, d.b, d.lambda1, d.lambda2)
        o = port.Options(sketch_rank=d.rank, rng_seed=d.seed, eps_abs=1e-4, eps_rel=1e-4, eps_dual_gap=1e-4,
                         max_iter=W + K, callback=lambda k: cb())
        t0 = time.perf_counter()
        res = port.solve(prob, o)
        setup = res.setup_s
        its = res.iterations
    if _limits is not None:
        _limits.restore_original_limits()
    t_setup = t0 + setup
    w = min(W, max(0, len(marks) - 1))
    start = marks[w - 1] if w > 0 else t_setup
    timed = len(marks) - w
    el = marks[-1] - start if timed > 0 else float("nan")
    return {"value": timed / el if timed > 0 else None, "kind": kind, "setup_s": setup, "timed_iters": timed,
            "threads": threads,
            "untimed_iters": w, "timed_s": el, "s_per_iter": el / timed if timed > 0 else None,
            "iterations_run": its}


def host_info():
    """lscpu model / sockets / cores, host RAM, BLAS library and threads."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        info.update(model=kv.get("Model name"), sockets=kv.get("Socket(s)"),
                    cores_per_socket=kv.get("Core(s) per socket"), threads_per_core=kv.get("Thread(s) per core"))
    except Exception:
        pass
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal"):
                    info["ram_gb"] = round(int(line.split()[1]) / 1024 ** 2, 1)
    except Exception:
        pass
    try:
        from threadpoolctl import threadpool_info

        blas = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if blas:
            info["blas"] = f"{blas[0].get('internal_api')} {blas[0].get('version')}"
            info["blas_threads"] = max(i.get("num_threads", 1) for i in blas)
    except Exception:
        pass
    return info


def config_block(cfg, d, world):
    """The workload description, identical in both arms' lines."""
    if getattr(d, "A", None) is None:
        N, n = d.N, d.n
    else:
        n = d.P.shape[0] if d.kind == "boxqp" else d.A.shape[1]
        N = d.A.shape[0]
    return {"workload": f"config {cfg}: {d.kind} {N}x{n} FP64, rank {d.rank}, tol 1e-4, solve to tolerance",
            "config_index": cfg, "rows": N, "features": n, "sketch_rank": d.rank,
            "parallelism": f"row-shard x{world}" if world > 1 else "single GPU",
            "metric_definition": "ADMM iterations / (total - setup) s (BASELINE.md §2)",
            "l2_policy": _l2_policy(8 * N * n)}


def _l2_policy(nbytes):
    mb = nbytes / 1e6
    if mb > 126:
        return "A (%.0f MB) larger than the 126 MB L2; no flush" % mb
    return ("A (%.0f MB) fits in the 126 MB L2 and stays resident across iterations, as in any "
            "solve of this size; no flush" % mb)


def run_reference(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return  # the CPU reference runs once, on rank 0
    cfg = args.config
    sample_note = ""
    if cfg == 5:
        # 160 GB does not fit a host run: the reference solves config 5's row
        # block 0 (12500 x 200000, the rows one GPU holds at N = 8) as a LASSO
        from paper_2310_08333_b200 import datagen

        Ab, noise = datagen.cfg5_block(0)
        b = Ab @ datagen.cfg5_truth() + noise
        lam = 0.1 * float(np.max(np.abs(Ab.T @ b)))
        d = datagen.ConfigData(5, "lasso", "square", Ab, b, lam, 0.0, rank=300, seed=4)
        sample_note = "config 5 row block 0 (12500 x 200000) as its own LASSO (160 GB exceeds a host run); "
    else:
        d, _ = build_problem(cfg)
    W, K = args.warmup, args.steps
    r = cpu_sample(d, W, K)
    hi = host_info()
    line = {
        "impl": "reference", "metric": "ADMM iters/s", "value": r["value"], "unit": "iters/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * r["s_per_iter"] if r["s_per_iter"] else None,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(cfg, d, world) if cfg != 5 else config_block(5, _cfg5_desc(), world),
        "cpu_baseline": {"value": r["value"], "unit": "iters/s",
                         "cores": r.get("threads") or hi.get("blas_threads", os.cpu_count()),
                         "kind": r["kind"],
                         "sample": f"{sample_note}one setup ({r['setup_s']:.1f} s), then {r['untimed_iters']} "
                                   f"untimed + {r['timed_iters']} timed ADMM iterations (one step = one "
                                   f"iteration); " + ("the unmodified nysopt package (baseline/_ref)"
                                                      if r["kind"] == "reference" else "oracle port") +
                                   ", NumPy/OpenBLAS on all host threads",
                         "setup_s": r["setup_s"], "host": hi},
        "e2e": {"value": r["value"], "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _cfg5_desc():
    from paper_2310_08333_b200 import datagen

    c = datagen.CONFIGS[5]
    return DevData(5, "lasso", "square", c["N"], c["n"], c["rank"], c["seed"], 0.0, None)


# ------------------------------------------------------------------ GPU arm --


def kernel_name(kx, d, n, rows_loc, world):
    """The kernel that runs the x-update's Hessian application for this shape."""
    persistent = (os.environ.get("NYS_CG_PERSIST", "1") != "0" and n <= 13312 and (d.kind == "boxqp" or world == 1))
    try:
        import paper_2310_08333_b200.dist as _dist

        persistent = persistent and not (_dist.FORCE_COLLECTIVES and d.kind != "boxqp")
    except ImportError:
        pass
    if persistent:
        return "cg_persist_kernel", "one Hessian application of the persistent PCG, incl. its CG vector phases"
    plan = kx.hvp_plan_name(rows_loc, n) if hasattr(kx, "hvp_plan_name") else "hvp"
    return plan, "one Hessian application A^T(d o A v) (+ shift v, p.Ap) incl. its partial-sum reduction"


def run_ours(args):
    import torch

    rank, world, local = _env_rank()
    ndev = max(1, torch.cuda.device_count())
    if world > 1:
        if os.environ.get("NYS_DIST_BACKEND", "nccl") == "nccl" and ndev < world:
            raise SystemExit(f"{world} ranks need {world} GPUs (found {ndev}); "
                             "NYS_DIST_BACKEND=gloo lets ranks share a GPU (test mode)")
        torch.cuda.set_device(local % ndev)
        # NCCL over NVLink; NYS_DIST_BACKEND=gloo lets several ranks share one GPU
        # to exercise this multi-rank code path (host-staged collectives, not a measurement)
        torch.distributed.init_process_group(os.environ.get("NYS_DIST_BACKEND", "nccl"),
                                             device_id=torch.device("cuda", local % ndev)
                                             if os.environ.get("NYS_DIST_BACKEND", "nccl") == "nccl" else None)
    else:
        torch.cuda.set_device(0)
        if args.collectives:
            # the row-sharded engine and its NCCL exchange steps on one rank (what a one-GPU box
            # allows): measures the sharded schedule's own cost, no NVLink transfer in it
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29591")
            torch.distributed.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
            import paper_2310_08333_b200.dist as _dist

            _dist.FORCE_COLLECTIVES = True
    import paper_2310_08333_b200 as nys
    from paper_2310_08333_b200.kernels import get_kernels

    kx = get_kernels()
    cfg = args.config
    want_cpu = rank == 0 and world == 1 and not args.no_cpu
    host_rows = None  # this rank's rows on the host (pinned) for the e2e leg
    if cfg == 5:
        # 160 GB: generated in HBM per rank (each rank holds only its row blocks)
        d, opts, A_dev = build_cfg5(world, rank)
        args.no_e2e = True
    elif cfg == 4 and args.collectives and args.as_rank_of > 1:
        # per-rank cost of an N-rank run, measured on one GPU: this process holds the rows of rank 0
        # of N and solves the statistically equivalent stand-in (sqrt(N) A_loc, sqrt(N) b_loc: the
        # rows are i.i.d., so A'^T A' ~ A^T A and A'^T b' ~ A^T b, with the global lambda) through
        # the sharded engine and NCCL.  Same kernels, shapes and exchange calls as that rank would
        # run; not the global problem, so iterations / CG counts are reported, not asserted.
        import math

        import numpy as np

        d, opts, A_dev = build_cfg4_device(args.as_rank_of, 0, False)
        r0, r1 = d.row0, d.row0 + A_dev.shape[0]
        A_dev.mul_(math.sqrt(args.as_rank_of))
        d.b = np.ascontiguousarray(d.b[r0:r1]) * math.sqrt(args.as_rank_of)
        d.N, d.row0 = A_dev.shape[0], 0
        args.no_e2e = True
        want_cpu = False
    elif cfg == 4:
        need_host = (not args.no_e2e) or want_cpu
        d, opts, A_dev = build_cfg4_device(world, rank if world > 1 else 0, need_host and world == 1)
        if not args.no_e2e:
            if world == 1:
                host_rows = d.A_host
            else:
                host_rows = torch.empty(tuple(A_dev.shape), dtype=torch.float64, pin_memory=True)
                host_rows.copy_(A_dev)
    else:
        d, opts = build_problem(cfg)
        host_A = d.P if d.kind == "boxqp" else d.A
        # A resident in HBM for the kernel-side metric (each rank: its row shard inside solve)
        A_dev = torch.from_numpy(host_A).cuda()
        host_rows = torch.from_numpy(host_A).pin_memory() if not args.no_e2e else None
    prob = make_gpu_problem(d, A_dev, world)

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
    setup_s = 0.0
    barrier()
    st = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(st)
        for _ in range(args.steps):
            res = nys.solve(prob, opts)
            iters += res.iterations
            setup_s += res.timings.setup_s
        e1.record(st)
        barrier()
    el_s = e0.elapsed_time(e1) / 1e3
    loop_s = maxred(el_s - setup_s)  # iterations / (total - setup), slowest rank
    el_s = maxred(el_s)
    launches = kx.kernel_launches() - launches0
    value = iters / loop_s
    tts = el_s / args.steps

    # one extra, instrumented solve: every Hessian-application launch of the
    # x-update is bracketed by CUDA events on the solve's stream (with the
    # persistent solver one launch is a whole CG solve and counts its operator
    # applications; predicated no-op launches are excluded)
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
    rows_loc = A_dev.shape[0] if d.kind != "boxqp" else n
    alg_bytes = 8 * rows_loc * n + 8 * (2 * n + rows_loc)
    peak, peak_kind = _peaks()
    kname, unit_desc = kernel_name(kx, d, n, rows_loc, world)
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
                "traffic": traffic_db.get(f"cfg{cfg}_{kname}") if world == 1 else None,
                "alg_bytes_per_unit": alg_bytes, "unit_of_work": unit_desc, "ms_per_unit": avg_ms,
                "units_timed": k_count, "share_of_step": k_total_ms / inst_ms,
                "timing": "CUDA events on the solve stream around every Hessian-application launch of one "
                          "extra instrumented solve (not the timed steps)"}
    # the HVP kernel alone, back to back on the same A and row weights
    hvp_alone = None
    if d.kind != "boxqp" and world == 1:
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
        hk = kx.hvp_plan_name(A_dev.shape[0], n) if hasattr(kx, "hvp_plan_name") else "hvp"
        hvp_alone = {"kernel": hk, "achieved": ha, "peak": peak, "unit": "GB/s", "frac": ha / peak,
                     "ms_per_launch": hms, "traffic": traffic_db.get(f"cfg{cfg}_hvp"),
                     "timing": f"CUDA events around {reps} back-to-back launches"}

    # e2e: public API with host buffers (pinned), upload + readback inside each step
    e2e = None
    if host_rows is not None:
        kx.h2d = kx.d2h = 0
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        e_iters = 0
        steps_e = max(1, args.steps)
        host_view = host_rows if isinstance(d, DevData) else host_rows.numpy()
        t0.record(st)
        for _ in range(steps_e):
            p2 = make_gpu_problem(d, host_view, world)
            r2 = nys.solve(p2, opts)
            e_iters += r2.iterations
        t1.record(st)
        barrier()
        e_s = maxred(t0.elapsed_time(t1) / 1e3)
        a_bytes = host_rows.numel() * 8 if isinstance(d, DevData) else host_rows.numel() * 8 // world
        b_bytes = 0 if d.kind == "boxqp" else d.b.nbytes // world
        e2e = {"value": e_iters / e_s, "unit": "iters/s", "h2d_bytes_per_step": int(a_bytes + b_bytes + kx.h2d / steps_e),
               "d2h_bytes_per_step": int(kx.d2h / steps_e), "time_to_tolerance_s": e_s / steps_e,
               "definition": "iterations / whole public-API solve wall time (upload and setup included)"}
    if cfg == 5:
        e2e = {"unavailable": "config 5 is generated in HBM per rank (160 GB); there is no host copy to upload"}
    cpu = None
    if want_cpu and cfg != 5:
        A_host = d.A_host.numpy() if isinstance(d, DevData) else None
        W, K = CPU_SAMPLE
        r = cpu_sample(d, W, K, A_host=A_host)
        hi = host_info()
        cpu = {"value": r["value"], "unit": "iters/s", "cores": r.get("threads") or hi.get("blas_threads", os.cpu_count()),
               "kind": r["kind"], "setup_s": r["setup_s"], "host": hi,
               "sample": f"config {cfg}: one setup ({r['setup_s']:.1f} s), then {r['untimed_iters']} untimed + "
                         f"{r['timed_iters']} timed ADMM iterations ({r['timed_s']:.1f} s), iterations / time "
                         "after setup; " + ("the unmodified nysopt package (baseline/_ref)"
                                            if r["kind"] == "reference" else "oracle port") + ", NumPy/OpenBLAS"}

    if rank == 0:
        line = {
            "metric": "ADMM iters/s", "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el_s / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(cfg, d, world),
            "result": {"time_to_tolerance_s": tts, "setup_s_per_solve": setup_s / args.steps,
                       "iterations": res.iterations, "status": res.status.value, "objective": res.objective,
                       "sketches": res.device_stats.get("sketches")},
            "roofline": roof, "hvp_alone": hvp_alone, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if getattr(args, "collectives", False) and world == 1:
            line["config"]["parallelism"] = ("row-sharded engine on one rank, exchange steps over NCCL "
                                             "(world-size-1 group; --collectives)")
            if args.as_rank_of > 1:
                line["config"]["parallelism"] += (f"; rows of ONE rank of {args.as_rank_of} "
                                                  "(scaled stand-in problem: a per-rank cost projection, "
                                                  "not the global solve)")
                line["result"]["cg_iterations"] = int(sum(h.cg_iters for h in res.history))
        print(json.dumps(line), flush=True)
    if world > 1 or (torch.distributed.is_available() and torch.distributed.is_initialized()):
        torch.distributed.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args):
    """``--gpus N`` without a launcher: re-exec through torch.distributed.run
    (one rank per GPU, rendezvous on 127.0.0.1).  Under a launcher the world
    size must match ``--gpus``."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if args.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
                   *sys.argv[1:]]
            os.execv(sys.executable, cmd)
        return
    if int(world) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--as-rank-of", type=int, default=1,
                    help="with --collectives, config 4: hold the rows of one rank of N and solve the "
                         "statistically equivalent stand-in (per-rank cost projection)")
    ap.add_argument("--collectives", action="store_true",
                    help="N = 1 only: run the row-sharded engine with its NCCL exchange steps on a world-size-1 group")
    args = ap.parse_args()
    relaunch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
