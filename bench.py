"""Plan-search benchmark: candidate plans evaluated / s and wall-time to the best plan.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1|2|3|4|5] [--impl ours|reference]

A step = one complete solve of the configured workload (config 1: the exhaustive
search of all 3.25e10 candidates of the paper workload; config 2: every solve of
one introspection run of it -- the initial solve plus the re-solve at each tick;
sampled configs: a fixed candidate budget), sharded over the ranks, combined with
an NCCL all-reduce MIN.
Rank 0 prints one JSON line.  `--impl reference` times the CPU oracle port
(oracle/oracle.c, OpenMP on every host thread) on a bounded sample of the same
workload -- the reference's own solver does not exist.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--budget", type=int, default=0, help="sampled configs: candidates per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=8.0, help="CPU baseline sample length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-index-leg", action="store_true", help="config 1: skip the per-candidate k_cand leg")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """`nvidia-smi -lms 50` running in the background across the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)          # first sample lands before the timed region starts
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        rows = [[x.strip() for x in l.split(",")] for l in self.lines]
        rows = [r for r in rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- workload
def workload(cfg: int, budget: int):
    from paper_2311_02840_b200.problem import SolveOptions
    from paper_2311_02840_b200.workloads import CONFIGS, config_workload

    w, t, c = config_workload(cfg)
    if cfg in (1, 2):
        opts = SolveOptions(kernel="tree")                      # exhaustive full scan (evaluated/s)
    else:
        default = {3: 1 << 27, 4: 1 << 26, 5: 1 << 26}[cfg]
        opts = SolveOptions(search="sampled", budget=budget or default, seed=7)
    return w, t, c, opts


def respawn_if_needed(args) -> None:
    """`--gpus N` outside torchrun: re-exec this script under torch.distributed.run with N ranks
    (one process per GPU, 127.0.0.1 rendezvous), so `python bench.py --gpus N` always runs N ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def dist_setup(n_gpus: int):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"bench.py: --gpus {n_gpus} but WORLD_SIZE={world} (launch with torchrun "
                         f"--nproc-per-node {n_gpus}, or without torchrun to let bench.py spawn the ranks)")
    if world > 1 and os.environ.get("SATURN_BENCH_GPU_OVERRIDE") is None and torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks need {world} GPUs, {torch.cuda.device_count()} visible")
    if world > 1:
        import torch.distributed as dist

        # SATURN_BENCH_GPU_OVERRIDE=k maps every rank onto cuda:k with the gloo backend: a
        # functional check of the sharded path on a one-GPU box (ranks never wait on each
        # other inside a kernel; only the host-side collectives meet).  Never a bench number.
        override = os.environ.get("SATURN_BENCH_GPU_OVERRIDE")
        if override is not None:
            local = int(override)
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- CPU baseline
def cpu_baseline(cfg: int, seconds: float, w, t, opts):
    """C oracle port on every host thread over a bounded prefix (or sample) of the workload."""
    from oracle import coracle, saturn_oracle

    op = saturn_oracle.build(t.entries, w)
    cp = coracle.CProblem(op)
    threads = os.cpu_count() or 1
    src = "index" if cfg == 1 else "substream"
    n = 20000
    while True:
        t0 = time.perf_counter()
        cp.search(src, opts.seed, 0, n, threads)
        dt = time.perf_counter() - t0
        if dt > 0.5 or n > 1 << 34:
            break
        n *= 4
    rate = n / dt
    n2 = max(n, int(rate * seconds))
    t0 = time.perf_counter()
    cp.search(src, opts.seed, 0, n2, threads)
    dt2 = time.perf_counter() - t0
    return {"value": n2 / dt2, "unit": "plans/s", "cores": threads, "kind": "port",
            "sample": f"{'first' if cfg == 1 else 'substream(7, i) for i <'} {n2} candidates of config {cfg} "
                      f"({dt2:.1f} s, oracle/oracle.c literal per-GPU list scheduler, OpenMP)"}


def milp_baseline(w, t, gpu_makespan=None):
    """The reference's solver class on the CPU: the time-indexed MILP of SPEC.md:182-200 solved
    by HiGHS (scipy.optimize.milp) -- wall time to the provably optimal makespan (configs 1, 3).
    The MILP admits every gang schedule (backfilling included), so its optimum lower-bounds the
    list-scheduling optimum: equality with the GPU plan's makespan certifies that plan optimal."""
    from oracle import saturn_oracle

    op = saturn_oracle.build(t.entries, w)
    t0 = time.perf_counter()
    opt = saturn_oracle.milp_optimum(op, time_limit=120.0)
    out = {"seconds": time.perf_counter() - t0, "optimum_intervals": opt, "solver": "HiGHS (scipy.optimize.milp)",
            "formulation": "time-indexed MILP, SPEC.md:182-200, after the exact option prune", "threads": "HiGHS default"}
    if gpu_makespan is not None:
        out["gpu_plan_certified_optimal"] = gpu_makespan == opt
    return out


def python_baseline(cfg: int, w, t, opts, seconds: float = 3.0):
    """Pure-Python oracle (the reference's language), 1 core, for context."""
    from oracle import saturn_oracle

    op = saturn_oracle.build(t.entries, w)
    src = "index" if cfg == 1 else "substream"
    n, t0 = 0, time.perf_counter()
    step = 500
    while time.perf_counter() - t0 < seconds:
        saturn_oracle.search(op, src, opts.seed, n, n + step)
        n += step
    return {"value": n / (time.perf_counter() - t0), "unit": "plans/s", "cores": 1, "kind": "port",
            "sample": f"first {n} candidates, oracle/saturn_oracle.py"}


def run_reference(args):
    rank, world, _ = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), 0
    if rank != 0:
        return
    w, t, c, opts = workload(args.config, args.budget)
    from oracle import coracle, saturn_oracle

    op = saturn_oracle.build(t.entries, w)
    cp = coracle.CProblem(op)
    threads = os.cpu_count() or 1
    src = "index" if args.config in (1, 2) else "substream"
    # calibrate a per-step sample of ~`per_step` seconds so K+W steps finish in minutes
    per_step = min(15.0, 150.0 / max(1, args.steps + args.warmup))
    n = 20000
    while True:
        t0 = time.perf_counter()
        cp.search(src, opts.seed, 0, n, threads)
        dt = time.perf_counter() - t0
        if dt > 0.3 or n > 1 << 34:
            break
        n *= 4
    n_step = max(n, int(n / dt * per_step))
    for i in range(args.warmup):
        cp.search(src, opts.seed, 0, max(1, n_step // 10), threads)
    times = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        cp.search(src, opts.seed, i * n_step, (i + 1) * n_step, threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = n_step * args.steps / tot
    line = {
        "impl": "reference", "metric": "candidate plans evaluated/sec", "value": value, "unit": "plans/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int32" if opts.time_mode == "grid" else "f64", "data": "synthetic",
        "config": {"workload": c["name"], "sample_per_step": n_step},
        "cpu_baseline": {"value": value, "unit": "plans/s", "cores": threads, "kind": "port",
                         "sample": f"{n_step} candidates per step ({src} order) of {c['name']}, oracle/oracle.c, "
                                   f"OpenMP {threads} threads"},
        "e2e": {"value": value, "unit": "plans/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "time_to_best_s_extrapolated": (op.space / value) if args.config == 1 else None,
    }
    print(json.dumps(line))


NCU_KEYS = {"issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "threads_per_warp_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
            "warp_insts": "smsp__inst_executed.sum",
            "kernel_ms": "gpu__time_duration.sum"}


def ncu_capture(kernel: str, cfg: int):
    """The newest committed `ncu --set full` summary of this kernel at this config
    (profiles/rNN_ncu_full_<kernel>_cfg<k>.json): (DRAM bytes per launch, issue / pipe
    utilisation dict, source path), or Nones."""
    import glob

    hits = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_ncu_full_{kernel}_cfg{cfg}.json")),
                  key=lambda f: os.path.basename(f).split("_")[0])
    if not hits:
        return None, None, None
    with open(hits[-1]) as f:
        rep = json.load(f)
    for k in rep.get("kernels", []):
        if kernel in k.get("kernel", ""):
            util = {short: k[m]["value"] for short, m in NCU_KEYS.items() if isinstance(k.get(m), dict)}
            return k.get("traffic_bytes"), util, os.path.relpath(hits[-1], ROOT)
    return None, None, None


# ----------------------------------------------------------------------------- ours
class DeviceSolve:
    """One search of a step, marshalled once (launch parameters resident), sharded over ranks."""

    def __init__(self, eng, prob, opts, rank, world):
        from paper_2311_02840_b200 import engine as EN

        self.EN, self.eng, self.prob, self.opts, self.world = EN, eng, prob, opts, world
        self.mode, n_idx = eng.plan_search(prob, opts)
        self.idx_bits, _ = prob.key_bits(n_idx)
        self.nprob = EN.NativeProblem(prob, self.idx_bits)
        self.use_tree = self.mode == "exhaustive" and eng._tree_ok(prob)
        G, N, J = prob.G, prob.N, prob.J
        if self.use_tree:
            # per rank ~4 warp tasks per resident warp at least (dynamic cursor balance)
            self.info = eng.tree_plan(self.nprob, eng.full_scan_prefix(self.nprob, world))
            self.a, self.b = eng.tree_shard(self.nprob, self.info.prefix_len, rank, world)   # work-balanced
            self.n_cand = self.info.n_candidates
            # algorithmic INT32 work of the prefix-shared walk, counted on
            # the minimal enumeration tree (every (ordered job prefix, options) node placed once:
            # the 1-job-prefix layout), so lanes re-placing their prefix earn nothing:
            #   internal placement: node pick (N) + 2G slot min/max + add + makespan max = N + 2G + 2
            #   leaf placement (last job, no state update): node pick + add + max = N + 2
            mini = eng.tree_plan(self.nprob, 1)
            merges = mini.n_job_steps - mini.n_candidates
            self.ops = (merges // world) * (N + 2 * G + 2) + (self.n_cand // world) * (N + 2)
            self.kernel = "k_tree"
        else:
            self.a, self.b = EN._shard(n_idx, rank, world)
            self.n_cand = n_idx
            self.ops = (n_idx // world) * J * (N + 2 * G + 2)
            self.kernel = "k_cand"
        self.best = eng.reset_best(eng.torch.empty(2, dtype=eng.torch.int64, device=eng.device))

    def launch(self):
        EN, eng = self.EN, self.eng
        eng.reset_best(self.best)
        if self.use_tree:
            eng.search_tree(self.nprob, self.info.prefix_len, self.a, self.b, self.best)
        elif self.mode == "exhaustive":
            eng.search_index(self.nprob, self.a, self.b, self.best)
        else:
            eng.search_sampled(self.nprob, EN.SRC_SUBSTREAM, self.opts.seed, self.a, self.b, self.best)

    def combine(self, group):
        # the engine's key hand-off (sat_key_finish, + NCCL MIN across ranks): no library
        # elementwise kernels inside the timed step
        key, _ = self.eng._key_finish(self.best, self.nprob.grid, group, self.world, self.idx_bits, 0)
        return key.cpu().tolist()[:2]


def introspection_run(t, w, opts, group=None, record=None):
    """Config 2: plan_saturn, then execute with a re-solve every R = predicted/10 and rho = 30 s
     -- the public API end to end.  Returns (report, candidates evaluated)."""
    from paper_2311_02840_b200 import planners
    from paper_2311_02840_b200 import simulator as SIM

    evaluated = [0]

    def replan(table, workload, ctx):
        sol = planners.solve(table, workload, None, opts, ctx, group=group)
        evaluated[0] += sol.search.evaluated
        if record is not None:
            record.append(ctx)
        return sol.plan

    sol0 = planners.solve(t, w, None, opts, group=group)
    evaluated[0] += sol0.search.evaluated
    rep = SIM.simulate(w, t, sol0.plan, SIM.SimOptions(introspection_interval=sol0.plan.predicted_makespan / 10,
                                                       checkpoint_overhead=30.0, replanner=replan))
    return rep, evaluated[0]


def per_candidate_leg(eng, prob, opts, rank, world, group, peak_i32, tree_key, reps: int = 2):
    """The exhaustive space once more through the per-candidate kernel (k_cand, index source):
    every candidate decoded and list-scheduled from scratch, no prefix sharing -- the SURVEY.md
    8(d) work model (J x (N + 2G + 2) INT32 ops per plan) applies to it as written.  Same key as
    the tree walk required."""
    import torch

    from paper_2311_02840_b200 import engine as EN

    n = prob.space
    bits, _ = prob.key_bits(n)
    nprob = EN.NativeProblem(prob, bits)
    a, b = EN._shard(n, rank, world)
    best = eng.reset_best(torch.empty(2, dtype=torch.int64, device=eng.device))
    stream = torch.cuda.current_stream()
    eng.search_index(nprob, a, b, best)                                   # warm-up
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        eng.reset_best(best)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.search_index(nprob, a, b, best)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    t_dev = max_over_ranks(min(times), world)
    k = int(EN._combine(best, True, group, world)[0])
    key = (k >> bits, k & ((1 << bits) - 1))
    ops_per_plan = prob.J * (prob.N + 2 * prob.G + 2)
    rate = n / t_dev
    return {"kernel": "k_cand<int32, index> (one candidate per thread, decoded + scheduled from scratch)",
            "candidates": n, "device_s": t_dev, "value": rate, "unit": "plans/s",
            "ops_per_plan": ops_per_plan, "achieved_tops": rate * ops_per_plan / 1e12,
            "frac_of_int32_peak": rate * ops_per_plan / peak_i32,
            "key": list(key), "key_equals_tree": list(key) == list(tree_key)}


def run_ours(args):
    import torch

    from paper_2311_02840_b200 import engine as EN
    from paper_2311_02840_b200 import planners
    from paper_2311_02840_b200.problem import build_problem

    rank, world, local = dist_setup(args.gpus)
    group = None
    w, t, c, opts = workload(args.config, args.budget)
    eng = planners.get_engine(local)
    report = None
    if args.config == 2:
        ctxs = []
        report, _ = introspection_run(t, w, opts, group, record=ctxs)
        problems = [build_problem(t, w, opts)] + [build_problem(t, w, opts, ctx) for ctx in ctxs]
    else:
        problems = [build_problem(t, w, opts)]
    solves = [DeviceSolve(eng, p, opts, rank, world) for p in problems]
    head = solves[0]
    n_cand = sum(s.n_cand for s in solves)
    stream = torch.cuda.current_stream()
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")

    for _ in range(args.warmup):
        for s in solves:
            s.launch()
        for s in solves:
            s.combine(group)
    torch.cuda.synchronize()

    # ---- device-resident timed region: K steps, L2 flushed between steps ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = eng.launches
    keys = []
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            e0, e1, e2 = ev[i]
            e0.record(stream)
            for s in solves:
                s.launch()
            e1.record(stream)
            keys.append([s.combine(group) for s in solves])
            e2.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = eng.launches - launches0
    step_s = [e0.elapsed_time(e2) / 1e3 for e0, _, e2 in ev]
    kern_s = [e0.elapsed_time(e1) / 1e3 for e0, e1, _ in ev]
    t_max = max_over_ranks(sum(step_s), world)
    kern_avg = max_over_ranks(sum(kern_s) / len(kern_s), world)
    value = n_cand * args.steps / t_max
    key = keys[-1][0]
    assert all(k == keys[-1] for k in keys), "non-deterministic search result"
    idx_bits = head.idx_bits
    ms = key[0] >> idx_bits if head.nprob.grid else None

    # ---- e2e: the public API with host inputs (marshal, launch, NCCL, decode, check) ----
    e2e_times = []
    e2e_cand = n_cand
    barrier(world)
    for i in range(max(2, min(args.steps, 5))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if args.config == 2:
            _, e2e_cand = introspection_run(t, w, opts, group)
            api = "planners.solve (plan_saturn) + simulator.simulate with engine re-solves (resolve)"
        else:
            planners.solve(t, w, None, opts, group=group)
            api = "paper_2311_02840_b200.planners.solve (plan_saturn)"
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(statistics.median(e2e_times[1:]), world)
    # ---- wall-time to the best-makespan plan: the default exact solve (bound-and-prune) ----
    ttb = None
    api = "paper_2311_02840_b200.planners.solve (plan_saturn)"
    if args.config in (1, 2):
        from paper_2311_02840_b200.problem import SolveOptions

        bopts = SolveOptions()                                  # auto = bnb for these problems
        dev, wall, stats = [], [], None
        for i in range(max(3, min(args.steps, 5))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if args.config == 2:
                introspection_run(t, w, bopts, group)
            else:
                sol_b = planners.solve(t, w, None, bopts, group=group)
                dev.append(sol_b.search.device_seconds)
                stats = sol_b.search.stats
            torch.cuda.synchronize()
            wall.append(time.perf_counter() - t0)
        ttb = {"method": "bound-and-prune (sat_search_bnb), same plan as the full scan",
               "wall_s": max_over_ranks(statistics.median(wall[1:]), world),
               "device_s": max_over_ranks(statistics.median(dev[1:]), world) if dev else None,
               "stats": stats,
               "api": api.replace("(plan_saturn)", "(plan_saturn, default options)")}
        if ttb["device_s"]:
            # candidates covered (scheduled or cut by a bound) per second,
            # reported apart from the full scan's evaluated/s
            ttb["covered_per_s"] = head.n_cand / ttb["device_s"]
    else:
        # spaces beyond exact search: the default solve is local search from greedy starts;
        # report the plan it reaches, the lower bound and the time (next to the sampled sweep)
        from paper_2311_02840_b200.problem import SolveOptions

        dev, wall, sol_l = [], [], None
        for i in range(7):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sol_l = planners.solve(t, w, None, SolveOptions(), group=group)
            torch.cuda.synchronize()
            wall.append(time.perf_counter() - t0)
            dev.append(sol_l.search.device_seconds)
        starts = "greedy" if sol_l.search.source == EN.SRC_GREEDY else "sampled"
        ttb = {"method": f"local search from {starts} starts (sat_local_search), {sol_l.search.evaluated} walkers"
                         + (", optimality by the state-space search" if sol_l.search.proven else
                            (", optimality by the lower bound" if sol_l.status == "Optimal" else "")),
               "makespan_intervals": sol_l.makespan, "lower_bound_intervals": sol_l.lower_bound,
               "status": sol_l.status, "sampled_step_makespan_intervals": ms,
               "wall_s": max_over_ranks(statistics.median(wall[1:]), world),
               "device_s": max_over_ranks(statistics.median(dev[1:]), world),
               "stats": sol_l.search.stats,
               "api": "paper_2311_02840_b200.planners.solve (plan_saturn, default options)"}

    # per solve in: the problem tables (host arrays), the tree kernel's by-value parameter block
    # and cursor reset, the decode id; out: best key + winner schedule (option, node, start per
    # job) + makespan
    tree_param = int(eng.lib.sat_tree_param_bytes())
    h2d = sum(s.nprob.param_bytes + 8 + (tree_param + 24 if s.use_tree else 0) for s in solves)
    d2h = sum(16 + 3 * 4 * s.prob.J + 8 for s in solves)

    # ---- roofline: INT32 min/max issue rate measured on this GPU ----
    # (k_tree launches whose pair pass is packed run VIMNMX.U16x2 / VIADDMNMX.U16x2: their
    # denominator is the same probe on 16-bit pairs, two lane-ops per lane-instruction)
    packed = bool(head.use_tree and head.info.pair_packed)

    def probe(fn):
        ops = torch.zeros(1, dtype=torch.int64, device="cuda")
        sink = torch.zeros(1, dtype=torch.int32, device="cuda")
        blocks, iters = eng.sm_count * 8, 4096
        fn(blocks, 256, iters, EN._vp(ops.data_ptr()), EN._vp(sink.data_ptr()), EN._vp(stream.cuda_stream))
        torch.cuda.synchronize()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        fn(blocks, 256, iters, EN._vp(ops.data_ptr()), EN._vp(sink.data_ptr()), EN._vp(stream.cuda_stream))
        p1.record(stream)
        torch.cuda.synchronize()
        return int(ops.item()) / (p0.elapsed_time(p1) / 1e3)

    peak_i32 = probe(eng.lib.sat_alu_probe)
    peak_ops = probe(eng.lib.sat_alu_probe16) if packed else peak_i32
    per_launch_ops = sum(s.ops for s in solves)
    achieved = per_launch_ops / kern_avg
    kernel_name = head.kernel
    traffic, ncu_util, traffic_src = ncu_capture(kernel_name, 1 if args.config == 2 else args.config)
    prob = head.prob
    # SURVEY.md 8(d)'s per-plan work model applied to every candidate of the step as if each were
    # scheduled from scratch: J x (N + 2G + 2) INT32 ops.  The tree walk shares prefixes, so for it
    # this exceeds the peak (the sharing is worth that factor); per-candidate kernels sit below 1.
    per_plan_ops = sum(s.n_cand * s.prob.J * (s.prob.N + 2 * s.prob.G + 2) for s in solves)
    per_plan_frac = per_plan_ops / kern_avg / peak_i32
    leg = None
    if args.config == 1 and head.use_tree and not args.no_index_leg:
        leg = per_candidate_leg(eng, prob, opts, rank, world, group, peak_i32,
                                (ms, key[0] & ((1 << idx_bits) - 1)))

    line = {
        "metric": "candidate plans evaluated/sec", "value": value, "unit": "plans/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int32" if head.nprob.grid else "f64", "data": "synthetic",
        "config": {"workload": c["name"], "jobs": prob.J, "nodes": prob.N, "gpus_per_node": int(prob.node_gpus[0]),
                   "search": head.mode, "candidates_per_step": n_cand, "solves_per_step": len(solves),
                   "kernel": kernel_name, "radix": [int(r) for r in prob.radix], "delta_s": prob.delta,
                   "l2": "256 MiB flush between steps, outside step events; working set = launch params",
                   "parallelism": f"candidate-space shards x{world}, NCCL all-reduce MIN"},
        "best": {"makespan_intervals": ms, "index": key[0] & ((1 << idx_bits) - 1) if head.nprob.grid else key[1],
                 "predicted_makespan_s": (ms * prob.delta) if ms is not None else None},
        "time_to_best_s": (ttb["device_s"] or ttb["wall_s"]) if ttb else t_max / args.steps / len(solves),
        "time_to_best": ttb or {"method": "full scan", "device_s": t_max / args.steps},
        "full_scan_s_per_solve": t_max / args.steps / len(solves),
        "e2e": {"value": e2e_cand / e2e_s, "unit": "plans/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "solve_wall_s": e2e_s, "api": api},
        "gpu_launches": launches,
        "kernel_ms": 1e3 * kern_avg,
        "roofline": {"bound": "int16x2-alu" if packed else "int32-alu", "achieved": achieved / 1e12,
                     "peak": peak_ops / 1e12, "unit": "TOP/s",
                     "frac": achieved / peak_ops, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": ("measured: sat_alu_probe16 VIMNMX.U16x2 chains on this GPU, 2 ops per "
                                     "lane-instruction (the pair pass runs on 16-bit pairs); MEASURED_PEAKS.json "
                                     "has no integer figure" if packed else
                                     "measured: sat_alu_probe IMNMX chains on this GPU (MEASURED_PEAKS.json has "
                                     "no INT32 figure)"),
                     "int32_peak": peak_i32 / 1e12, "frac_of_int32_peak": achieved / peak_i32,
                     "algorithmic_ops_per_launch": per_launch_ops,
                     "ops_model": ("tree walk on the minimal enumeration tree: internal placements x "
                                   "(N + 2G + 2) + leaves x (N + 2) (DESIGN.md 4.1)" if head.use_tree else
                                   "candidates x J x (N + 2G + 2) (SURVEY.md 8(d))"),
                     "per_plan_model_ops": per_plan_ops, "per_plan_model_frac": per_plan_frac,
                     "ncu": ncu_util, "ncu_source": traffic_src},
        "clocks": clk.summary(),
    }
    if head.use_tree:
        line["config"]["prefix_len"] = head.info.prefix_len
        line["config"]["walk_placements"] = head.info.n_job_steps
        line["config"]["counting"] = (
            "exhaustive prefix-shared enumeration (k_tree): every one of the candidates_per_step "
            "candidates' makespans is computed and enters the argmin, but candidates sharing an "
            "(order, options) prefix share its placements and the last job's options fold into "
            "per-gang minima -- ~7 ALU ops per candidate instead of J x (N + 2G + 2); the "
            "per-candidate kernel over the same space is per_candidate_leg")
    elif head.mode == "exhaustive":
        line["config"]["counting"] = "exhaustive, one candidate per thread decoded and scheduled from scratch"
    else:
        line["config"]["counting"] = "sampled candidates substream(seed, i), each scheduled from scratch"
    if leg is not None:
        line["per_candidate_leg"] = leg
    if report is not None:
        line["introspection"] = {"makespan_s": report.makespan, "replans": report.replan_count,
                                 "checkpoints": report.checkpoint_count,
                                 "candidates_per_solve": [s.n_cand for s in solves]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(1 if args.config == 2 else args.config, args.cpu_seconds, w, t, opts)
        if head.mode == "exhaustive" and line["cpu_baseline"].get("value"):
            # the CPU full scan's time to the best plan, extrapolated from the
            # bounded sample's rate (the port scans candidates at a uniform cost)
            line["cpu_baseline"]["full_scan_s_extrapolated"] = head.n_cand / line["cpu_baseline"]["value"]
        line["cpu_baseline_python"] = python_baseline(1 if args.config == 2 else args.config, w, t, opts)
        if args.config in (1, 3):
            try:
                line["cpu_time_to_best_milp"] = milp_baseline(
                    w, t, ttb.get("makespan_intervals", ms) if ttb else ms)
            except Exception as exc:          # scipy / HiGHS missing: say so, keep the line
                line["cpu_time_to_best_milp"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        respawn_if_needed(args)
        run_ours(args)


if __name__ == "__main__":
    main()
