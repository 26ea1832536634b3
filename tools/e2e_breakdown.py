"""Wall-time breakdown of one public-API solve (build -> search -> decode -> check), no profiler.

usage: python tools/e2e_breakdown.py [config] [tree|default]
Each stage is bracketed by torch.cuda.synchronize(); medians over 30 solves after 5 warm-ups.
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200 import domain as D  # noqa: E402
from paper_2311_02840_b200.engine import NativeProblem  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions, build_problem  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
mode = sys.argv[2] if len(sys.argv) > 2 else "tree"
w, t, _ = config_workload(cfg)
opts = SolveOptions(kernel="tree") if mode == "tree" else SolveOptions()
eng = PL.get_engine(None)

stages = {k: [] for k in ("build", "search", "decode", "check", "solve_total")}
for rep in range(35):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = build_problem(t, w, opts)
    t1 = time.perf_counter()
    res = eng.search(prob, opts)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    nprob = NativeProblem(prob, res.idx_bits)
    src = 0 if res.exhaustive else res.source
    plan, options, ms, runtimes = PL._decode(eng, prob, nprob, w, src, res.seed, ident=res.index) \
        if res.kernel != "local" else (None, None, None, None)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    if plan is not None:
        D.check_plan(plan, w, runtimes)
    t4 = time.perf_counter()
    PL.solve(t, w, None, opts)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    if rep >= 5:
        for k, v in zip(stages, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)):
            v_ms = v * 1e3
            stages[k].append(v_ms)
print(f"config {cfg} mode {mode}: median ms per stage")
for k, v in stages.items():
    print(f"  {k:12s} {statistics.median(v):8.3f}")
