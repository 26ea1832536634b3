"""Seed bound cost inside the default exact solve (bound-and-prune) for 8-11 one-node jobs:
device time of the seed (2^20 sampled candidates, plus a 4096-walker local search from 10 jobs)
against the whole solve."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import engine as EN  # noqa: E402
from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions, build_problem  # noqa: E402
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table  # noqa: E402
from paper_2311_02840_b200.workloads import synthetic_workload  # noqa: E402

eng = EN.Engine(0)
for J in (8, 9, 10, 11):
    w = synthetic_workload(J, 1, 8)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w)
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        U = eng.seed_bound(prob)
        torch.cuda.synchronize()
        seed_s = time.perf_counter() - t0
    s = PL.solve(t, w, None, SolveOptions(kernel="bnb", max_exhaustive=1 << 62))
    print(f"J={J} lower_bound={prob.lower_bound()} seed_bound={U} seed {seed_s * 1e3:.2f} ms; "
          f"solve dev {s.search.device_seconds * 1e3:.2f} ms makespan {s.makespan}", flush=True)
