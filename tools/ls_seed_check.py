"""Diagnostic: the local-search solve honours SolveOptions.seed (different walker starts)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

w, t, c = config_workload(3)
for seed in (7, 11, 12345):
    s = PL.solve(t, w, None, SolveOptions(search="local", walkers=4096, wave=4096, seed=seed))
    print(seed, s.search.seed, s.search.index, s.makespan, s.search.stats, flush=True)
