"""Config 3: best makespan the local search reaches vs walkers (lower bound 29)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

w, t, c = config_workload(3)
for seed in (7, 11):
    for n in (1 << 16, 1 << 18, 1 << 20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = PL.solve(t, w, None, SolveOptions(search="local", walkers=n, wave=1 << 14, seed=seed))
        torch.cuda.synchronize()
        print(f"seed={seed} walkers={n} makespan={s.makespan} bound={s.lower_bound} status={s.status} "
              f"time={time.perf_counter() - t0:.2f}s stats={s.search.stats}", flush=True)
