"""cProfile of the public-API solve (planners.solve, default options) for one config.

usage: python tools/solve_cprofile.py [config] [n]
Prints the median wall per solve (no profiler) and then the top host functions by own time
over n profiled solves (after warm-up).  Host-side evidence for the wall-time to best.
"""
import cProfile
import os
import pstats
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
w, t, _ = config_workload(cfg)
for _ in range(5):
    PL.solve(t, w)
torch.cuda.synchronize()
wall = []
for _ in range(n):
    t0 = time.perf_counter()
    s = PL.solve(t, w)
    wall.append(time.perf_counter() - t0)
print(f"config {cfg}: median wall {statistics.median(wall) * 1e3:.3f} ms, device {s.search.device_seconds * 1e3:.3f} ms, "
      f"status {s.status}, makespan {s.makespan}")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    PL.solve(t, w)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(30)
