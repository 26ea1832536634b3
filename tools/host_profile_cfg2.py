"""Host-side profile of config 2's public-API run (plan_saturn + the introspection driver with
engine re-solves), as bench.py's e2e times it; wall per run printed first (no profiler)."""
import cProfile
import os
import pstats
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

w, t, c = config_workload(2)
_, _, _, opts = bench.workload(2, None)
for _ in range(3):
    bench.introspection_run(t, w, opts)
walls = []
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bench.introspection_run(t, w, opts)
    torch.cuda.synchronize()
    walls.append((time.perf_counter() - t0) * 1e3)
print(f"wall ms per run: median {statistics.median(walls):.3f}")
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    bench.introspection_run(t, w, opts)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
