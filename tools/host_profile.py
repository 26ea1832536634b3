"""Host-side profile of one default exact solve of config 1 (plan_saturn through the public API)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

w, t, c = config_workload(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
for _ in range(5):
    PL.solve(t, w)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    PL.solve(t, w)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(28)
