"""cProfile of the default public-API solve (plan_saturn) of a config: where the host wall time
outside the device search goes.  python tools/host_profile_solve.py CFG"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
w, t, _ = config_workload(cfg)
for _ in range(3):
    PL.solve(t, w)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    s = PL.solve(t, w)
    torch.cuda.synchronize()
pr.disable()
print("device ms per solve", 1e3 * s.search.device_seconds)
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
