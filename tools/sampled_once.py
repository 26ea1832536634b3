"""One sampled search of a config's candidate stream (substream(7, i), i < budget) through the
per-candidate kernel, for ncu captures: python tools/sampled_once.py CFG [log2 budget]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

cfg = int(sys.argv[1])
w, t, _ = config_workload(cfg)
budget = 1 << int(sys.argv[2] if len(sys.argv) > 2 else 24)
s = PL.solve(t, w, None, SolveOptions(search="sampled", budget=budget, seed=7))
print(cfg, s.search.kernel, s.search.makespan, f"{1e3 * s.search.device_seconds:.2f} ms")
