"""One default solve of a config (for ncu captures / launch lists): python tools/one_solve.py CFG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

w, t, _ = config_workload(int(sys.argv[1]))
s = PL.solve(t, w, None, SolveOptions(**eval(os.environ.get("OPTS", "{}"))))
print(sys.argv[1], s.status, s.makespan, f"{1e3 * s.search.device_seconds:.2f} ms", s.search.stats)
