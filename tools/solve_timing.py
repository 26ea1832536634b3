"""Device / wall time of the default solve (plan_saturn) per config, with its search stats:
the time-to-best figures of the bench's time_to_best block, on demand.

    python tools/solve_timing.py [configs...]     (default 1 3 4 5)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

reps = int(os.environ.get("REPS", "5"))
for cfg in [int(x) for x in (sys.argv[1:] or ["1", "3", "4", "5"])]:
    w, t, _ = config_workload(cfg)
    opts = SolveOptions(**eval(os.environ.get("OPTS", "{}")))
    PL.solve(t, w, None, opts)
    dev, wall = [], []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = PL.solve(t, w, None, opts)
        torch.cuda.synchronize()
        wall.append(time.perf_counter() - t0)
        dev.append(s.search.device_seconds)
    st = dict(s.search.stats or {})
    proof = st.pop("proof", None)
    print(f"cfg{cfg} kernel={s.search.kernel} status={s.status} makespan={s.makespan} lb={s.lower_bound} "
          f"dev_ms={1e3 * min(dev):.2f} (median {1e3 * sorted(dev)[len(dev) // 2]:.2f}) "
          f"wall_ms={1e3 * min(wall):.2f} stats={st} proof={proof}", flush=True)
