"""Local-search time to the proven optimum vs the first wave size (configs 3-5), and where the
wall time of plan_saturn goes (search / whole solve)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions, build_problem  # noqa: E402
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table  # noqa: E402
from paper_2311_02840_b200.workloads import TECHNIQUES_4, TECHNIQUES_6, synthetic_workload  # noqa: E402

SHAPES = {3: (16, 1, 8, TECHNIQUES_4), 4: (32, 4, 8, TECHNIQUES_4), 5: (64, 1, 32, TECHNIQUES_6)}
for cfg in [int(x) for x in (sys.argv[1:] or ["3", "4", "5"])]:
    J, N, G, T = SHAPES[cfg]
    w = synthetic_workload(J, N, G, T)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    for wave in [int(x) for x in os.environ.get("WAVES", "256,1024,4096,16384").split(",")]:
        opts = SolveOptions(wave=wave)
        PL.solve(t, w, None, opts)
        eng = PL.get_engine(None)
        prob = build_problem(t, w, opts)
        torch.cuda.synchronize()
        dev, wall, srch = [], [], []
        for _ in range(3):
            t0 = time.perf_counter()
            s = PL.solve(t, w, None, opts)
            torch.cuda.synchronize()
            wall.append(time.perf_counter() - t0)
            dev.append(s.search.device_seconds)
            t1 = time.perf_counter()
            eng.search(prob, opts)
            torch.cuda.synchronize()
            srch.append(time.perf_counter() - t1)
        print(f"cfg{cfg} wave={wave} makespan={s.makespan} status={s.status} dev_ms={1e3 * min(dev):.2f} "
              f"search_wall_ms={1e3 * min(srch):.2f} solve_wall_ms={1e3 * min(wall):.2f} stats={s.search.stats}",
              flush=True)
