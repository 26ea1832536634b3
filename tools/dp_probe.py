"""sat_search_dp on a config at given targets: status, levels, states, device ms.
python tools/dp_probe.py CFG T [T ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import engine as EN  # noqa: E402
from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import build_problem  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

cfg = int(sys.argv[1])
w, t, _ = config_workload(cfg)
prob = build_problem(t, w)
eng = PL.get_engine(0)
nprob = EN.NativeProblem(prob, 1)
budget = int(os.environ.get("DP_STATES", 1 << 22))
for T in [int(x) for x in sys.argv[2:]]:
    ts = []
    for rep in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record()
        st, info, cand = eng.dp_search(nprob, T, budget)
        e1.record()
        e1.synchronize()
        ts.append((e0.elapsed_time(e1), 1e3 * (time.perf_counter() - w0)))
    ts.sort()
    print(f"cfg{cfg} T={T} status={EN.DP_STATUS[st]} levels={info.levels} states={info.states} "
          f"widest={info.widest_level} makespan={info.makespan} dev_ms={ts[2][0]:.3f} wall_ms={ts[2][1]:.3f}")
