"""One wide (several-node) state-space search call, for timing and ncu: a synthetic workload,
a target, a state budget, prover or exact states.

usage: python tools/dp_wide_probe.py J N G seed target log2_budget [exact]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import engine as EN  # noqa: E402
from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import build_problem  # noqa: E402
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table  # noqa: E402
from paper_2311_02840_b200.workloads import synthetic_workload  # noqa: E402

J, N, G, seed, T, lg = (int(x) for x in sys.argv[1:7])
exact = len(sys.argv) > 7 and sys.argv[7] == "exact"
w = synthetic_workload(J, N, G, seed=seed)
t = build_profile_table(w, SyntheticExecutor(w.cluster))
prob = build_problem(t, w)
eng = PL.get_engine(0)
nprob = EN.NativeProblem(prob, 1)
eng.dp_search(nprob, T, 1 << lg, exact=exact)          # warm (the budget's workspace, module load)
torch.cuda.synchronize()
t0 = time.perf_counter()
st, info, cand = eng.dp_search(nprob, T, 1 << lg, exact=exact)
dt = time.perf_counter() - t0
print(f"J={J} N={N} G={G} seed={seed} T={T} budget=2^{lg} exact={exact}: {EN.DP_STATUS[st]} levels={info.levels} "
      f"states={info.states} widest={info.widest_level} {dt * 1e3:.1f} ms = {info.states / dt / 1e6:.1f} M states/s")
