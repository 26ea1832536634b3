"""Bound-and-prune time on config 1 vs the quality of the seed bound."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import engine as EN  # noqa: E402
from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import build_problem  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

w, t, c = config_workload(1)
prob = build_problem(t, w)
eng = PL.get_engine(0)
bits = (prob.space - 1).bit_length()
nprob = EN.NativeProblem(prob, bits)
print("sampled seed bound (2^16):", eng.seed_bound(prob), " (2^20):", eng.seed_bound(prob, 1 << 20))
for P in (4, 5):
    info = eng.tree_plan(nprob, P)
    for U in (30, 31, 32, 34, 40, None):
        times = []
        for rep in range(4):
            best = eng.reset_best()
            if U is not None:
                best[0:1].fill_((U << bits) | ((1 << bits) - 1))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ws = eng.search_bnb(nprob, P, 0, info.n_tasks, best)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        k = int(best[0].item())
        st = ws[:24].view(torch.int64).cpu().tolist()
        print(f"P={P} seed U={U}: {min(times[1:]):.3f} ms  key ms={k >> bits} idx={k & ((1 << bits) - 1)} "
              f"pruned={st[1]}/{info.n_tasks} pairs={st[2]}", flush=True)
