"""Full-scan time of the cfg1 tree walk for each lane-prefix length (layout choice evidence)."""
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
bits, _ = prob.key_bits(prob.space)
nprob = EN.NativeProblem(prob, bits)
for P in range(1, prob.J - 1):
    info = eng.tree_plan(nprob, P)
    best = eng.reset_best()
    for _ in range(2):
        eng.search_tree(nprob, P, 0, info.n_tasks, best)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        eng.search_tree(nprob, P, 0, info.n_tasks, best)
    e1.record()
    torch.cuda.synchronize()
    k = int(best[0].item())
    print(f"P={P} tasks={info.n_tasks} placements={info.n_job_steps} ms={e0.elapsed_time(e1) / 3:.3f} "
          f"key_ms={k >> bits}", flush=True)
