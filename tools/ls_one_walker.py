"""One cfg-N local-search walker alone (the latency-bound critical path of a wave), for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import engine as EN  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions, build_problem  # noqa: E402
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table  # noqa: E402
from paper_2311_02840_b200.workloads import TECHNIQUES_4, TECHNIQUES_6, synthetic_workload  # noqa: E402

SHAPES = {3: (16, 1, 8, TECHNIQUES_4), 4: (32, 4, 8, TECHNIQUES_4), 5: (64, 1, 32, TECHNIQUES_6)}
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
walkers = int(sys.argv[2]) if len(sys.argv) > 2 else 1
J, N, G, T = SHAPES[cfg]
w = synthetic_workload(J, N, G, T)
t = build_profile_table(w, SyntheticExecutor(w.cluster))
prob = build_problem(t, w, SolveOptions())
eng = EN.Engine(0)
bits, _ = prob.key_bits(1 << 20)
nprob = EN.NativeProblem(prob, bits)
best = eng.reset_best()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
eng.local_search(nprob, EN.SRC_SUBSTREAM, 7, 0, walkers, 4096, best, stop_ms=int(prob.lower_bound()))
e1.record()
torch.cuda.synchronize()
print(f"cfg{cfg} walkers={walkers} ms={EN.ls_key_fields(int(best[0].item()), bits)[0]} dev_ms={e0.elapsed_time(e1):.2f}")
