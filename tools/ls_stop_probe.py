"""Local-search wave time on a config as a function of its stop makespan (the first wave only):
python tools/ls_stop_probe.py CFG STOP [STOP ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import engine as EN  # noqa: E402
from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions, build_problem  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

cfg = int(sys.argv[1])
w, t, _ = config_workload(cfg)
opts = SolveOptions(search="local")
prob = build_problem(t, w, opts)
eng = PL.get_engine(0)
wave = 8192 if prob.J < 24 else 2 * eng.sm_count
bits, _ = prob.key_bits(opts.walkers)
nprob = EN.NativeProblem(prob, bits)
for stop in [int(x) for x in sys.argv[2:]]:
    ts = []
    for rep in range(6):
        best = eng.reset_best()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.local_search(nprob, EN.SRC_SUBSTREAM, opts.seed, 0, wave, opts.max_rounds, best, stop_ms=stop)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    k = int(best[0].item())
    print(f"cfg{cfg} stop={stop} wave={wave} key={EN.ls_key_fields(k, bits)} ms={sorted(ts)[len(ts) // 2]:.3f} (all {[round(x, 3) for x in ts]})")
