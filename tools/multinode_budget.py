"""State budget of the state-space proof on the multi-node workloads the default solve leaves
Local (tools/multinode_optimality.py shapes): status, makespan and wall per budget.

usage: python tools/multinode_budget.py [n_workloads]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions  # noqa: E402
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table  # noqa: E402
from paper_2311_02840_b200.workloads import synthetic_workload  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
shapes = [(J, N, G) for J in (8, 10, 12, 14) for N, G in ((2, 4), (2, 8), (3, 4), (4, 8))]
for i in range(n):
    J, N, G = shapes[i % len(shapes)]
    w = synthetic_workload(J, N, G, seed=100 + i)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    s0 = PL.solve(t, w)
    if s0.status == "Optimal":
        continue
    out = [f"J={J:2d} N={N} G={G} seed={100 + i}: default {s0.status} ms={s0.makespan:.0f} lb={s0.lower_bound:.0f}"]
    for lg in (23, 25, 27):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = PL.solve(t, w, None, SolveOptions(dp_states=1 << lg))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        att = (s.search.stats or {}).get("proof", {}).get("attempts", [])
        last = att[-1] if att else {}
        out.append(f"2^{lg}: {s.status} ms={s.makespan:.0f} {dt * 1e3:.0f} ms "
                   f"[{len(att)} attempts, last T={last.get('target')} {last.get('status')} "
                   f"{last.get('states', 0) / 1e6:.1f}M states{' exact' if last.get('exact') else ''}]")
    print(" | ".join(out), flush=True)
