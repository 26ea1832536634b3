"""How often the default solve proves its plan optimal on multi-node workloads beyond exhaustive
search, with and without the exact multi-node state-space mode (SolveOptions.dp_exact).

usage: python tools/multinode_optimality.py [n_workloads]
Random synthetic workloads (synthetic_workload shapes: 8-14 jobs, 2-4 nodes of 4 or 8 GPUs,
seeded); per workload the status, makespan, lower bound and wall time of planners.solve.
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions  # noqa: E402
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table  # noqa: E402
from paper_2311_02840_b200.workloads import synthetic_workload  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
shapes = [(J, N, G) for J in (8, 10, 12, 14) for N, G in ((2, 4), (2, 8), (3, 4), (4, 8))]
rows = []
for i in range(n):
    J, N, G = shapes[i % len(shapes)]
    w = synthetic_workload(J, N, G, seed=100 + i)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    res = {}
    for exact in (False, True):
        PL.solve(t, w, None, SolveOptions(dp_exact=exact))        # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = PL.solve(t, w, None, SolveOptions(dp_exact=exact))
        torch.cuda.synchronize()
        res[exact] = (s.status, s.makespan, s.lower_bound, time.perf_counter() - t0,
                      (s.search.stats or {}).get("winner", ""))
    rows.append((J, N, G, res))
    a, b = res[False], res[True]
    print(f"J={J:2d} N={N} G={G}: prover only {a[0]:8s} ms={a[1]:.0f} lb={a[2]:.0f} {a[3]*1e3:7.1f} ms | "
          f"+ exact {b[0]:8s} ms={b[1]:.0f} {b[3]*1e3:7.1f} ms {b[4]}", flush=True)
for exact in (False, True):
    opt = sum(r[3][exact][0] == "Optimal" for r in rows)
    print(f"dp_exact={exact}: Optimal on {opt} of {len(rows)}; median wall "
          f"{statistics.median(r[3][exact][3] for r in rows) * 1e3:.1f} ms; "
          f"sum of makespans {sum(r[3][exact][1] for r in rows):.0f}")
