"""Exact bound-and-prune on the 12-job mirrors (1 node) vs the default local search."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import planners as PL  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions  # noqa: E402
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table  # noqa: E402
from paper_2311_02840_b200.workloads import generate_workload  # noqa: E402

for preset in ("wikitext_mirror", "imagenet_mirror"):
    w = generate_workload(preset, 1, 7)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    for label, opts in (("local", SolveOptions()), ("bnb", SolveOptions(kernel="bnb", max_bnb=1 << 60))):
        PL.solve(t, w, None, opts)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = PL.solve(t, w, None, opts)
        torch.cuda.synchronize()
        print(preset, label, s.status, s.makespan, s.lower_bound, "dev %.3f s wall %.3f s" %
              (s.search.device_seconds, time.perf_counter() - t0), s.search.stats, flush=True)
