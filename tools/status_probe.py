"""Status and time of the default solve on the small golden workloads and the SPEC.md:428-436
mirror presets (1 and 2 nodes): python tools/status_probe.py"""
import sys, os, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch
from helpers import golden_workload
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table
from paper_2311_02840_b200 import workloads as WL
cases = []
for n in ["small5_1x4", "small4_2x2", "hetero6", "tiny3_1x3"]:
    w, _ = golden_workload(n); cases.append((n, w))
for name in dir(WL):
    pass
try:
    for ds in ("wikitext_mirror", "imagenet_mirror"):
        for nodes in (1, 2):
            w = WL.generate_workload(ds, nodes, seed=7) if hasattr(WL, "generate_workload") else None
            if w is not None: cases.append((f"{ds}_{nodes}n", w))
except Exception as e:
    print("gen fail", e)
for n, w in cases:
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    PL.solve(t, w)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s = PL.solve(t, w)
    torch.cuda.synchronize()
    print(n, len(w.jobs), len(w.cluster.nodes), s.search.kernel, s.status, s.makespan, s.lower_bound, f"{1e3*(time.perf_counter()-t0):.1f} ms", f"space={s.problem.space:.3e}")
