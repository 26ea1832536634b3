cat > /tmp/t2.py <<'PY'
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200.problem import SolveOptions, build_problem
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table
from paper_2311_02840_b200.workloads import synthetic_workload
for J in (8, 9, 10, 11):
    w = synthetic_workload(J, 1, 8)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    p = build_problem(t, w)
    print("J", J, "space %.3e" % p.space, p.key_bits(p.space), flush=True)
    try:
        for i in range(2):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            s = PL.solve(t, w, None, SolveOptions(kernel="bnb", max_exhaustive=1 << 62))
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print("  bnb", s.makespan, s.search.index, "dev %.3f ms wall %.3f ms" % (s.search.device_seconds * 1e3, dt * 1e3), s.search.stats, flush=True)
        if p.space < 2e12:
            s2 = PL.solve(t, w, None, SolveOptions(kernel="tree", max_exhaustive=1 << 62))
            print("  tree", s2.makespan, s2.search.index, "dev %.3f ms" % (s2.search.device_seconds * 1e3), flush=True)
    except Exception as e:
        print("  error", type(e).__name__, e, flush=True)
PY
timeout 600 python /tmp/t2.py > gpurun_out/bnb_scale.log 2>&1
