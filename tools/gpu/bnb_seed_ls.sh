timeout 600 python tools/bnb_mirror_timing.py > gpurun_out/bnb_mirror.log 2>&1
cat > /tmp/j.py <<'PY'
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200.problem import SolveOptions
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table
from paper_2311_02840_b200.workloads import synthetic_workload
for J in (9, 10, 11):
    w = synthetic_workload(J, 1, 8); t = build_profile_table(w, SyntheticExecutor(w.cluster))
    PL.solve(t, w); torch.cuda.synchronize(); t0 = time.perf_counter()
    s = PL.solve(t, w); torch.cuda.synchronize()
    print(J, s.search.kernel, s.makespan, s.search.index, "dev %.3f s wall %.3f s" % (s.search.device_seconds, time.perf_counter() - t0), s.search.stats, flush=True)
PY
timeout 600 python /tmp/j.py > gpurun_out/bnb_j.log 2>&1
