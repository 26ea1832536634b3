timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/gputests.log
cat > /tmp/t.py <<'PY'
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200.problem import SolveOptions
from paper_2311_02840_b200.workloads import config_workload
w, t, c = config_workload(1)
for k in ("tree", "bnb"):
    for i in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s = PL.solve(t, w, None, SolveOptions(kernel=k))
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(k, s.makespan, s.search.index, "dev %.3f ms wall %.3f ms" % (s.search.device_seconds * 1e3, dt * 1e3), s.search.stats)
PY
python /tmp/t.py > gpurun_out/bnb_timing.log 2>&1
