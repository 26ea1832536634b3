cat > /tmp/lsq.py <<'PY'
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200.problem import SolveOptions
from paper_2311_02840_b200.workloads import config_workload
for k in (3, 4, 5):
    w, t, c = config_workload(k)
    for mode, n, rounds in (("sampled", 1 << 27, 0), ("local", 1 << 12, 4096), ("local", 1 << 14, 4096), ("local", 1 << 16, 4096)):
        if k == 5 and mode == "local" and n > (1 << 14):
            continue
        opts = SolveOptions(search=mode, budget=n, walkers=n, max_rounds=rounds or 4096)
        PL.solve(t, w, None, SolveOptions(search=mode, budget=1024, walkers=64))
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s = PL.solve(t, w, None, opts)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"cfg{k} {mode:8s} n={n:>10d} makespan={s.makespan:.0f} dev={s.search.device_seconds*1e3:.1f}ms wall={dt*1e3:.1f}ms", flush=True)
PY
timeout 900 python /tmp/lsq.py > gpurun_out/ls_quality.log 2>&1
