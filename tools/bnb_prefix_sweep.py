"""Bound-and-prune lane-prefix sweep on config 1: device span and wall of planners.solve per prefix rule (min warp tasks)."""
import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_02840_b200 import planners as PL, engine as EN
from paper_2311_02840_b200.workloads import config_workload
w, t, _ = config_workload(1)
eng = PL.get_engine(0)
orig = EN.Engine.bnb_prefix
for mt in (1 << 10, 1 << 12, 1 << 13, 1 << 14, 1 << 15, 1 << 16, 1 << 17):
    EN.Engine.bnb_prefix = lambda self, nprob, min_tasks=0, mt=mt: orig(self, nprob, mt)
    dev, wall = [], []
    for r in range(12):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s = PL.solve(t, w)
        torch.cuda.synchronize(); wall.append(time.perf_counter() - t0); dev.append(s.search.device_seconds)
    print(f"min_tasks={mt}: P={s.search.stats['prefix_len']} tasks={s.search.stats['tasks']} pruned={s.search.stats.get('pruned_tasks')} "
          f"dev {statistics.median(dev[2:])*1e3:.3f} ms wall {statistics.median(wall[2:])*1e3:.3f} ms ms={s.makespan} idx={s.search.index}", flush=True)
