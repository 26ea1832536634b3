import cProfile, pstats, sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200.problem import SolveOptions
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table
from paper_2311_02840_b200.workloads import TECHNIQUES_6, TECHNIQUES_4, synthetic_workload
for (J,N,G,T) in [(64,1,32,TECHNIQUES_6),(32,4,8,TECHNIQUES_4)]:
    w = synthetic_workload(J, N, G, T)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    PL.solve(t, w); PL.solve(t, w); torch.cuda.synchronize()
    pr = cProfile.Profile(); pr.enable()
    for _ in range(3): PL.solve(t, w)
    torch.cuda.synchronize(); pr.disable()
    pstats.Stats(pr).sort_stats("cumtime").print_stats(28)
