import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2311_02840_b200 import engine as EN, planners
from paper_2311_02840_b200.problem import build_problem, SolveOptions
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table
from paper_2311_02840_b200.workloads import synthetic_workload
eng = EN.Engine(0)
w = synthetic_workload(5, 1, 4)
t = build_profile_table(w, SyntheticExecutor(w.cluster))
prob = build_problem(t, w)
for ident in (0, 61440):
    for bits in (62, prob.key_bits(prob.space)[0]):
        nprob = EN.NativeProblem(prob, bits)
        print('schedule', ident, bits, flush=True)
        r = eng.schedule(nprob, EN.SRC_INDEX, ids=[ident]); print(r[3], flush=True)
res = eng.search(prob, SolveOptions()); print(res, flush=True)
nprob = EN.NativeProblem(prob, prob.key_bits(prob.space)[0])
print(eng.schedule(nprob, EN.SRC_INDEX, ids=[res.index]), flush=True)
