"""Final makespan and rounds of each of the first N local-search walkers (configs 4, 5), one walker per launch:
the distribution behind the wave / tie-break choices.  python tools/walk_distribution.py N"""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_02840_b200 import engine as EN
from paper_2311_02840_b200.problem import SolveOptions, build_problem
from paper_2311_02840_b200.workloads import config_workload
eng = EN.Engine(0)
for cfg in (4, 5):
    w, t, _ = config_workload(cfg)
    prob = build_problem(t, w, SolveOptions())
    lb = int(prob.lower_bound())
    bits, _ = prob.key_bits(1 << 20)
    nprob = EN.NativeProblem(prob, bits)
    off = ctypes.c_size_t()
    eng.lib.sat_ls_counter_offset(nprob.ref, ctypes.byref(off))
    rows = []
    for wk in range(int(sys.argv[1])):
        best = eng.reset_best()
        eng.local_search(nprob, EN.SRC_SUBSTREAM, 7, wk, wk + 1, 4096, best, stop_ms=lb)
        torch.cuda.synchronize()
        rounds = int(eng._ws[off.value:off.value + 8].view(torch.int64).item())
        ms = EN.ls_key_fields(int(best[0].item()), bits)[0]
        rows.append((ms, rounds))
    print("cfg", cfg, "lb", lb, repr(rows), flush=True)
