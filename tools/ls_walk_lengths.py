"""Walk lengths of the first local-search walkers (configs 4 / 5, stop at the lower bound):
rounds of 32 moves each walker scans, its final makespan, and single-walker device time --
the critical path of a local-search wave is the longest walk below the winning walker id."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import engine as EN  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions, build_problem  # noqa: E402
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table  # noqa: E402
from paper_2311_02840_b200.workloads import TECHNIQUES_4, TECHNIQUES_6, synthetic_workload  # noqa: E402

SHAPES = {3: (16, 1, 8, TECHNIQUES_4), 4: (32, 4, 8, TECHNIQUES_4), 5: (64, 1, 32, TECHNIQUES_6)}
eng = EN.Engine(0)
for cfg in [int(x) for x in (sys.argv[1:] or ["4", "5"])]:
    J, N, G, T = SHAPES[cfg]
    w = synthetic_workload(J, N, G, T)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w, SolveOptions())
    lb = int(prob.lower_bound())
    res = eng.search(prob, SolveOptions(search="local"))
    bits, _ = prob.key_bits(1 << 20)
    nprob = EN.NativeProblem(prob, bits)
    off = ctypes.c_size_t()
    eng.lib.sat_ls_counter_offset(nprob.ref, ctypes.byref(off))
    rows = []
    for wk in range(48):
        best = eng.reset_best()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.local_search(nprob, EN.SRC_SUBSTREAM, 7, wk, wk + 1, 4096, best, stop_ms=lb)
        e1.record()
        torch.cuda.synchronize()
        rounds = int(eng._ws[off.value:off.value + 8].view(torch.int64).item())
        ms = EN.ls_key_fields(int(best[0].item()), bits)[0]
        rows.append((wk, ms, rounds, e0.elapsed_time(e1)))
    print(f"cfg{cfg} lb={lb} winner={res.index} ms={res.makespan} dev_ms={1e3 * res.search.device_seconds if hasattr(res, 'search') else res.device_seconds:.2f}")
    for r in rows:
        print(f"  walker {r[0]:3d} final={r[1]:3d} rounds={r[2]:5d} dev_ms={r[3]:.2f} us/round={1e3 * r[3] / max(1, r[2]):.2f}")
