"""Where a local-search walk's time goes (library built with -DSAT_LS_PROFILE, see
tools/build_variant.sh): per config, one walker alone and the default first wave -- steps,
improving steps, cycles evaluating moves (incl. the group barrier) vs applying moves, and the
mean position of the improving round inside its step.

    SATURN_ENGINE_LIB=.../lsprof.so python tools/ls_profile.py [configs]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import engine as EN  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions, build_problem  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

eng = EN.Engine(0)
for cfg in [int(x) for x in (sys.argv[1:] or ["3", "4", "5"])]:
    w, t, _ = config_workload(cfg)
    prob = build_problem(t, w, SolveOptions())
    lb = int(prob.lower_bound())
    bits, _ = prob.key_bits(1 << 20)
    nprob = EN.NativeProblem(prob, bits)
    off = ctypes.c_size_t()
    eng.lib.sat_ls_counter_offset(nprob.ref, ctypes.byref(off))
    for lo, hi in ((18, 19), (33, 34), (0, 16384)):
        best = eng.reset_best()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.local_search(nprob, EN.SRC_SUBSTREAM, 7, lo, hi, 4096, best, stop_ms=lb)
        e1.record()
        torch.cuda.synchronize()
        c = eng._ws[off.value:off.value + 48].view(torch.int64).cpu().tolist()
        rounds, steps, imp, ev, ap, pos = c
        print(f"cfg{cfg} walkers [{lo},{hi}) dev_ms={e0.elapsed_time(e1):.2f} rounds={rounds} steps={steps} "
              f"improving={imp} eval_cyc/step={ev / max(1, steps):.0f} apply_cyc/improving={ap / max(1, imp):.0f} "
              f"mean_improving_round={pos / max(1, imp):.2f} best={EN.ls_key_fields(int(best[0].item()), bits)[0]}", flush=True)
