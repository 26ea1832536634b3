"""Sampled-search throughput of the per-candidate kernel (k_cand) per config -- device time of
2^26 candidates of substream(7, i), best of 3 -- plus a bit-exactness check of a 4096-candidate
window against the C oracle.  python tools/sampled_rate.py [configs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import coracle as C  # noqa: E402
from oracle import saturn_oracle as O  # noqa: E402
from paper_2311_02840_b200 import engine as EN  # noqa: E402
from paper_2311_02840_b200.problem import SolveOptions, build_problem  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

eng = EN.Engine(0)
for cfg in [int(x) for x in (sys.argv[1:] or ["3", "4", "5"])]:
    w, t, _ = config_workload(cfg)
    prob = build_problem(t, w, SolveOptions())
    n = 1 << 26
    bits, _ = prob.key_bits(n)
    nprob = EN.NativeProblem(prob, bits)
    times = []
    for _ in range(4):
        best = eng.reset_best()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.search_sampled(nprob, EN.SRC_SUBSTREAM, 7, 0, n, best)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    dt = min(times[1:])
    best = eng.reset_best()
    eng.search_sampled(nprob, EN.SRC_SUBSTREAM, 7, 1000, 5096, best)
    k = int(best[0].item())
    got = (float(k >> bits), k & ((1 << bits) - 1))
    want = C.CProblem(O.build(t.entries, w)).search("substream", 7, 1000, 5096)
    ops = prob.J * (prob.N + 2 * prob.G + 2)
    print(f"cfg{cfg}: {n / dt:.3e} plans/s ({1e3 * dt:.2f} ms), 8(d) ops {n * ops / dt / 1e12:.2f} TOP/s, "
          f"window key {'==' if got == want else '!='} oracle", flush=True)
