"""One small problem through every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck; one tool per run).  Checks results against the CPU oracle too, so a sanitizer run
that silently perturbed execution would also fail here.

    compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""

import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from helpers import golden_workload  # noqa: E402
from test_engine_gpu import bnb_key, gpu_key, to_search_problem, workload_problem  # noqa: E402
from test_oracle import random_problem  # noqa: E402

from oracle import coracle as C  # noqa: E402
from paper_2311_02840_b200 import engine as EN  # noqa: E402


def main():
    eng = EN.Engine(0)
    rng = random.Random(5)
    checks = 0
    # one node (tree, bnb, k_cand One16 / One), two nodes (Multi16 / Multi), float mode
    for nodes, scale in (([4], 1), ([4], 30000), ([3, 2], 1), ([4, 4], 1)):
        op = random_problem(rng, 4, nodes, max_opts=3, max_d=7, hetero=len(nodes) == 2 and nodes[0] == 3)
        op.dur = [[[d * scale for d in row] for row in job] for job in op.dur]
        op.runtime = [[list(r) for r in job] for job in op.dur]
        prob = to_search_problem(op)
        want = C.CProblem(op).search()
        assert gpu_key(eng, prob, "index") == want
        if len(nodes) == 1:
            assert gpu_key(eng, prob, "tree") == want
            assert bnb_key(eng, prob) == want
        got = gpu_key(eng, prob, "sampled", 0, 500, source=EN.SRC_SUBSTREAM, seed=3, n_idx=500)
        assert got == C.CProblem(op).search("substream", 3, 0, 500)
        got = gpu_key(eng, prob, "sampled", 0, 500, source=EN.SRC_SEED, seed=3, n_idx=500)
        assert got == C.CProblem(op).search("seed", 3, 0, 500)
        checks += 4
    w, t, prob, op = workload_problem("small5_1x4", time_mode="float")
    n = min(prob.space, 20000)
    got = gpu_key(eng, prob, "index", 0, n)
    assert got[1] == C.CProblem(op).search(hi=n)[1]
    # recorded schedules (sat_schedule, k_generic)
    w, t, prob, op = workload_problem("small4_2x2")
    nprob = EN.NativeProblem(prob, 62)
    opt, node, start, ms = eng.schedule(nprob, EN.SRC_SUBSTREAM, seed=7, ids=[0, 1, 2, 3])
    cp = C.CProblem(op)
    for r in range(4):
        o, order = cp.decode(r, "substream", 7)
        assert ms[r] == cp.eval(o, order)[0]
    print(f"sanitize_small ok: {checks + 5} checks")


if __name__ == "__main__":
    main()
