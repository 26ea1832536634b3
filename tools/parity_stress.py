"""Extended parity sweep on one GPU (beyond the pytest suite's fixed trials): random one-node
problems through the tree kernel (packed and 32-bit pair pass, every lane-prefix length) and
bound-and-prune, random 1-4-node problems through the index kernel and the sampled stream,
local-search walkers (1 / 4 / 8 / 16 / 32 warps per walker), and the state-space search (one node:
INFEASIBLE at the oracle optimum - 1, FEASIBLE at it with a candidate the oracle replays within the
target; several nodes: the prover never calls a reachable target infeasible) -- every key compared
with the CPU oracle.  Prints one summary line per family; any mismatch raises."""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import coracle as C  # noqa: E402
from paper_2311_02840_b200 import engine as EN  # noqa: E402
from test_engine_gpu import bnb_key, gpu_key, to_search_problem  # noqa: E402
from test_oracle import random_problem  # noqa: E402

N_TRIALS = int(os.environ.get("STRESS_TRIALS", "150"))
eng = EN.Engine(0)
rng = random.Random(int(os.environ.get("STRESS_SEED", "2026")))

t0, checks = time.time(), 0
for trial in range(N_TRIALS):
    gsz = rng.choice([2, 3, 4, 5, 6, 7, 8, 10, 12, 16, 20, 32])
    J = rng.randint(3, 7)
    op = random_problem(rng, J, [gsz], max_opts=4 if J < 6 else 3, max_d=rng.choice([5, 12, 40]))
    if trial % 3 == 0:
        op.init_free = [sorted(rng.randint(0, 6) for _ in range(gsz))]
    prob = to_search_problem(op)
    want = C.CProblem(op).search()
    for packed in ("1", "0"):
        os.environ["SATURN_TREE_PACKED"] = packed
        for P in range(1, J - 1):
            got = gpu_key(eng, prob, "tree", prefix=P)
            assert got == want, ("tree", trial, packed, P, got, want)
            checks += 1
        got = bnb_key(eng, prob)
        assert got == want, ("bnb", trial, packed, got, want)
        checks += 1
os.environ.pop("SATURN_TREE_PACKED", None)
print(f"tree + bnb: {N_TRIALS} random one-node problems, {checks} keys equal the oracle ({time.time() - t0:.0f} s)",
      flush=True)

t0, checks = time.time(), 0
for trial in range(N_TRIALS):
    nodes = [[rng.randint(1, 8)], [rng.randint(1, 4), rng.randint(1, 4)], [2, 3, 1],
             [rng.randint(1, 8) for _ in range(4)]][trial % 4]
    op = random_problem(rng, rng.randint(1, 5), nodes, max_opts=4, max_d=9, hetero=trial % 3 == 0)
    if trial % 2:
        op.release = [rng.randint(0, 5) for _ in range(op.J)]
        op.init_free = [[rng.randint(0, 6) for _ in range(n)] for n in nodes]
    prob = to_search_problem(op)
    cp = C.CProblem(op)
    assert gpu_key(eng, prob, "index") == cp.search(), ("index", trial)
    n = 5000
    got = gpu_key(eng, prob, "sampled", 0, n, source=EN.SRC_SUBSTREAM, seed=trial, n_idx=n)
    assert got == cp.search("substream", trial, 0, n), ("sampled", trial)
    checks += 2
print(f"index + sampled: {N_TRIALS} random 1-4-node problems (releases, initial free times, heterogeneous), "
      f"{checks} keys equal the oracle ({time.time() - t0:.0f} s)", flush=True)

t0, checks = time.time(), 0
for trial in range(max(8, N_TRIALS // 5)):
    nodes = [[rng.choice([4, 8, 12, 16, 24, 32])], [rng.randint(2, 4), rng.randint(2, 4)]][trial % 2]
    op = random_problem(rng, rng.randint(4, 9), nodes, max_opts=4, max_d=9)
    if trial % 3 == 1:
        op.release = [rng.randint(0, 4) for _ in range(op.J)]
        op.init_free = [[rng.randint(0, 3) for _ in range(n)] for n in nodes]
    prob = to_search_problem(op)
    bits, _ = prob.key_bits(1 << 10)
    nprob = EN.NativeProblem(prob, bits)
    cp = C.CProblem(op)
    stop = int(prob.lower_bound()) if trial % 2 else -1
    for group in ("1", "4", "8", "16", "32"):
        os.environ["SATURN_LS_GROUP"] = group
        for walker in (0, 7):
            _, o, r, _ = cp.local_search(walker, "substream", trial, 4096, stop_ms=stop)
            got = eng.local_search_state(nprob, EN.SRC_SUBSTREAM, trial, walker, 4096, stop_ms=stop)
            assert got == (o, r), ("ls", trial, group, walker)
            checks += 1
os.environ.pop("SATURN_LS_GROUP", None)
print(f"local search: {checks} walks (1 / 4 / 8 / 16 / 32 warps per walker, with and without the stop) equal the oracle "
      f"({time.time() - t0:.0f} s)", flush=True)

t0, checks, proven = time.time(), 0, 0
for trial in range(N_TRIALS):
    if trial % 2 == 0:
        gsz = rng.choice([1, 2, 3, 4, 6, 8, 12, 16])
        op = random_problem(rng, rng.randint(2, 6), [gsz], max_opts=3, max_d=rng.choice([6, 12]))
        if trial % 3 == 0:
            op.init_free = [sorted(rng.randint(0, 5) for _ in range(gsz))]
        if trial % 5 == 1:
            op.release = [rng.randint(0, 6) for _ in range(op.J)]
        prob = to_search_problem(op)
        cp = C.CProblem(op)
        opt = int(cp.search()[0])
        nprob = EN.NativeProblem(prob, 1)
        st, _, _ = eng.dp_search(nprob, opt - 1, 1 << 20)
        assert st == EN.SAT_DP_INFEASIBLE, ("dp", trial, opt)
        st, info, cand = eng.dp_search(nprob, opt, 1 << 20)
        assert st == EN.SAT_DP_FEASIBLE and cand is not None, ("dp", trial, opt)
        assert cp.eval(*cand)[0] <= opt, ("dp replay", trial)
        checks += 2
    else:
        nodes = [[2, 2], [4, 4], [3, 2], [2, 2, 2], [4, 2, 1], [4, 4, 4], [4, 4, 4, 4], [8, 8]][trial % 8]
        op = random_problem(rng, rng.randint(2, 5), nodes, max_opts=3, max_d=8, hetero=trial % 3 == 0)
        if trial % 4 == 1:
            op.release = [rng.randint(0, 4) for _ in range(op.J)]
        prob = to_search_problem(op)
        opt = int(C.CProblem(op).search()[0])
        nprob = EN.NativeProblem(prob, 1)
        for target in (opt - 1, opt):
            st, _, _ = eng.dp_search(nprob, target, 1 << 20)
            assert st != EN.SAT_DP_BUDGET
            assert st == EN.SAT_DP_FEASIBLE or target < opt, ("prover", trial, target, opt)
            checks += 1
            proven += target == opt - 1 and st == EN.SAT_DP_INFEASIBLE
        # exact states (SAT_DP_EXACT): infeasible at opt - 1, a candidate reaching opt
        st, _, _ = eng.dp_search(nprob, opt - 1, 1 << 20, exact=True)
        assert st == EN.SAT_DP_INFEASIBLE, ("exact", trial, opt)
        st, info, cand = eng.dp_search(nprob, opt, 1 << 20, exact=True)
        assert st == EN.SAT_DP_FEASIBLE and cand is not None, ("exact", trial, opt)
        assert C.CProblem(op).eval(*cand)[0] == info.makespan <= opt, ("exact replay", trial)
        checks += 2
print(f"state-space search: {N_TRIALS} random problems (1-16-GPU nodes and 2-3-node clusters, releases, initial "
      f"free times), {checks} answers consistent with the oracle optimum; multi-node optimum proven on "
      f"{proven} of {N_TRIALS // 2} by the prover and on every one by exact states, each with a candidate "
      f"the oracle replays ({time.time() - t0:.0f} s)", flush=True)
