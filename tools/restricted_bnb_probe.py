"""Probe: prove the lower bound M infeasible by bound-and-prune over the slack-restricted space.

At target makespan M the slack is S = M*G - (committed + sum of every job's least area).  Any
schedule with makespan <= M uses, for each job, an option of area <= least area + S, so the
search can drop every other option; bound-and-prune seeded with M then either finds a
candidate <= M or proves there is none.  Config 3: S = 0 at M = 29 (radix 1-2 per job)."""
import dataclasses
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02840_b200 import engine as EN  # noqa: E402
from paper_2311_02840_b200.problem import build_problem  # noqa: E402
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table  # noqa: E402
from paper_2311_02840_b200.workloads import synthetic_workload  # noqa: E402


def restricted(prob, M):
    G = int(prob.node_gpus[0])
    init = prob.init_free_i32[0, :G]
    area = [[int(prob.gpus[j, o]) * int(prob.dur_i32[j, o, 0]) for o in range(prob.radix[j])] for j in range(prob.J)]
    slack = M * G - int(init.sum()) - sum(min(a) for a in area)
    keep = [[o for o in range(prob.radix[j]) if area[j][o] <= min(area[j]) + slack] for j in range(prob.J)]
    C = max(len(k) for k in keep)
    gpus = np.zeros((prob.J, C), np.int32)
    mask = np.zeros((prob.J, C), np.uint32)
    dur = np.zeros((prob.J, C, 1), np.int32)
    rt = np.zeros((prob.J, C, 1))
    for j, ks in enumerate(keep):
        for i, o in enumerate(ks):
            gpus[j, i], mask[j, i] = prob.gpus[j, o], prob.node_mask[j, o]
            dur[j, i, 0], rt[j, i, 0] = prob.dur_i32[j, o, 0], prob.runtime[j, o, 0]
    sub = dataclasses.replace(prob, radix=np.array([len(k) for k in keep], np.int32), gpus=gpus, node_mask=mask,
                              dur_i32=dur, runtime=rt, options=[[prob.options[j][o] for o in ks] for j, ks in enumerate(keep)],
                              option_src=[[prob.option_src[j][o] for o in ks] for j, ks in enumerate(keep)],
                              extra={})
    return sub, slack


J = int(sys.argv[1]) if len(sys.argv) > 1 else 16
w = synthetic_workload(J, 1, 8)
t = build_profile_table(w, SyntheticExecutor(w.cluster))
prob = build_problem(t, w)
eng = EN.Engine(0)
M = int(prob.lower_bound())
for target in (M, M + 1):
    sub, slack = restricted(prob, target)
    bits, _ = sub.key_bits(sub.space)
    nprob = EN.NativeProblem(sub, bits)
    P = int(os.environ.get("PREFIX", "0")) or eng.bnb_prefix(nprob, 1 << 15)
    info = eng.tree_plan(nprob, P)
    best = eng.reset_best()
    seed_key = (target << bits) | ((1 << bits) - 1)
    best[0:1].fill_(seed_key)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ws = eng.search_bnb(nprob, info.prefix_len, 0, info.n_tasks, best)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    k = int(best[0].item()) & ((1 << 64) - 1)
    found = k != seed_key
    cnt = ws[:24].view(torch.int64).cpu().tolist()
    print(f"J={J} target={target} slack={slack} radix={sub.radix.tolist()} space={sub.space:.3e} P={P} "
          f"tasks={info.n_tasks} -> {'FOUND makespan %d' % (k >> bits) if found else 'none: infeasible'} "
          f"in {dt * 1e3:.1f} ms (pruned tasks {cnt[1]}, pair nodes {cnt[2]})", flush=True)
