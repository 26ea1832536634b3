"""Per-rank device time of the sharded cfg1 full scan / bound-and-prune, one rank at a time
on one GPU: what each rank's kernel takes on its own B200 at N = 1, 2, 4, 8 (the NCCL
all-reduce of one 8-byte key is not included).  Prints, per world size and lane-prefix
length, the max and mean rank time; max over ranks is the job's device time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_02840_b200 import engine as EN  # noqa: E402
from paper_2311_02840_b200.problem import build_problem  # noqa: E402
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table  # noqa: E402
from paper_2311_02840_b200.workloads import synthetic_workload  # noqa: E402

w = synthetic_workload(8, 1, 8)
t = build_profile_table(w, SyntheticExecutor(w.cluster))
prob = build_problem(t, w)
eng = EN.Engine(0)
idx_bits, _ = prob.key_bits(prob.space)
nprob = EN.NativeProblem(prob, idx_bits)
stream = torch.cuda.current_stream()


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


keys = set()
modes = sys.argv[1:] or ["tree"]
for mode in modes:
    for world in (1, 2, 4, 8):
        if mode == "tree":
            default = eng.full_scan_prefix(nprob, world) or eng.tree_plan(nprob).prefix_len
        else:
            default = eng.bnb_prefix(nprob, 1 << 15)
        for P in sorted({4, 5, 6, default}):
            info = eng.tree_plan(nprob, P)
            ms = []
            best_all = []
            for r in range(world):
                a, b = eng.tree_shard(nprob, P, r, world)
                best = eng.reset_best()
                if mode == "tree":
                    ms.append(timed(lambda: eng.search_tree(nprob, P, a, b, eng.reset_best(best))))
                else:
                    seed_ms = eng.seed_bound(prob)
                    def run():
                        eng.reset_best(best)
                        best[0:1].fill_((seed_ms << idx_bits) | ((1 << idx_bits) - 1))
                        eng.search_bnb(nprob, P, a, b, best)
                    ms.append(timed(run))
                best_all.append(int(best[0].item()) & ((1 << 64) - 1))
            keys.add(min(best_all))
            print(f"{mode} world={world} P={P}{' (engine)' if P == default else ''} tasks={info.n_tasks} "
                  f"max_rank_ms={max(ms):.3f} mean_rank_ms={sum(ms) / len(ms):.3f} "
                  f"plans/s={prob.space / (max(ms) / 1e3):.3e} ranks_ms={[round(x, 3) for x in ms]}", flush=True)
print("distinct combined keys:", len(keys))
