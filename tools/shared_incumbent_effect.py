"""Work saved by the cross-rank shared incumbent (engine.SharedIncumbent), measured on ONE GPU:
W ranks (separate processes, gloo, all on cuda:0 -- a functional setting, so device times are
not multi-GPU numbers) run the same sharded solve with and without the shared cell, and report
the work every rank did: bound-and-prune pair nodes scheduled and tasks cut (cfg1 and a 10-job
one-node problem), local-search rounds (cfg4, cfg5).  Same keys either way.

    python tools/shared_incumbent_effect.py [world]
"""
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch.multiprocessing as mp  # noqa: E402

CASES = [("cfg1", {}), ("j10", {}), ("cfg4", {}), ("cfg5", {})]


def _worker(rank, world, port, share, q):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paper_2311_02840_b200 import planners as PL
    from paper_2311_02840_b200.problem import SolveOptions
    from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table
    from paper_2311_02840_b200.workloads import config_workload, synthetic_workload

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    out = []
    for name, kw in CASES:
        if name == "j10":
            w = synthetic_workload(10, 1, 8)
            t = build_profile_table(w, SyntheticExecutor(w.cluster))
        else:
            w, t, _ = config_workload(int(name[3:]))
        opts = SolveOptions(share_incumbent=share, **kw)
        PL.solve(t, w, None, opts)                        # warm-up
        sol = PL.solve(t, w, None, opts)
        st = dict(sol.search.stats or {})
        out.append((name, sol.search.kernel, sol.makespan, sol.search.index,
                    st.get("pair_nodes"), st.get("pruned_tasks"), st.get("rounds"), sol.search.device_seconds))
    q.put((rank, out))
    dist.destroy_process_group()


def run(world, share):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ps = [ctx.Process(target=_worker, args=(r, world, port, share, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=900) for _ in range(world))
    for p in ps:
        p.join(60)
    return got


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    res = {share: run(world, share) for share in (False, True)}
    for i, (name, _) in enumerate(CASES):
        rows = {share: [res[share][r][i] for r in range(world)] for share in (False, True)}
        keys = {share: (rows[share][0][2], rows[share][0][3]) for share in rows}
        assert keys[False] == keys[True], (name, keys)
        kern = rows[True][0][1]
        if kern == "bnb":
            a = [r[4] for r in rows[False]], [r[4] for r in rows[True]]
            print(f"{name} ({kern}, world {world}): pair nodes per rank {a[0]} -> {a[1]} "
                  f"(total {sum(a[0])} -> {sum(a[1])}); same key {keys[True]}")
        else:
            a = [r[6] for r in rows[False]], [r[6] for r in rows[True]]
            print(f"{name} ({kern}, world {world}): local-search rounds per rank {a[0]} -> {a[1]} "
                  f"(total {sum(a[0])} -> {sum(a[1])}); same key {keys[True]}")
