"""Pin the winner IDENTITY (makespan, lowest index) of the headline exhaustive solves on the CPU.

Writes tests/golden/winners.json.  Run here (build container, 8 threads: ~1-2 min):

    python tests/golden/make_winners.py

For each solve the certificate has two independent halves, neither using the GPU:

1. the optimum VALUE M* -- the time-indexed MILP of SPEC.md:182-200 solved to optimality by HiGHS
   (``oracle.saturn_oracle.milp_optimum``; it admits every gang schedule, so M* lower-bounds every
   list-scheduled candidate);
2. the lowest index reaching it -- ``oracle/oracle.c`` (the literal per-GPU-id list scheduler,
   OpenMP) scans the candidate index space from 0 in chunks and stops at the first chunk whose
   minimum makespan is M*; the chunk minimum's (lowest) index is the winner, and every earlier
   index was evaluated and found > M*.  This is SPEC.md:249's lexicographic tie-break.

Config 1 (BASELINE.json configs[0]) is the initial solve.  Config 2 is the introspection run of
config 1 (R = predicted / 10, rho = 30 s): this script executes it with
``simulator.simulate`` driven by these CPU certificates (the re-solve contexts are deterministic
functions of the plans), and records every re-solve's context and winner.  The GPU suite
(tests/test_winners_gpu.py) replays the same run with the engine as replanner and requires the
identical context / key sequence.
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import coracle as C                      # noqa: E402
from oracle import saturn_oracle as O                # noqa: E402
from paper_2311_02840_b200 import domain as D        # noqa: E402
from paper_2311_02840_b200 import simulator as SIM   # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402

CHUNK = 1 << 23


def certify(op, threads=0, log=print):
    """(M*, lowest index with makespan M*, scanned, milp seconds, scan seconds)."""
    t0 = time.perf_counter()
    m_star = O.milp_optimum(op, time_limit=600.0)
    t_milp = time.perf_counter() - t0
    cp = C.CProblem(op)
    t0 = time.perf_counter()
    lo = 0
    while lo < op.space:
        hi = min(op.space, lo + CHUNK)
        ms, idx = cp.search("index", 0, lo, hi, threads)
        assert ms >= m_star, (ms, m_star, idx)      # a candidate below the MILP optimum cannot exist
        if ms == m_star:
            break
        lo = hi
    else:
        raise RuntimeError(f"no candidate reaches the MILP optimum {m_star} (list scheduling gap)")
    t_scan = time.perf_counter() - t0
    log(f"  M* = {m_star} (HiGHS {t_milp:.1f} s), lowest index {idx} of {op.space} "
        f"(scanned {hi} in {t_scan:.1f} s)")
    return int(m_star), int(idx), int(hi), t_milp, t_scan


def plan_from_key(op, index):
    opts, order = O.decode_index(op, index)
    ms, starts, nodes = O.list_schedule(op, opts, order, record=True)
    entries = {}
    for j, jid in enumerate(op.job_ids):
        tech, g = op.options[j][opts[j]]
        entries[jid] = D.PlanEntry(D.RunConfig(tech, g), op.node_ids[nodes[j]], starts[j] * op.delta)
    return D.Plan(entries, ms * op.delta)


def main():
    w, t, _ = config_workload(1)
    out = {"_doc": __doc__.strip().splitlines()[0], "chunk": CHUNK}
    print("config 1:")
    op = O.build(t.entries, w)
    m, idx, scanned, tm, ts = certify(op)
    out["cfg1"] = {"makespan": m, "index": idx, "space": op.space, "scanned": scanned,
                   "milp_s": round(tm, 2), "scan_s": round(ts, 2)}

    solves = []

    def record(ctx, op_, key, scanned_):
        solves.append({"remaining": dict(sorted(ctx.remaining.items())) if ctx else None,
                       "current": {k: list(v) for k, v in sorted(ctx.current.items())} if ctx else None,
                       "space": op_.space, "makespan": key[0], "index": key[1], "scanned": scanned_})

    def replan(table, workload, ctx):
        print(f"re-solve {len(solves)}: {len(ctx.remaining)} jobs")
        op_ = O.build(table.entries, workload, context=(dict(ctx.remaining), dict(ctx.current),
                                                         ctx.checkpoint_cost))
        m_, i_, sc, _, _ = certify(op_)
        record(ctx, op_, (m_, i_), sc)
        return plan_from_key(op_, i_)

    record(None, op, (m, idx), scanned)
    p0 = plan_from_key(op, idx)
    rep = SIM.simulate(w, t, p0, SIM.SimOptions(introspection_interval=p0.predicted_makespan / 10,
                                                checkpoint_overhead=30.0, replanner=replan))
    out["cfg2"] = {"interval_s": p0.predicted_makespan / 10, "checkpoint_s": 30.0, "solves": solves,
                   "makespan_s": rep.makespan.hex(), "replans": rep.replan_count,
                   "checkpoints": rep.checkpoint_count}
    with open(os.path.join(HERE, "winners.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")
    print(f"wrote winners.json: cfg1 {out['cfg1']['makespan']}@{out['cfg1']['index']}, "
          f"cfg2 {len(solves)} solves, executed makespan {rep.makespan}")


if __name__ == "__main__":
    main()
