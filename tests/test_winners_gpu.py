"""Winner identity on the headline exhaustive configs, against CPU certificates.

tests/golden/winners.json (tests/golden/make_winners.py) holds, for config 1 and for every
solve of config 2's introspection run, the optimum makespan proven by HiGHS and the lowest
candidate index reaching it found by the C oracle scanning the index space from 0 (SPEC.md:249
tie-break).  Every exact GPU search must return exactly that key."""

import json
import os

import pytest

from paper_2311_02840_b200 import domain as D
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200 import simulator as SIM
from paper_2311_02840_b200.problem import SolveOptions
from paper_2311_02840_b200.workloads import config_workload

pytestmark = pytest.mark.gpu

WIN = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "winners.json")))


@pytest.mark.parametrize("kernel", ["tree", "bnb", "index"])
def test_cfg1_winner_identity(kernel):
    """Full scan (k_tree), bound-and-prune and the per-candidate index kernel (k_cand over all
    3.25e10 candidates) all return the certified (30, lowest index)."""
    w, t, _ = config_workload(1)
    sol = PL.solve(t, w, None, SolveOptions(kernel=kernel))
    want = WIN["cfg1"]
    assert sol.search.kernel == kernel and sol.status == "Optimal"
    assert (sol.makespan, sol.search.index) == (want["makespan"], want["index"])
    if kernel != "bnb":
        assert sol.search.evaluated == want["space"]
    else:
        # the seed bound is the optimum, so every task is cut against 30 from the start: the
        # counters are deterministic (and must survive the winner replay queued behind the search)
        assert (sol.search.stats["pruned_tasks"], sol.search.stats["pair_nodes"]) == (44920, 35858)


@pytest.mark.parametrize("kernel", ["auto", "tree"])
def test_cfg2_introspection_resolves_identity(kernel):
    """Config 2: the introspection run with engine re-solves makes the certified decision at
    every tick (same context, same winner key) and executes to the same makespan, bit for bit."""
    w, t, _ = config_workload(1)
    opts = SolveOptions(kernel=kernel)
    seen = []

    def replan(table, workload, ctx):
        sol = PL.solve(table, workload, None, opts, ctx)
        seen.append((ctx, sol))
        return sol.plan

    s0 = PL.solve(t, w, None, opts)
    rep = SIM.simulate(w, t, s0.plan, SIM.SimOptions(introspection_interval=s0.plan.predicted_makespan / 10,
                                                     checkpoint_overhead=30.0, replanner=replan))
    want = WIN["cfg2"]
    assert s0.plan.predicted_makespan / 10 == want["interval_s"]
    got = [(None, s0)] + seen
    assert len(got) == len(want["solves"])
    for (ctx, sol), rec in zip(got, want["solves"]):
        if ctx is not None:
            assert dict(sorted(ctx.remaining.items())) == rec["remaining"]
            assert {k: list(v) for k, v in sorted(ctx.current.items())} == rec["current"]
        assert sol.status == "Optimal"
        assert (sol.makespan, sol.search.index) == (rec["makespan"], rec["index"])
    assert rep.makespan.hex() == want["makespan_s"]
    assert (rep.replan_count, rep.checkpoint_count) == (want["replans"], want["checkpoints"])
