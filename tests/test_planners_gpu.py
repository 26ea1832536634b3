"""End-to-end planners on the GPU engine: reference-facing API, plan validity, SPEC examples."""

import math

import numpy as np
import pytest

from helpers import golden, golden_workload, import_reference, reference_available

from oracle import coracle as C
from oracle import saturn_oracle as O
import paper_2311_02840_b200 as S
from paper_2311_02840_b200 import domain as D
from paper_2311_02840_b200 import engine as EN
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200.problem import SolveOptions
from paper_2311_02840_b200.profiling import ProfileTable, SyntheticExecutor, build_profile_table

pytestmark = pytest.mark.gpu


def setup(name):
    w, _ = golden_workload(name)
    return w, build_profile_table(w, SyntheticExecutor(w.cluster))


def test_plan_saturn_cfg1_optimal_and_valid():
    w, t = setup("cfg1")
    sol = PL.solve(t, w, None, SolveOptions(kernel="tree"))
    assert sol.status == "Optimal"
    assert sol.makespan == 30 == golden()["milp"]["cfg1"]["optimum_intervals"]
    assert sol.search.kernel == "tree" and sol.search.evaluated == 32514048000
    default = PL.solve(t, w)                                   # auto = bound-and-prune
    assert default.search.kernel == "bnb" and default.plan == sol.plan
    D.check_plan(sol.plan, w, sol.runtimes)
    assert math.isclose(sol.plan.predicted_makespan, 30 * sol.problem.delta)
    # the decoded plan is exactly the oracle's replay of the winning index
    op = O.build(t.entries, w)
    opts, order = O.decode_index(op, sol.search.index)
    ms, starts, nodes = C.CProblem(op).eval(opts, order)
    for j, jid in enumerate(op.job_ids):
        e = sol.plan.entries[jid]
        assert (e.config.technique, e.config.gpus) == op.options[j][opts[j]]
        assert e.start_time == starts[j] * op.delta


def test_spec_two_job_example():
    """SPEC.md:199/283/292/373: Saturn makespan 10, Current Practice 12, Optimus 10."""
    techs = (D.TechniqueSpec(name="t", archetype="sharded", serial_fraction=0.0, comm_overhead=0.0),)
    jobs = (D.JobSpec("a", 1, 1.0, 1.0), D.JobSpec("b", 1, 1.0, 1.0))
    cl = D.ClusterSpec((D.NodeSpec("n", 2, 80.0),))
    w = D.Workload(jobs, cl, techs)
    t = ProfileTable({("a", "t", 1): 10.0, ("a", "t", 2): 6.0, ("b", "t", 1): 10.0, ("b", "t", 2): 6.0}, "ingested")
    opts = SolveOptions(delta=1.0, k_max=1000)
    sat = S.plan_saturn(t, w, None, opts)
    assert sat.predicted_makespan == 10.0
    assert all(e.config.gpus == 1 and e.start_time == 0 for e in sat.entries.values())
    cp = S.plan_current_practice(t, w, None, opts)
    assert cp.predicted_makespan == 12.0
    opt = S.plan_optimus(t, w, None, opts)
    assert opt.predicted_makespan == 10.0
    # one job -> its best config at t=0
    w1 = D.Workload(jobs[:1], cl, techs)
    p1 = S.plan_saturn(t, w1, None, opts)
    assert p1.entries["a"].config.gpus == 2 and p1.entries["a"].start_time == 0.0


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5"])
def test_sampled_saturn_and_baselines(name):
    w, t = setup(name)
    sol = PL.solve(t, w, None, SolveOptions(search="sampled", budget=200000))
    assert sol.status in ("Sampled", "Optimal") and sol.makespan <= sol.search.makespan
    D.check_plan(sol.plan, w, sol.runtimes)
    opt = PL._explicit_solution(t, w, SolveOptions(), None, PL.optimus_allocation, None)
    cp = PL._explicit_solution(t, w, SolveOptions(), None, PL.current_practice_allocation, None)
    for s in (opt, cp):
        D.check_plan(s.plan, w, s.runtimes)
    rnd = S.plan_random(t, w, None, seed=7)
    assert set(rnd.entries) == {j.id for j in w.jobs}
    # the baselines' allocations equal the oracle's restatement
    op = O.build(t.entries, w, prune=False)
    assert PL.optimus_allocation(opt.problem) == tuple(O.optimus(op))
    assert PL.current_practice_allocation(cp.problem) == tuple(O.current_practice(op))
    # and their engine makespans equal the oracle's list schedule
    cpo = C.CProblem(op)
    assert opt.makespan == cpo.eval(*O.optimus(op))[0]
    assert cp.makespan == cpo.eval(*O.current_practice(op))[0]


def test_plan_random_matches_oracle_draws():
    w, t = setup("cfg3")
    op = O.build(t.entries, w, prune=False)
    for seed in (0, 7, 2**63 + 1):
        plan = S.plan_random(t, w, None, seed=seed)
        opts, order = O.candidate(op, "seed", seed, 0)
        ms, starts, nodes = C.CProblem(op).eval(opts, order)
        assert math.isclose(plan.predicted_makespan, ms * op.delta)
        for j, jid in enumerate(op.job_ids):
            assert (plan.entries[jid].config.technique, plan.entries[jid].config.gpus) == op.options[j][opts[j]]
    best = PL.plan_random_best(t, w, None, seed0=100, n_seeds=50000)
    want = C.CProblem(op).search("seed", 100, 0, 50000)
    assert (best.makespan, best.search.index) == want


def test_resolve_runs_and_keeps_running_job_cheaper():
    w, t = setup("cfg1")
    first = PL.solve(t, w)
    # five unfinished jobs keep the oracle's exhaustive check to seconds
    remaining = {j.id: j.total_batches // 2 for j in w.jobs[:5]}
    running = {jid: (e.config.technique, e.config.gpus, e.node)
               for jid, e in first.plan.entries.items() if e.start_time == 0.0 and jid in remaining}
    ctx = D.RunningContext(remaining=remaining, current=running, checkpoint_cost=30.0)
    sol = PL.solve(t, w, None, None, ctx)
    assert sol.status == "Optimal" and set(sol.plan.entries) == set(remaining)
    op = O.build(t.entries, w, context=(remaining, running, 30.0))
    assert sol.makespan == C.CProblem(op).search()[0]


def test_distinct_time_modes_agree_on_valid_plans():
    w, t = setup("small5_1x4")
    g = PL.solve(t, w, None, SolveOptions(time_mode="grid"))
    f = PL.solve(t, w, None, SolveOptions(time_mode="float"))
    D.check_plan(f.plan, w, f.runtimes)
    # float optimum never exceeds the grid optimum (grid rounds durations up)
    assert f.plan.predicted_makespan <= g.plan.predicted_makespan + 1e-9


@pytest.mark.skipif(not reference_available(), reason="reference package not present (GPU box)")
def test_drop_in_with_reference_objects():
    core, profiling, rng = import_reference()
    w, _ = golden_workload("small5_1x4")
    rw = core.Workload.model_validate({"jobs": [j.__dict__ for j in w.jobs],
                                       "cluster": {"nodes": [n.__dict__ for n in w.cluster.nodes]},
                                       "techniques": [t.__dict__ for t in w.techniques]})
    rt = profiling.build_profile_table(rw, profiling.SyntheticExecutor(rw.cluster))
    plan = S.plan_saturn(rt, rw)
    assert type(plan) is core.Plan
    runtimes = {}
    for jid, e in plan.entries.items():
        runtimes[jid] = profiling.estimate_runtime(rt, rw.job(jid), e.config, rw.job(jid).total_batches)
    core.check_plan(plan, rw, runtimes)


def test_plan_saturn_bnb_equals_exhaustive():
    for name in ("cfg1", "small5_1x4"):
        w, t = setup(name)
        ex = PL.solve(t, w)
        bb = PL.solve(t, w, None, SolveOptions(kernel="bnb"))
        assert bb.search.kernel == "bnb" and bb.status == "Optimal"
        assert (bb.makespan, bb.search.index) == (ex.makespan, ex.search.index)
        assert bb.plan == ex.plan
        assert bb.search.stats["pair_nodes"] > 0


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_local_search_plan_beats_its_own_starts(name):
    """search="local" from sampled starts: each walker ends at or below its start, so the best
    walker is at least as good as sampling the same candidates; the decoded plan is valid and
    replays to the key.  The default greedy starts do at least as well here."""
    w, t = setup(name)
    n = 2048
    loc = PL.solve(t, w, None, SolveOptions(search="local", walkers=n, ls_start="sampled"))
    gre = PL.solve(t, w, None, SolveOptions(search="local", walkers=n))
    assert gre.search.source == EN.SRC_GREEDY and gre.makespan <= loc.makespan
    D.check_plan(gre.plan, w, gre.runtimes)
    smp = PL.solve(t, w, None, SolveOptions(search="sampled", budget=n))
    assert loc.status in ("Local", "Optimal") and loc.makespan <= smp.makespan
    assert loc.lower_bound <= loc.makespan
    assert (loc.status == "Optimal") == (loc.makespan == loc.lower_bound)
    D.check_plan(loc.plan, w, loc.runtimes)


def test_default_solve_of_large_configs_is_local_and_bounded():
    """auto on spaces beyond exact search = local search; cfg4 / cfg5 meet the lower bound
    (proven optimal); cfg3 reaches the HiGHS-certified optimum, one above the bound, and the
    state-space search proves it (status Optimal)."""
    for name, by_dp in (("cfg3", True), ("cfg4", False), ("cfg5", False)):
        w, t = setup(name)
        sol = PL.solve(t, w)
        assert sol.search.kernel == "local"
        D.check_plan(sol.plan, w, sol.runtimes)
        assert sol.status == "Optimal" and sol.makespan == sol.lower_bound
        assert sol.search.proven == by_dp
        if by_dp:
            assert sol.makespan == golden()["milp"][name]["optimum_intervals"]
            assert sol.makespan == sol.problem.lower_bound() + 1


def test_evaluate_fixed_reproduces_planner_plans():
    w, t = setup("cfg1")
    sol = PL.solve(t, w)
    fixed = PL.evaluate_fixed(t, w, sol.options, sol.order, prune=True)
    assert fixed.plan == sol.plan and fixed.makespan == sol.makespan
    prob = PL._baseline_problem(t, w, SolveOptions())
    options, order = PL.optimus_allocation(prob)
    assert PL.evaluate_fixed(t, w, options, order).plan == PL.plan_optimus(t, w)


def test_bnb_beyond_the_worst_case_key_width():
    """A 12-job one-node mirror (space 3.9e16): the worst-case makespan bound would not fit the
    packed key next to the index, the seed bound does -- exact bound-and-prune when asked for."""
    from paper_2311_02840_b200.workloads import generate_workload

    w = generate_workload("wikitext_mirror", 1, 7)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    exact = PL.solve(t, w, None, SolveOptions(kernel="bnb", max_bnb=1 << 60))
    assert exact.search.kernel == "bnb" and exact.status == "Optimal"
    local = PL.solve(t, w)                                  # default: local search for this size
    assert exact.makespan <= local.makespan
    assert exact.lower_bound == exact.makespan


@pytest.mark.parametrize("shape", [(1, [1]), (1, [8]), (2, [2]), (3, [8, 4, 2]), (5, [8, 4, 2]),
                                   (4, [1, 1, 1, 1]), (3, [32]), (6, [4, 4])])
def test_public_api_edge_shapes(shape):
    """plan_saturn on unusual shapes (single job, single GPU nodes, mixed node sizes, a 32-GPU
    node): a valid plan whose makespan is the oracle's exhaustive optimum."""
    from paper_2311_02840_b200.workloads import TECHNIQUES_4

    n_jobs, sizes = shape
    jobs = tuple(D.JobSpec(f"j{j}", 100 * (1 + j), 1.0 + 0.3 * j, 10.0 + 25.0 * (j % 2), 2.0) for j in range(n_jobs))
    nodes = tuple(D.NodeSpec(f"n{i}", g, 40.0) for i, g in enumerate(sizes))
    w = D.Workload(jobs, D.ClusterSpec(nodes), TECHNIQUES_4)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    sol = PL.solve(t, w)
    D.check_plan(sol.plan, w, sol.runtimes)
    op = O.build(t.entries, w)
    if op.space <= 3_000_000:
        assert sol.makespan == C.CProblem(op).search()[0], (shape, sol.search.kernel)
    assert sol.lower_bound <= sol.makespan


@pytest.mark.parametrize("cfg", [3, 4])
def test_batched_replay_equals_single_replays(cfg):
    """The winner and the Optimus / current-practice incumbents replay in one sat_schedule
    launch: each row of the batch equals its own single-candidate replay and the oracle's
    evaluation of the same (options, order)."""
    from paper_2311_02840_b200.engine import SRC_EXPLICIT, NativeProblem
    from paper_2311_02840_b200.problem import build_problem
    from paper_2311_02840_b200.workloads import config_workload

    w, t, _ = config_workload(cfg)
    prob = build_problem(t, w, SolveOptions())
    sol = PL.solve_problem(prob, w, SolveOptions())
    eng = PL.get_engine()
    nexp = NativeProblem(prob, 62)
    rows = [np.array(list(sol.options) + list(sol.order), dtype=np.uint8)]
    for builder in (PL.optimus_allocation, PL.current_practice_allocation):
        o, r = builder(prob)
        rows.append(np.array(list(o) + list(r), dtype=np.uint8))
    batch = PL._decode(eng, prob, nexp, w, SRC_EXPLICIT, 0, explicit=np.stack(rows))
    op = O.build(t.entries, w)
    cp = C.CProblem(op)
    for row, got in zip(rows, batch):
        single = PL._decode(eng, prob, nexp, w, SRC_EXPLICIT, 0, explicit=row)
        assert got[0] == single[0] and got[1:] == single[1:]
        ms, _, _ = cp.eval([int(x) for x in row[:prob.J]], [int(x) for x in row[prob.J:]])
        assert got[2] == ms
    assert batch[0][2] == sol.makespan


@pytest.mark.parametrize("name,opts", [("cfg1", SolveOptions(kernel="tree")),
                                       ("small5_1x4", SolveOptions(kernel="index")),
                                       ("cfg1", SolveOptions(search="sampled", budget=1 << 16, seed=3))])
def test_device_replay_equals_host_decode(name, opts):
    """search(replay=True) schedules the winner from the device-side key; the result equals the
    replay of the host-read index (the path it replaces) and the solve's plan."""
    from paper_2311_02840_b200.engine import SRC_INDEX, NativeProblem
    from paper_2311_02840_b200.problem import build_problem

    w, t = setup(name)
    prob = build_problem(t, w, opts)
    eng = PL.get_engine()
    res = eng.search(prob, opts, replay=True)
    assert res.replay is not None
    src = SRC_INDEX if res.exhaustive else res.source
    host = eng.schedule(NativeProblem(prob, res.idx_bits), src, res.seed, ids=[res.index])
    for a, b in zip(res.replay, host):
        assert a.dtype == b.dtype and np.array_equal(a, b)
    assert float(res.replay[3][0]) == res.makespan
    sol = PL.solve(t, w, None, opts)
    assert sol.makespan == res.makespan and sol.options == [int(x) for x in host[0][0]]


@pytest.mark.parametrize("kernel", ["auto", "index"])
def test_random_workloads_plan_equals_oracle_optimum(kernel):
    """plan_saturn on random 4-6-job workloads (1-2 nodes): the winning index, makespan and
    every job's (option, node, start) equal the C oracle's exhaustive search and replay.
    kernel=auto takes bound-and-prune on one node (host-index replay) and the index kernel on
    two; kernel=index takes the full scan with the device-queued replay."""
    from paper_2311_02840_b200.workloads import random_workload

    checked = 0
    for seed in range(60):
        w = random_workload(1000 + seed, n_jobs=4 + seed % 3)
        t = build_profile_table(w, SyntheticExecutor(w.cluster))
        op = O.build(t.entries, w)
        if math.prod(op.radix) * math.factorial(op.J) > 3e7:      # keep the CPU search short
            continue
        checked += 1
        cp = C.CProblem(op)
        ms, ident = cp.search()
        sol = PL.solve(t, w, None, SolveOptions(search="exhaustive", kernel=kernel))
        assert sol.status == "Optimal" and sol.makespan == ms and sol.search.index == ident
        opts, order = cp.decode(ident)
        ms2, starts, nodes = cp.eval(opts, order)
        assert ms2 == ms and sol.options == opts
        for j, jid in enumerate(op.job_ids):
            e = sol.plan.entries[jid]
            assert e.start_time == starts[j] * sol.problem.delta
            assert e.node == sol.problem.node_ids[nodes[j]]
    assert checked >= 30
