"""State-space search (sat_search_dp) against the CPU oracle.

For every problem: with M* = the oracle's exhaustive optimum (lowest makespan over the whole
candidate space, oracle/oracle.c), the DP must report INFEASIBLE at target M* - 1 and FEASIBLE
at M* -- and the candidate it returns, replayed by the oracle's own list scheduler, must have
makespan <= the target.  The returned candidate is deterministic (same one on every run).  The
headline use: config 3's optimum (30, certified by HiGHS on the CPU) is proven on the GPU, so
plan_saturn(cfg3) returns status Optimal."""

import random

import pytest

from helpers import golden
from test_engine_gpu import to_search_problem, workload_problem
from test_oracle import random_problem

from oracle import coracle as C
from paper_2311_02840_b200 import engine as EN
from paper_2311_02840_b200 import errors as E
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200.problem import SolveOptions, build_problem
from paper_2311_02840_b200.workloads import config_workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    return EN.Engine(0)


def dp(eng, prob, target, max_states=1 << 20):
    return eng.dp_search(EN.NativeProblem(prob, 1), target, max_states)


def check_around_optimum(eng, op, prob):
    opt = C.CProblem(op).search()[0]
    st, info, cand = dp(eng, prob, int(opt) - 1)
    assert st == EN.SAT_DP_INFEASIBLE, (opt, info.levels)
    for target in (int(opt), int(opt) + 2):
        st, info, cand = dp(eng, prob, target)
        assert st == EN.SAT_DP_FEASIBLE
        opts, order = cand
        assert sorted(order) == list(range(op.J))
        ms, _, _ = C.CProblem(op).eval(opts, order)
        assert ms <= target and ms == info.makespan
        assert dp(eng, prob, target)[2] == cand            # deterministic reconstruction
    return opt


def test_dp_random_one_node(eng):
    rng = random.Random(2024)
    for trial in range(60):
        gsz = [1, 2, 3, 4, 5, 8, 16, 32][trial % 8]
        J = [2, 3, 4, 5, 6][trial % 5]
        # (keys must fit 63 bits: 2^J x C(T + G, G); 32-GPU nodes get short jobs)
        op = random_problem(rng, J, [gsz], max_opts=4 if J < 6 else 3, max_d=12 if gsz < 32 else 2)
        if trial % 3 == 0:
            op.init_free = [sorted(rng.randint(0, 5) for _ in range(gsz))]
        if trial % 4 == 1:
            op.release = [rng.randint(0, 6) for _ in range(op.J)]
        check_around_optimum(eng, op, to_search_problem(op))


@pytest.mark.parametrize("name", ["small5_1x4", "tiny3_1x3"])
def test_dp_workloads(eng, name):
    w, t, prob, op = workload_problem(name)
    assert check_around_optimum(eng, op, prob) == golden()["milp"][name]["optimum_intervals"]


def test_dp_cfg1_optimum():
    """Config 1: nothing at 29, a 30-interval candidate at 30 (= HiGHS, = the full scan)."""
    eng = PL.get_engine(0)
    w, t, _ = config_workload(1)
    prob = build_problem(t, w)
    assert dp(eng, prob, 29, 1 << 22)[0] == EN.SAT_DP_INFEASIBLE
    st, info, cand = dp(eng, prob, 30, 1 << 22)
    assert st == EN.SAT_DP_FEASIBLE and info.makespan == 30


def test_dp_proves_cfg3_optimal():
    """Config 3 (16 jobs, 3e23 candidates): local search reaches 30, the trivial bound says 29;
    the state-space search shows no candidate reaches 29, so the plan is Optimal -- the value
    HiGHS certifies on the CPU (tests/golden)."""
    eng = PL.get_engine(0)
    w, t, _ = config_workload(3)
    prob = build_problem(t, w)
    st, info, _ = dp(eng, prob, 29, 1 << 22)
    assert st == EN.SAT_DP_INFEASIBLE and info.levels <= prob.J
    sol = PL.solve(t, w)
    assert sol.status == "Optimal" and sol.makespan == 30 == golden()["milp"]["cfg3"]["optimum_intervals"]
    assert sol.lower_bound == 30 and sol.search.proven
    assert sol.search.stats["proof"]["attempts"][-1]["status"] == "infeasible"


def test_dp_budget_and_unsupported(eng):
    w, t, _ = config_workload(3)
    prob = build_problem(t, w)
    st, info, _ = dp(eng, prob, 29, 1000)
    assert st == EN.SAT_DP_BUDGET
    w4, t4, _ = config_workload(4)                       # several nodes: the prover (no candidate)
    p4 = build_problem(t4, w4)
    assert dp(eng, p4, 7)[0] == EN.SAT_DP_INFEASIBLE     # below the area bound: decided on the host
    rng = random.Random(5)                               # > 8 nodes: beyond the prover
    op = random_problem(rng, 3, [1] * 9, max_opts=2, max_d=4)
    with pytest.raises(E.TooLarge):
        dp(eng, to_search_problem(op), 3)


def test_dp_budget_exhaustion_stops_early(eng):
    """Out of budget at one level, the remaining work of that level is dropped: config 3 at
    T = 31 overflows 4 M states at level 5 in about a millisecond (it took 0.3 s while the
    level kept inserting into the hash set after the overflow)."""
    import time

    w, t, _ = config_workload(3)
    prob = build_problem(t, w)
    dp(eng, prob, 31, 1 << 22)                           # warm (workspace, tables)
    t0 = time.perf_counter()
    st, info, _ = dp(eng, prob, 31, 1 << 22)
    assert st == EN.SAT_DP_BUDGET and info.levels < prob.J
    assert time.perf_counter() - t0 < 0.1


def test_solve_without_proof_keeps_local_status():
    w, t, _ = config_workload(3)
    sol = PL.solve(t, w, None, SolveOptions(prove=False))
    assert sol.status == "Local" and sol.makespan == 30 and not sol.search.proven


def test_dp_multinode_prover_is_sound():
    """Several nodes (heterogeneous, interchangeable, releases, initial free times; the
    homogeneous 2 x 4, 3 x 4, 4 x 4 and 2 x 8 shapes run the register-resident specialisation of
    the wide kernel): the wide prover never calls a reachable target infeasible -- every INFEASIBLE at T has the oracle's
    exhaustive optimum above T -- and it is FEASIBLE from the optimum up.  It proves the optimum
    (INFEASIBLE at M* - 1) on most problems."""
    eng = EN.Engine(0)
    rng = random.Random(31)
    proven = total = 0
    for trial in range(40):
        nodes = [[2, 2], [4, 4], [3, 2], [2, 2, 2], [4, 2, 1], [8, 8], [4, 4, 4], [4, 4, 4, 4]][trial % 8]
        op = random_problem(rng, rng.randint(2, 5), nodes, max_opts=3, max_d=8, hetero=trial % 3 == 0)
        if trial % 4 == 1:
            op.release = [rng.randint(0, 4) for _ in range(op.J)]
        if trial % 5 == 2:
            op.init_free = [sorted(rng.randint(0, 3) for _ in range(n)) for n in nodes]
        prob = to_search_problem(op)
        opt = int(C.CProblem(op).search()[0])
        for target in range(max(0, opt - 3), opt + 2):
            st, info, cand = dp(eng, prob, target)
            assert cand is None and st != EN.SAT_DP_BUDGET
            if st == EN.SAT_DP_INFEASIBLE:
                assert target < opt, (trial, target, opt)
            if target >= opt:
                assert st == EN.SAT_DP_FEASIBLE, (trial, target, opt)
        total += 1
        proven += dp(eng, prob, opt - 1)[0] == EN.SAT_DP_INFEASIBLE
    assert proven >= total * 3 // 4, (proven, total)


def test_dp_multinode_exact_equals_oracle():
    """SAT_DP_EXACT (ABI v8) on several nodes: labelled states expanded by the list scheduler's
    own node choice, so the search is exact -- INFEASIBLE at M* - 1 on EVERY problem, FEASIBLE
    at M* and above with a candidate the oracle replays to makespan <= target (= the reported
    makespan), rebuilt deterministically.  Heterogeneous and interchangeable nodes, releases,
    initial free times."""
    eng = EN.Engine(0)
    rng = random.Random(57)
    for trial in range(40):
        nodes = [[2, 2], [4, 4], [3, 2], [2, 2, 2], [4, 2, 1], [8, 8], [4, 4, 4, 4], [4, 4, 4]][trial % 8]
        op = random_problem(rng, rng.randint(2, 5), nodes, max_opts=3, max_d=8, hetero=trial % 3 == 0)
        if trial % 4 == 1:
            op.release = [rng.randint(0, 4) for _ in range(op.J)]
        if trial % 5 == 2:
            op.init_free = [sorted(rng.randint(0, 3) for _ in range(n)) for n in nodes]
        prob = to_search_problem(op)
        nprob = EN.NativeProblem(prob, 1)
        opt = int(C.CProblem(op).search()[0])
        st, info, cand = eng.dp_search(nprob, opt - 1, 1 << 20, exact=True)
        assert st == EN.SAT_DP_INFEASIBLE, (trial, opt, info.levels)
        for target in (opt, opt + 2):
            st, info, cand = eng.dp_search(nprob, target, 1 << 20, exact=True)
            assert st == EN.SAT_DP_FEASIBLE and cand is not None, (trial, target, opt)
            opts, order = cand
            assert sorted(order) == list(range(op.J))
            ms, _, _ = C.CProblem(op).eval(opts, order)
            assert ms <= target and ms == info.makespan, (trial, target, ms, info.makespan)
            assert eng.dp_search(nprob, target, 1 << 20, exact=True)[2] == cand     # deterministic


def test_prove_below_multinode_returns_the_optimum():
    """prove_below on several nodes from a candidate above the optimum: the prover's
    inconclusive answers hand over to exact states, and the descent ends AT the exhaustive
    optimum with a candidate reaching it, proven (one interval less is infeasible)."""
    eng = EN.Engine(0)
    rng = random.Random(58)
    for trial in range(12):
        nodes = [[4, 4], [2, 2, 2], [8, 4]][trial % 3]
        op = random_problem(rng, rng.randint(3, 5), nodes, max_opts=3, max_d=8, hetero=trial % 2 == 0)
        prob = to_search_problem(op)
        opt = int(C.CProblem(op).search()[0])
        proven, ms, cand, stats = eng.prove_below(prob, opt + 3, SolveOptions(), lb=0)
        assert proven and ms == opt, (trial, ms, opt, stats["attempts"])
        opts, order = cand
        assert C.CProblem(op).eval(opts, order)[0] == opt


def test_hetero6_local_plan_proven_or_improved():
    """hetero6 (6 jobs, 8 + 4 GPU nodes, 2.3e11 candidates): the default solve is the local
    search; its makespan must equal the exhaustive optimum (index kernel over the whole space)
    and, when the prover closes the gap, carry status Optimal."""
    w, t, prob, op = workload_problem("hetero6")
    sol = PL.solve(t, w)
    full = PL.solve(t, w, None, SolveOptions(search="exhaustive", kernel="index", max_exhaustive=1 << 40))
    assert full.status == "Optimal"
    assert sol.makespan == full.makespan
    proof = (sol.search.stats or {}).get("proof")
    assert proof is not None
    assert sol.status == ("Optimal" if proof["proven"] else "Local")


@pytest.mark.parametrize("at_bound", [True, False])
def test_local_search_with_proof_random_one_node(eng, at_bound):
    """Local search forced onto small one-node problems with a deliberately weak wave (8
    walkers, 2 rounds): the state-space search -- at the lower bound on a side stream during
    the first wave (dp_at_bound), then below the wave's best -- must still end at the oracle's
    exhaustive optimum with a proof, and the returned (options, order) must replay to it."""
    rng = random.Random(77)
    seen = set()
    for trial in range(30):
        gsz = [2, 3, 4, 8][trial % 4]
        op = random_problem(rng, rng.randint(3, 6), [gsz], max_opts=3, max_d=10)
        if trial % 3 == 1:
            op.release = [rng.randint(0, 5) for _ in range(op.J)]
        prob = to_search_problem(op)
        opt = C.CProblem(op).search()[0]
        res = eng.search(prob, SolveOptions(search="local", walkers=64, wave=8, max_rounds=2,
                                            dp_at_bound=at_bound))
        assert res.proven or res.makespan <= prob.lower_bound(), (trial, res.stats)
        assert res.makespan == opt, (trial, res.makespan, opt)
        opts, order = res.state
        assert C.CProblem(op).eval(opts, order)[0] == opt
        proof = res.stats.get("proof")
        if proof and proof["attempts"] and proof["attempts"][0]["target"] == int(prob.lower_bound()):
            seen.add(proof["attempts"][0]["status"])
    if at_bound:       # both outcomes of the side-stream attempt at the bound occur
        assert {"feasible", "infeasible"} <= seen, seen


def test_multinode_solve_improved_and_proven_by_exact_states():
    """A 2-node workload beyond exhaustive search (8 jobs, 2 x 4 GPUs, 1.1e13 candidates) where
    the local search stops one interval above the optimum (profiles/r02m_multinode_optimality.txt):
    with the prover alone the solve stays Local at 24; the exact multi-node mode hands over a
    23-interval candidate and proves it (22 unreachable) -- status Optimal, the plan validated by
    check_plan and replayed by the oracle's list scheduler to the same makespan."""
    from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table
    from paper_2311_02840_b200.workloads import synthetic_workload
    from oracle import saturn_oracle

    w = synthetic_workload(8, 2, 4, seed=100)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    base = PL.solve(t, w, None, SolveOptions(dp_exact=False))
    sol = PL.solve(t, w)
    assert sol.status == "Optimal" and sol.makespan < base.makespan, (sol.makespan, base.makespan)
    assert sol.makespan == sol.lower_bound
    assert sol.search.stats.get("winner") == "sat_search_dp"
    op = saturn_oracle.build(t.entries, w)
    assert C.CProblem(op).eval(list(sol.options), list(sol.order))[0] == sol.makespan
