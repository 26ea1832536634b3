"""Pin the oracle's search semantics: list-schedule optimum == independent optima.

* HiGHS on the time-indexed MILP -- golden values and live runs,
* brute_force_schedule on <= 3-job instances,
* the exact dominance prune keeps the optimum value (single node),
* the C oracle equals the Python oracle (windows, full small spaces, streams).
"""

import math
import random

import pytest

from helpers import golden, golden_workload

from oracle import coracle as C
from oracle import saturn_oracle as O
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table


def random_problem(rng, J, nodes, max_opts=3, max_d=6, hetero=False):
    gpus, eligible, dur, opts = [], [], [], []
    for _ in range(J):
        k = rng.randint(1, max_opts)
        gs, el, du, op = [], [], [], []
        for o in range(k):
            g = rng.randint(1, max(nodes))
            row_el = [n >= g and (not hetero or rng.random() < 0.8) for n in nodes]
            if not any(row_el):
                row_el = [n >= g for n in nodes]
            d = rng.randint(1, max_d)
            gs.append(g)
            el.append(row_el)
            du.append([d + (rng.randint(0, 2) if hetero else 0) if e else math.inf for e in row_el])
            op.append(("t%d" % o, g))
        gpus.append(gs); eligible.append(el); dur.append(du); opts.append(op)
    return O.Problem(job_ids=[f"j{j}" for j in range(J)], node_ids=[f"n{i}" for i in range(len(nodes))],
                     node_gpus=list(nodes), options=opts, gpus=gpus, eligible=eligible,
                     runtime=[[list(x) for x in r] for r in dur], dur=dur, delta=1.0, grid=True,
                     release=[0] * J, init_free=[[0] * n for n in nodes])


def test_golden_milp_values_match_oracle_search():
    """The recorded HiGHS optimum equals the oracle's exhaustive list-schedule optimum."""
    g = golden()["milp"]
    for name in ("small5_1x4", "small4_2x2", "tiny3_1x3"):
        w, _ = golden_workload(name)
        t = build_profile_table(w, SyntheticExecutor(w.cluster))
        prob = O.build(t.entries, w)
        assert prob.radix == g[name]["radix"]
        ms, _ = C.CProblem(prob).search()
        assert ms == g[name]["optimum_intervals"], name


def test_cfg3_optimum_certificate():
    """Config 3 (16 jobs, space 3e23): the recorded HiGHS optimum is 30 intervals, one above
    the area / longest-job bound; the MILP admits every gang schedule, so infeasibility at
    horizon 29 proves no list schedule reaches 29 (tools/cfg3_milp_bound.py)."""
    g = golden()["milp"]["cfg3"]
    w, _ = golden_workload("cfg3")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = O.build(t.entries, w)
    assert prob.radix == g["radix"] and g["optimum_intervals"] == 30
    with pytest.raises(RuntimeError, match="nfeasible"):
        O.milp_optimum(prob, horizon=29, time_limit=120.0)


def test_single_node_random_vs_highs():
    rng = random.Random(11)
    for _ in range(40):
        prob = random_problem(rng, rng.randint(2, 4), [rng.randint(2, 4)])
        ms, _ = O.search(prob)
        assert ms == O.milp_optimum(prob)


def test_two_node_random_vs_highs():
    rng = random.Random(5)
    for _ in range(40):
        prob = random_problem(rng, rng.randint(2, 4), [rng.randint(1, 3), rng.randint(1, 3)],
                              hetero=rng.random() < 0.5)
        ms, _ = O.search(prob)
        assert ms == O.milp_optimum(prob)


def test_brute_force_agrees():
    rng = random.Random(3)
    for _ in range(25):
        prob = random_problem(rng, rng.randint(1, 3), [rng.randint(2, 3)], max_d=4)
        assert O.search(prob)[0] == O.brute_force_schedule(prob) == O.milp_optimum(prob)


def test_spec_two_job_example():
    """2 jobs on a 2-GPU node, T(g=1)=10, T(g=2)=6, delta=1 -> M=10 (CP gives 12)."""
    prob = O.Problem(job_ids=["a", "b"], node_ids=["n"], node_gpus=[2], options=[[("t", 1), ("t", 2)]] * 2,
                     gpus=[[1, 2], [1, 2]], eligible=[[[True], [True]]] * 2, runtime=[[[10], [6]]] * 2,
                     dur=[[[10], [6]]] * 2, delta=1.0, grid=True, release=[0, 0], init_free=[[0, 0]])
    assert O.search(prob)[0] == 10
    assert O.brute_force_schedule(prob) == 10
    opts, order = O.current_practice(prob)
    assert O.list_schedule(prob, opts, order) == 12


def test_prune_keeps_optimum():
    rng = random.Random(8)
    for _ in range(30):
        J = rng.randint(2, 4)
        nodes = [rng.randint(2, 4)]
        prob = random_problem(rng, J, nodes, max_opts=4)
        full = O.search(prob)[0]
        # prune in place: per g cheapest, then strictly decreasing in g
        kept = []
        for j in range(J):
            per_g = {}
            for o, g in enumerate(prob.gpus[j]):
                d = prob.dur[j][o][0]
                if g not in per_g or d < per_g[g][1]:
                    per_g[g] = (o, d)
            keep, last = [], None
            for g in sorted(per_g):
                if last is None or per_g[g][1] < last:
                    keep.append(per_g[g][0]); last = per_g[g][1]
            kept.append(sorted(keep))
        pr = O.Problem(job_ids=prob.job_ids, node_ids=prob.node_ids, node_gpus=prob.node_gpus,
                       options=[[prob.options[j][o] for o in kept[j]] for j in range(J)],
                       gpus=[[prob.gpus[j][o] for o in kept[j]] for j in range(J)],
                       eligible=[[prob.eligible[j][o] for o in kept[j]] for j in range(J)],
                       runtime=[[prob.runtime[j][o] for o in kept[j]] for j in range(J)],
                       dur=[[prob.dur[j][o] for o in kept[j]] for j in range(J)], delta=1.0, grid=True,
                       release=prob.release, init_free=prob.init_free)
        assert O.search(pr)[0] == full


def test_c_oracle_matches_python():
    rng = random.Random(21)
    for trial in range(12):
        nodes = [rng.randint(1, 4)] if trial % 2 else [rng.randint(1, 3), rng.randint(1, 3)]
        prob = random_problem(rng, rng.randint(1, 5), nodes, hetero=trial % 3 == 0)
        prob.release = [rng.randint(0, 3) for _ in range(prob.J)]
        prob.init_free = [[rng.randint(0, 4) for _ in range(n)] for n in nodes]
        cp = C.CProblem(prob)
        hi = min(prob.space, 3000)
        assert cp.search(hi=hi) == tuple(map(float, O.search(prob, hi=hi))) or \
            cp.search(hi=hi)[0] == O.search(prob, hi=hi)[0]
        ms = cp.makespans(lo=0, hi=hi)
        for ident in range(0, hi, max(1, hi // 50)):
            opts, order = O.decode_index(prob, ident)
            assert ms[ident] == O.list_schedule(prob, opts, order)
            assert cp.decode(ident) == (opts, order)
        for src, seed in (("substream", 7), ("seed", 123)):
            a = cp.search(src, seed, 0, 300)
            b = O.search(prob, src, seed, 0, 300)
            assert a == (float(b[0]), b[1])
            for ident in (0, 17, 299):
                assert cp.decode(ident, src, seed) == O.candidate(prob, src, seed, ident)


def test_c_oracle_float_mode_bit_exact():
    w, _ = golden_workload("small5_1x4")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = O.build(t.entries, w, grid=False)
    cp = C.CProblem(prob)
    ms = cp.makespans(lo=1000, hi=1400)
    for i in range(0, 400, 37):
        opts, order = O.decode_index(prob, 1000 + i)
        assert ms[i].hex() == float(O.list_schedule(prob, opts, order)).hex()


def test_optimus_spec_examples():
    """gain example; 2 identical jobs on 2 GPUs -> 1 GPU each."""
    prob = O.Problem(job_ids=["a", "b"], node_ids=["n"], node_gpus=[2], options=[[("t", 1), ("t", 2)]] * 2,
                     gpus=[[1, 2], [1, 2]], eligible=[[[True], [True]]] * 2,
                     runtime=[[[1000.0], [500.0]]] * 2, dur=[[[2], [1]]] * 2, delta=500.0, grid=True,
                     release=[0, 0], init_free=[[0, 0]])
    b = O.best_by_g(prob, 0)
    assert b[1][0] - b[2][0] == 500.0
    opts, order = O.optimus(prob)
    assert [prob.gpus[j][opts[j]] for j in range(2)] == [1, 1]
    assert O.list_schedule(prob, opts, order) == 2
