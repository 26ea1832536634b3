"""Host marshalling (problem.py) == the oracle's independent restatement, bit for bit."""

import math

import numpy as np
import pytest

from helpers import golden, golden_workload, unhex

from oracle import saturn_oracle as O
from paper_2311_02840_b200 import domain as D
from paper_2311_02840_b200 import errors as E
from paper_2311_02840_b200.problem import SolveOptions, build_problem
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table

NAMES = ["cfg1", "cfg3", "cfg4", "cfg5", "small5_1x4", "small4_2x2", "hetero6", "tiny3_1x3"]


def compare(prob, oprob):
    assert prob.job_ids == oprob.job_ids
    assert prob.node_ids == oprob.node_ids
    assert prob.delta.hex() == float(oprob.delta).hex()
    assert list(prob.radix) == oprob.radix
    grid = prob.time_mode == "grid"
    for j in range(prob.J):
        for o in range(int(prob.radix[j])):
            cfg = prob.options[j][o][0]
            assert (cfg.technique, cfg.gpus) == oprob.options[j][o]
            assert int(prob.gpus[j, o]) == oprob.gpus[j][o]
            for n in range(prob.N):
                el = bool((int(prob.node_mask[j, o]) >> n) & 1)
                assert el == oprob.eligible[j][o][n]
                if el:
                    assert prob.runtime[j, o, n].hex() == float(oprob.runtime[j][o][n]).hex()
                    if grid:
                        assert int(prob.dur_i32[j, o, n]) == oprob.dur[j][o][n]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("mode", ["grid", "float"])
def test_build_problem_matches_oracle(name, mode):
    w, _ = golden_workload(name)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w, SolveOptions(time_mode=mode))
    oprob = O.build(t.entries, w, grid=mode == "grid")
    compare(prob, oprob)
    assert prob.pruned == (len(w.cluster.nodes) == 1)


@pytest.mark.parametrize("name", ["cfg1", "small5_1x4", "tiny3_1x3"])
def test_build_problem_unpruned_matches_oracle(name):
    w, _ = golden_workload(name)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w, SolveOptions(prune=False))
    compare(prob, O.build(t.entries, w, prune=False))
    assert not prob.pruned


def test_cfg1_shape_and_delta():
    """cfg1 radices 4,7,5,6,5,8,4,6, space 3.25e10, delta 2255.40625668252 s."""
    w, _ = golden_workload("cfg1")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w)
    assert list(prob.radix) == [4, 7, 5, 6, 5, 8, 4, 6]
    assert prob.space == 32514048000
    assert prob.delta.hex() == golden()["milp"]["cfg1"]["delta"]
    assert prob.key_bits(prob.space) == (35, 9)


@pytest.mark.parametrize("rho", [0.0, 30.0, 5000.0])
def test_resolve_transform_matches_oracle(rho):
    """Re-solve: remaining batches, finished jobs dropped, +rho on changed assignments."""
    w, _ = golden_workload("hetero6")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    remaining = {"j00": 1234, "j01": 0, "j02": 20000, "j03": 7, "j05": 15000}
    current = {"j00": ("ddp", 2, "n0"), "j03": ("fsdp", 4, "n1")}
    ctx = D.RunningContext(remaining=remaining, current=current, checkpoint_cost=rho)
    for mode in ("grid", "float"):
        prob = build_problem(t, w, SolveOptions(time_mode=mode), running_context=ctx)
        oprob = O.build(t.entries, w, grid=mode == "grid", context=(remaining, current, rho))
        compare(prob, oprob)
        assert prob.job_ids == ["j00", "j02", "j03", "j05"]


def test_resolve_single_node_prune_with_rho():
    w, _ = golden_workload("cfg1")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    remaining = {j.id: j.total_batches // 3 for j in w.jobs}
    current = {"j01": ("gpipe", 5, "n0"), "j04": ("ddp", 3, "n0")}
    ctx = D.RunningContext(remaining=remaining, current=current, checkpoint_cost=30.0)
    prob = build_problem(t, w, running_context=ctx)
    compare(prob, O.build(t.entries, w, context=(remaining, current, 30.0)))


def test_index_codec_roundtrip():
    w, _ = golden_workload("small5_1x4")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w)
    oprob = O.build(t.entries, w)
    rng = np.random.default_rng(0)
    for ident in list(rng.integers(0, prob.space, 200)) + [0, prob.space - 1]:
        ident = int(ident)
        opts, order = prob.decode_index(ident)
        assert (opts, order) == O.decode_index(oprob, ident)
        assert prob.encode_index(opts, order) == ident


def test_errors():
    w, _ = golden_workload("cfg1")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    with pytest.raises(E.HorizonOverflow):
        build_problem(t, w, SolveOptions(delta=10.0))
    with pytest.raises(E.InvariantViolation):
        build_problem(t, w, SolveOptions(time_mode="bogus"))
    empty = type(t)({k: v for k, v in t.entries.items() if k[0] != "j03"}, "synthetic")
    with pytest.raises(E.NoFeasibleConfig):
        build_problem(empty, w)
    w4, _ = golden_workload("cfg4")
    t4 = build_profile_table(w4, SyntheticExecutor(w4.cluster))
    with pytest.raises(E.InvariantViolation):
        build_problem(t4, w4, SolveOptions(prune=True))
    big = D.Workload(jobs=w4.jobs, cluster=D.ClusterSpec(nodes=tuple(
        D.NodeSpec(f"n{i}", 8, 40.0) for i in range(5))), techniques=w4.techniques)
    tb = build_profile_table(big, SyntheticExecutor(big.cluster))
    with pytest.raises(E.TooLarge):
        build_problem(tb, big)


def test_lower_bound_never_exceeds_the_optimum():
    """problem.lower_bound() <= the exhaustive optimum (oracle) on random 1- and 2-node problems."""
    import random

    from oracle import coracle as C
    from test_engine_gpu import to_search_problem
    from test_oracle import random_problem

    rng = random.Random(41)
    for trial in range(40):
        nodes = [[rng.randint(1, 6)], [rng.randint(1, 4), rng.randint(1, 4)]][trial % 2]
        op = random_problem(rng, rng.randint(1, 4), nodes, max_opts=3, max_d=8, hetero=trial % 3 == 0)
        if trial % 4 == 1:
            op.release = [rng.randint(0, 4) for _ in range(op.J)]
            op.init_free = [[rng.randint(0, 3) for _ in range(n)] for n in nodes]
        ms, _ = C.CProblem(op).search()
        assert to_search_problem(op).lower_bound() <= ms, trial


def _lower_bound_literal(p):
    """The bound of SearchProblem.lower_bound restated as plain loops (committed free time,
    each job's earliest end over its options and eligible nodes, area over all GPUs)."""
    import math

    grid = p.time_mode == "grid"
    d = p.dur_i32 if grid else p.runtime
    init = p.init_free_i32 if grid else p.init_free_f64
    rel = p.release_i32 if grid else p.release_f64
    real = [float(init[n, i]) for n in range(p.N) for i in range(int(p.node_gpus[n]))]
    lb, area = (max(real) if real else 0.0), sum(real)
    for j in range(p.J):
        ends, areas = [], []
        for o in range(int(p.radix[j])):
            g = int(p.gpus[j, o])
            for n in range(p.N):
                if (int(p.node_mask[j, o]) >> n) & 1:
                    kth = sorted(float(init[n, i]) for i in range(int(p.node_gpus[n])))[g - 1]
                    ends.append(max(float(rel[j]), kth) + float(d[j, o, n]))
                    areas.append(g * float(d[j, o, n]))
        lb = max(lb, min(ends))
        area += min(areas)
    lb = max(lb, area / float(sum(int(x) for x in p.node_gpus)))
    return float(math.ceil(lb - 1e-9)) if grid else lb


def test_lower_bound_equals_literal_restatement():
    """The vectorised, memoised lower_bound equals the loop restatement bit for bit (grid and
    float time, releases, initial free times, heterogeneous eligibility)."""
    import random

    from test_engine_gpu import to_search_problem
    from test_oracle import random_problem

    rng = random.Random(43)
    for trial in range(60):
        nodes = [[rng.randint(1, 8)], [rng.randint(1, 4), rng.randint(1, 4)], [2, 3, 1]][trial % 3]
        op = random_problem(rng, rng.randint(1, 6), nodes, max_opts=4, max_d=20, hetero=trial % 2 == 0)
        op.grid = trial % 5 != 0
        if trial % 4 == 1:
            op.release = [rng.randint(0, 6) for _ in range(op.J)]
            op.init_free = [[rng.randint(0, 5) for _ in range(n)] for n in nodes]
        p = to_search_problem(op)
        want = _lower_bound_literal(p)
        assert p.lower_bound() == want, trial
        assert p.lower_bound() == want, trial            # memoised value


def test_optimus_marginal_gain_spec_examples():
    """latency halving g=1 -> 2, 1000 batches, base 1 s -> 500 s; g at the node
    maximum -> 0; a slower g+1 -> clamped to 0."""
    from paper_2311_02840_b200 import planners as PL
    from paper_2311_02840_b200.profiling import ProfileTable

    job = D.JobSpec("a", 1000, 1.0, 1.0)
    t = ProfileTable({("a", "t", 1): 1.0, ("a", "t", 2): 0.5, ("a", "u", 2): 0.6, ("a", "t", 3): 0.55,
                      ("a", "t", 4): float("inf")}, "x")
    assert PL.optimus_marginal_gain(t, job, 1, 1000) == 500.0
    assert PL.optimus_marginal_gain(t, job, 1) == 500.0                 # default: total batches
    assert PL.optimus_marginal_gain(t, job, 2, 1000) == 0.0              # 0.55 > 0.5: harmful GPU
    assert PL.optimus_marginal_gain(t, job, 3, 1000) == 0.0              # g+1 infeasible
    assert PL.optimus_marginal_gain(t, job, 8, 1000) == 0.0              # beyond the table


@pytest.mark.parametrize("row_min", [0, 1 << 30])
@pytest.mark.parametrize("mode", ["grid", "float"])
def test_one_node_array_marshalling_matches_oracle(mode, row_min, monkeypatch):
    """Both one-node marshalling paths (rows as arrays with the array prune; short rows as
    tuples) against the oracle's build on random one-node workloads, one table entry made
    infeasible and one dropped."""
    from paper_2311_02840_b200 import problem as P
    from paper_2311_02840_b200.workloads import random_workload

    monkeypatch.setattr(P, "_ARRAY_ROW_MIN", row_min)
    monkeypatch.setattr(P, "_BATCH_ROWS", False)          # the per-job rows (batch: below)

    for seed in range(40):
        w = random_workload(seed, n_nodes=1)
        t = build_profile_table(w, SyntheticExecutor(w.cluster))
        keys = sorted(t.entries)
        if seed % 3 == 1 and len(keys) > 2:
            t.entries[keys[seed % len(keys)]] = math.inf
        if seed % 3 == 2 and len(keys) > 2:
            del t.entries[keys[(7 * seed) % len(keys)]]
        try:
            oprob = O.build(t.entries, w, grid=mode == "grid")
        except Exception as exc:  # noqa: BLE001 -- both sides must refuse the same way
            with pytest.raises(type(exc)):
                build_problem(t, w, SolveOptions(time_mode=mode))
            continue
        compare(build_problem(t, w, SolveOptions(time_mode=mode)), oprob)


def test_dominance_prune_arrays_equals_list_prune():
    from paper_2311_02840_b200.problem import _dominance_prune, _dominance_prune_arrays

    rng = np.random.default_rng(5)
    for _ in range(500):
        n = int(rng.integers(1, 40))
        g = rng.integers(1, 9, n)
        cost = rng.integers(1, 12, n).astype(np.float64)      # many ties
        want = _dominance_prune([(i, int(g[i]), float(cost[i])) for i in range(n)])
        assert _dominance_prune_arrays(g, cost) == want


def test_resolve_random_contexts_match_oracle():
    """Re-solve marshalling on random workloads and random running contexts (some jobs done,
    some running on a random feasible (technique, g, node), rho 0 / 30) against the oracle."""
    from paper_2311_02840_b200.profiling import feasible_entries
    from paper_2311_02840_b200.workloads import random_workload

    for seed in range(30):
        w = random_workload(seed)
        t = build_profile_table(w, SyntheticExecutor(w.cluster))
        rng = np.random.default_rng(seed)
        remaining, current = {}, {}
        for job in w.jobs:
            remaining[job.id] = int(rng.integers(0, job.total_batches + 1)) if rng.random() < 0.8 else 0
            ents = feasible_entries(t, job, w)
            if remaining[job.id] and ents and rng.random() < 0.6:
                cfg, _ = ents[int(rng.integers(len(ents)))]
                node = w.cluster.nodes[int(rng.integers(len(w.cluster.nodes)))]
                current[job.id] = (cfg.technique, cfg.gpus, node.id)
        if not any(remaining.values()):
            continue
        rho = 30.0 if seed % 2 else 0.0
        ctx = D.RunningContext(remaining=remaining, current=current, checkpoint_cost=rho)
        for mode in ("grid", "float"):
            try:
                oprob = O.build(t.entries, w, grid=mode == "grid", context=(remaining, current, rho))
            except Exception as exc:  # noqa: BLE001 -- both sides must refuse the same way
                with pytest.raises(type(exc)):
                    build_problem(t, w, SolveOptions(time_mode=mode), running_context=ctx)
                continue
            compare(build_problem(t, w, SolveOptions(time_mode=mode), running_context=ctx), oprob)


def test_best_runtime_by_g_equals_loop_restatement():
    """The incumbents' per-g best runtime (one array pass) equals its per-option loop: least
    runtime over eligible nodes, then least over techniques at each g, earliest option on ties."""
    from paper_2311_02840_b200 import planners as PL
    from paper_2311_02840_b200.workloads import config_workload, random_workload

    def loop(prob, j):
        out = {}
        for o in range(int(prob.radix[j])):
            g = int(prob.gpus[j, o])
            rt = min(prob.runtime[j, o, n] for n in range(prob.N) if (int(prob.node_mask[j, o]) >> n) & 1)
            if g not in out or rt < out[g][0]:
                out[g] = (rt, o)
        return out

    probs = [build_problem(t, w) for w, t, _ in (config_workload(k) for k in (1, 4))]
    for seed in range(40):
        w = random_workload(seed)
        t = build_profile_table(w, SyntheticExecutor(w.cluster))
        probs.append(build_problem(t, w, SolveOptions(time_mode="float" if seed % 2 else "grid")))
    for prob in probs:
        got = PL._best_runtime_all(prob)
        for j in range(prob.J):
            want = loop(prob, j)
            assert got[j].keys() == want.keys() == PL._best_runtime_by_g(prob, j).keys()
            for g in want:
                assert got[j][g][1] == want[g][1] and float(got[j][g][0]).hex() == float(want[g][0]).hex()


@pytest.mark.parametrize("mode", ["grid", "float"])
def test_batch_marshalling_equals_per_job_rows(mode, monkeypatch):
    """`_batch_rows` (whole-problem numpy; every solve without running configurations) builds
    exactly the arrays, options and delta of the per-job rows: configs 1-5, and random 1-4-node
    workloads with infeasible / missing table entries and re-solve contexts that only shrink
    the remaining batches; errors are raised the same way."""
    from paper_2311_02840_b200 import problem as P
    from paper_2311_02840_b200.workloads import config_workload, random_workload

    def build(flag, t, w, ctx=None, **kw):
        monkeypatch.setattr(P, "_BATCH_ROWS", flag)
        try:
            return build_problem(t, w, SolveOptions(time_mode=mode, **kw), ctx)
        except Exception as exc:  # noqa: BLE001
            return type(exc)

    def same(a, b):
        if isinstance(a, type) or isinstance(b, type):
            assert a == b
            return
        for f in ("radix", "gpus", "node_mask", "runtime", "dur_i32", "init_free_i32", "init_free_f64"):
            x, y = getattr(a, f), getattr(b, f)
            assert x.dtype == y.dtype and x.shape == y.shape and np.array_equal(x, y), f
        assert a.delta.hex() == b.delta.hex()
        assert (a.options, a.option_src, a.job_ids, a.pruned) == (b.options, b.option_src, b.job_ids, b.pruned)

    cases = []
    for c in (1, 2, 3, 4, 5):
        w, t, _ = config_workload(c)
        cases.append((t, w, None, {}))
        cases.append((t, w, None, {"prune": False}))
    for seed in range(40):
        w = random_workload(seed, n_nodes=1 + seed % 4)
        t = build_profile_table(w, SyntheticExecutor(w.cluster))
        keys = sorted(t.entries)
        if seed % 3 == 1 and len(keys) > 2:
            t.entries[keys[seed % len(keys)]] = math.inf
        if seed % 3 == 2 and len(keys) > 2:
            del t.entries[keys[(7 * seed) % len(keys)]]
        cases.append((t, w, None, {}))
        if seed % 2:
            rem = {j.id: (0 if k % 3 == 0 else max(1, int(j.total_batches) // (k + 2)))
                   for k, j in enumerate(w.jobs)}
            cases.append((t, w, D.RunningContext(remaining=rem, current={}, checkpoint_cost=30.0), {}))
    for t, w, ctx, kw in cases:
        same(build(True, t, w, ctx, **kw), build(False, t, w, ctx, **kw))


def test_table_view_never_serves_a_mutated_table():
    """The array view of a profile table's entries (`_TableView`) is reused across solves only
    while the dict's keys and latencies are provably unchanged: changing a latency, replacing
    a key makes the next marshalling re-read the table (same arrays as a fresh copy of the
    dict)."""
    import copy

    from paper_2311_02840_b200 import problem as P
    from paper_2311_02840_b200.workloads import config_workload

    w, t, _ = config_workload(4)

    def arrays(tab):
        p = build_problem(tab, w)
        return p.radix.tobytes(), p.dur_i32.tobytes(), p.runtime.tobytes(), p.delta

    base = arrays(t)
    assert arrays(t) == base and id(t.entries) in P._TABLE_VIEWS
    keys = [k for k, v in t.entries.items() if np.isfinite(v)]
    k0, k1 = keys[3], keys[-1]
    t.entries[k0] = t.entries[k0] * 0.5                          # a value change
    fresh = copy.copy(t)
    fresh.entries = dict(t.entries)
    assert arrays(t) == arrays(fresh) != base
    v1 = t.entries.pop(k1)                                       # delete + re-insert a key (order moves)
    t.entries[k1] = v1 * 3.0
    fresh.entries = dict(t.entries)
    assert arrays(t) == arrays(fresh)
    t.entries[k0] = 0.25                                         # a new float object, a new value
    v = P._TableView.of(t.entries)
    assert v.lat[v.keys.index(k0)] == 0.25 and P._TableView.of(t.entries) is v
