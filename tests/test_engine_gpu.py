"""GPU parity: the CUDA engine (through the C ABI) vs the CPU oracle, bit-exact keys.

Every test here runs on a B200 and fails (never skips) when the engine is missing.
"""

import math
import random

import numpy as np
import pytest

from helpers import golden, golden_workload
from test_oracle import random_problem

from oracle import coracle as C
from oracle import saturn_oracle as O
from paper_2311_02840_b200 import engine as EN
from paper_2311_02840_b200.problem import INF_I32, SearchProblem, SolveOptions, build_problem
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    return EN.Engine(0)


def to_search_problem(op: O.Problem) -> SearchProblem:
    """Product problem arrays holding exactly the oracle problem's numbers."""
    J, N = op.J, op.N
    C_ = max(op.radix)
    G = 1
    while G < max(op.node_gpus):
        G *= 2
    W = max(8, 1 << (N * G - 1).bit_length())
    gpus = np.zeros((J, C_), np.int32)
    mask = np.zeros((J, C_), np.uint32)
    rt = np.zeros((J, C_, N), np.float64)
    dur = np.zeros((J, C_, N), np.int32)
    for j in range(J):
        for o in range(op.radix[j]):
            gpus[j, o] = op.gpus[j][o]
            for n in range(N):
                if op.eligible[j][o][n]:
                    mask[j, o] |= np.uint32(1 << n)
                    rt[j, o, n] = op.dur[j][o][n]
                    if op.grid:
                        dur[j, o, n] = op.dur[j][o][n]
    init_i = np.full((N, G), INF_I32, np.int32)
    init_f = np.full((N, G), np.inf)
    for n in range(N):
        vals = sorted(op.init_free[n])
        init_i[n, : len(vals)] = vals
        init_f[n, : len(vals)] = vals
    return SearchProblem(job_ids=op.job_ids, jobs=[None] * J, node_ids=op.node_ids,
                         node_gpus=np.array(op.node_gpus, np.int32), G=G, W=W,
                         options=[[(None, 0.0)] * r for r in op.radix], option_src=[list(range(r)) for r in op.radix],
                         radix=np.array(op.radix, np.int32), gpus=gpus, node_mask=mask, runtime=rt, dur_i32=dur,
                         release_i32=np.array(op.release, np.int32), release_f64=np.array(op.release, np.float64),
                         init_free_i32=init_i, init_free_f64=init_f, time_mode="grid" if op.grid else "float",
                         delta=op.delta, pruned=False)


def gpu_key(eng, prob, kind, lo=None, hi=None, source=EN.SRC_SUBSTREAM, seed=7, prefix=0, n_idx=None):
    n_idx = prob.space if n_idx is None else n_idx
    idx_bits, _ = prob.key_bits(n_idx)
    nprob = EN.NativeProblem(prob, idx_bits)
    best = eng.reset_best()
    if kind == "index":
        eng.search_index(nprob, 0 if lo is None else lo, n_idx if hi is None else hi, best)
    elif kind == "tree":
        info = eng.tree_plan(nprob, prefix)
        eng.search_tree(nprob, info.prefix_len, 0, info.n_tasks, best)
    else:
        eng.search_sampled(nprob, source, seed, 0 if lo is None else lo, n_idx if hi is None else hi, best)
    k = best.cpu().numpy().view(np.uint64)
    if nprob.grid:
        key = int(k[0])
        return (float(key >> idx_bits), key & ((1 << idx_bits) - 1))
    return (float(k[0:1].view(np.float64)[0]), int(k[1]))


def workload_problem(name, **kw):
    w, _ = golden_workload(name)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    return w, t, build_problem(t, w, SolveOptions(**kw)), O.build(t.entries, w, grid=kw.get("time_mode", "grid") == "grid",
                                                                 prune=kw.get("prune"))


# --------------------------------------------------------------------------- exhaustive
def test_index_kernel_full_space_random(eng):
    rng = random.Random(101)
    for trial in range(30):
        nodes = [[rng.randint(1, 8)], [rng.randint(1, 4), rng.randint(1, 4)], [2, 3, 1],
                 [rng.randint(1, 8), rng.randint(1, 8), rng.randint(1, 8), rng.randint(1, 8)]][trial % 4]
        op = random_problem(rng, rng.randint(1, 5), nodes, max_opts=4, max_d=9, hetero=trial % 3 == 0)
        if trial % 2:
            op.release = [rng.randint(0, 5) for _ in range(op.J)]
            op.init_free = [[rng.randint(0, 6) for _ in range(n)] for n in nodes]
        want = C.CProblem(op).search()
        assert gpu_key(eng, to_search_problem(op), "index") == want, trial


@pytest.mark.parametrize("name", ["small5_1x4", "tiny3_1x3", "small4_2x2"])
def test_index_kernel_workloads(eng, name):
    w, t, prob, op = workload_problem(name)
    want = C.CProblem(op).search()
    assert gpu_key(eng, prob, "index") == want
    assert want[0] == golden()["milp"][name]["optimum_intervals"]


def test_tree_kernel_full_space_random(eng):
    rng = random.Random(7)
    for trial in range(24):
        gsz = [3, 4, 8, 5, 16, 2, 32, 1][trial % 8]
        J = [3, 4, 5, 6][trial % 4]
        op = random_problem(rng, J, [gsz], max_opts=4 if J < 6 else 3, max_d=12)
        if trial % 3 == 0:
            op.init_free = [[rng.randint(0, 5) for _ in range(gsz)]]
        prob = to_search_problem(op)
        want = C.CProblem(op).search()
        for P in range(1, J - 1):
            assert gpu_key(eng, prob, "tree", prefix=P) == want, (trial, P)


@pytest.mark.parametrize("name", ["small5_1x4", "tiny3_1x3"])
def test_tree_kernel_workloads(eng, name):
    w, t, prob, op = workload_problem(name)
    want = C.CProblem(op).search()
    assert gpu_key(eng, prob, "tree") == want


def test_cfg1_full_space_tree_equals_index_and_highs(eng):
    """All 3.25e10 candidates of the paper workload, both kernels; optimum = HiGHS 30."""
    w, t, prob, op = workload_problem("cfg1")
    a = gpu_key(eng, prob, "tree")
    b = gpu_key(eng, prob, "index")
    assert a == b
    assert a[0] == golden()["milp"]["cfg1"]["optimum_intervals"] == 30
    # the winner re-evaluated by the oracle has that makespan, and nothing before it does
    opts, order = O.decode_index(op, a[1])
    assert O.list_schedule(op, opts, order) == 30
    lo = max(0, a[1] - 200000)
    assert C.CProblem(op).search(lo=lo, hi=a[1] + 1) == a


def test_cfg1_random_windows(eng):
    w, t, prob, op = workload_problem("cfg1")
    cp = C.CProblem(op)
    rng = random.Random(3)
    for _ in range(6):
        lo = rng.randrange(0, prob.space - 300000)
        hi = lo + rng.randrange(1, 300000)
        assert gpu_key(eng, prob, "index", lo, hi) == cp.search(lo=lo, hi=hi)


def test_float_mode_full_space(eng):
    for name in ("small5_1x4", "small4_2x2", "hetero6"):
        w, t, prob, op = workload_problem(name, time_mode="float")
        n = min(prob.space, 400000)
        want = C.CProblem(op).search(hi=n)
        got = gpu_key(eng, prob, "index", 0, n)
        assert got[1] == want[1]
        assert float(got[0]).hex() == float(want[0]).hex()       # bit-exact, stricter than 1e-6


def test_wide_times_use_32bit_slots(eng):
    """One node with free times past 2^16 (the packed 16-bit layout must not be used) and
    right at its boundary: index and sampled searches still equal the oracle."""
    rng = random.Random(77)
    for trial in range(16):
        nodes = [[rng.randint(2, 8)], [rng.randint(9, 16)], [rng.randint(17, 32)], [1]][trial % 4]
        op = random_problem(rng, rng.randint(2, 5), nodes, max_opts=3, max_d=9)
        scale = [40000, 9000, 13107, 21845][trial % 4]          # bounds on both sides of 65535
        op.dur = [[[d * scale for d in row] for row in job] for job in op.dur]
        op.runtime = [[list(r) for r in job] for job in op.dur]
        if trial % 2:
            op.release = [rng.randint(0, 3) * scale for _ in range(op.J)]
            op.init_free = [[rng.randint(0, 2) * scale for _ in range(n)] for n in nodes]
        prob = to_search_problem(op)
        assert gpu_key(eng, prob, "index") == C.CProblem(op).search(), trial
        got = gpu_key(eng, prob, "sampled", 0, 3000, source=EN.SRC_SUBSTREAM, seed=trial, n_idx=3000)
        assert got == C.CProblem(op).search("substream", trial, 0, 3000), trial


def test_tree_packed_pair_pass_and_32bit_pass(eng, monkeypatch):
    """k_tree's pair pass runs on 16-bit pairs when every reachable free time is below 0x7000
    (node sizes <= 16) and on 32-bit slots otherwise: both equal the oracle, including
    horizons on both sides of the packing limit and the forced 32-bit pass."""
    rng = random.Random(505)
    for trial in range(24):
        gsz = [2, 3, 5, 8, 11, 16][trial % 6]
        J = [3, 4, 5][trial % 3]
        op = random_problem(rng, J, [gsz], max_opts=4, max_d=9)
        if trial % 4 == 1:                       # horizon = sum of each job's longest option
            horizon = sum(max(max(r) for r in job) for job in op.dur)
            scale = (0x7000 + rng.choice([-1, 0, 1, 40])) // horizon
            op.dur = [[[d * scale for d in row] for row in job] for job in op.dur]
            op.runtime = [[list(r) for r in job] for job in op.dur]
        if trial % 3 == 0:
            op.init_free = [sorted(rng.randint(0, 5) for _ in range(gsz))]
        prob = to_search_problem(op)
        want = C.CProblem(op).search()
        monkeypatch.delenv("SATURN_TREE_PACKED", raising=False)
        assert gpu_key(eng, prob, "tree") == want, trial
        assert bnb_key(eng, prob) == want, trial
        monkeypatch.setenv("SATURN_TREE_PACKED", "0")
        assert gpu_key(eng, prob, "tree") == want, trial
        assert bnb_key(eng, prob) == want, trial
    monkeypatch.delenv("SATURN_TREE_PACKED", raising=False)


# --------------------------------------------------------------------------- bound-and-prune
def bnb_key(eng, prob, prefix=None, seed_bound=True, shards=1):
    idx_bits, _ = prob.key_bits(prob.space)
    nprob = EN.NativeProblem(prob, idx_bits)
    P = eng.bnb_prefix(nprob) if prefix is None else prefix
    info = eng.tree_plan(nprob, P)
    keys = []
    for r in range(shards):
        best = eng.reset_best()
        if seed_bound:
            eng.seed_upper_bound(prob, nprob, best)
        a, b = EN._shard(info.n_tasks, r, shards)
        eng.search_bnb(nprob, info.prefix_len, a, b, best)
        keys.append(int(best.cpu().numpy().view(np.uint64)[0]))
    k = min(keys)
    return (float(k >> idx_bits), k & ((1 << idx_bits) - 1))


def test_bnb_equals_exhaustive_random(eng):
    """Pruning on bound > best keeps every tie: same (makespan, lowest index) as the full scan."""
    rng = random.Random(303)
    for trial in range(40):
        nodes = [rng.choice([2, 3, 4, 5, 8])]
        op = random_problem(rng, rng.randint(3, 6), nodes, max_opts=4, max_d=9)
        if trial % 3 == 0:
            op.init_free = [sorted(rng.randint(0, 5) for _ in range(nodes[0]))]
        prob = to_search_problem(op)
        want = C.CProblem(op).search()
        assert gpu_key(eng, prob, "tree") == want, trial
        assert bnb_key(eng, prob, seed_bound=trial % 2 == 0) == want, trial
        assert bnb_key(eng, prob, prefix=1, shards=3) == want, trial


@pytest.mark.parametrize("name", ["small5_1x4", "tiny3_1x3", "cfg1"])
def test_bnb_workloads(eng, name):
    w, t, prob, op = workload_problem(name)
    want = gpu_key(eng, prob, "tree")
    assert bnb_key(eng, prob) == want
    assert bnb_key(eng, prob, seed_bound=False) == want
    if name != "cfg1":
        assert want == C.CProblem(op).search()
    else:
        assert want[0] == golden()["milp"]["cfg1"]["optimum_intervals"]


# --------------------------------------------------------------------------- sampled
@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5", "hetero6"])
@pytest.mark.parametrize("source", [EN.SRC_SUBSTREAM, EN.SRC_SEED])
def test_sampled_kernel_vs_oracle(eng, name, source):
    w, t, prob, op = workload_problem(name)
    src = "substream" if source == EN.SRC_SUBSTREAM else "seed"
    cp = C.CProblem(op)
    for lo, hi, seed in ((0, 20000, 7), (10**9, 10**9 + 5000, 2**63 + 11)):
        got = gpu_key(eng, prob, "sampled", lo, hi, source=source, seed=seed, n_idx=hi)
        assert got == cp.search(src, seed, lo, hi), (lo, seed)


def test_sampled_float_mode(eng):
    w, t, prob, op = workload_problem("cfg4", time_mode="float")
    got = gpu_key(eng, prob, "sampled", 0, 5000, source=EN.SRC_SUBSTREAM, seed=7, n_idx=5000)
    want = C.CProblem(op).search("substream", 7, 0, 5000)
    assert got[1] == want[1] and float(got[0]).hex() == float(want[0]).hex()


# --------------------------------------------------------------------------- schedule / decode
@pytest.mark.parametrize("name", ["cfg1", "cfg4", "hetero6", "cfg5"])
def test_schedule_records_match_oracle(eng, name):
    w, t, prob, op = workload_problem(name)
    cp = C.CProblem(op)
    nprob = EN.NativeProblem(prob, 62)
    ids = [0, 1, 12345, 999999, 2**40 + 17]
    if name == "cfg1":
        opt, node, start, ms = eng.schedule(nprob, EN.SRC_INDEX, ids=[i % prob.space for i in ids])
        cands = [O.decode_index(op, i % prob.space) for i in ids]
    else:
        opt, node, start, ms = eng.schedule(nprob, EN.SRC_SUBSTREAM, seed=7, ids=ids)
        cands = [cp.decode(i, "substream", 7) for i in ids]
    for r, (o, order) in enumerate(cands):
        m, st, nd = cp.eval(o, order)
        assert ms[r] == m
        assert list(opt[r]) == list(o)
        assert [int(x) for x in node[r]] == nd
        assert [float(x) for x in start[r]] == st
    # explicit source reproduces the same rows
    ex = np.array([list(o) + list(order) for o, order in cands], dtype=np.uint8)
    opt2, node2, start2, ms2 = eng.schedule(nprob, EN.SRC_EXPLICIT, explicit=ex)
    assert (ms2 == ms).all() and (start2 == start).all() and (node2 == node).all()


# --------------------------------------------------------------------------- sharding
def test_shards_accumulate_to_full_key(eng):
    """Contiguous shards min-combined (as ranks would with NCCL MIN) == one full search."""
    w, t, prob, op = workload_problem("small5_1x4")
    full = gpu_key(eng, prob, "index")
    idx_bits, _ = prob.key_bits(prob.space)
    nprob = EN.NativeProblem(prob, idx_bits)
    for world in (2, 3, 8):
        keys = []
        for r in range(world):
            best = eng.reset_best()
            a, b = EN._shard(prob.space, r, world)
            eng.search_index(nprob, a, b, best)
            keys.append(int(best.cpu().numpy().view(np.uint64)[0]))
        k = min(keys)
        assert (float(k >> idx_bits), k & ((1 << idx_bits) - 1)) == full
    info = eng.tree_plan(nprob)
    for world in (2, 5):
        keys = []
        for r in range(world):
            best = eng.reset_best()
            a, b = EN._shard(info.n_tasks, r, world)
            eng.search_tree(nprob, info.prefix_len, a, b, best)
            keys.append(int(best.cpu().numpy().view(np.uint64)[0]))
        k = min(keys)
        assert (float(k >> idx_bits), k & ((1 << idx_bits) - 1)) == full


def test_edge_cases(eng):
    rng = random.Random(2)
    # single job, single option, single GPU
    op = random_problem(rng, 1, [1], max_opts=1)
    assert gpu_key(eng, to_search_problem(op), "index") == C.CProblem(op).search()
    # two jobs on 32 GPUs, all radix 1
    op = random_problem(rng, 2, [32], max_opts=1)
    assert gpu_key(eng, to_search_problem(op), "index") == C.CProblem(op).search()
    # empty range leaves the key empty
    prob = to_search_problem(op)
    nprob = EN.NativeProblem(prob, 8)
    best = eng.reset_best()
    eng.search_index(nprob, 1, 1, best)
    assert int(best.cpu().numpy().view(np.uint64)[0]) == 2**64 - 1
    # out-of-range indices are rejected
    from paper_2311_02840_b200 import errors as E
    with pytest.raises(E.InvariantViolation):
        eng.search_index(nprob, 0, prob.space + 1, best)


# --------------------------------------------------------------------------- local search
@pytest.mark.parametrize("name,seed", [("cfg1", 7), ("cfg3", 7), ("cfg3", 11), ("small4_2x2", 7), ("cfg4", 7),
                                       ("cfg4", 2**63 + 5), ("hetero6", 7), ("cfg5", 7)])
def test_local_search_walkers_match_oracle(eng, name, seed):
    """Every walker's whole descent (start = stream candidate, moves, tie-breaks, stop rule)
    equals the oracle's restatement: same final candidate and makespan; and the search key
    over a walker range equals the oracle's."""
    w, t, prob, op = workload_problem(name)
    cp = C.CProblem(op)
    rounds = 64 if name == "cfg5" else 4096
    W = 4 if name == "cfg5" else 48
    bits, _ = prob.key_bits(1 << 20)
    nprob = EN.NativeProblem(prob, bits)
    for walker in range(0, W, max(1, W // 6)):
        ms, o, r, _ = cp.local_search(walker, "substream", seed, rounds)
        go, gr = eng.local_search_state(nprob, EN.SRC_SUBSTREAM, seed, walker, rounds)
        assert (go, gr) == (o, r), (name, walker)
        assert cp.eval(go, gr)[0] == ms
    best = eng.reset_best()
    eng.local_search(nprob, EN.SRC_SUBSTREAM, seed, 0, W, rounds, best)
    k = int(best.cpu().numpy().view(np.uint64)[0])
    ms_, rr_, wk_ = EN.ls_key_fields(k, bits)          # (makespan, rounds scanned, walker)
    assert (float(ms_), wk_) == cp.ls_search("substream", seed, 0, W, rounds)
    assert rr_ == cp.local_search(wk_, "substream", seed, rounds)[3]


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5", "hetero6"])
def test_local_search_stop_at_bound(eng, name):
    """stop_ms = the lower bound: each walker's walk ends at its first candidate with that
    makespan (same final state as the oracle's restatement with the same rule), walkers fall
    out once they have scanned as many rounds as a published key at the bound, and the search
    key -- lowest (makespan, rounds, walker) -- over a walker range equals the oracle's."""
    w, t, prob, op = workload_problem(name)
    cp = C.CProblem(op)
    lb = int(prob.lower_bound())
    rounds = 256 if name == "cfg5" else 4096
    W = 8 if name == "cfg5" else 64
    bits, _ = prob.key_bits(1 << 20)
    nprob = EN.NativeProblem(prob, bits)
    for stop in (lb, lb + 2):
        for walker in range(0, W, max(1, W // 4)):
            ms, o, r, _ = cp.local_search(walker, "substream", 7, rounds, stop_ms=stop)
            assert eng.local_search_state(nprob, EN.SRC_SUBSTREAM, 7, walker, rounds, stop_ms=stop) == (o, r)
            full = cp.local_search(walker, "substream", 7, rounds)[0]
            assert ms == full or (ms <= stop and full <= ms), (name, walker, ms, full)
        best = eng.reset_best()
        eng.local_search(nprob, EN.SRC_SUBSTREAM, 7, 0, W, rounds, best, stop_ms=stop)
        k = int(best.cpu().numpy().view(np.uint64)[0])
        ms_, rr_, wk_ = EN.ls_key_fields(k, bits)
        got = (float(ms_), wk_)
        assert got == cp.ls_search("substream", 7, 0, W, rounds, stop_ms=stop)
        assert rr_ == cp.local_search(wk_, "substream", 7, rounds, stop_ms=stop)[3]
        full_key = cp.ls_search("substream", 7, 0, W, rounds)
        if full_key[0] > stop:                         # the bound was not reached: same key as the full walks
            assert got == full_key


@pytest.mark.parametrize("name,stop", [("cfg3", -1), ("cfg4", 8), ("hetero6", -1)])
def test_local_search_records_every_walker_state(eng, name, stop):
    """One launch over a walker range records every walker's final candidate (the winner's
    plan needs no replay): each equals the oracle's walk, and the engine's search result
    carries the winner's."""
    import torch

    w, t, prob, op = workload_problem(name)
    cp = C.CProblem(op)
    bits, _ = prob.key_bits(1 << 20)
    nprob = EN.NativeProblem(prob, bits)
    W, lo = 24, 5
    buf = torch.zeros(W * 2 * prob.J, dtype=torch.uint8, device="cuda")
    eng.local_search(nprob, EN.SRC_SUBSTREAM, 7, lo, lo + W, 4096, eng.reset_best(), state_out=buf, stop_ms=stop)
    got = buf.cpu().numpy().reshape(W, 2 * prob.J)
    for i in range(W):
        _, o, r, _ = cp.local_search(lo + i, "substream", 7, 4096, stop_ms=stop)
        assert got[i].tolist() == o + r, (name, i)
    for start in ("greedy", "sampled"):
        res = eng.search(prob, SolveOptions(search="local", walkers=64, wave=64, seed=7, ls_start=start))
        assert res.state is not None
        assert res.source == (EN.SRC_GREEDY if start == "greedy" else EN.SRC_SUBSTREAM)
        src = "greedy" if start == "greedy" else "substream"
        _, o, r, _ = cp.local_search(res.index, src, 7, 4096, stop_ms=res.stats["stop_ms"])
        assert (list(res.state[0]), list(res.state[1])) == (o, r)


@pytest.mark.parametrize("group", ["1", "4", "8", "16", "32"])
def test_local_search_wide_nodes_register_path(eng, group, monkeypatch):
    """Nodes of 9-32 GPUs (padded 16 / 32; with 8 warps per walker the move evaluation shifts
    in registers when the warp's lanes place equal gang sizes, in shared memory otherwise), with
    releases and initial free times: every walker's final candidate equals the oracle's."""
    monkeypatch.setenv("SATURN_LS_GROUP", group)
    rng = random.Random(17)
    for trial in range(8):
        nodes = [[16], [12], [32], [24]][trial % 4]
        op = random_problem(rng, rng.randint(4, 8), nodes, max_opts=4, max_d=9)
        if trial % 2:
            op.release = [rng.randint(0, 4) for _ in range(op.J)]
            op.init_free = [[rng.randint(0, 3) for _ in range(n)] for n in nodes]
        prob = to_search_problem(op)
        bits, _ = prob.key_bits(1 << 10)
        nprob = EN.NativeProblem(prob, bits)
        cp = C.CProblem(op)
        for walker in (0, 5, 9):
            ms, o, r, _ = cp.local_search(walker, "substream", 3, 4096)
            assert eng.local_search_state(nprob, EN.SRC_SUBSTREAM, 3, walker, 4096) == (o, r), (trial, walker)
        best = eng.reset_best()
        eng.local_search(nprob, EN.SRC_SUBSTREAM, 3, 0, 32, 4096, best)
        k = int(best.cpu().numpy().view(np.uint64)[0])
        ms_, _, wk_ = EN.ls_key_fields(k, bits)
        assert (float(ms_), wk_) == cp.ls_search("substream", 3, 0, 32, 4096), trial


def test_local_search_seed_source_and_release(eng):
    rng = random.Random(9)
    for trial in range(6):
        nodes = [[6], [4, 4], [8]][trial % 3]
        op = random_problem(rng, rng.randint(3, 7), nodes, max_opts=4, max_d=9, hetero=trial == 4)
        if trial % 2:
            op.release = [rng.randint(0, 4) for _ in range(op.J)]
            op.init_free = [[rng.randint(0, 3) for _ in range(n)] for n in nodes]
        prob = to_search_problem(op)
        bits, _ = prob.key_bits(1 << 10)
        nprob = EN.NativeProblem(prob, bits)
        cp = C.CProblem(op)
        for walker in (0, 3, 11):
            ms, o, r, _ = cp.local_search(walker, "seed", 5, 4096)
            assert eng.local_search_state(nprob, EN.SRC_SEED, 5, walker, 4096) == (o, r), (trial, walker)


@pytest.mark.parametrize("group", ["1", "16"])
def test_local_search_greedy_starts(eng, group, monkeypatch):
    """SAT_SRC_GREEDY (the default start): every job at its least-area option, jobs in the
    perturbed longest-first order of the walker's substream -- one node, several nodes,
    heterogeneous nodes, releases and initial free times, 1 and 16 warps per walker: each
    walker's final candidate, and the search key over a walker range with and without the stop
    at the bound, equal the oracle's restatement (greedy_start + the same walk)."""
    monkeypatch.setenv("SATURN_LS_GROUP", group)
    rng = random.Random(23)
    cases = [workload_problem(n)[2:] for n in ("cfg3", "cfg4", "hetero6")]
    for trial in range(8):
        nodes = [[8], [4, 4], [16], [6, 3], [2, 2, 2]][trial % 5]
        op = random_problem(rng, rng.randint(3, 9), nodes, max_opts=4, max_d=9, hetero=trial % 3 == 2)
        if trial % 2:
            op.release = [rng.randint(0, 4) for _ in range(op.J)]
            op.init_free = [sorted(rng.randint(0, 3) for _ in range(n)) for n in nodes]
        cases.append((to_search_problem(op), op))
    for prob, op in cases:
        cp = C.CProblem(op)
        bits, _ = prob.key_bits(1 << 10)
        nprob = EN.NativeProblem(prob, bits)
        lb = int(prob.lower_bound())
        for walker in (0, 1, 7):
            ms, o, r, _ = cp.local_search(walker, "greedy", 11, 4096)
            assert eng.local_search_state(nprob, EN.SRC_GREEDY, 11, walker, 4096) == (o, r), (prob.J, walker)
        for stop in (-1, lb):
            best = eng.reset_best()
            eng.local_search(nprob, EN.SRC_GREEDY, 11, 0, 24, 4096, best, stop_ms=stop)
            k = int(best.cpu().numpy().view(np.uint64)[0])
            ms_, rr_, wk_ = EN.ls_key_fields(k, bits)
            assert (float(ms_), wk_) == cp.ls_search("greedy", 11, 0, 24, 4096, stop_ms=stop)
            assert rr_ == cp.local_search(wk_, "greedy", 11, 4096, stop_ms=stop)[3]


def test_bnb_fixed_depth_walkers_equal_full_scan(eng):
    """Suffixes of 5-7 jobs (fixed-depth walkers D = 3..5) on a 9-job one-node problem: the
    bound-and-prune key equals the full scan's for every prefix length."""
    from paper_2311_02840_b200.workloads import synthetic_workload

    w = synthetic_workload(9, 1, 8)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w)
    want = gpu_key(eng, prob, "tree")
    for prefix in (2, 3, 4, 5, 6):
        assert bnb_key(eng, prob, prefix=prefix) == want, prefix
