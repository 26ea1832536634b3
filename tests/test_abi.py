"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/ declares.

No compute call needs a GPU here: only the pure-host entry points are exercised."""

import ctypes
import math
import os
import re

import pytest

from helpers import golden_workload

from paper_2311_02840_b200 import build as B
from paper_2311_02840_b200 import engine as EN
from paper_2311_02840_b200.problem import build_problem
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "saturn_engine.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*(sat_\w+)\s*\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return EN.load_library()


def test_header_declarations_bound(lib):
    names = declared()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n
        assert n in EN._SIGS, f"{n} not bound in engine._SIGS"


def test_host_only_entry_points(lib):
    assert lib.sat_abi_version() == 8
    for st in range(6):
        assert lib.sat_error_string(st)


def test_sass_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {B.OUT} 2>&1").read()
    assert "sm_100a" in out


def test_tree_plan_layout_host_only(lib):
    w, _ = golden_workload("cfg1")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w)
    nprob = EN.NativeProblem(prob, 35)
    info = EN.SatTreeInfo()
    assert lib.sat_tree_plan(nprob.ref, 0, ctypes.byref(info)) == 0
    assert info.n_candidates == prob.space == 32514048000
    assert info.prefix_len == 4 and info.n_sets == math.comb(8, 4)
    assert info.n_tasks >= 1 << 15
    # placements of the prefix-shared walk are far fewer than J per candidate
    assert prob.space < info.n_job_steps < 2 * prob.space
    for P in (1, 3, 6):
        assert lib.sat_tree_plan(nprob.ref, P, ctypes.byref(info)) == 0
        assert info.prefix_len == P and info.n_candidates == prob.space
    assert lib.sat_tree_plan(nprob.ref, 7, ctypes.byref(info)) == EN.SAT_ERR_INVALID


def test_tree_plan_reports_packed_pair_pass(lib, monkeypatch):
    """The pair pass packs two 16-bit free times per word when every reachable free time
    (latest initial free time + each job's longest option) is below 0x7000."""
    w, _ = golden_workload("cfg1")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w)
    nprob = EN.NativeProblem(prob, 35)
    info = EN.SatTreeInfo()
    assert ctypes.sizeof(info) == 40
    assert lib.sat_tree_plan(nprob.ref, 0, ctypes.byref(info)) == 0
    assert info.pair_packed == 1
    monkeypatch.setenv("SATURN_TREE_PACKED", "0")
    assert lib.sat_tree_plan(nprob.ref, 0, ctypes.byref(info)) == 0
    assert info.pair_packed == 0
    monkeypatch.delenv("SATURN_TREE_PACKED")
    horizon = sum(int(max(nprob.dur[j, :prob.radix[j], 0])) for j in range(prob.J))
    nprob.dur[:] *= 0x7000 // horizon + 1                      # past the limit (same buffer)
    assert lib.sat_tree_plan(nprob.ref, 0, ctypes.byref(info)) == 0
    assert info.pair_packed == 0


def test_validation_codes(lib):
    w, _ = golden_workload("small5_1x4")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w)
    nprob = EN.NativeProblem(prob, 20)
    info = EN.SatTreeInfo()
    nprob.radix[2] = 0
    assert lib.sat_tree_plan(nprob.ref, 0, ctypes.byref(info)) == EN.SAT_ERR_NO_OPTIONS
    nprob.radix[2] = prob.radix[2]
    nprob.struct.G = 3
    assert lib.sat_tree_plan(nprob.ref, 0, ctypes.byref(info)) == EN.SAT_ERR_INVALID
    w4, _ = golden_workload("small4_2x2")
    t4 = build_profile_table(w4, SyntheticExecutor(w4.cluster))
    p4 = EN.NativeProblem(build_problem(t4, w4), 20)
    assert lib.sat_tree_plan(p4.ref, 0, ctypes.byref(info)) == EN.SAT_ERR_UNSUPPORTED


def test_tree_shard_partitions_and_balances_work(lib):
    """sat_tree_shard: contiguous ranges covering every warp task once, each with ~1/world of
    the full-scan device cost (host-only entry point).  Cost model: a pair node = a fixed part
    + one group per gang of each of its two jobs; an upper-level node = one merge; a task = the
    prefix decode (constants from the k_tree source profile)."""
    w, _ = golden_workload("cfg1")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w)
    bits, _ = prob.key_bits(prob.space)
    nprob = EN.NativeProblem(prob, bits)
    info = EN.SatTreeInfo()
    assert lib.sat_tree_plan(nprob.ref, 5, ctypes.byref(info)) == 0
    radix, J, P = [int(r) for r in prob.radix], prob.J, 5
    memo = {}

    def walk(rem):
        jobs = [j for j in range(J) if rem >> j & 1]
        if len(jobs) < 2:
            return 0.0
        if rem not in memo:
            if len(jobs) == 2:
                memo[rem] = 110.0 + 14.0 * (radix[jobs[0]] + radix[jobs[1]])
            else:
                memo[rem] = sum(radix[j] * (25.0 + walk(rem & ~(1 << j))) for j in jobs)
        return memo[rem]

    per_task = []       # cost of every warp task, in layout order (sets in mask order)
    for S in range(1 << J):
        if bin(S).count("1") != P:
            continue
        npref = math.factorial(P) * math.prod(radix[j] for j in range(J) if S >> j & 1)
        per_task += [250.0 + walk(((1 << J) - 1) & ~S)] * ((npref + 31) // 32)
    assert len(per_task) == info.n_tasks
    total = sum(per_task)
    for world in (2, 3, 8):
        prev = 0
        for r in range(world):
            lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
            assert lib.sat_tree_shard(nprob.ref, 5, world, r, ctypes.byref(lo), ctypes.byref(hi)) == 0
            assert lo.value == prev
            prev = hi.value
            share = sum(per_task[lo.value:hi.value]) / (total / world)
            assert 0.98 < share < 1.02, (world, r, share)
        assert prev == info.n_tasks
    assert lib.sat_tree_shard(nprob.ref, 5, 2, 2, ctypes.byref(lo), ctypes.byref(hi)) == EN.SAT_ERR_INVALID


def test_no_options_status_names_the_job(lib):
    """SAT_ERR_NO_OPTIONS from the library becomes NoFeasibleConfig carrying the offending job's
    id (errors.py:23-26), not a placeholder."""
    from paper_2311_02840_b200 import errors as E

    w, _ = golden_workload("small5_1x4")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w)
    prob.radix[2] = 0                                   # job 2 loses every option
    nprob = EN.NativeProblem(prob, 30)
    nbytes = ctypes.c_size_t()
    st = lib.sat_workspace_bytes(nprob.ref, ctypes.byref(nbytes))
    assert st == EN.SAT_ERR_NO_OPTIONS
    eng = EN.Engine.__new__(EN.Engine)                 # host-only: no device needed to map a status
    eng.lib = lib
    with pytest.raises(E.NoFeasibleConfig) as exc:
        eng._check(st, nprob=nprob)
    assert prob.job_ids[2] in str(exc.value)


def test_tree_layout_memo_is_transparent(lib):
    """The per-process tree-layout memo returns the same plan for repeated and interleaved calls."""
    w, _ = golden_workload("cfg1")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    prob = build_problem(t, w)
    nprob = EN.NativeProblem(prob, 35)
    first = {}
    for rep in range(3):
        for P in (0, 1, 2, 3, 4, 5, 6):
            info = EN.SatTreeInfo()
            assert lib.sat_tree_plan(nprob.ref, P, ctypes.byref(info)) == 0
            got = (info.prefix_len, info.n_sets, info.n_tasks, info.n_candidates, info.n_job_steps)
            assert first.setdefault(P, got) == got
            lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
            assert lib.sat_tree_shard(nprob.ref, P, 3, 1, ctypes.byref(lo), ctypes.byref(hi)) == 0
            assert 0 < lo.value < hi.value < info.n_tasks
