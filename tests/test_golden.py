"""Pin the oracle AND the product's host mirror to vectors produced by the reference itself.

tests/golden/reference_golden.json is written by tests/golden/make_golden.py, which
runs the reference package (jointsched core / profiling / rng) -- see that file.
"""

import hashlib
import json
import math

import pytest

from helpers import golden, golden_workload, unhex

from oracle import saturn_oracle as O
from paper_2311_02840_b200 import domain as D
from paper_2311_02840_b200 import errors as E
from paper_2311_02840_b200 import profiling as P
from paper_2311_02840_b200 import rng as R
from paper_2311_02840_b200.workloads import CONFIGS, synthetic_workload

NAMES = ["cfg1", "cfg3", "cfg4", "cfg5", "small5_1x4", "small4_2x2", "hetero6", "tiny3_1x3"]


def fhex(x):
    return "inf" if math.isinf(x) else float(x).hex()


def digest(obj):
    return hashlib.sha256(json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


# ------------------------------------------------------------------ rng (rng.py:20-56)
@pytest.mark.parametrize("impl", ["oracle", "product"])
def test_rng_vectors(impl):
    g = golden()["rng"]
    mk = (lambda s: O.Rng(s)) if impl == "oracle" else (lambda s: R.SplitMix64(s))
    sub = O.substream if impl == "oracle" else R.substream
    s = mk(0)
    assert [hex(s.next_u64()) for _ in range(3)] == g["splitmix0_first3"]
    s = mk(7)
    assert [s.below(10) for _ in range(10)] == g["below10_seed7"]
    s = mk(7)
    items = list(range(8))
    s.shuffle(items)
    assert items == g["shuffle8_seed7"]
    assert hex(sub(7, 1, 2).next_u64()) == g["substream_7_1_2_first"]
    s = sub(7, 1)
    assert [fhex(s.uniform()) for _ in range(64)] == g["uniform_substream_7_1_first64"]
    for d in g["random_draws"]:
        s = mk(int(d["seed"])) if "seed" in d else sub(*d["substream"])
        assert [s.below(r) for r in d["radix"]] == d["opts"]
        order = list(range(len(d["radix"])))
        s.shuffle(order)
        assert order == d["order"]


# ------------------------------------------------------------------ SPEC known answers
def test_spec_examples_product():
    g = golden()["spec"]
    job = D.JobSpec(id="a", total_batches=10000, base_batch_time=1.0, model_memory=1.0)
    t = D.TechniqueSpec(name="t", archetype="sharded", serial_fraction=0.2, comm_overhead=0.01)
    lat = P.synthetic_latency(job, t, 4, 100.0)
    assert fhex(lat) == g["latency_0.43"]
    t3 = D.TechniqueSpec(name="o", archetype="offloaded", serial_fraction=0.0, comm_overhead=0.0,
                         offload_multiplier=3.0)
    assert fhex(P.synthetic_latency(job, t3, 1, 100.0)) == g["latency_offload_3"]
    tab = P.ProfileTable({("a", "t", 4): lat}, "synthetic")
    assert fhex(P.estimate_runtime(tab, job, D.RunConfig("t", 4), 10000)) == g["estimate_4300"]
    j32 = D.JobSpec(id="m", total_batches=1, base_batch_time=1.0, model_memory=32.0, activation_memory=4.0)
    sh = D.TechniqueSpec(name="s", archetype="sharded", serial_fraction=0.0, comm_overhead=0.0)
    rp = D.TechniqueSpec(name="r", archetype="replicated", serial_fraction=0.0, comm_overhead=0.0)
    of = D.TechniqueSpec(name="o", archetype="offloaded", serial_fraction=0.0, comm_overhead=0.0)
    j500 = D.JobSpec(id="b", total_batches=1, base_batch_time=1.0, model_memory=500.0)
    assert [D.memory_feasible(j32, sh, 4, 12.0), D.memory_feasible(j32, rp, 8, 12.0),
            D.memory_feasible(j500, of, 1, 12.0)] == g["memory"]
    with pytest.raises(E.InfeasibleEntry):
        P.ProfileTable({("a", "t", 4): math.inf}, "x").latency("a", "t", 4)
    with pytest.raises(E.MissingEntry):
        P.ProfileTable({}, "x").latency("a", "t", 4)


def test_spec_examples_oracle():
    g = golden()["spec"]

    class C:  # minimal cluster for the oracle's latency()
        nodes = (D.NodeSpec("n", 8, 100.0),)
    job = D.JobSpec(id="a", total_batches=10000, base_batch_time=1.0, model_memory=1.0)
    t = D.TechniqueSpec(name="t", archetype="sharded", serial_fraction=0.2, comm_overhead=0.01)
    assert fhex(O.latency(job, t, 4, C)) == g["latency_0.43"]
    assert fhex(10000 * O.latency(job, t, 4, C)) == g["estimate_4300"]


# ------------------------------------------------------------------ profile tables
def _records(entries, w, table_entries):
    fe = {}
    rt = {}
    fc = {}
    for j in w.jobs:
        fc[j.id] = [[c.technique, c.gpus] for c in D.feasible_configs(j, w.cluster, w.techniques)]
        rows = P.feasible_entries(table_entries, j, w)
        fe[j.id] = [[c.technique, c.gpus, fhex(lat)] for c, lat in rows]
        rt[j.id] = [fhex(P.estimate_runtime(table_entries, j, c, j.total_batches)) for c, _ in rows]
    return {"entries": entries, "feasible_configs": fc, "feasible_entries": fe, "runtime_total": rt}


@pytest.mark.parametrize("name", NAMES)
def test_product_profile_table_matches_reference(name):
    w, rec = golden_workload(name)
    table = P.build_profile_table(w, P.SyntheticExecutor(w.cluster))
    entries = [[k[0], k[1], k[2], fhex(v)] for k, v in table.entries.items()]
    got = _records(entries, w, table)
    assert fhex(table.profiling_cost) == rec["profiling_cost"]
    if "sha256" in rec:
        assert len(entries) == rec["n_entries"]
        for k, h in rec["sha256"].items():
            assert digest(got[k]) == h, k
    else:
        for k in ("entries", "feasible_configs", "feasible_entries", "runtime_total"):
            assert got[k] == rec[k], k


@pytest.mark.parametrize("name", NAMES)
def test_oracle_profile_table_matches_reference(name):
    w, rec = golden_workload(name)
    ent = O.profile_entries(w)
    entries = [[k[0], k[1], k[2], fhex(v)] for k, v in ent.items()]
    fe = {j.id: [[t, g, fhex(lat)] for t, g, lat in O.options_of(ent, j, w)] for j in w.jobs}
    if "sha256" in rec:
        assert digest(entries) == rec["sha256"]["entries"]
        assert digest(fe) == rec["sha256"]["feasible_entries"]
    else:
        assert entries == rec["entries"]
        assert fe == rec["feasible_entries"]


@pytest.mark.parametrize("k", [1, 3, 4, 5])
def test_workload_recipe_matches_reference(k):
    """workloads.synthetic_workload == the reference-built recipe (golden)."""
    c = CONFIGS[k]
    w = synthetic_workload(c["jobs"], c["nodes"], c["gpus"], c["techs"])
    gw, _ = golden_workload(f"cfg{k}")
    assert w == gw


# ------------------------------------------------------------------ check_plan verdicts
@pytest.mark.parametrize("name", ["cfg1", "small4_2x2", "hetero6"])
def test_check_plan_verdicts(name):
    w, rec = golden_workload(name)
    for case in rec["check_plan"]:
        entries = {k: D.PlanEntry(D.RunConfig(v[0], v[1]), v[2], unhex(v[3])) for k, v in case["entries"].items()}
        plan = D.Plan(entries=entries, predicted_makespan=unhex(case["predicted"]))
        rts = {k: unhex(v) for k, v in case["runtimes"].items()}
        try:
            D.check_plan(plan, w, rts)
            verdict = "ok"
        except E.SchedulerError as exc:
            verdict = type(exc).__name__
        assert verdict == case["verdict"], case["kind"]


def test_validate_workload_errors():
    w, _ = golden_workload("cfg1")
    D.validate_workload(w)
    dup = D.Workload(jobs=w.jobs + (w.jobs[0],), cluster=w.cluster, techniques=w.techniques)
    with pytest.raises(E.DuplicateId):
        D.validate_workload(dup)
    rep_only = (D.TechniqueSpec(name="r", archetype="replicated", serial_fraction=0.0, comm_overhead=0.0),)
    big = D.JobSpec(id="x", total_batches=1, base_batch_time=1.0, model_memory=200.0)
    with pytest.raises(E.NoFeasibleConfig):
        D.validate_workload(D.Workload(jobs=(big,), cluster=w.cluster, techniques=rep_only))
    with pytest.raises(E.InvariantViolation):
        D.TechniqueSpec(name="bad", archetype="sharded", serial_fraction=0.1, comm_overhead=0.0,
                        offload_multiplier=2.0)
