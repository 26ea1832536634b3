"""The package's host-side restatements behave exactly like the reference's own code on random
inputs (CPU; the reference package comes from baseline/_ref or the reference source tree):

* ``domain.check_plan`` (array passes) vs ``core.check_plan`` (core.py:254-287): same verdict
  class and message on random valid and broken plans;
* ``formats.parse_profiles`` (columnar reader) vs ``profiling.load_profiles``
  (profiling.py:173-209): same table, or the same error class, line number and message, on
  randomly corrupted CSV text;
* ``profiling.build_profile_table`` (row-wise cost model) vs the reference's: bit-identical
  entries and profiling charge on random workloads.
"""

import random

import pytest

from helpers import import_reference, reference_available

from paper_2311_02840_b200 import domain as D
from paper_2311_02840_b200 import errors as E
from paper_2311_02840_b200 import formats as F
from paper_2311_02840_b200 import profiling as P

pytestmark = pytest.mark.skipif(not reference_available(), reason="run tools/install_reference.sh")


def _random_workload(rng, n_jobs=None):
    techs = [D.TechniqueSpec(name="ddp", archetype="replicated", serial_fraction=0.02, comm_overhead=0.01),
             D.TechniqueSpec(name="fsdp", archetype="sharded", serial_fraction=rng.choice([0.0, 0.05]),
                             comm_overhead=0.03, min_gpus=rng.choice([1, 2])),
             D.TechniqueSpec(name="gpipe", archetype="pipelined", serial_fraction=0.15, comm_overhead=0.005),
             D.TechniqueSpec(name="spill", archetype="offloaded", serial_fraction=0.02, comm_overhead=0.01,
                             offload_multiplier=rng.choice([1.5, 2.5]))]
    rng.shuffle(techs)
    nodes = tuple(D.NodeSpec(f"n{i}", rng.choice([2, 4, 8]), rng.choice([24.0, 40.0, 80.0]))
                  for i in range(rng.randint(1, 3)))
    jobs = tuple(D.JobSpec(f"j{i:02d}", rng.randint(1, 20000), rng.uniform(0.1, 5.0), rng.uniform(1, 200),
                           rng.uniform(0, 10)) for i in range(n_jobs or rng.randint(1, 6)))
    return D.Workload(jobs, D.ClusterSpec(nodes), tuple(techs))


def _to_ref(core, w):
    return core.Workload.model_validate({"jobs": [j.__dict__ for j in w.jobs],
                                         "cluster": {"nodes": [n.__dict__ for n in w.cluster.nodes]},
                                         "techniques": [t.__dict__ for t in w.techniques]})


def _verdict(fn):
    try:
        fn()
        return ("ok", "")
    except Exception as exc:  # noqa: BLE001 -- compare class name and message
        return (type(exc).__name__, str(exc))


def test_build_profile_table_bit_identical():
    core, profiling, _ = import_reference()
    rng = random.Random(5)
    for _ in range(60):
        w = _random_workload(rng)
        mine = P.build_profile_table(w, P.SyntheticExecutor(w.cluster))
        rw = _to_ref(core, w)
        ref = profiling.build_profile_table(rw, profiling.SyntheticExecutor(rw.cluster))
        assert list(mine.entries) == list(ref.entries)
        assert [v.hex() for v in mine.entries.values()] == [v.hex() for v in ref.entries.values()]
        assert mine.profiling_cost.hex() == ref.profiling_cost.hex()


def _random_plan(rng, w, table):
    entries, rts = {}, {}
    for job in w.jobs:
        rows = P.feasible_entries(table, job, w)
        cfg, lat = rng.choice(rows)
        g = cfg.gpus
        if rng.random() < 0.05:
            g = g + rng.choice([-1, 8])
        node = rng.choice(w.cluster.nodes).id
        entries[job.id] = D.PlanEntry(D.RunConfig(cfg.technique, max(1, g)), node,
                                      float(rng.choice([0, 1, 2, 5, 10, rng.uniform(0, 20)])))
        rts[job.id] = rng.choice([lat * 3, 5.0, 1.0, 0.0, -2.0 if rng.random() < 0.05 else 2.0])
    last = max(e.start_time + rts[j] for j, e in entries.items())
    pred = last + rng.choice([0.0, 1.0, -1e-3, -1.0, 1e-7])
    if rng.random() < 0.05:
        entries.pop(next(iter(entries)))
    return entries, max(0.0, pred), rts


def test_check_plan_same_verdicts_as_reference():
    core, profiling, _ = import_reference()
    rng = random.Random(11)
    seen = set()
    for _ in range(600):
        w = _random_workload(rng)
        t = P.build_profile_table(w, P.SyntheticExecutor(w.cluster))
        rw = _to_ref(core, w)
        entries, pred, rts = _random_plan(rng, w, t)
        mine = D.Plan(entries, pred)
        ref = core.Plan(entries={k: core.PlanEntry(config=core.RunConfig(technique=e.config.technique,
                                                                          gpus=e.config.gpus),
                                                    node=e.node, start_time=e.start_time)
                                 for k, e in entries.items()}, predicted_makespan=pred)
        a = _verdict(lambda: D.check_plan(mine, w, rts))
        b = _verdict(lambda: core.check_plan(ref, rw, rts))
        assert a == b
        seen.add(a[0])
    assert {"ok", "CapacityViolation", "InvalidPlan"} <= seen


def _mutate(rng, text):
    lines = text.split("\n")
    for _ in range(rng.randint(0, 3)):
        i = rng.randrange(len(lines))
        ln = lines[i]
        op = rng.randrange(9)
        if op == 0:
            lines[i] = ln + ",x"
        elif op == 1 and ln:
            f = ln.split(",")
            if len(f) == 4:
                f[2] = rng.choice(["0", "-1", "two", " 3 ", "+2", "1_0", ""])
                lines[i] = ",".join(f)
        elif op == 2 and ln:
            f = ln.split(",")
            if len(f) == 4:
                f[3] = rng.choice(["0", "-0.5", "nan?", " inf", "inf", "1e-3", "Infinity", "-inf"])
                lines[i] = ",".join(f)
        elif op == 3 and i > 0:
            lines.insert(i, lines[rng.randrange(1, len(lines))])
        elif op == 4:
            lines.insert(i, "   ")
        elif op == 5 and i == 0:
            lines[0] = rng.choice(["job,technique,gpus", " job,technique,gpus,latency_s ", ""])
        elif op == 6:
            lines[i] = ln.replace(",", ", ")
    return "\n".join(lines)


def test_profile_csv_reader_same_as_reference(tmp_path):
    core, profiling, _ = import_reference()
    from jointsched import errors as RE  # noqa: F401 -- error classes compared by name + message

    rng = random.Random(3)
    kinds = set()
    for k in range(400):
        w = _random_workload(rng, n_jobs=rng.randint(1, 3))
        t = P.build_profile_table(w, P.SyntheticExecutor(w.cluster))
        text = _mutate(rng, F.dump_profiles(t))
        p = tmp_path / f"p{k}.csv"
        p.write_text(text, encoding="utf-8")

        def mine():
            return F.parse_profiles(text)

        def ref():
            return profiling.load_profiles(p)

        a, b = _verdict(mine), _verdict(ref)
        assert a == b, text
        kinds.add(a[0])
        if a[0] == "ok":
            ma, rb = mine(), ref()
            assert list(ma.entries.items()) == list(rb.entries.items()) and ma.provenance == rb.provenance
            err = getattr(E, "ParseError")
            assert err is not None
        else:
            la, lb = None, None
            try:
                mine()
            except E.SchedulerError as exc:
                la = exc.line_no
            try:
                ref()
            except Exception as exc:  # noqa: BLE001
                lb = exc.line_no
            assert la == lb
    assert {"ok", "ParseError", "NegativeLatency"} <= kinds


def test_profile_csv_writer_same_bytes_as_reference(tmp_path):
    core, profiling, _ = import_reference()
    rng = random.Random(9)
    for k in range(20):
        w = _random_workload(rng)
        rw = _to_ref(core, w)
        rt = profiling.build_profile_table(rw, profiling.SyntheticExecutor(rw.cluster))
        profiling.save_profiles(rt, tmp_path / "r.csv")
        F.save_profiles(P.build_profile_table(w, P.SyntheticExecutor(w.cluster)), tmp_path / "m.csv")
        assert (tmp_path / "r.csv").read_bytes() == (tmp_path / "m.csv").read_bytes()
