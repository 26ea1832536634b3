"""The drop-in boundary with the reference's OWN objects on the B200.

The reference package (``jointsched`` core / profiling / rng / errors, unmodified) is installed
into ``baseline/_ref`` by ``tools/install_reference.sh`` and travels to the GPU box with the repo
snapshot.  Its pydantic ``Workload`` / ``ProfileTable`` (``build_profile_table``,
profiling.py:122-144, or ``load_profiles``, profiling.py:173-209) and ``RunningContext``
(core.py:211-223) go straight into this package's planners; the plans that come back are
``core.Plan`` objects (core.py:114-120), validated by the reference's own ``core.check_plan``
(core.py:254-287), and must be the very plans the engine returns for this package's mirror
objects (same index order and tie-break) -- and, where a CPU check is affordable, the oracle's.
"""

import json
import math
import os

import pytest

from helpers import golden, golden_workload, import_reference, reference_available

from oracle import coracle as C
from oracle import saturn_oracle as O
from paper_2311_02840_b200 import domain as D
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200 import simulator as SIM
from paper_2311_02840_b200.problem import SolveOptions
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not reference_available(), reason="run tools/install_reference.sh")]

WINNERS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "winners.json")


def ref_workload(core, w):
    """The mirror workload as the reference's pydantic model (core.py:123-142)."""
    return core.Workload.model_validate({"jobs": [j.__dict__ for j in w.jobs],
                                         "cluster": {"nodes": [n.__dict__ for n in w.cluster.nodes]},
                                         "techniques": [t.__dict__ for t in w.techniques]})


def ref_setup(name):
    core, profiling, _ = import_reference()
    w, _ = golden_workload(name)
    rw = ref_workload(core, w)
    rt = profiling.build_profile_table(rw, profiling.SyntheticExecutor(rw.cluster))
    return core, profiling, w, rw, rt


def entries_of(plan):
    return {jid: (e.config.technique, e.config.gpus, e.node, e.start_time) for jid, e in plan.entries.items()}


def ref_runtimes(profiling, rt, rw, plan, ctx=None):
    """Per-job runtime of the plan's configs by the reference's estimate_runtime (profiling.py:147),
    plus rho for a running job whose (technique, g, node) changed."""
    out = {}
    for jid, e in plan.entries.items():
        rem = rw.job(jid).total_batches if ctx is None else ctx.remaining[jid]
        r = profiling.estimate_runtime(rt, rw.job(jid), e.config, rem)
        if ctx is not None and jid in ctx.current and ctx.current[jid] != (e.config.technique, e.config.gpus, e.node):
            r += ctx.checkpoint_cost
        out[jid] = r
    return out


@pytest.mark.parametrize("name", ["small5_1x4", "small4_2x2", "hetero6", "cfg1"])
def test_plan_saturn_reference_objects(name):
    core, profiling, w, rw, rt = ref_setup(name)
    plan = PL.plan_saturn(rt, rw)
    assert type(plan) is core.Plan
    core.check_plan(plan, rw, ref_runtimes(profiling, rt, rw, plan))
    # the same plan as for the mirror objects
    mirror = PL.solve(build_profile_table(w, SyntheticExecutor(w.cluster)), w)
    assert entries_of(plan) == entries_of(mirror.plan)
    assert plan.predicted_makespan == mirror.plan.predicted_makespan
    if name == "cfg1":
        win = json.load(open(WINNERS))["cfg1"]
        assert mirror.status == "Optimal" and (mirror.makespan, mirror.search.index) == (win["makespan"], win["index"])
    else:
        op = O.build(rt.entries, rw)
        if op.space <= 10 ** 7:                 # the oracle's full scan finishes in seconds
            assert (mirror.makespan, mirror.search.index) == C.CProblem(op).search()


def test_job_list_call_shape():
    """SPEC.md:276's ``plan_saturn(table, jobs, cluster, techniques=...)`` for both object families
    (the job-list view offers the ``technique`` / ``job`` lookups check_plan needs)."""
    core, profiling, w, rw, rt = ref_setup("small4_2x2")
    a = PL.plan_saturn(rt, list(rw.jobs), rw.cluster, techniques=rw.techniques)
    b = PL.plan_saturn(rt, rw)
    assert type(a) is core.Plan and entries_of(a) == entries_of(b)
    sol = PL.solve(rt, list(rw.jobs), rw.cluster, techniques=list(rw.techniques))
    assert entries_of(sol.plan) == entries_of(b)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    m = PL.plan_saturn(t, list(w.jobs), w.cluster, techniques=w.techniques)
    assert type(m) is D.Plan and entries_of(m) == entries_of(b)
    from paper_2311_02840_b200 import milp

    bb = milp.branch_and_bound(milp.build_milp(t, list(w.jobs), w.cluster, techniques=w.techniques))
    assert bb.status == "Optimal"


def test_resolve_with_reference_running_context():
    core, profiling, w, rw, rt = ref_setup("cfg1")
    first = PL.plan_saturn(rt, rw)
    remaining = {j.id: j.total_batches // 2 for j in rw.jobs[:5]}     # five unfinished jobs
    running = {jid: (e.config.technique, e.config.gpus, e.node)
               for jid, e in first.entries.items() if e.start_time == 0.0 and jid in remaining}
    assert running
    ctx = core.RunningContext(remaining=remaining, current=running, checkpoint_cost=30.0)
    sol = PL.solve(rt, rw, None, None, ctx)
    plan = sol.plan
    assert type(plan) is core.Plan and set(plan.entries) == set(remaining)
    sub = core.Workload(jobs=[rw.job(j) for j in sorted(remaining)], cluster=rw.cluster, techniques=rw.techniques)
    rts = ref_runtimes(profiling, rt, rw, plan, ctx)
    assert all(math.isclose(rts[j], sol.runtimes[j], rel_tol=0, abs_tol=0) for j in rts)
    core.check_plan(plan, sub, rts)
    # = the mirror re-solve, = the oracle's exhaustive lowest-index scan of the re-solve space
    mctx = D.RunningContext(remaining=dict(remaining), current=dict(running), checkpoint_cost=30.0)
    mw, _ = golden_workload("cfg1")
    msol = PL.solve(build_profile_table(mw, SyntheticExecutor(mw.cluster)), mw, None, None, mctx)
    assert entries_of(plan) == entries_of(msol.plan)
    op = O.build(rt.entries, rw, context=(remaining, running, 30.0))
    assert (sol.makespan, sol.search.index) == C.CProblem(op).search()
    assert PL.resolve(rt, rw, ctx) == plan


def test_baseline_planners_reference_objects():
    core, profiling, w, rw, rt = ref_setup("small4_2x2")
    for plan in (PL.plan_random(rt, rw, seed=3), PL.plan_optimus(rt, rw), PL.plan_current_practice(rt, rw)):
        assert type(plan) is core.Plan
        core.check_plan(plan, rw, ref_runtimes(profiling, rt, rw, plan))


def test_reference_errors_cross_the_boundary():
    """Reference objects get the reference's own error classes (errors.py:23-26, 84-85)."""
    core, profiling, w, rw, rt = ref_setup("small4_2x2")
    from jointsched import errors as RE

    big = rw.jobs[0].model_copy(update={"id": "zz", "model_memory": 1e6})
    bad = core.Workload(jobs=[j for j in rw.jobs if j.model_memory < 50] + [big], cluster=rw.cluster,
                        techniques=[t for t in rw.techniques if t.archetype != "offloaded"])
    with pytest.raises(RE.NoFeasibleConfig) as exc:
        PL.plan_saturn(rt, bad)
    assert "zz" in str(exc.value)
    many = core.Workload(jobs=[rw.jobs[0].model_copy(update={"id": f"k{i:02d}"}) for i in range(30)],
                         cluster=rw.cluster, techniques=rw.techniques)
    with pytest.raises(RE.TooLarge):
        PL.solve(profiling.build_profile_table(many, profiling.SyntheticExecutor(many.cluster)), many, None,
                 SolveOptions(search="exhaustive"))


def test_reference_csv_tables_feed_the_engine(tmp_path):
    """Measured tables flow in unchanged: the reference's own save_profiles / load_profiles
    (profiling.py:173-215) round trip feeds plan_saturn, same plan as the in-memory table."""
    core, profiling, w, rw, rt = ref_setup("hetero6")
    p = tmp_path / "prof.csv"
    profiling.save_profiles(rt, p)
    loaded = profiling.load_profiles(p)
    a, b = PL.plan_saturn(loaded, rw), PL.plan_saturn(rt, rw)
    assert entries_of(a) == entries_of(b)


def test_simulate_with_reference_objects_equals_mirror():
    """The introspection driver hands the replanner the reference's own
    RunningContext when the workload is the reference's; the run is the mirror run, byte for byte."""
    core, profiling, w, rw, rt = ref_setup("small5_1x4")
    seen = []

    def replan(table, workload, ctx):
        seen.append(type(ctx))
        return PL.resolve(table, workload, ctx)

    p0 = PL.plan_saturn(rt, rw)
    rep = SIM.simulate(rw, rt, p0, SIM.SimOptions(introspection_interval=p0.predicted_makespan / 10,
                                                  checkpoint_overhead=30.0, replanner=replan))
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    m0 = PL.plan_saturn(t, w)
    mrep = SIM.simulate(w, t, m0, SIM.SimOptions(introspection_interval=m0.predicted_makespan / 10,
                                                 checkpoint_overhead=30.0, replanner="saturn"))
    assert seen and all(c is core.RunningContext for c in seen)
    assert rep.replan_count == mrep.replan_count > 0
    assert rep.to_json() == mrep.to_json()


def test_local_search_beyond_the_prover_reference_objects():
    """A reference workload whose shape the state-space prover does not take (9 nodes): the
    default solve falls back to the local search's result (the prover's TooLarge is the caller's
    own error class and must not escape)."""
    core, profiling, _ = import_reference()
    w, _ = golden_workload("small5_1x4")
    rw = ref_workload(core, w)
    nodes = [core.NodeSpec(id=f"m{i}", gpu_count=1, gpu_memory=80.0) for i in range(9)]
    jobs = [rw.jobs[0].model_copy(update={"id": f"k{i:02d}", "model_memory": 10.0}) for i in range(14)]
    big = core.Workload(jobs=jobs, cluster=core.ClusterSpec(nodes=nodes), techniques=rw.techniques)
    rt = profiling.build_profile_table(big, profiling.SyntheticExecutor(big.cluster))
    sol = PL.solve(rt, big)
    assert sol.search.kernel == "local" and sol.status in ("Local", "Optimal")
    core.check_plan(sol.plan, big, ref_runtimes(profiling, rt, big, sol.plan))
