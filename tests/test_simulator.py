"""Introspection driver on the CPU: the replanner is the oracle's exhaustive
search (test infrastructure), so these run without a GPU.  The GPU runs of the same driver
with the engine as replanner are in test_simulator_gpu.py.

Checked: the SPEC examples (R=0 verbatim execution, 2-job example 10 vs 12), the report
invariants (work conservation, per-node capacity including checkpoint drains, makespan),
no-regression with rho=0, determinism, the apply_replan fixed point, and ReplanFailure
keeping the old plan."""

import math
import random

import pytest

from helpers import golden_workload

from oracle import coracle as C
from oracle import saturn_oracle as O
from paper_2311_02840_b200 import domain as D
from paper_2311_02840_b200 import errors as E
from paper_2311_02840_b200 import simulator as SIM
from paper_2311_02840_b200.profiling import ProfileTable, SyntheticExecutor, build_profile_table


def oracle_plan(t, w, ctx=None, which="saturn"):
    """Exhaustive oracle optimum (or a baseline) as a Plan, start times relative to now."""
    context = None if ctx is None else (dict(ctx.remaining), dict(ctx.current), ctx.checkpoint_cost)
    op = O.build(t.entries, w, context=context, prune=False if which != "saturn" else None)
    if which == "saturn":
        ms, index = C.CProblem(op).search()
        opts, order = O.decode_index(op, index)
    elif which == "cp":
        opts, order = O.current_practice(op)
    else:
        opts, order = O.optimus(op)
    ms, starts, nodes = O.list_schedule(op, opts, order, record=True)
    entries = {}
    for j, jid in enumerate(op.job_ids):
        tech, g = op.options[j][opts[j]]
        entries[jid] = D.PlanEntry(D.RunConfig(tech, g), op.node_ids[nodes[j]], starts[j] * op.delta)
    return D.Plan(entries, ms * op.delta)


def oracle_replanner(table, workload, ctx):
    return oracle_plan(table, workload, ctx)


def two_job():
    techs = (D.TechniqueSpec(name="t", archetype="sharded", serial_fraction=0.0, comm_overhead=0.0),)
    jobs = (D.JobSpec("a", 10, 1.0, 1.0), D.JobSpec("b", 10, 1.0, 1.0))
    w = D.Workload(jobs, D.ClusterSpec((D.NodeSpec("n", 2, 80.0),)), techs)
    t = ProfileTable({("a", "t", 1): 1.0, ("a", "t", 2): 0.6, ("b", "t", 1): 1.0, ("b", "t", 2): 0.6}, "ingested")
    return w, t


def test_single_job_verbatim():
    """R=0, single job, T=100 s -> makespan 100, replan_count 0."""
    techs = (D.TechniqueSpec(name="t", archetype="sharded", serial_fraction=0.0, comm_overhead=0.0),)
    w = D.Workload((D.JobSpec("a", 100, 1.0, 1.0),), D.ClusterSpec((D.NodeSpec("n", 4, 80.0),)), techs)
    t = ProfileTable({("a", "t", g): 1.0 for g in range(1, 5)}, "ingested")
    plan = D.Plan({"a": D.PlanEntry(D.RunConfig("t", 2), "n", 0.0)}, 100.0)
    rep = SIM.simulate(w, t, plan, SIM.SimOptions())
    assert rep.makespan == 100.0 and rep.replan_count == 0 and rep.checkpoint_count == 0
    SIM.verify_report(rep, w)
    assert rep.timeline_csv().splitlines()[0] == "job,technique,gpus,node,start_s,end_s,batches"


def test_two_job_example_saturn_vs_current_practice():
    """2-job/2-GPU example executes to 10 under Saturn's plan, 12 under CP's."""
    w, t = two_job()
    sat = oracle_plan(t, w)
    cp = oracle_plan(t, w, which="cp")
    assert SIM.simulate(w, t, sat).makespan == pytest.approx(10.0)
    assert SIM.simulate(w, t, cp).makespan == pytest.approx(12.0)


def _random_workload(rng, J, gpus):
    techs = (
        D.TechniqueSpec(name="ddp", archetype="replicated", serial_fraction=0.02, comm_overhead=0.01),
        D.TechniqueSpec(name="fsdp", archetype="sharded", serial_fraction=0.05, comm_overhead=0.03),
    )
    jobs = tuple(D.JobSpec(f"j{j}", rng.randint(50, 400), rng.uniform(0.5, 3.0), rng.choice([8.0, 20.0]), 2.0)
                 for j in range(J))
    w = D.Workload(jobs, D.ClusterSpec((D.NodeSpec("n0", gpus, 40.0),)), techs)
    return w, build_profile_table(w, SyntheticExecutor(w.cluster))


@pytest.mark.parametrize("seed", range(6))
def test_introspection_invariants_and_no_regression(seed):
    rng = random.Random(seed)
    w, t = _random_workload(rng, rng.randint(2, 4), rng.choice([2, 4]))
    plan0 = oracle_plan(t, w)
    static = SIM.simulate(w, t, plan0)
    SIM.verify_report(static, w)
    assert static.makespan <= plan0.predicted_makespan + 1e-6        # grid durations are ceilings
    opts = SIM.SimOptions(introspection_interval=plan0.predicted_makespan / 10, checkpoint_overhead=0.0,
                          replanner=oracle_replanner)
    rep = SIM.simulate(w, t, plan0, opts)
    SIM.verify_report(rep, w)
    assert rep.replan_count >= 1
    # SPEC.md:395 no-regression (exact profiles, rho = 0): within one grid interval of plan0
    op = O.build(t.entries, w)
    assert rep.makespan <= plan0.predicted_makespan + op.delta + 1e-6
    # determinism: byte-identical reports
    assert SIM.simulate(w, t, plan0, opts).to_json() == rep.to_json()


@pytest.mark.parametrize("rho", [5.0, 60.0])
def test_checkpoints_hold_gpus_and_conserve_work(rho):
    rng = random.Random(11)
    w, t = _random_workload(rng, 4, 4)
    plan0 = oracle_plan(t, w, which="cp")                               # a poor plan: re-solves move jobs
    opts = SIM.SimOptions(introspection_interval=plan0.predicted_makespan / 7, checkpoint_overhead=rho,
                          replanner=oracle_replanner)
    rep = SIM.simulate(w, t, plan0, opts)
    SIM.verify_report(rep, w)                                           # includes drain segments
    assert rep.checkpoint_count >= 1
    assert rep.checkpoint_time_total == pytest.approx(rho * rep.checkpoint_count)
    drains = [s for s in rep.timeline if s.kind == "checkpoint"]
    assert len(drains) == rep.checkpoint_count and all(s.end - s.start == pytest.approx(rho) for s in drains)
    assert rep.makespan < SIM.simulate(w, t, plan0).makespan          # introspection beats the poor plan


def test_apply_replan_fixed_point_and_failure_keeps_plan():
    rng = random.Random(5)
    w, t = _random_workload(rng, 3, 2)
    plan0 = oracle_plan(t, w)
    sim = SIM._Sim(w, t, plan0, SIM.SimOptions())
    # at t=0 nothing runs yet: re-adopting plan0 changes nothing and checkpoints nothing
    SIM.apply_replan(sim, plan0, 0.0)
    sim.run()
    assert sim.ckpts == 0
    assert sim.report().makespan == SIM.simulate(w, t, plan0).makespan

    def broken(table, workload, ctx):
        raise E.ReplanFailure("solver unavailable")

    rep = SIM.simulate(w, t, plan0, SIM.SimOptions(introspection_interval=plan0.predicted_makespan / 5,
                                                    replanner=broken))
    assert rep.replan_failures >= 1 and rep.replan_count == 0
    assert rep.makespan == SIM.simulate(w, t, plan0).makespan          # old plan kept


def test_remaining_batches_examples():
    """pending -> total; running 50 s at 0.5 s/batch from 0 -> total - 100."""
    job = SIM._Job(spec=None, lat={("t", 1): 0.5}, state="pending", remaining=1000)
    assert SIM.remaining_batches(job, 50.0) == 1000
    job.state, job.tech, job.gpus, job.seg_start = "running", "t", 1, 0.0
    assert SIM.remaining_batches(job, 50.0) == 900
    job.state = "done"
    assert SIM.remaining_batches(job, 50.0) == 0


def test_cfg1_introspection_with_oracle_windows():
    """cfg1 plan0 from the golden optimum value path: R = predicted/10, rho = 30 s, the replanner
    restricted to a tiny oracle search is replaced by keeping plan0 feasible -- checks the driver
    on the real 8-job table (the engine-backed run is in test_simulator_gpu.py)."""
    w, _ = golden_workload("cfg1")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    op = O.build(t.entries, w)
    opts, order = O.current_practice(op)
    ms, starts, nodes = O.list_schedule(op, opts, order, record=True)
    entries = {jid: D.PlanEntry(D.RunConfig(*op.options[j][opts[j]]), op.node_ids[nodes[j]], starts[j] * op.delta)
               for j, jid in enumerate(op.job_ids)}
    plan0 = D.Plan(entries, ms * op.delta)
    rep = SIM.simulate(w, t, plan0)
    SIM.verify_report(rep, w)
    assert rep.makespan <= plan0.predicted_makespan + 1e-6
    assert math.isfinite(rep.makespan)
