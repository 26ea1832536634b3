"""Introspection driver with the GPU engine as the replanner (config 2 of BASELINE.json).

The engine-backed simulation must be byte-identical to the same simulation driven by the
CPU oracle's exhaustive re-solves (same index order and tie-break => same plans => same
timeline), for Saturn re-solves and for Optimus-Dynamic."""

import random

import pytest

from test_simulator import _random_workload, oracle_plan, oracle_replanner

from helpers import golden_workload
from oracle import saturn_oracle as O
from paper_2311_02840_b200 import domain as D
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200 import simulator as SIM
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table

pytestmark = pytest.mark.gpu


def oracle_optimus(table, workload, ctx):
    return oracle_plan(table, workload, ctx, which="optimus")


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("rho", [0.0, 30.0])
def test_engine_resolve_simulation_equals_oracle(seed, rho):
    rng = random.Random(100 + seed)
    w, t = _random_workload(rng, rng.randint(3, 5), rng.choice([2, 4, 8]))
    plan0 = PL.plan_saturn(t, w)
    assert plan0 == oracle_plan(t, w)
    R = plan0.predicted_makespan / 10
    eng = SIM.simulate(w, t, plan0, SIM.SimOptions(introspection_interval=R, checkpoint_overhead=rho))
    ora = SIM.simulate(w, t, plan0, SIM.SimOptions(introspection_interval=R, checkpoint_overhead=rho,
                                                   replanner=oracle_replanner))
    SIM.verify_report(eng, w)
    assert eng.replan_failures == 0
    assert eng.to_json() == ora.to_json()


@pytest.mark.parametrize("seed", range(3))
def test_optimus_dynamic_simulation_equals_oracle(seed):
    rng = random.Random(200 + seed)
    w, t = _random_workload(rng, rng.randint(3, 6), rng.choice([4, 8]))
    plan0 = PL.plan_optimus(t, w)
    assert plan0 == oracle_plan(t, w, which="optimus")
    R = plan0.predicted_makespan / 10
    eng = SIM.simulate(w, t, plan0, SIM.SimOptions(introspection_interval=R, replanner="optimus",
                                                   planner="optimus_dynamic"))
    ora = SIM.simulate(w, t, plan0, SIM.SimOptions(introspection_interval=R, replanner=oracle_optimus,
                                                   planner="optimus_dynamic"))
    SIM.verify_report(eng, w)
    assert eng.to_json() == ora.to_json()


def test_cfg1_introspection_run():
    """Config 2: the paper workload with R = predicted/10 and rho = 30 s."""
    w, _ = golden_workload("cfg1")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    plan0 = PL.plan_saturn(t, w)
    static = SIM.simulate(w, t, plan0)
    rep = SIM.simulate(w, t, plan0, SIM.SimOptions(introspection_interval=plan0.predicted_makespan / 10,
                                                   checkpoint_overhead=30.0))
    SIM.verify_report(static, w)
    SIM.verify_report(rep, w)
    assert rep.replan_count >= 5 and rep.replan_failures == 0
    delta = O.build(t.entries, w).delta
    assert rep.makespan <= static.makespan + delta
    # every planner's executed makespan is no better than Saturn's static plan - delta
    for plan in (PL.plan_optimus(t, w), PL.plan_current_practice(t, w), PL.plan_random(t, w, seed=7)):
        assert SIM.simulate(w, t, plan).makespan >= static.makespan - delta
