"""jointsched.milp facade on the engine: branch_and_bound = brute_force_schedule = oracle."""

import pytest

from helpers import golden, golden_workload

from oracle import coracle as C
from oracle import saturn_oracle as O
from paper_2311_02840_b200 import domain as D
from paper_2311_02840_b200 import milp
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200.profiling import ProfileTable, SyntheticExecutor, build_profile_table

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cfg1", "small5_1x4", "small4_2x2", "tiny3_1x3"])
def test_bnb_equals_brute_force_equals_oracle(name):
    w, _ = golden_workload(name)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    inst = milp.build_milp(t, w)
    bb = milp.branch_and_bound(inst)
    bf = milp.brute_force_schedule(inst)
    assert bb.status == bf.status == "Optimal"
    assert bb.assignment == bf.assignment and bb.objective == bf.objective
    if name == "cfg1":                        # 3.25e10 candidates: the CPU oracle would take minutes
        ms = golden()["milp"][name]["optimum_intervals"]
    else:
        ms, _ = C.CProblem(O.build(t.entries, w)).search()
        assert ms == golden()["milp"][name]["optimum_intervals"]
    assert bb.objective == ms * inst.delta
    plan = milp.decode_plan(inst, bb)
    assert plan == PL.plan_saturn(t, w)
    # decode from the assignment alone (c, n, i) reproduces the plan
    bare = milp.MilpSolution(bb.assignment, bb.objective, bb.status, bb.node_count)
    assert milp.decode_plan(inst, bare) == plan
    assert bb.node_count > 0


def test_spec_two_job_example():
    """2 jobs on a 2-GPU node, T(g=1)=10, T(g=2)=6, delta=1 -> M = 10."""
    techs = (D.TechniqueSpec(name="t", archetype="sharded", serial_fraction=0.0, comm_overhead=0.0),)
    w = D.Workload((D.JobSpec("a", 1, 1.0, 1.0), D.JobSpec("b", 1, 1.0, 1.0)),
                   D.ClusterSpec((D.NodeSpec("n", 2, 80.0),)), techs)
    t = ProfileTable({("a", "t", 1): 10.0, ("a", "t", 2): 6.0, ("b", "t", 1): 10.0, ("b", "t", 2): 6.0}, "x")
    inst = milp.build_milp(t, w, delta=1.0, k_max=1000)
    sol = milp.branch_and_bound(inst)
    assert sol.status == "Optimal" and sol.objective == 10.0
    assert sol.assignment == {"a": (0, "n", 0), "b": (0, "n", 0)}
    assert milp.brute_force_schedule(inst).objective == 10.0
