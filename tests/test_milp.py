"""The jointsched.milp facade: instance building on the CPU; the GPU-backed
solvers in test_milp_gpu.py."""

import pytest

from helpers import golden, golden_workload

from paper_2311_02840_b200 import domain as D
from paper_2311_02840_b200 import errors as E
from paper_2311_02840_b200 import milp
from paper_2311_02840_b200.profiling import ProfileTable, SyntheticExecutor, build_profile_table


def test_build_milp_cfg1_grid_and_horizon():
    w, _ = golden_workload("cfg1")
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    inst = milp.build_milp(t, w)
    assert inst.delta.hex() == golden()["milp"]["cfg1"]["delta"]
    assert inst.horizon == 48                 # SPEC.md:195 K with delta = sum(min T) / K_max
    d = inst.durations()
    assert all(isinstance(v, int) and v >= 1 for v in d.values())


def test_build_milp_spec_examples():
    techs = (D.TechniqueSpec(name="t", archetype="sharded", serial_fraction=0.0, comm_overhead=0.0),)
    cl = D.ClusterSpec((D.NodeSpec("n", 2, 80.0),))
    # 1 job, 1 config, T = 10 s, delta = 10 s -> K = 1
    w1 = D.Workload((D.JobSpec("a", 1, 1.0, 1.0),), D.ClusterSpec((D.NodeSpec("n", 1, 80.0),)), techs)
    t1 = ProfileTable({("a", "t", 1): 10.0}, "ingested")
    inst = milp.build_milp(t1, w1, delta=10.0)
    assert inst.horizon == 1 and inst.durations() == {("a", "t", 1): 1}
    # explicit delta too small for K_max -> HorizonOverflow (errors.py:77-81)
    w = D.Workload((D.JobSpec("a", 1, 1.0, 1.0), D.JobSpec("b", 1, 1.0, 1.0)), cl, techs)
    t = ProfileTable({("a", "t", 1): 10.0, ("a", "t", 2): 6.0, ("b", "t", 1): 10.0, ("b", "t", 2): 6.0}, "x")
    with pytest.raises(E.HorizonOverflow):
        milp.build_milp(t, w, delta=0.1, k_max=48)
    assert milp.build_milp(t, w, delta=1.0, k_max=1000).horizon == 12
