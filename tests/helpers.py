"""Shared test helpers: golden fixtures -> this package's domain objects."""

from __future__ import annotations

import json
import math
import os

from paper_2311_02840_b200 import domain as D
from paper_2311_02840_b200.profiling import ProfileTable

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.json")
REF_SRC = "/root/reference/pkg/src"

_gold = None


def golden():
    global _gold
    if _gold is None:
        with open(GOLDEN) as f:
            _gold = json.load(f)
    return _gold


def unhex(s: str) -> float:
    return math.inf if s == "inf" else float.fromhex(s)


def workload_from_json(d) -> D.Workload:
    jobs = tuple(D.JobSpec(**j) for j in d["jobs"])
    nodes = tuple(D.NodeSpec(**n) for n in d["cluster"]["nodes"])
    techs = tuple(D.TechniqueSpec(**t) for t in d["techniques"])
    return D.Workload(jobs=jobs, cluster=D.ClusterSpec(nodes=nodes), techniques=techs)


def golden_workload(name):
    rec = golden()["workloads"][name]
    return workload_from_json(rec["workload"]), rec


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "jointsched"))


def import_reference():
    import sys
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from jointsched import core, profiling, rng  # noqa: F401
    return core, profiling, rng
