"""Shared test helpers: golden fixtures -> this package's domain objects."""

from __future__ import annotations

import json
import math
import os

from paper_2311_02840_b200 import domain as D
from paper_2311_02840_b200.profiling import ProfileTable

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.json")
# the reference package: installed into baseline/_ref (git-ignored, travels to the GPU box with
# the snapshot; tools/install_reference.sh) or, in the build container, its source tree
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIRS = (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")

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


def reference_dir():
    for d in REF_DIRS:
        if os.path.isfile(os.path.join(d, "jointsched", "core.py")):
            return d
    return None


def reference_available() -> bool:
    return reference_dir() is not None


def import_reference():
    import sys
    d = reference_dir()
    if d is None:
        raise RuntimeError("reference package missing: run tools/install_reference.sh")
    if d not in sys.path:
        sys.path.insert(0, d)
    from jointsched import core, profiling, rng  # noqa: F401
    return core, profiling, rng
