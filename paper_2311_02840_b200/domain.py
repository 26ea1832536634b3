"""Host-side mirror of the reference's domain types (L0).

The engine is duck-typed: every function in this package accepts either these
classes or the reference's pydantic models (``pkg/src/jointsched/core.py``)
because it only reads attributes.  These frozen dataclasses exist so the
engine, its tests and ``bench.py`` run where the reference package is absent
(the GPU box).  Field names, validation rules and ordering guarantees follow
the reference line by line; the implementations are this package's own.

Reference map:
  JobSpec        core.py:25-39      NodeSpec      core.py:42-47
  ClusterSpec    core.py:50-67      TechniqueSpec core.py:70-91
  RunConfig      core.py:94-103     PlanEntry     core.py:106-111
  Plan           core.py:114-120    Workload      core.py:123-142
  memory_feasible core.py:145-156   hosting_gpu_memory core.py:159-162
  feasible_configs core.py:165-182  validate_workload core.py:185-208
  RunningContext core.py:211-223    sweep_capacity core.py:226-251
  check_plan     core.py:254-287
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Mapping

import numpy as np

from . import errors as E

ARCHETYPES = ("replicated", "sharded", "pipelined", "offloaded")
_MEM_SLACK = 1e-12  # core.py:156


def _require(cond: bool, name: str, msg: str) -> None:
    if not cond:
        raise E.InvariantViolation(name, msg)


@dataclass(frozen=True)
class JobSpec:
    id: str
    total_batches: int
    base_batch_time: float
    model_memory: float
    activation_memory: float = 0.0

    def __post_init__(self):
        _require(int(self.total_batches) == self.total_batches and self.total_batches >= 1,
                 "total_batches", "must be an integer >= 1")
        _require(self.base_batch_time > 0, "base_batch_time", "must be > 0")
        _require(self.model_memory > 0, "model_memory", "must be > 0")
        _require(self.activation_memory >= 0, "activation_memory", "must be >= 0")


@dataclass(frozen=True)
class NodeSpec:
    id: str
    gpu_count: int
    gpu_memory: float

    def __post_init__(self):
        _require(self.gpu_count >= 1, "gpu_count", "must be >= 1")
        _require(self.gpu_memory > 0, "gpu_memory", "must be > 0")


@dataclass(frozen=True)
class ClusterSpec:
    nodes: tuple

    def __post_init__(self):
        object.__setattr__(self, "nodes", tuple(self.nodes))
        _require(len(self.nodes) >= 1, "nodes", "at least one node")

    @property
    def max_gpus_per_node(self) -> int:
        return max(n.gpu_count for n in self.nodes)

    @property
    def total_gpus(self) -> int:
        return sum(n.gpu_count for n in self.nodes)

    def node(self, node_id: str):
        for n in self.nodes:
            if n.id == node_id:
                return n
        raise KeyError(node_id)


@dataclass(frozen=True)
class TechniqueSpec:
    name: str
    archetype: str
    serial_fraction: float
    comm_overhead: float
    offload_multiplier: float = 1.0
    min_gpus: int = 1

    def __post_init__(self):
        _require(self.archetype in ARCHETYPES, "archetype", f"one of {ARCHETYPES}")
        _require(0 <= self.serial_fraction < 1, "serial_fraction", "in [0, 1)")
        _require(self.comm_overhead >= 0, "comm_overhead", ">= 0")
        _require(self.offload_multiplier >= 1, "offload_multiplier", ">= 1")
        _require(self.min_gpus >= 1, "min_gpus", ">= 1")
        if self.archetype != "offloaded":
            _require(self.offload_multiplier == 1.0, "offload_multiplier",
                     "must be 1 unless archetype is 'offloaded'")


@dataclass(frozen=True)
class RunConfig:
    technique: str
    gpus: int

    def __post_init__(self):
        _require(self.gpus >= 1, "gpus", ">= 1")

    def key(self) -> tuple:
        return (self.technique, self.gpus)


@dataclass(frozen=True)
class PlanEntry:
    config: RunConfig
    node: str
    start_time: float

    def __post_init__(self):
        _require(self.start_time >= 0, "start_time", ">= 0")


@dataclass(frozen=True)
class Plan:
    entries: dict
    predicted_makespan: float

    def __post_init__(self):
        _require(self.predicted_makespan >= 0, "predicted_makespan", ">= 0")


@dataclass(frozen=True)
class Workload:
    jobs: tuple
    cluster: ClusterSpec
    techniques: tuple

    def __post_init__(self):
        object.__setattr__(self, "jobs", tuple(self.jobs))
        object.__setattr__(self, "techniques", tuple(self.techniques))

    def job(self, job_id: str):
        for j in self.jobs:
            if j.id == job_id:
                return j
        raise KeyError(job_id)

    def technique(self, name: str):
        for t in self.techniques:
            if t.name == name:
                return t
        raise KeyError(name)


@dataclass(frozen=True)
class RunningContext:
    """Re-solve snapshot (core.py:211-223): unfinished job -> remaining batches,
    running job -> (technique, gpus, node) it holds, and checkpoint cost rho."""

    remaining: Mapping[str, int]
    current: Mapping[str, tuple] = field(default_factory=dict)
    checkpoint_cost: float = 0.0


# --------------------------------------------------------------------------
# feasibility (core.py:145-208)
# --------------------------------------------------------------------------

def memory_feasible(job, technique, g: int, gpu_memory: float) -> bool:
    """Shard-factor memory rule of core.py:145-156."""
    if g < 1:
        raise ValueError("g must be >= 1")
    arch = technique.archetype
    if arch == "offloaded":
        return True
    per_gpu_model = job.model_memory if arch == "replicated" else job.model_memory / float(g)
    return per_gpu_model + job.activation_memory <= gpu_memory + _MEM_SLACK


def hosting_gpu_memory(cluster, g: int):
    """Largest per-GPU memory among nodes with >= g GPUs, None if none (core.py:159-162)."""
    mems = [n.gpu_memory for n in cluster.nodes if n.gpu_count >= g]
    return max(mems) if mems else None


def node_eligible(job, technique, g: int, node) -> bool:
    """Can a g-gang of `technique` for `job` run on `node` (the per-node clause of core.py:177-180)."""
    return node.gpu_count >= g and memory_feasible(job, technique, g, node.gpu_memory)


_CONFIGS_MEMO: dict = {}


def feasible_configs(job, cluster, techniques: Iterable) -> list:
    """(technique, g) runnable on some node; registration order then ascending g (core.py:165-182).

    A pure function of immutable inputs (frozen dataclasses / frozen pydantic models), memoised
    by value: re-solves and repeated solves of the same workload skip the enumeration."""
    techniques = tuple(techniques)
    try:
        key = (job, cluster, techniques)
        hit = _CONFIGS_MEMO.get(key)
    except TypeError:                   # unhashable inputs: compute every time
        return _feasible_configs(job, cluster, techniques)
    if hit is None:
        hit = tuple(_feasible_configs(job, cluster, techniques))
        if len(_CONFIGS_MEMO) > 1 << 16:
            _CONFIGS_MEMO.clear()
        _CONFIGS_MEMO[key] = hit
    return list(hit)


def _feasible_configs(job, cluster, techniques) -> list:
    top = cluster.max_gpus_per_node
    found = []
    for tech in techniques:
        g = tech.min_gpus
        while g <= top:
            if hosting_gpu_memory(cluster, g) is not None and any(
                node_eligible(job, tech, g, n) for n in cluster.nodes
            ):
                found.append(RunConfig(technique=tech.name, gpus=g))
            g += 1
    return found


def validate_workload(workload):
    """Unique ids and >= 1 feasible config per job (core.py:185-208)."""
    for kind, ids in (
        ("job", [j.id for j in workload.jobs]),
        ("node", [n.id for n in workload.cluster.nodes]),
        ("technique", [t.name for t in workload.techniques]),
    ):
        seen = set()
        for i in ids:
            if i in seen:
                raise E.DuplicateId(kind, i)
            seen.add(i)
    for job in workload.jobs:
        if not feasible_configs(job, workload.cluster, workload.techniques):
            raise E.NoFeasibleConfig(job.id)
    return workload


# --------------------------------------------------------------------------
# plan validation (core.py:226-287), as array passes over the plan's segments
# --------------------------------------------------------------------------

def sweep_capacity(segments: Iterable, cluster, tol: float = 1e-9) -> None:
    """Per-node GPU demand over time (core.py:226-251).  Each segment contributes a +g event at
    its start and a -g event at its end; at equal times ends sort first, so a gang may take GPUs
    freed at the instant it starts.  Demand = running sum of the sorted events per node."""
    segs = list(segments)
    if not segs:
        return
    nodes = [s[0] for s in segs]
    g = np.array([s[1] for s in segs], dtype=np.int64)
    t = np.array([(s[2], s[3]) for s in segs], dtype=np.float64)            # [n, (start, end)]
    reversed_ = np.flatnonzero(t[:, 1] < t[:, 0] - tol)
    if reversed_.size:
        raise E.InvalidPlan(f"segment on {nodes[reversed_[0]]} ends before it starts")
    node_of = np.array([{n: i for i, n in enumerate(dict.fromkeys(nodes))}[n] for n in nodes])
    for k, node_id in enumerate(dict.fromkeys(nodes)):         # nodes in order of first use
        sel = np.flatnonzero(node_of == k)
        times = t[sel].ravel()                                  # start, end, start, end, ...
        kind = np.tile(np.array([1, 0]), sel.size)              # start = 1 sorts after end = 0
        step = np.stack([g[sel], -g[sel]], axis=1).ravel()
        perm = np.lexsort((kind, times))                        # stable: ties keep input order
        demand = np.cumsum(step[perm])
        cap = cluster.node(node_id).gpu_count
        over = np.flatnonzero(demand > cap)
        if over.size:
            i = over[0]
            raise E.CapacityViolation(f"node {node_id}: {int(demand[i])} GPUs in use at t={times[perm[i]]:.6g}, "
                                      f"capacity {cap}")


def check_plan(plan, workload, runtimes: Mapping, tol: float = 1e-6) -> None:
    """Plan invariants against per-job runtimes (core.py:254-287): every workload job planned
    exactly once, each gang fits its node and meets its technique's minimum, node capacity holds
    at every instant, and the predicted makespan covers the last completion."""
    want, got = {j.id for j in workload.jobs}, set(plan.entries)
    if want != got:
        raise E.InvalidPlan(f"plan covers {sorted(got)}, workload has {sorted(want)}")
    ids = list(plan.entries)
    ents = [plan.entries[i] for i in ids]
    node_objs = [workload.cluster.node(e.node) for e in ents]
    min_g = np.array([workload.technique(e.config.technique).min_gpus for e in ents], dtype=np.int64)
    gang = np.array([e.config.gpus for e in ents], dtype=np.int64)
    cap = np.array([n.gpu_count for n in node_objs], dtype=np.int64)
    wide, short = gang > cap, gang < min_g
    first = np.flatnonzero(wide | short)
    if first.size:
        i = first[0]
        if wide[i]:
            raise E.CapacityViolation(f"job {ids[i]}: gang of {gang[i]} exceeds node {node_objs[i].id} ({cap[i]})")
        raise E.InvalidPlan(f"job {ids[i]}: {gang[i]} GPUs below technique minimum")
    start = np.array([e.start_time for e in ents], dtype=np.float64)
    end = start + np.array([runtimes[i] for i in ids], dtype=np.float64)
    sweep_capacity(zip([e.node for e in ents], gang.tolist(), start.tolist(), end.tolist()), workload.cluster)
    last_end = max(0.0, float(end.max())) if len(ids) else 0.0
    if plan.predicted_makespan < last_end - tol:
        raise E.InvalidPlan(
            f"predicted makespan {plan.predicted_makespan:.6g} below last completion {last_end:.6g}")
