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
# plan validation (core.py:226-287)
# --------------------------------------------------------------------------

def sweep_capacity(segments: Iterable, cluster, tol: float = 1e-9) -> None:
    """Per-node event sweep; at equal t an end (kind 0) is applied before a start (kind 1)."""
    per_node: dict = {}
    for node_id, gpus, start, end in segments:
        if end < start - tol:
            raise E.InvalidPlan(f"segment on {node_id} ends before it starts")
        ev = per_node.setdefault(node_id, [])
        ev.append((start, 1, gpus))
        ev.append((end, 0, -gpus))
    for node_id, ev in per_node.items():
        cap = cluster.node(node_id).gpu_count
        busy = 0
        for t, _kind, delta in sorted(ev, key=lambda e: (e[0], e[1])):
            busy += delta
            if busy > cap:
                raise E.CapacityViolation(f"node {node_id}: {busy} GPUs in use at t={t:.6g}, capacity {cap}")


def check_plan(plan, workload, runtimes: Mapping, tol: float = 1e-6) -> None:
    """Coverage, gang fit, min_gpus, capacity sweep, predicted >= last end (core.py:254-287)."""
    want = {j.id for j in workload.jobs}
    got = set(plan.entries)
    if want != got:
        raise E.InvalidPlan(f"plan covers {sorted(got)}, workload has {sorted(want)}")
    segs = []
    last_end = 0.0
    for job_id, entry in plan.entries.items():
        tech = workload.technique(entry.config.technique)
        node = workload.cluster.node(entry.node)
        if entry.config.gpus > node.gpu_count:
            raise E.CapacityViolation(
                f"job {job_id}: gang of {entry.config.gpus} exceeds node {node.id} ({node.gpu_count})")
        if entry.config.gpus < tech.min_gpus:
            raise E.InvalidPlan(f"job {job_id}: {entry.config.gpus} GPUs below technique minimum")
        end = entry.start_time + runtimes[job_id]
        segs.append((entry.node, entry.config.gpus, entry.start_time, end))
        last_end = max(last_end, end)
    sweep_capacity(segs, workload.cluster)
    if plan.predicted_makespan < last_end - tol:
        raise E.InvalidPlan(
            f"predicted makespan {plan.predicted_makespan:.6g} below last completion {last_end:.6g}")
