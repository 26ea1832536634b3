"""Trial Runner / Library plugin contract mirror (L1).

Reference map (``pkg/src/jointsched/profiling.py``):
  synthetic_latency   :25-43    Executor protocol :46-55
  SyntheticExecutor   :58-76    TableExecutor     :79-94
  ProfileTable        :97-119   build_profile_table :122-144
  estimate_runtime    :147-151  feasible_entries  :154-161
  ensure_complete     :164-170

The plan-search engine consumes any object with an ``entries`` dict keyed by
``(job_id, technique, gpus)`` -- the reference ``ProfileTable`` works as is.
"""

from __future__ import annotations

import math
from typing import Protocol

from . import errors as E
from .domain import feasible_configs, hosting_gpu_memory, memory_feasible

INFEASIBLE = math.inf


def synthetic_latency(job, technique, g: int, gpu_memory: float) -> float:
    """mu * base * ((1 - sigma)/g + sigma + kappa*(g - 1)), or inf if it does not fit."""
    if not memory_feasible(job, technique, g, gpu_memory):
        return INFEASIBLE
    s = technique.serial_fraction
    k = technique.comm_overhead
    return technique.offload_multiplier * job.base_batch_time * ((1.0 - s) / g + s + k * (g - 1))


class Executor(Protocol):
    """The Library's two-function plugin surface (profiling.py:46-55)."""

    provenance: str

    def profile(self, job, technique, g: int) -> float: ...

    def execute(self, job, technique, g: int, batches: int) -> float: ...


class SyntheticExecutor:
    provenance = "synthetic"

    def __init__(self, cluster):
        self._cluster = cluster

    def profile(self, job, technique, g: int) -> float:
        mem = hosting_gpu_memory(self._cluster, g)
        return INFEASIBLE if mem is None else synthetic_latency(job, technique, g, mem)

    def execute(self, job, technique, g: int, batches: int) -> float:
        lat = self.profile(job, technique, g)
        if math.isinf(lat):
            raise E.InfeasibleEntry((job.id, technique.name, g))
        return batches * lat


class ProfileTable:
    """(job, technique, gpus) -> per-batch seconds; inf marks a misfit."""

    def __init__(self, entries: dict, provenance: str, profiling_cost: float = 0.0):
        self.entries = entries
        self.provenance = provenance
        self.profiling_cost = profiling_cost

    def latency(self, job_id: str, technique: str, g: int) -> float:
        key = (job_id, technique, g)
        try:
            lat = self.entries[key]
        except KeyError:
            raise E.MissingEntry(key) from None
        if math.isinf(lat):
            raise E.InfeasibleEntry(key)
        return lat

    def is_feasible(self, job_id: str, technique: str, g: int) -> bool:
        return math.isfinite(self.entries.get((job_id, technique, g), INFEASIBLE))

    def __len__(self) -> int:
        return len(self.entries)


class TableExecutor:
    provenance = "ingested"

    def __init__(self, table):
        self._table = table

    def profile(self, job, technique, g: int) -> float:
        key = (job.id, technique.name, g)
        if key not in self._table.entries:
            raise E.MissingEntry(key)
        return self._table.entries[key]

    def execute(self, job, technique, g: int, batches: int) -> float:
        return batches * self._table.latency(job.id, technique.name, g)


def build_profile_table(workload, executor) -> ProfileTable:
    """One profile() per feasible (job, config); cost = sum of 2 x latency (profiling.py:122-144)."""
    entries: dict = {}
    cost = 0.0
    for job in workload.jobs:
        for cfg in feasible_configs(job, workload.cluster, workload.techniques):
            tech = workload.technique(cfg.technique)
            key = (job.id, cfg.technique, cfg.gpus)
            try:
                lat = executor.profile(job, tech, cfg.gpus)
            except Exception as exc:  # noqa: BLE001 -- abort with the offending key
                raise E.ExecutorFailure(key, exc) from exc
            if math.isfinite(lat) and lat <= 0:
                raise E.ExecutorFailure(key, ValueError(f"non-positive latency {lat}"))
            entries[key] = lat
            if math.isfinite(lat):
                cost += 2.0 * lat
    return ProfileTable(entries, executor.provenance, cost)


def estimate_runtime(table, job, config, remaining_batches: int) -> float:
    if remaining_batches < 0:
        raise ValueError("remaining_batches must be >= 0")
    return remaining_batches * table.latency(job.id, config.technique, config.gpus)


def feasible_entries(table, job, workload) -> list:
    """[(RunConfig, latency)] with finite latency, canonical order (profiling.py:154-161)."""
    get, jid, finite = table.entries.get, job.id, math.isfinite
    return [(cfg, lat) for cfg in feasible_configs(job, workload.cluster, workload.techniques)
            for lat in (get((jid, cfg.technique, cfg.gpus), INFEASIBLE),) if finite(lat)]


def ensure_complete(table, workload) -> None:
    for job in workload.jobs:
        for cfg in feasible_configs(job, workload.cluster, workload.techniques):
            key = (job.id, cfg.technique, cfg.gpus)
            if key not in table.entries:
                raise E.MissingEntry(key)
