"""Trial Runner side (L1): the profile table the plan search runs over.

The engine reads a table only through its ``entries`` mapping
``(job id, technique, gpus) -> seconds per batch`` (``inf`` = does not fit), so the
reference's own ``ProfileTable`` (profiling.py:97-119) -- built by its
``build_profile_table`` or read by its ``load_profiles`` -- plugs in unchanged.
This module is the package's own Library side for runs without the reference
installed (the bench, ``smoke()``): same contract, different construction.

* The cost model (profiling.py:25-43) is evaluated as arrays: one job's whole
  (technique, g) row in one numpy expression (the same IEEE operations in the
  same order as the scalar formula, so every entry is bit-identical).
* ``build_profile_table`` asks an executor for a row at a time when it can
  (``profile_row``) and falls back to one ``profile`` call per configuration for
  any other executor (the plugin contract, profiling.py:46-55).  The profiling
  charge (2 x latency per finite entry) is folded left to right in entry order,
  as the reference accumulates it.

Reference map: synthetic latency :25-43, Executor :46-55, SyntheticExecutor :58-76,
TableExecutor :79-94, ProfileTable :97-119, build_profile_table :122-144,
estimate_runtime :147-151, feasible_entries :154-161, ensure_complete :164-170.
"""

from __future__ import annotations

import functools
import math
import operator
from dataclasses import dataclass
from typing import Protocol

import numpy as np

from . import errors as E
from .domain import feasible_configs, hosting_gpu_memory, memory_feasible

INFEASIBLE = math.inf


def _amdahl_row(mu: float, base: float, sigma: float, kappa: float, g: np.ndarray) -> np.ndarray:
    """mu * base * ((1 - sigma)/g + sigma + kappa*(g - 1)) for a vector of gang sizes."""
    return (mu * base) * (((1.0 - sigma) / g + sigma) + kappa * (g - 1.0))


def synthetic_latency(job, technique, g: int, gpu_memory: float) -> float:
    """Analytic seconds per batch of a g-gang, or ``inf`` when it does not fit (profiling.py:25-43)."""
    if not memory_feasible(job, technique, g, gpu_memory):
        return INFEASIBLE
    row = _amdahl_row(technique.offload_multiplier, job.base_batch_time, technique.serial_fraction,
                      technique.comm_overhead, np.array([float(g)]))
    return float(row[0])


class Executor(Protocol):
    """The Library's two-function plugin surface (profiling.py:46-55)."""

    provenance: str

    def profile(self, job, technique, g: int) -> float: ...

    def execute(self, job, technique, g: int, batches: int) -> float: ...


class SyntheticExecutor:
    """The analytic executor bound to a cluster's GPU memory; ``profile_row`` evaluates a
    whole (technique, [g ...]) row at once."""

    provenance = "synthetic"

    def __init__(self, cluster):
        self._cluster = cluster
        self._mem = {}

    def _memory(self, g: int):
        if g not in self._mem:
            self._mem[g] = hosting_gpu_memory(self._cluster, g)
        return self._mem[g]

    def profile_row(self, job, technique, gs) -> list:
        gs = list(gs)
        lat = _amdahl_row(technique.offload_multiplier, job.base_batch_time, technique.serial_fraction,
                          technique.comm_overhead, np.asarray(gs, dtype=np.float64)).tolist()
        for i, g in enumerate(gs):
            mem = self._memory(g)
            if mem is None or not memory_feasible(job, technique, g, mem):
                lat[i] = INFEASIBLE
        return lat

    def profile(self, job, technique, g: int) -> float:
        return self.profile_row(job, technique, [g])[0]

    def execute(self, job, technique, g: int, batches: int) -> float:
        lat = self.profile(job, technique, g)
        if lat == INFEASIBLE:
            raise E.InfeasibleEntry((job.id, technique.name, g))
        return batches * lat


@dataclass
class ProfileTable:
    """(job id, technique, gpus) -> seconds per batch; ``inf`` marks a configuration that does
    not fit.  ``profiling_cost`` = simulated seconds spent profiling (2 batches per entry)."""

    entries: dict
    provenance: str
    profiling_cost: float = 0.0

    def latency(self, job_id: str, technique: str, g: int) -> float:
        key = (job_id, technique, g)
        lat = self.entries.get(key)
        if lat is None:
            raise E.MissingEntry(key)
        if lat == INFEASIBLE:
            raise E.InfeasibleEntry(key)
        return lat

    def is_feasible(self, job_id: str, technique: str, g: int) -> bool:
        return math.isfinite(self.entries.get((job_id, technique, g), INFEASIBLE))

    def __len__(self) -> int:
        return len(self.entries)


class TableExecutor:
    """Replays an ingested table through the executor contract (profiling.py:79-94)."""

    provenance = "ingested"

    def __init__(self, table):
        self._table = table

    def profile(self, job, technique, g: int) -> float:
        try:
            return self._table.entries[(job.id, technique.name, g)]
        except KeyError:
            raise E.MissingEntry((job.id, technique.name, g)) from None

    def execute(self, job, technique, g: int, batches: int) -> float:
        return batches * self._table.latency(job.id, technique.name, g)


def _positive(key, v):
    if math.isfinite(v) and not v > 0:
        raise E.ExecutorFailure(key, ValueError(f"non-positive latency {v}"))
    return v


def _profiled_row(executor, job, tech, gs) -> list:
    """Latencies of one (job, technique) row.  The first configuration (in g order) whose profile
    raises or returns a non-positive latency aborts the build with its key."""
    row_fn = getattr(executor, "profile_row", None)
    if row_fn is not None:
        try:
            got = list(row_fn(job, tech, gs))
        except Exception:               # noqa: BLE001 -- redo per configuration to name the key
            got = None
        if got is not None:
            return [_positive((job.id, tech.name, g), v) for g, v in zip(gs, got)]
    out = []
    for g in gs:
        try:
            v = executor.profile(job, tech, g)
        except Exception as exc:  # noqa: BLE001
            raise E.ExecutorFailure((job.id, tech.name, g), exc) from exc
        out.append(_positive((job.id, tech.name, g), v))
    return out


def build_profile_table(workload, executor) -> ProfileTable:
    """One latency per feasible (job, technique, g), in feasible_configs order (profiling.py:122-144)."""
    techs = {t.name: t for t in workload.techniques}
    keys, lats = [], []
    for job in workload.jobs:
        # the job's canonical configs as per-technique rows (registration order, then ascending g)
        rows: dict = {}
        for cfg in feasible_configs(job, workload.cluster, workload.techniques):
            rows.setdefault(cfg.technique, []).append(cfg.gpus)
        for name, gs in rows.items():
            lats.extend(_profiled_row(executor, job, techs[name], gs))
            keys.extend((job.id, name, g) for g in gs)
    charge = functools.reduce(operator.add, (2.0 * v for v in lats if math.isfinite(v)), 0.0)
    return ProfileTable(dict(zip(keys, lats)), executor.provenance, charge)


def estimate_runtime(table, job, config, remaining_batches: int) -> float:
    """remaining batches x profiled seconds per batch (profiling.py:147-151)."""
    if remaining_batches < 0:
        raise ValueError("remaining_batches must be >= 0")
    return remaining_batches * table.latency(job.id, config.technique, config.gpus)


def feasible_entries(table, job, workload) -> list:
    """[(RunConfig, latency)] with finite latency, canonical order (profiling.py:154-161)."""
    cfgs = feasible_configs(job, workload.cluster, workload.techniques)
    lats = [table.entries.get((job.id, c.technique, c.gpus), INFEASIBLE) for c in cfgs]
    return [pair for pair in zip(cfgs, lats) if math.isfinite(pair[1])]


def ensure_complete(table, workload) -> None:
    """Every feasible configuration of every job must be in the table (profiling.py:164-170)."""
    missing = ((j.id, c.technique, c.gpus) for j in workload.jobs
               for c in feasible_configs(j, workload.cluster, workload.techniques))
    for key in missing:
        if key not in table.entries:
            raise E.MissingEntry(key)
