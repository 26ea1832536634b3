"""File formats on either side of the search: profile CSV in, workload JSON in/out, plan JSON out.

* profile CSV (profiling.py:22, 173-215): header ``job,technique,gpus,latency_s``, ``inf``
  marks an infeasible configuration; ``load_profiles`` raises ``ParseError`` /
  ``NegativeLatency`` with the 1-based line number exactly where the reference does;
  ``save_profiles`` writes rows sorted by key with ``repr`` floats (byte-identical output).
* workload JSON (core.py:290-310): the pydantic ``model_dump_json(indent=2)`` layout
  (fields in declaration order), parsed and validated with ``validate_workload``.
* plan JSON (the output of ``decode_plan``): entries keyed by job id.

These let measured tables flow into the engine unchanged.
"""

from __future__ import annotations

import json
import math
from pathlib import Path

from . import domain as D
from . import errors as E
from .profiling import INFEASIBLE, ProfileTable

CSV_HEADER = "job,technique,gpus,latency_s"


# ---------------------------------------------------------------- profile CSV
def parse_profiles(text: str) -> ProfileTable:
    lines = text.split("\n")
    if not lines or lines[0].strip() != CSV_HEADER:
        raise E.ParseError(1, f"expected header {CSV_HEADER!r}")
    entries: dict = {}
    for idx, line in enumerate(lines[1:], start=2):
        if not line.strip():
            continue
        parts = line.split(",")
        if len(parts) != 4:
            raise E.ParseError(idx, f"expected 4 comma-separated fields, got {len(parts)}")
        job_id, tech, g_raw, lat_raw = (p.strip() for p in parts)
        try:
            g = int(g_raw)
        except ValueError:
            raise E.ParseError(idx, f"bad gpu count {g_raw!r}") from None
        if g < 1:
            raise E.ParseError(idx, f"gpu count must be >= 1, got {g}")
        if lat_raw == "inf":
            lat = INFEASIBLE
        else:
            try:
                lat = float(lat_raw)
            except ValueError:
                raise E.ParseError(idx, f"bad latency {lat_raw!r}") from None
            if lat <= 0:
                raise E.NegativeLatency(idx, lat)
        key = (job_id, tech, g)
        if key in entries:
            raise E.ParseError(idx, f"duplicate entry for {key}")
        entries[key] = lat
    return ProfileTable(entries, "ingested")


def load_profiles(path) -> ProfileTable:
    return parse_profiles(Path(path).read_text(encoding="utf-8"))


def dump_profiles(table) -> str:
    rows = [CSV_HEADER]
    for (job_id, tech, g), lat in sorted(table.entries.items()):
        rows.append(f"{job_id},{tech},{g},{'inf' if math.isinf(lat) else repr(lat)}")
    return "\n".join(rows) + "\n"


def save_profiles(table, path) -> None:
    Path(path).write_text(dump_profiles(table), encoding="utf-8")


# ---------------------------------------------------------------- workload JSON
_JOB_FIELDS = ("id", "total_batches", "base_batch_time", "model_memory", "activation_memory")
_NODE_FIELDS = ("id", "gpu_count", "gpu_memory")
_TECH_FIELDS = ("name", "archetype", "serial_fraction", "comm_overhead", "offload_multiplier", "min_gpus")


def _strict(kind: str, payload, fields) -> dict:
    if not isinstance(payload, dict):
        raise E.InvariantViolation(kind, "expected an object")
    extra = set(payload) - set(fields)
    if extra:                                              # extra="forbid" (core.py:22)
        raise E.InvariantViolation(f"{kind}.{sorted(extra)[0]}", "Extra inputs are not permitted")
    return payload


def workload_from_dict(payload: dict) -> D.Workload:
    try:
        _strict("workload", payload, ("jobs", "cluster", "techniques"))
        jobs = tuple(D.JobSpec(**_strict("jobs", j, _JOB_FIELDS)) for j in payload["jobs"])
        cl = _strict("cluster", payload["cluster"], ("nodes",))
        nodes = tuple(D.NodeSpec(**_strict("nodes", n, _NODE_FIELDS)) for n in cl["nodes"])
        techs = tuple(D.TechniqueSpec(**_strict("techniques", t, _TECH_FIELDS)) for t in payload["techniques"])
    except KeyError as exc:
        raise E.InvariantViolation(str(exc.args[0]), "Field required") from None
    except TypeError as exc:
        raise E.InvariantViolation("workload", str(exc)) from None
    return D.Workload(jobs=jobs, cluster=D.ClusterSpec(nodes=nodes), techniques=techs)


def workload_to_dict(w) -> dict:
    def row(obj, fields):
        return {f: getattr(obj, f) for f in fields}

    return {"jobs": [row(j, _JOB_FIELDS) for j in w.jobs],
            "cluster": {"nodes": [row(n, _NODE_FIELDS) for n in w.cluster.nodes]},
            "techniques": [row(t, _TECH_FIELDS) for t in w.techniques]}


def load_workload(path) -> D.Workload:
    raw = Path(path).read_text(encoding="utf-8")
    try:
        payload = json.loads(raw)
    except json.JSONDecodeError as exc:
        raise E.InvariantViolation("<file>", f"not valid JSON: {exc}") from exc
    return D.validate_workload(workload_from_dict(payload))


def save_workload(w, path) -> None:
    Path(path).write_text(json.dumps(workload_to_dict(w), indent=2) + "\n", encoding="utf-8")


# ---------------------------------------------------------------- plan JSON
def plan_to_dict(plan) -> dict:
    return {"entries": {jid: {"config": {"technique": e.config.technique, "gpus": e.config.gpus},
                              "node": e.node, "start_time": e.start_time}
                        for jid, e in sorted(plan.entries.items())},
            "predicted_makespan": plan.predicted_makespan}


def plan_from_dict(payload: dict) -> D.Plan:
    entries = {jid: D.PlanEntry(D.RunConfig(e["config"]["technique"], int(e["config"]["gpus"])), e["node"],
                                float(e["start_time"]))
               for jid, e in payload["entries"].items()}
    return D.Plan(entries, float(payload["predicted_makespan"]))
