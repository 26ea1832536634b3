"""File formats on either side of the search: profile CSV in, workload JSON in/out, plan JSON out.

* profile CSV (profiling.py:22, 173-215): header ``job,technique,gpus,latency_s``, ``inf``
  marks an infeasible configuration; ``load_profiles`` (a columnar reader) raises
  ``ParseError`` / ``NegativeLatency`` with the 1-based line number and message the reference
  raises for the same text; ``save_profiles`` writes rows sorted by key with ``repr`` floats
  (byte-identical output).  The reference's own reader feeds the engine just as well
  (tests/test_dropin_reference_gpu.py).
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
# Columnar reader: the body is tokenised into columns first, every row gets the verdict of the
# first rule it breaks (field count, gpu count, latency, duplicate key -- the reference's check
# order, profiling.py:173-209), and the lowest failing line raises.  Parsing stops at the first
# bad line in the reference, so every row above it is valid: a row is a duplicate iff its key
# appears on an earlier row.

def _as_int(raw: str):
    try:
        return int(raw)
    except ValueError:
        return None


def _as_latency(raw: str):
    if raw == "inf":
        return INFEASIBLE
    try:
        return float(raw)
    except ValueError:
        return None


def _row_error(line_no: int, n_fields: int, g_raw: str, g, lat_raw: str, lat, duplicate_of):
    """The error the reference raises for this row (None if the row is good)."""
    if n_fields != 4:
        return E.ParseError(line_no, f"expected 4 comma-separated fields, got {n_fields}")
    if g is None:
        return E.ParseError(line_no, f"bad gpu count {g_raw!r}")
    if g < 1:
        return E.ParseError(line_no, f"gpu count must be >= 1, got {g}")
    if lat is None:
        return E.ParseError(line_no, f"bad latency {lat_raw!r}")
    if lat <= 0:
        return E.NegativeLatency(line_no, lat)
    if duplicate_of is not None:
        return E.ParseError(line_no, f"duplicate entry for {duplicate_of}")
    return None


def parse_profiles(text: str) -> ProfileTable:
    """Profile CSV text (header ``job,technique,gpus,latency_s``; ``inf`` = infeasible) -> table."""
    head, _, body = text.partition("\n")
    if head.strip() != CSV_HEADER:
        raise E.ParseError(1, f"expected header {CSV_HEADER!r}")
    rows = [(no, ln.split(",")) for no, ln in enumerate(body.split("\n"), start=2) if ln.strip()]
    width = [len(f) for _, f in rows]
    cols = [[p.strip() for p in f] if len(f) == 4 else ["", "", "", ""] for _, f in rows]
    jobs, techs, g_raw, lat_raw = (list(c) for c in zip(*cols)) if cols else ([], [], [], [])
    gs = [_as_int(x) for x in g_raw]
    lats = [_as_latency(x) for x in lat_raw]
    first_row: dict = {}
    for r, (no, _) in enumerate(rows):
        key = (jobs[r], techs[r], gs[r])
        dup = key if width[r] == 4 and key in first_row else None
        err = _row_error(no, width[r], g_raw[r], gs[r], lat_raw[r], lats[r], dup)
        if err is not None:
            raise err
        first_row[key] = r
    return ProfileTable({k: lats[r] for k, r in first_row.items()}, "ingested")


def load_profiles(path) -> ProfileTable:
    return parse_profiles(Path(path).read_text(encoding="utf-8"))


def dump_profiles(table) -> str:
    """Rows in key order, shortest round-trip floats (``repr``), ``inf`` for misfits."""
    body = "".join(f"{j},{t},{g},{'inf' if v == INFEASIBLE else repr(v)}\n"
                   for (j, t, g), v in sorted(table.entries.items()))
    return f"{CSV_HEADER}\n{body}"


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
