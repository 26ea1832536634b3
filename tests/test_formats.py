"""Ingest / output formats against fixtures written by the reference itself
(tests/golden/make_formats.py): byte-identical writers, identical parses and errors."""

import json
import math
import os

import pytest

from helpers import golden, workload_from_json

from paper_2311_02840_b200 import errors as E
from paper_2311_02840_b200 import formats as F
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table

FIX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "formats_golden.json")))


@pytest.mark.parametrize("name", ["cfg1", "hetero6"])
def test_writers_byte_identical_to_reference(name, tmp_path):
    w = workload_from_json(golden()["workloads"][name]["workload"])
    F.save_workload(w, tmp_path / "w.json")
    assert (tmp_path / "w.json").read_text() == FIX["workloads"][name]["workload_json"]
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    F.save_profiles(t, tmp_path / "p.csv")
    assert (tmp_path / "p.csv").read_text() == FIX["workloads"][name]["profile_csv"]


@pytest.mark.parametrize("name", ["cfg1", "hetero6"])
def test_readers_roundtrip_reference_files(name, tmp_path):
    (tmp_path / "w.json").write_text(FIX["workloads"][name]["workload_json"])
    w = F.load_workload(tmp_path / "w.json")
    assert w == workload_from_json(golden()["workloads"][name]["workload"])
    (tmp_path / "p.csv").write_text(FIX["workloads"][name]["profile_csv"])
    t = F.load_profiles(tmp_path / "p.csv")
    ref = build_profile_table(w, SyntheticExecutor(w.cluster))
    assert t.entries == ref.entries and t.provenance == "ingested"


@pytest.mark.parametrize("name", sorted(FIX["bad_csv"]))
def test_profile_csv_errors_match_reference(name):
    case = FIX["bad_csv"][name]
    if "error" in case:
        with pytest.raises(getattr(E, case["error"])) as info:
            F.parse_profiles(case["text"])
        assert info.value.line_no == case["line_no"] and str(info.value) == case["message"]
    else:
        t = F.parse_profiles(case["text"])
        got = [[list(k), "inf" if math.isinf(v) else v.hex()] for k, v in sorted(t.entries.items())]
        assert got == case["entries"]


def test_workload_json_rejects_extra_and_missing_fields():
    d = golden()["workloads"]["cfg1"]["workload"]
    bad = json.loads(json.dumps(d))
    bad["jobs"][0]["colour"] = "red"
    with pytest.raises(E.InvariantViolation):
        F.workload_from_dict(bad)
    bad = json.loads(json.dumps(d))
    del bad["cluster"]
    with pytest.raises(E.InvariantViolation):
        F.workload_from_dict(bad)


def test_plan_json_roundtrip():
    from paper_2311_02840_b200 import domain as D

    p = D.Plan({"a": D.PlanEntry(D.RunConfig("t", 2), "n0", 12.5), "b": D.PlanEntry(D.RunConfig("u", 1), "n1", 0.0)},
               40.0)
    assert F.plan_from_dict(json.loads(json.dumps(F.plan_to_dict(p)))) == p
