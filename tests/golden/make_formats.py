"""Golden fixtures for the ingest / output formats, produced by the REFERENCE package.

Run in the build container (needs /root/reference):  python tests/golden/make_formats.py
Writes tests/golden/formats_golden.json:
  * workload JSON written by core.save_workload (core.py:309-310) for two workloads,
  * profile CSV written by profiling.save_profiles (profiling.py:211-215) for them,
  * what profiling.load_profiles (profiling.py:173-208) makes of malformed CSVs
    (error class and line number) and of a valid one (entries as hex floats).
"""

from __future__ import annotations

import json
import math
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

from jointsched import core, profiling  # noqa: E402
from jointsched import errors as ref_errors  # noqa: E402

GOLD = os.path.join(HERE, "reference_golden.json")

BAD_CSVS = {
    "no_header": "job,tech,gpus,lat\na,t,1,1.0\n",
    "short_row": "job,technique,gpus,latency_s\na,t,1\n",
    "bad_gpus": "job,technique,gpus,latency_s\na,t,1,1.0\na,t,x,2.0\n",
    "zero_gpus": "job,technique,gpus,latency_s\na,t,0,1.0\n",
    "bad_latency": "job,technique,gpus,latency_s\na,t,1,fast\n",
    "negative": "job,technique,gpus,latency_s\na,t,1,1.0\n\na,t,2,-3.5\n",
    "zero_latency": "job,technique,gpus,latency_s\na,t,1,0\n",
    "duplicate": "job,technique,gpus,latency_s\na,t,1,1.0\na, t ,1,2.0\n",
    "valid": "job,technique,gpus,latency_s\n a ,t,1,1.5\na,t,2,inf\nb,u,4,0.1\n\n",
}


def fhex(x):
    return "inf" if math.isinf(x) else float(x).hex()


def main():
    gold = json.load(open(GOLD))
    out = {"workloads": {}, "bad_csv": {}}
    tmp = tempfile.mkdtemp()
    for name in ("cfg1", "hetero6"):
        w = core.workload_from_dict(gold["workloads"][name]["workload"])
        core.save_workload(w, os.path.join(tmp, "w.json"))
        t = profiling.build_profile_table(w, profiling.SyntheticExecutor(w.cluster))
        profiling.save_profiles(t, os.path.join(tmp, "p.csv"))
        out["workloads"][name] = {"workload_json": open(os.path.join(tmp, "w.json")).read(),
                                  "profile_csv": open(os.path.join(tmp, "p.csv")).read()}
    for name, text in BAD_CSVS.items():
        path = os.path.join(tmp, name + ".csv")
        open(path, "w").write(text)
        try:
            t = profiling.load_profiles(path)
            out["bad_csv"][name] = {"text": text, "entries": [[list(k), fhex(v)] for k, v in sorted(t.entries.items())]}
        except ref_errors.SchedulerError as exc:
            out["bad_csv"][name] = {"text": text, "error": type(exc).__name__,
                                    "line_no": getattr(exc, "line_no", None), "message": str(exc)}
    with open(os.path.join(HERE, "formats_golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
