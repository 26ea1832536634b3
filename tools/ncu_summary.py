"""Summarise an ncu report (.ncu-rep) or a launch-list CSV into profiles/ (run in the build container).

    python tools/ncu_summary.py full  <report.ncu-rep> <out.json> [label]
    python tools/ncu_summary.py launches <launches.csv> <out.json> [label]

`full`: the counters the north star asks for (issue utilisation, ALU / FMA pipe
share, lane efficiency, shared-memory wavefronts, DRAM bytes) for each profiled
kernel.  `launches`: per-kernel launch count, total and share of device time
from an `ncu --metrics gpu__time_duration.sum` list.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes.sum.per_second",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__maximum_warps_per_active_cycle_pct",
    "smsp__warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__warps_issue_stalled_selected_per_issue_active.ratio",
]


def _num(s: str):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return s


def full(rep: str, label: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        rec = {"kernel": vals[head.index("Kernel Name")]}
        for m in FULL_METRICS:
            if m in head:
                i = head.index(m)
                rec[m] = {"value": _num(vals[i]), "unit": units[i]}
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = rec.get("dram__bytes_read.sum")
        wr = rec.get("dram__bytes_write.sum")
        if rd and wr:
            rec["traffic_bytes"] = rd["value"] * scale.get(rd["unit"], 1) + wr["value"] * scale.get(wr["unit"], 1)
        kernels.append(rec)
    return {"label": label, "source": rep.split("/")[-1], "kind": "ncu --set full --clock-control none",
            "kernels": kernels}


def launches(path: str, label: str) -> dict:
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        ns = float(r["Metric Value"].replace(",", ""))
        a = agg.setdefault(name, {"launches": 0, "total_ns": 0.0})
        a["launches"] += 1
        a["total_ns"] += ns
    total = sum(a["total_ns"] for a in agg.values()) or 1.0
    ks = [{"kernel": k, "launches": a["launches"], "total_ms": a["total_ns"] / 1e6,
           "avg_ms": a["total_ns"] / 1e6 / a["launches"], "share": a["total_ns"] / total}
          for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["total_ns"])]
    return {"label": label, "source": path.split("/")[-1],
            "kind": "ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised)",
            "total_ms": total / 1e6, "kernels": ks}


def main():
    mode, src, dst = sys.argv[1:4]
    label = sys.argv[4] if len(sys.argv) > 4 else ""
    res = full(src, label) if mode == "full" else launches(src, label)
    with open(dst, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
