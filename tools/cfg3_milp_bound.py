"""Is the config-3 local-search plan optimal?  The list-scheduling optimum is >= the
time-indexed MILP optimum (any non-preemptive gang schedule, backfilling
allowed), so if HiGHS proves the MILP infeasible with horizon K = found - 1, the plan the
engine found is optimal.  CPU only; prints HiGHS' verdict and time."""

import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])

from oracle import saturn_oracle  # noqa: E402
from paper_2311_02840_b200.workloads import config_workload  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 29
    limit = float(sys.argv[3]) if len(sys.argv) > 3 else 1800.0
    w, t, _ = config_workload(cfg)
    op = saturn_oracle.build(t.entries, w)
    t0 = time.perf_counter()
    try:
        opt = saturn_oracle.milp_optimum(op, horizon=k, time_limit=limit)
        verdict = f"feasible within K={k}: MILP optimum {opt}"
    except RuntimeError as e:
        verdict = f"K={k}: {e}"
    print(f"config {cfg}: {verdict} ({time.perf_counter() - t0:.1f} s, HiGHS)")


if __name__ == "__main__":
    main()
