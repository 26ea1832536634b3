"""Checkpoint / resume of the exact searches: a search stopped after any
number of chunks and resumed from its saved cursor returns exactly the one-shot key and plan."""

import os

import pytest

from helpers import golden_workload

from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200 import resume as R
from paper_2311_02840_b200.problem import SolveOptions, build_problem
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table
from paper_2311_02840_b200.workloads import config_workload

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,kernel", [("cfg1", "tree"), ("cfg1", "auto"), ("small4_2x2", "auto"),
                                         ("small5_1x4", "tree")])
def test_chunked_resume_equals_one_shot(name, kernel, tmp_path):
    if name.startswith("cfg"):
        w, t, _ = config_workload(int(name[3:]))
    else:
        w, _ = golden_workload(name)
        t = build_profile_table(w, SyntheticExecutor(w.cluster))
    opts = SolveOptions(kernel=kernel)
    one = PL.solve(t, w, None, opts)
    eng = PL.get_engine(0)
    prob = build_problem(t, w, opts)
    cur = R.start_cursor(eng, prob, opts)
    path = tmp_path / "cursor.json"
    steps = 0
    while not cur.done:                       # 1/7 of the range per "session", saved and reloaded
        R.run_cursor(eng, prob, cur, chunk=max(1, cur.end // 7), max_chunks=1)
        cur.save(path)
        cur = R.SearchCursor.load(path)
        steps += 1
    assert steps == cur.chunks and cur.chunks >= min(7, cur.end)
    assert R.cursor_result(prob, cur) == (one.makespan, one.search.index)


def test_solve_suspends_and_resumes(tmp_path):
    """plan_saturn with a time budget: Suspended with a checkpoint on disk, then Optimal with
    the one-shot plan once resumed (the checkpoint is removed)."""
    w, t, _ = config_workload(1)
    opts = SolveOptions(kernel="tree")
    one = PL.solve(t, w, None, opts)
    path = str(tmp_path / "cfg1.ckpt")
    first = PL.solve(t, w, None, opts, checkpoint=path, time_budget_s=0.002)
    assert first.status == "Suspended" and os.path.exists(path)
    assert first.cursor.next < first.cursor.end
    sol = first
    for _ in range(20000):
        sol = PL.solve(t, w, None, opts, checkpoint=path, time_budget_s=0.05)
        if sol.status != "Suspended":
            break
    assert sol.status == "Optimal" and not os.path.exists(path)
    assert (sol.makespan, sol.plan) == (one.makespan, one.plan)
