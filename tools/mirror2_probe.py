import sys, os
sys.path.insert(0, os.getcwd())
from paper_2311_02840_b200 import planners as PL, workloads as WL
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table
from paper_2311_02840_b200 import engine as EN
for ds in ("wikitext_mirror",):
    w = WL.generate_workload(ds, 2, seed=7)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    s = PL.solve(t, w)
    print(s.status, s.makespan, s.lower_bound, s.search.stats)
    eng = PL.get_engine(0)
    for T in (16, 17):
        for ms in (1 << 22, 1 << 24):
            st, info, c = eng.dp_search(EN.NativeProblem(s.problem, 1), T, ms)
            print(T, ms, EN.DP_STATUS[st], info.levels, info.states, info.widest_level)
