"""Table 2 mirror: Saturn (with introspection) / Optimus-Dynamic / Current
Practice / Random executed makespans on the generated mirror presets, 1 and 2 nodes."""
import sys, os, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_acceptance_gpu import _compare, _table
from paper_2311_02840_b200 import planners as PL, simulator as SIM
from paper_2311_02840_b200.workloads import generate_workload
for preset in ("wikitext_mirror", "imagenet_mirror"):
    for n in (1, 2):
        w = generate_workload(preset, n, 7)
        t0 = time.time()
        reps = _compare(w)
        print(preset, n, [round(r.makespan / 3600, 2) for r in reps], "h", "%.1fs" % (time.time() - t0), flush=True)
