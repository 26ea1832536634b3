timeout 600 python tools/table2_mirror.py > gpurun_out/table2.log 2>&1
cat > /tmp/lsp.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2311_02840_b200 import planners as PL
from paper_2311_02840_b200.problem import SolveOptions
from paper_2311_02840_b200.workloads import config_workload
k = int(sys.argv[1])
w, t, c = config_workload(k)
s = PL.solve(t, w, None, SolveOptions(search="local", walkers=1024, wave=1024))
print(k, s.makespan, s.search.device_seconds, s.search.stats)
PY
for c in 4 5; do python /tmp/lsp.py $c > gpurun_out/lsp_plain$c.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ls -c 1 -o gpurun_out/ls_cfg$c python /tmp/lsp.py $c > gpurun_out/ncu_ls$c.log 2>&1; done
