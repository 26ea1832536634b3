# GPU suite + smoke + wall per public-API solve (and its cProfile) + bench lines cfg1/3/4/5.
T=${1:-hc}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/${T}_gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/${T}_smoke.log
for c in 1 3 4 5; do timeout 300 python tools/solve_cprofile.py $c 30 > gpurun_out/${T}_solve_cprofile_cfg$c.txt 2>&1; done
for c in 1 3 4 5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_cfg$c.log 2>&1; done
head -1 gpurun_out/${T}_solve_cprofile_cfg*.txt
tail -2 gpurun_out/${T}_gputests.log gpurun_out/${T}_smoke.log
