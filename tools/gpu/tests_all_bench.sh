timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/smoke.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg1.log 2>&1
for c in 2 3 4 5; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1; done
