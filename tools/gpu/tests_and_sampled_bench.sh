timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/gputests.log
for c in 3 4 5; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1; done
