# Final round-2 capture: GPU suite, smoke, every bench line (both arms), cfg1 launch list,
# bounds-checked build over the suite, one-solve launch list of config 3.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/smoke.log
bash tools/gpu/bench_all.sh r02t
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain1.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02t_launches_cfg1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02t_launches_solve_cfg3.csv python tools/one_solve.py 3 > /dev/null 2>&1
bash tools/gpu/debug_bounds.sh
tail -n 2 gpurun_out/gputests.log gpurun_out/smoke.log gpurun_out/debug_gputests.log gpurun_out/debug_small.log
