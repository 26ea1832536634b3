# full evidence: tests, smoke, every bench config, reference arm, launch list, ncu captures
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_cfg1.log 2>&1
for c in 2 3 4 5; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain1.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain1b.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tree -c 2 -o gpurun_out/tree_cfg1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_tree.log 2>&1
for c in 3 4 5; do python bench.py --config $c --budget 16777216 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain$c.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_cand|k_ls' -s 1 -c 2 -o gpurun_out/cand_cfg$c python bench.py --config $c --budget 16777216 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cand$c.log 2>&1; done
ls -la gpurun_out
