# wide state-space search after a kernel change: its tests, the parity stress DP families, rates
timeout 600 python -m pytest tests/test_dp_gpu.py -x -q > gpurun_out/dpw_tests.log 2>&1; echo rc=$? >> gpurun_out/dpw_tests.log
STRESS_TRIALS=1000 STRESS_SEED=93 timeout 900 python tools/parity_stress.py > gpurun_out/dpw_stress.txt 2>&1; echo rc=$? >> gpurun_out/dpw_stress.txt
rm -f gpurun_out/dpw_rates.txt
for a in "14 3 4 114 15 25" "14 2 4 112 23 25" "14 2 8 113 15 23" "12 2 4 124 22 23 exact" "14 4 8 115 12 23"; do
  timeout 300 python tools/dp_wide_probe.py $a >> gpurun_out/dpw_rates.txt 2>&1
done
tail -n 2 gpurun_out/dpw_tests.log; tail -n 2 gpurun_out/dpw_stress.txt; cat gpurun_out/dpw_rates.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dp_expand_wide -s 22 -c 1 -o gpurun_out/dpw \
  python tools/dp_wide_probe.py 14 3 4 114 15 25 > gpurun_out/ncu_dpw.log 2>&1
ncu -i gpurun_out/dpw.ncu-rep --page source --csv > gpurun_out/dpw_source.csv 2>/dev/null
ncu -i gpurun_out/dpw.ncu-rep --page details > gpurun_out/dpw_details.txt 2>/dev/null
rm -f gpurun_out/dpw.ncu-rep
timeout 300 python tools/dp_probe.py 3 29 30 > gpurun_out/dp_cfg3.txt 2>&1; cat gpurun_out/dp_cfg3.txt
timeout 300 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); t=d['time_to_best']; print('cfg3 ttb', t['device_s'], t['wall_s'], t['status'])"
timeout 600 python tools/multinode_optimality.py 32 > gpurun_out/mn_opt2.txt 2>&1; tail -2 gpurun_out/mn_opt2.txt
