# After the Multi16 placement specialisation: GPU suite, smoke, parity stress, bench lines,
# ncu of k_cand / k_ls at config 4.
R=${1:-r02k}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/${R}_gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/${R}_smoke.log
STRESS_TRIALS=1500 STRESS_SEED=91 timeout 900 python tools/parity_stress.py > gpurun_out/${R}_parity_stress.txt 2>&1; echo stress_exit=$? >> gpurun_out/${R}_parity_stress.txt
for c in 4 3 5 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_bench_cfg$c.log 2>&1; done
timeout 300 python tools/solve_cprofile.py 4 30 > gpurun_out/${R}_solve_cprofile_cfg4.txt 2>&1
summ() {
  python tools/ncu_summary.py full gpurun_out/$1.ncu-rep gpurun_out/$2 "$3" > /dev/null 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>/dev/null
  rm -f gpurun_out/$1.ncu-rep
}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cand -s 1 -c 1 -o gpurun_out/cand_cfg4 \
  python bench.py --config 4 --budget 16777216 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cand4.log 2>&1
summ cand_cfg4 ${R}_ncu_full_k_cand_cfg4.json "$R: k_cand sampled 2^24, config 4 (specialised Multi16 placement)"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ls -c 1 -o gpurun_out/ls_cfg4 \
  python tools/one_solve.py 4 > gpurun_out/ncu_ls4.log 2>&1
summ ls_cfg4 ${R}_ncu_full_k_ls_cfg4.json "$R: k_ls, first launch of the default config-4 solve (specialised Multi16 placement)"
tail -n 3 gpurun_out/${R}_gputests.log gpurun_out/${R}_smoke.log gpurun_out/${R}_parity_stress.txt
