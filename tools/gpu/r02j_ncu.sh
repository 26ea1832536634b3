# Round-2 kernel captures of the current code: k_cand sampled (configs 3, 4), k_ls of the default
# solve (configs 4, 5), launch lists of the default solves (configs 3-5), host cProfile of the
# public-API solve.  Summaries land in gpurun_out/ (tools/ncu_summary.py), reports are removed.
R=r02j
summ() {  # rep json label
  python tools/ncu_summary.py full gpurun_out/$1.ncu-rep gpurun_out/$2 "$3" > /dev/null 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page details > gpurun_out/$1_details.txt 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>/dev/null
  rm -f gpurun_out/$1.ncu-rep
}
for c in 3 4; do
  python bench.py --config $c --budget 16777216 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain$c.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cand -s 1 -c 1 -o gpurun_out/cand_cfg$c \
    python bench.py --config $c --budget 16777216 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cand$c.log 2>&1
  summ cand_cfg$c ${R}_ncu_full_k_cand_cfg$c.json "$R: k_cand sampled 2^24, config $c"
done
for c in 4 5; do
  python tools/one_solve.py $c > gpurun_out/solve_plain$c.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ls -c 1 -o gpurun_out/ls_cfg$c \
    python tools/one_solve.py $c > gpurun_out/ncu_ls$c.log 2>&1
  summ ls_cfg$c ${R}_ncu_full_k_ls_cfg$c.json "$R: k_ls, first launch of the default config-$c solve (greedy starts)"
done
for c in 3 4 5; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_solve_cfg$c.csv \
    python tools/one_solve.py $c > gpurun_out/ncu_launch_solve$c.log 2>&1
done
for c in 1 3 4 5; do timeout 300 python tools/solve_cprofile.py $c 30 > gpurun_out/${R}_solve_cprofile_cfg$c.txt 2>&1; done
du -sh gpurun_out
