# full evidence: tests, smoke, every bench config, reference arm, launch list, ncu captures.
# ncu reports are summarised on the box (tools/ncu_summary.py) and removed: gpurun_out must
# stay under 64 MiB to come back.
R=${ROUND_TAG:-r01d}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_cfg1.log 2>&1
for c in 2 3 4 5; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain1.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
summ() {  # rep json label
  python tools/ncu_summary.py full gpurun_out/$1.ncu-rep gpurun_out/$2 "$3" > /dev/null 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page details > gpurun_out/$1_details.txt 2>/dev/null
  rm -f gpurun_out/$1.ncu-rep
}
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain1b.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tree -c 1 -o gpurun_out/tree_cfg1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_tree.log 2>&1
summ tree_cfg1 ${R}_ncu_full_k_tree_cfg1.json "$R: k_tree<8> full scan, config 1"
for c in 3 4 5; do python bench.py --config $c --budget 16777216 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain$c.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cand -s 1 -c 1 -o gpurun_out/cand_cfg$c python bench.py --config $c --budget 16777216 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cand$c.log 2>&1; summ cand_cfg$c ${R}_ncu_full_k_cand_cfg$c.json "$R: k_cand sampled 2^24, config $c"; done
python tools/ls_seed_check.py > gpurun_out/plain_ls.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ls -c 1 -o gpurun_out/ls_cfg3 python tools/ls_seed_check.py > gpurun_out/ncu_ls3.log 2>&1
summ ls_cfg3 ${R}_ncu_full_k_ls_cfg3.json "$R: k_ls local search, config 3, one 4096-walker wave"
python tools/ls_one_walker.py 5 4096 > gpurun_out/plain_ls5.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ls -c 1 -o gpurun_out/ls_cfg5 python tools/ls_one_walker.py 5 4096 > gpurun_out/ncu_ls5.log 2>&1
summ ls_cfg5 ${R}_ncu_full_k_ls_cfg5.json "$R: k_ls local search, config 5, one 4096-walker wave (4 warps per walker, stop at the bound)"
timeout 600 python tools/shard_emulation.py tree bnb > gpurun_out/${R}_shard_emulation.txt 2>&1
bash tools/ls_group_sweep.sh > gpurun_out/${R}_ls_group_sweep.txt 2>&1
du -sh gpurun_out; ls -la gpurun_out
