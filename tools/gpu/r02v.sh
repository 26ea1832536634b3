# After the no-release placement path: GPU suite, smoke, parity stress, bench lines of the
# sampled configs (both arms), the k_cand cfg3 capture.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02v_gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/r02v_gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02v_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/r02v_smoke.log
STRESS_TRIALS=2000 STRESS_SEED=96 timeout 900 python tools/parity_stress.py > gpurun_out/r02v_parity_stress.txt 2>&1; echo stress_exit=$? >> gpurun_out/r02v_parity_stress.txt
for c in 3 4 5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r02v_bench_cfg$c.log 2>&1; done
python bench.py --config 3 --budget 16777216 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cand -s 1 -c 1 -o gpurun_out/cand_cfg3 \
  python bench.py --config 3 --budget 16777216 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cand3.log 2>&1
python tools/ncu_summary.py full gpurun_out/cand_cfg3.ncu-rep gpurun_out/r02v_ncu_full_k_cand_cfg3.json "r02v: k_cand sampled 2^24, config 3 (no-release placement path)" > /dev/null 2>&1
rm -f gpurun_out/cand_cfg3.ncu-rep
tail -n 2 gpurun_out/r02v_gputests.log gpurun_out/r02v_smoke.log; tail -n 2 gpurun_out/r02v_parity_stress.txt
