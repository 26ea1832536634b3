# Late round-2 verification: GPU suite, smoke, long parity stress, multi-node optimality sweep.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02p_gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/r02p_gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02p_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/r02p_smoke.log
STRESS_TRIALS=4000 STRESS_SEED=2028 timeout 1500 python tools/parity_stress.py > gpurun_out/r02p_parity_stress.txt 2>&1; echo stress_exit=$? >> gpurun_out/r02p_parity_stress.txt
timeout 900 python tools/multinode_optimality.py 32 > gpurun_out/r02p_multinode_optimality.txt 2>&1
tail -n 2 gpurun_out/r02p_gputests.log gpurun_out/r02p_smoke.log; tail -n 5 gpurun_out/r02p_parity_stress.txt; tail -n 2 gpurun_out/r02p_multinode_optimality.txt
