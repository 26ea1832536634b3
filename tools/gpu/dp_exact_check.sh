# Exact multi-node state-space search (ABI v8): its tests first, then the GPU suite, smoke and
# the parity stress with the exact family.
timeout 600 python -m pytest tests/test_dp_gpu.py -x -q > gpurun_out/dpx_tests.log 2>&1; echo dp_tests_exit=$? >> gpurun_out/dpx_tests.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/dpx_gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/dpx_gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dpx_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/dpx_smoke.log
STRESS_TRIALS=1000 STRESS_SEED=92 timeout 900 python tools/parity_stress.py > gpurun_out/dpx_parity_stress.txt 2>&1; echo stress_exit=$? >> gpurun_out/dpx_parity_stress.txt
tail -n 4 gpurun_out/dpx_tests.log; tail -n 3 gpurun_out/dpx_gputests.log; tail -n 2 gpurun_out/dpx_smoke.log; tail -n 3 gpurun_out/dpx_parity_stress.txt
