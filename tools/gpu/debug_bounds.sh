# Bounds-checked library (SAT_ASSERT on every shared-memory region index) through the small
python -m paper_2311_02840_b200.build --debug > gpurun_out/debug_build.log 2>&1 || exit 1
# all-kernel script and the whole GPU parity suite; compute-sanitizer is closed on this pool.
export SATURN_ENGINE_LIB=$PWD/paper_2311_02840_b200/_lib/libsaturn_b200_debug.so
timeout 300 python tools/sanitize_small.py > gpurun_out/debug_small.log 2>&1; echo rc=$? >> gpurun_out/debug_small.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/debug_gputests.log 2>&1; echo rc=$? >> gpurun_out/debug_gputests.log
timeout 300 python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/debug_cfg5.log 2>&1; echo rc=$? >> gpurun_out/debug_cfg5.log
timeout 300 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/debug_cfg4.log 2>&1; echo rc=$? >> gpurun_out/debug_cfg4.log
