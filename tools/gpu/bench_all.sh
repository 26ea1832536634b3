# Every bench line of the round (configs 1-5, our arm and the reference arm) on one box.
# Usage (under gpurun): bash tools/gpu/bench_all.sh <tag>
TAG=${1:-r02}
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_cfg$c.log 2>&1
  timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_reference_cfg$c.log 2>&1
done
for c in 1 2 3 4 5; do tail -c 400 gpurun_out/${TAG}_bench_cfg$c.log; echo; done
