# Functional check of the sharded (multi-rank) path on ONE GPU: two ranks share cuda:0 through
# gloo (SATURN_BENCH_GPU_OVERRIDE); results must equal the single-rank run.  Not a bench number.
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/shard_n1.log 2>&1
SATURN_BENCH_GPU_OVERRIDE=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/shard_n2.log 2>&1
SATURN_BENCH_GPU_OVERRIDE=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 \
  --master-addr 127.0.0.1 --master-port 29534 bench.py --config 4 --gpus 3 --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/shard_n3_cfg4.log 2>&1
timeout 300 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/shard_n1_cfg4.log 2>&1
cat > /tmp/h6.py <<'PY'
import sys, os, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch
from helpers import golden_workload
from paper_2311_02840_b200 import engine as EN, planners as PL
from paper_2311_02840_b200.problem import build_problem, SolveOptions
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table
w, _ = golden_workload("hetero6")
t = build_profile_table(w, SyntheticExecutor(w.cluster))
p = build_problem(t, w)
eng = PL.get_engine(0)
bits, _ = p.key_bits(p.space)
nprob = EN.NativeProblem(p, bits)
for n in (1 << 26, 1 << 28):
    best = eng.reset_best(); torch.cuda.synchronize(); t0 = time.perf_counter()
    eng.search_index(nprob, 0, n, best); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print("hetero6 index", n, "%.3e plans/s" % (n / dt), flush=True)
    sp = EN.NativeProblem(p, 30)
    best = eng.reset_best(); torch.cuda.synchronize(); t0 = time.perf_counter()
    eng.search_sampled(sp, EN.SRC_SUBSTREAM, 7, 0, n, best); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print("hetero6 sampled", n, "%.3e plans/s" % (n / dt), flush=True)
PY
timeout 300 python /tmp/h6.py > gpurun_out/hetero6_rate.log 2>&1
