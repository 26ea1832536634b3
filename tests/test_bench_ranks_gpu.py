"""`python bench.py --gpus 2` on a one-GPU box: bench.py re-executes itself under
torch.distributed.run with two ranks; SATURN_BENCH_GPU_OVERRIDE=0 maps both onto cuda:0 through
gloo (a functional check of the sharded path -- never a bench number).  The two-rank line must
report n_gpus 2 and the same best key, makespan and time-to-best status as the one-rank line
(configs 1 and 4: the exhaustive tree scan sharded by tasks, the sampled stream sharded by
candidate ranges, bound-and-prune / local search with the shared incumbent cell)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args, env_extra=None):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=420)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("cfg", [1, 4])
def test_bench_two_ranks_equal_one(cfg):
    common = ["--config", str(cfg), "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-index-leg",
              "--budget", str(1 << 22)]
    one = _line(common)
    two = _line(common + ["--gpus", "2"], {"SATURN_BENCH_GPU_OVERRIDE": "0"})
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["best"] == one["best"]
    assert two["time_to_best"].get("status") == one["time_to_best"].get("status")
    if cfg == 4:
        assert two["time_to_best"]["makespan_intervals"] == one["time_to_best"]["makespan_intervals"]
