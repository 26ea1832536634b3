"""Multi-rank logic on CPU (gloo, world_size 2): shard partition + all-reduce MIN combine.

The GPU path issues exactly this combine over NCCL after each rank's kernel; here each
rank's partial key comes from the C oracle on its shard."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import golden_workload

from oracle import coracle as C
from oracle import saturn_oracle as O
from paper_2311_02840_b200 import engine as EN
from paper_2311_02840_b200.profiling import SyntheticExecutor, build_profile_table


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pack(ms, ident, grid, idx_bits):
    if ms == float("inf"):
        return torch.tensor([-1, -1], dtype=torch.int64)
    if grid:
        return torch.tensor([(int(ms) << idx_bits) | ident, -1], dtype=torch.int64)
    bits = int(np.array([ms], dtype=np.float64).view(np.int64)[0])
    return torch.tensor([bits, ident], dtype=torch.int64)


def _worker(rank, world, port, name, grid, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, _ = golden_workload(name)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    op = O.build(t.entries, w, grid=grid)
    n = min(op.space, 60000)
    a, b = EN._shard(n, rank, world)
    ms, ident = C.CProblem(op).search(lo=a, hi=b) if b > a else (float("inf"), 0)
    key = EN._combine(_pack(ms, ident, grid, 40), grid, None, world)
    out[rank] = key
    dist.destroy_process_group()


@pytest.mark.parametrize("grid", [True, False])
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_allreduce_min_matches_single_rank(grid, world):
    name = "small5_1x4"
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    ps = [ctx.Process(target=_worker, args=(r, world, _free_port() if r < 0 else PORTS[world], name, grid, out))
          for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    w, _ = golden_workload(name)
    t = build_profile_table(w, SyntheticExecutor(w.cluster))
    op = O.build(t.entries, w, grid=grid)
    ms, ident = C.CProblem(op).search(hi=min(op.space, 60000))
    for r in range(world):
        key = out[r]
        if grid:
            assert (key[0] >> 40, key[0] & ((1 << 40) - 1)) == (int(ms), ident)
        else:
            got = float(np.array([key[0]], dtype=np.int64).view(np.float64)[0])
            assert got.hex() == float(ms).hex() and key[1] == ident


PORTS = {2: _free_port(), 3: _free_port()}


def test_shard_partition_covers_range():
    for n in (0, 1, 7, 10**12 + 3):
        for world in (1, 2, 3, 8):
            parts = [EN._shard(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
