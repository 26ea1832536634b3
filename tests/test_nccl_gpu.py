"""The NCCL leg of the sharded search on the one GPU a test box has: a one-rank NCCL group
runs the same all-reduce calls the N-GPU combine makes (int64 MIN of the packed key; fp64
makespan bits then index for float mode) and bench.py's max-over-ranks, so the collective
types and ops are checked on the real backend (the multi-rank logic itself is covered by the
gloo tests in test_sharding.py)."""

import os
import socket

import numpy as np
import pytest
import torch

from paper_2311_02840_b200 import engine as EN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist

    if dist.is_initialized():
        pytest.skip("a process group already exists")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


def test_combine_grid_key_over_nccl(nccl_group):
    key = (30 << 35) | 123456
    best = torch.tensor([key, 0], dtype=torch.int64, device="cuda")
    assert EN._combine(best, True, nccl_group, 2)[0] == key
    empty = torch.tensor([-1, -1], dtype=torch.int64, device="cuda")      # nothing found on a rank
    assert EN._combine(empty, True, nccl_group, 2)[0] == EN.INT64_MAX


def test_combine_float_key_over_nccl(nccl_group):
    ms = np.array([65699.5], dtype=np.float64).view(np.int64)[0]
    best = torch.tensor([int(ms), 77], dtype=torch.int64, device="cuda")
    out = EN._combine(best, False, nccl_group, 2)
    assert out == [int(ms), 77]


def test_max_over_ranks_over_nccl(nccl_group):
    import torch.distributed as dist

    t = torch.tensor([1.25], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=nccl_group)
    assert float(t.item()) == 1.25


def _finish(eng, best, world, group, idx_bits, n_idx, extra=None, check=True):
    key, ids = eng._key_finish(best, True, group, world, idx_bits, n_idx, extra=extra, want_ids=True,
                               check_range=check)
    return key.cpu().tolist(), int(ids.cpu()[0])


def test_key_finish_matches_combine(nccl_group):
    """sat_key_finish (ABI v7) = `_combine_dev` + the replay-id rule it replaced: empty -> INT64_MAX,
    id = low idx_bits (0 when empty or, for exhaustive spaces, out of range); counters appended;
    the world > 1 path all-reduces between the two launches."""
    from paper_2311_02840_b200 import planners as PL

    eng = PL.get_engine(0)
    bits = 35
    key = (30 << bits) | 38747577
    cnt = torch.tensor([7, 11, 13], dtype=torch.int64, device="cuda")
    for world in (1, 2):
        best = torch.tensor([key, 5], dtype=torch.int64, device="cuda")
        out, rid = _finish(eng, best, world, nccl_group, bits, 1 << 34, extra=cnt.view(torch.uint8))
        assert out[:2] == EN._combine(best, True, nccl_group, world)
        assert out[2:] == [7, 11, 13] and rid == 38747577
        empty = torch.tensor([-1, -1], dtype=torch.int64, device="cuda")
        out, rid = _finish(eng, empty, world, nccl_group, bits, 1 << 34)
        assert out == [EN.INT64_MAX, EN.INT64_MAX] and rid == 0
        # an index past the space (exhaustive check) decodes as 0; without the check it stands
        far = torch.tensor([(30 << bits) | ((1 << bits) - 1), 0], dtype=torch.int64, device="cuda")
        assert _finish(eng, far, world, nccl_group, bits, 1000)[1] == 0
        assert _finish(eng, far, world, nccl_group, bits, 1000, check=False)[1] == (1 << bits) - 1
