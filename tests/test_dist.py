"""N > 1 host logic on CPU with the gloo backend (world_size 2): sequence
sharding covers [0, B) exactly once, the max-over-ranks timing reduction,
and the output all-gather reassembles the per-rank blocks in order."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2303_06865_b200 import dist as fd


@pytest.mark.parametrize("B", [1, 4, 18, 143, 144])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_partition(B, world):
    seen = []
    for r in range(world):
        b, e = fd.shard(B, world, r)
        assert 0 <= b <= e <= B
        seen.extend(range(b, e))
        assert fd.rank_batch(B, world, r, "strong") == e - b
        assert fd.rank_batch(B, world, r, "weak") == B
    assert seen == list(range(B))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = fd.max_over_ranks(10.0 + rank)
        b, e = fd.shard(B, world, rank)
        out = torch.arange(b, e, dtype=torch.float32).view(-1, 1).repeat(1, 3)
        full = fd.gather_outputs(out, B)
        q.put((rank, t, full[:, 0].tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B", [5, 144])
def test_gloo_world2(B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, col in res:
        assert t == 11.0                       # max over ranks
        assert col == [float(i) for i in range(B)]
