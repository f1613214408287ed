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


def test_bench_rank_rows_and_defaults():
    """bench.py's sharding: strong scaling splits the fixed global batch (configs[3]: 144 over
    the GPUs), weak gives every rank its own block of the per-GPU batch; owner() inverts shard()."""
    import importlib.util
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for world in (1, 2, 4, 8):
        rows = [bench.rank_rows(144, world, r, "strong", 144) for r in range(world)]
        assert rows[0][0] == 0 and rows[-1][1] == 144
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        for r, (b0, b1) in enumerate(rows):
            assert all(fd.owner(144, world, x) == r for x in range(b0, b1))
        weak = [bench.rank_rows(144 * world, world, r, "weak", 144) for r in range(world)]
        assert weak == [(144 * r, 144 * (r + 1)) for r in range(world)]
    old = sys.argv
    try:
        sys.argv = ["bench.py", "--gpus", "8"]
        assert bench.parse().scaling == "strong"
        sys.argv = ["bench.py", "--config", "opt-30b"]
        assert bench.parse().scaling == "weak"
    finally:
        sys.argv = old


def test_bench_world_size_mismatch_fails():
    """--gpus N must match the launched world size (no silent single-process run)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE=3" in (r.stderr + r.stdout)
