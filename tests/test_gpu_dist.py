"""Multi-rank parity on the GPU (SURVEY 4 test layer 5): the global batch sharded over two
ranks -- two processes on the same device, gloo for the gather (NCCL needs one GPU per rank) --
gives, once the per-rank outputs are gathered, exactly the single-process outputs, bit for bit.

Each rank draws its shard of the global inputs (synth.fill_rows) and runs prompt fill and three
fused decode steps (flexq_append_decode_attention) over its own caches.  The test-only schedule
override FLEXQ_ATTN_SPLIT=0,0,0 makes every launch hand out whole heads, so a head's arithmetic
does not depend on how many heads share the launch (the default schedule may cut a small
launch's heads into pieces, which merges in a different rounding order)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

B_GLOBAL, H, D, S, N, STEPS = 8, 16, 128, 300, 4, 3
SEED = 4242


def run_shard(b0: int, b1: int) -> np.ndarray:
    """Prompt fill + STEPS fused decode steps for global rows [b0, b1) -> outputs [steps][b][H][D]."""
    from paper_2303_06865_b200 import flexq as fq
    from paper_2303_06865_b200 import synth
    dev = torch.device("cuda:0")
    cache = fq.KVCache(b1 - b0, H, D, S, N, device=dev)
    kp = synth.fill_rows(SEED, synth.tensor_id(0, synth.K_PROMPT), (B_GLOBAL, H, S, D), b0, b1, device=dev)
    vp = synth.fill_rows(SEED, synth.tensor_id(0, synth.V_PROMPT), (B_GLOBAL, H, S, D), b0, b1, device=dev)
    fq.flexq_append_kv(kp, vp, cache, pos=0)
    outs = []
    for i in range(1, STEPS + 1):
        rows = lambda kind: synth.fill_rows(SEED, synth.tensor_id(0, kind, i), (B_GLOBAL, H, D), b0, b1,  # noqa: E731
                                            device=dev)
        outs.append(fq.flexq_append_decode_attention(rows(synth.Q), rows(synth.K_NEW), rows(synth.V_NEW), cache,
                                                     S + i))
    torch.cuda.synchronize()
    return torch.stack(outs).cpu().numpy()


def _rank_main(rank: int, world: int, port: int, out_path: str):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), FLEXQ_ATTN_SPLIT="0,0,0")
    import torch.distributed as dist
    from paper_2303_06865_b200 import dist as fd
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    b0, b1 = fd.shard(B_GLOBAL, world, rank)
    local = torch.from_numpy(run_shard(b0, b1)).permute(1, 0, 2, 3).contiguous()   # [b][steps][H][D]
    full = fd.gather_outputs(local, B_GLOBAL)
    if rank == 0:
        np.save(out_path, full.permute(1, 0, 2, 3).contiguous().numpy())
    dist.barrier()
    dist.destroy_process_group()


def _single_main(_: int, out_path: str):
    os.environ["FLEXQ_ATTN_SPLIT"] = "0,0,0"
    np.save(out_path, run_shard(0, B_GLOBAL))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_match_single_process_bitwise(tmp_path):
    sharded, single = str(tmp_path / "sharded.npy"), str(tmp_path / "single.npy")
    mp.spawn(_rank_main, args=(2, _free_port(), sharded), nprocs=2, join=True)
    mp.spawn(_single_main, args=(single,), nprocs=1, join=True)
    a, b = np.load(sharded), np.load(single)
    assert a.shape == b.shape == (STEPS, B_GLOBAL, H, D)
    assert np.array_equal(a.view(np.uint16), b.view(np.uint16)), \
        f"{int((a.view(np.uint16) != b.view(np.uint16)).sum())} outputs differ"


def test_bench_two_ranks_same_device(tmp_path):
    """bench.py's N > 1 path end to end on one GPU (two ranks, gloo): strong scaling of the global
    batch, the gathered row checked against rank 0's from-scratch recomputation."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--same-device", "--layers", "4", "--steps", "3", "--warmup", "3", "--no-e2e",
           "--no-cpu-baseline", "--no-sweep", "--no-offload", "--no-weak"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["config"]["global_batch"] == 144
    assert line["dist"]["comm_size"] == 2
    assert line["output_check"]["within_reading_Q"], line["output_check"]
