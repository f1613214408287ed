"""Time flexq_decode_attention alone on one configuration (tuning helper).

    FLEXQ_ATTN_CFG=32,3 python scripts/attn_sweep.py --config opt-175b --layers 8

Rotates over `layers` independent caches (working set >> L2) and reports the
average launch time and algorithmic GB/s (workloads.attention_bytes).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2303_06865_b200 import flexq as fq  # noqa: E402
from paper_2303_06865_b200 import synth  # noqa: E402
from paper_2303_06865_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="opt-175b")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--fused", action="store_true", help="time flexq_append_decode_attention")
    a = ap.parse_args()
    w = wl.CONFIGS[a.config]
    B = a.batch or w.batch
    H, D, s, n = w.heads, w.head_dim, w.prompt_len, w.gen_len
    dev = torch.device("cuda:0")
    caches = [fq.KVCache(B, H, D, s, n, device=dev) for _ in range(a.layers)]
    k = synth.fill(5, 1, (B, H, s + n - 1, D), device=dev)
    v = synth.fill(5, 2, (B, H, s + n - 1, D), device=dev)
    for c in caches:
        fq.flexq_append_kv(k, v, c, pos=0)
    del k, v
    q = synth.fill(5, 3, (B, H, D), device=dev)
    out = torch.empty_like(q)
    ws = fq.make_workspace(caches[0])
    cur = s + n - 1
    st = torch.cuda.current_stream()
    kn = synth.fill(5, 4, (B, H, D), device=dev)
    vn = synth.fill(5, 5, (B, H, D), device=dev)

    def call(c):
        if a.fused:
            fq.flexq_append_decode_attention(q, kn, vn, c, cur, out=out, workspace=ws)
        else:
            fq.flexq_decode_attention(q, c, cur, out=out, workspace=ws)
    g = torch.cuda.CUDAGraph()
    for c in caches:
        call(c)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for c in caches:
            call(c)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.reps):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (a.reps * a.layers)
    nb = wl.attention_bytes(B, H * D, cur) + (wl.append_bytes(B, H * D) if a.fused else 0)
    print(json.dumps({"cfg": os.environ.get("FLEXQ_ATTN_CFG", "default"), "fused": a.fused, "config": a.config,
                      "batch": B,
                      "cur_len": cur, "us": round(us, 2), "GBps": round(nb / us / 1e3, 1)}))


if __name__ == "__main__":
    main()
