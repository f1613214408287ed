"""Time flexq_decode_attention_topk alone (tuning / profiling helper)."""
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
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--layout", default="token_major", choices=["dense", "token_major"])
    ap.add_argument("--dense", action="store_true", help="time flexq_decode_attention on the same caches")
    a = ap.parse_args()
    w = wl.CONFIGS[a.config]
    B, H, D, s, n = w.batch, w.heads, w.head_dim, w.prompt_len, w.gen_len
    dev = torch.device("cuda:0")
    caches = [fq.KVCache(B, H, D, s, n, device=dev, layout=a.layout) for _ in range(a.layers)]
    k = synth.fill(5, 1, (B, H, s + n - 1, D), device=dev)
    v = synth.fill(5, 2, (B, H, s + n - 1, D), device=dev)
    for c in caches:
        fq.flexq_append_kv(k, v, c, pos=0)
    del k, v
    q = synth.fill(5, 3, (B, H, D), device=dev)
    out = torch.empty_like(q)
    ws = fq.make_workspace(caches[0]) if a.dense else fq.make_topk_workspace(caches[0])
    cur = s + n - 1
    keep = fq.topk_keep(cur)

    def call(c):
        if a.dense:
            fq.flexq_decode_attention(q, c, cur, out=out, workspace=ws)
        else:
            fq.flexq_decode_attention_topk(q, c, cur, keep, out=out, workspace=ws)
    for c in caches:
        call(c)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for c in caches:
            call(c)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (a.reps * a.layers)
    print(json.dumps({"config": a.config, "layout": a.layout, "dense": a.dense, "cur_len": cur, "keep": keep,
                      "us": round(us, 2)}))


if __name__ == "__main__":
    main()
