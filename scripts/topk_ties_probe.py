"""Top-K timing on caches whose last 31 tokens share one K row (the bench's decode step rewrites the
same k_new every step) against caches of distinct rows (tuning helper)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2303_06865_b200 import flexq as fq  # noqa: E402
from paper_2303_06865_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--same", action="store_true", help="tokens 512..542 share one K / V row")
    a = ap.parse_args()
    B, H, D, s, n = 144, 96, 128, 512, 32
    dev = torch.device("cuda:0")
    cur = s + n - 1
    caches = []
    for j in range(a.layers):
        c = fq.KVCache(B, H, D, s, n, device=dev, layout="token_major")
        k = synth.fill(5, 10 + j, (B, H, cur, D), device=dev)
        v = synth.fill(5, 20 + j, (B, H, cur, D), device=dev)
        if a.same:
            k[:, :, s:] = k[:, :, s:s + 1]
            v[:, :, s:] = v[:, :, s:s + 1]
        fq.flexq_append_kv(k, v, c, pos=0)
        del k, v
        caches.append(c)
    q = synth.fill(5, 3, (B, H, D), device=dev)
    out = torch.empty_like(q)
    keep = fq.topk_keep(cur)
    ws = fq.make_topk_workspace(caches[0])
    g = torch.cuda.CUDAGraph()
    for c in caches:
        fq.flexq_decode_attention_topk(q, c, cur, keep, out=out, workspace=ws)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for c in caches:
            fq.flexq_decode_attention_topk(q, c, cur, keep, out=out, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"same_tail": a.same, "keep": keep, "us": round(e0.elapsed_time(e1) * 1e3 / (10 * a.layers), 2),
                      "lib": os.environ.get("FLEXQ_LIB", "default")}))


if __name__ == "__main__":
    main()
