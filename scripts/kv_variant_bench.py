"""Decode attention over the NEXT-3 variant caches (b in {2, 3, 4, 8} x g in {32, 64, 128}) at one
configuration, against the b = 4, g = 64 tensor-core kernel on the same shape.

    python scripts/kv_variant_bench.py --config opt-175b --layers 4

Each variant rotates over `layers` caches (working set >> L2), replayed as a CUDA graph; reports
the average launch time and the algorithmic bytes / s: 2 B H cur_len (D b / 8 + 4 D / g) (K and
V codes + meta of every attended token) + q and out, the variant's analogue of
workloads.attention_bytes.  One JSON line per variant.
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

VARIANTS = [(4, 64)] + [(b, g) for b in (2, 3, 4, 8) for g in (32, 64, 128) if (b, g) != (4, 64)]


def variant_bytes(B, H, D, cur, bits, group):
    return 2 * B * H * cur * (D * bits // 8 + 4 * D // group) + 2 * B * H * D * 2


def run(cfg, bits, group, layers, reps, dev):
    B, H, D, s, n = cfg.batch, cfg.heads, cfg.head_dim, cfg.prompt_len, cfg.gen_len
    cur = s + n - 1
    caches = [fq.KVCache(B, H, D, s, n, device=dev, bits=bits, group_size=group) for _ in range(layers)]
    k = synth.fill(5, 1, (B, H, cur, D), device=dev)
    v = synth.fill(5, 2, (B, H, cur, D), device=dev)
    for c in caches:
        fq.flexq_append_kv(k, v, c, pos=0)
    del k, v
    q = synth.fill(5, 3, (B, H, D), device=dev)
    out = torch.empty_like(q)
    ws = fq.make_workspace(caches[0])
    for c in caches:
        fq.flexq_decode_attention(q, c, cur, out=out, workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for c in caches:
            fq.flexq_decode_attention(q, c, cur, out=out, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * layers)
        best = us if best is None else min(best, us)
    nb = variant_bytes(B, H, D, cur, bits, group) if (bits, group) != (4, 64) else wl.attention_bytes(B, H * D, cur)
    del caches, g
    torch.cuda.empty_cache()
    return {"bits": bits, "group": group, "config": cfg.name if hasattr(cfg, "name") else None, "cur_len": cur,
            "kernel": "tensor-core b4g64" if (bits, group) == (4, 64) else "variant (CUDA cores)",
            "us": round(best, 2), "bytes": nb, "GBps": round(nb / best / 1e3, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="opt-175b")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="", help="b,g (one variant)")
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.config]
    dev = torch.device("cuda:0")
    todo = VARIANTS if not a.only else [tuple(int(x) for x in a.only.split(","))]
    for bits, group in todo:
        if cfg.head_dim % group:
            continue
        r = run(cfg, bits, group, a.layers, a.reps, dev)
        r["config"] = a.config
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
