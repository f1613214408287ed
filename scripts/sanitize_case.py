"""Small end-to-end run of every kernel for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python scripts/sanitize_case.py

Covers: quantize/dequantize with a ragged row count (and the b/g variants),
prompt fill + 1-token append, attention with split-K (few heads) and without,
Top-K, the fused append + attention, a cache whose capacity is not a multiple
of the token stride (cur_len = T_cap, last head: the metadata bulk copy rounds
up into the stride padding), the KV-cache variants, weight packing, the tcgen05 dequant-GEMM and the small-batch dequant-GEMV.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2303_06865_b200 import flexq as fq  # noqa: E402
from paper_2303_06865_b200 import synth  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    x = synth.fill(1, 1, (37, 192), device=dev)
    c, m = fq.flexq_quantize(x)
    fq.flexq_dequantize(c, m)
    for (B, H, D, s, n) in [(2, 3, 128, 100, 3), (1, 2, 64, 61, 0), (8, 40, 128, 33, 2)]:
        if n == 0:
            n = 1
        cache = fq.KVCache(B, H, D, s, n, device=dev)
        k = synth.fill(2, 1, (B, H, s, D), device=dev)
        v = synth.fill(2, 2, (B, H, s, D), device=dev)
        fq.flexq_append_kv(k, v, cache, pos=0)
        for i in range(n):
            kn = synth.fill(2, 10 + i, (B, H, 1, D), device=dev)
            fq.flexq_append_kv(kn, kn, cache, pos=s + i)
        q = synth.fill(2, 3, (B, H, D), device=dev)
        ws = fq.make_workspace(cache)
        for cur in (1, s, s + n):
            fq.flexq_decode_attention(q, cache, cur, workspace=ws)
        # NEXT-1 Top-K and NEXT-3 fused append + attention on the same cache
        fq.flexq_decode_attention_topk(q, cache, s, keep=fq.topk_keep(s))
        # the token-major layout (Top-K's): append, Top-K gather of contiguous rows, dense attention
        tm = fq.KVCache(B, H, D, s, n, device=dev, layout="token_major")
        fq.flexq_append_kv(k, v, tm, pos=0)
        fq.flexq_decode_attention_topk(q, tm, s, keep=fq.topk_keep(s))
        fq.flexq_append_decode_attention(q, q, q, tm, s + n)
        fq.flexq_append_decode_attention(q, q, q, cache, s + n, workspace=ws)
        # interop: export the cache to the plain layout, import a token range back
        kc, km, vc, vm = fq.flexq_kv_export(cache)
        fq.flexq_kv_import(cache, kc, km, vc, vm, t0=min(5, s), n_tok=min(37, s + n - min(5, s)))
    # NEXT-3 quantizer variants
    for b, g in ((2, 32), (3, 128), (8, 64)):
        c, m = fq.flexq_quantize(x[:, :128].contiguous(), bits=b, group_size=g)
        fq.flexq_dequantize(c, m, bits=b, group_size=g)
    # NEXT-3 KV-cache variants: append, attention with and without splits (cur_len up to T_cap,
    # last head: the staged chunks end at the buffer end), the one-call decode step; b = 8 stages K
    for (b, g, D, B, H, s, n) in ((3, 32, 128, 1, 3, 300, 3), (8, 128, 128, 2, 2, 160, 1), (2, 64, 64, 8, 40, 61, 2)):
        cache = fq.KVCache(B, H, D, s, n, device=dev, bits=b, group_size=g)
        k = synth.fill(4, b, (B, H, s, D), device=dev)
        fq.flexq_append_kv(k, k, cache, pos=0)
        q = synth.fill(4, 9, (B, H, D), device=dev)
        ws = fq.make_workspace(cache)
        for cur in (1, s):
            fq.flexq_decode_attention(q, cache, cur, workspace=ws)
        fq.flexq_append_decode_attention(q, q, q, cache, s + n, workspace=ws)
    # NEXT-2 decode linear layer: a full tile and split-k remainder tiles, two row chunks
    K, N = 256, 512
    w = synth.fill(3, 1, (K, N), device=dev)
    c, m = fq.flexq_quantize(w)
    panels = fq.flexq_pack_weight(c, m)
    for M in (5, 12, 20, 170):   # 5, 12: the small-batch panel-streaming kernel (8 panels, 8 CTAs)
        fq.flexq_dequant_gemm(synth.fill(3, 2 + M, (M, K), device=dev), panels, N)
    torch.cuda.synchronize()
    print("sanitize case ok")


if __name__ == "__main__":
    main()
