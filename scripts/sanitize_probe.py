"""Run one piece of sanitize_case under a sanitizer (tuning helper): python scripts/sanitize_probe.py topk|gemv|attn"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2303_06865_b200 import flexq as fq  # noqa: E402
from paper_2303_06865_b200 import synth  # noqa: E402

dev = torch.device("cuda:0")
what = sys.argv[1]
if what == "topk":
    B, H, D, s, n = 2, 3, 128, 100, 3
    for layout in ("dense", "token_major"):
        c = fq.KVCache(B, H, D, s, n, device=dev, layout=layout)
        k = synth.fill(2, 1, (B, H, s, D), device=dev)
        fq.flexq_append_kv(k, k, c, pos=0)
        q = synth.fill(2, 3, (B, H, D), device=dev)
        fq.flexq_decode_attention_topk(q, c, s, keep=fq.topk_keep(s))
elif what == "gemv":
    K, N = 256, 512
    w = synth.fill(3, 1, (K, N), device=dev)
    cc, m = fq.flexq_quantize(w)
    p = fq.flexq_pack_weight(cc, m)
    for M in (5, 12):
        fq.flexq_dequant_gemm(synth.fill(3, 2 + M, (M, K), device=dev), p, N)
elif what == "attn":
    B, H, D, s, n = 2, 3, 128, 100, 3
    for layout in ("dense", "token_major"):
        c = fq.KVCache(B, H, D, s, n, device=dev, layout=layout)
        k = synth.fill(2, 1, (B, H, s, D), device=dev)
        fq.flexq_append_kv(k, k, c, pos=0)
        q = synth.fill(2, 3, (B, H, D), device=dev)
        fq.flexq_append_decode_attention(q, q, q, c, s + 1)
elif what == "tm":
    B, H, D, s, n = 2, 3, 128, 100, 3
    c = fq.KVCache(B, H, D, s, n, device=dev, layout="token_major")
    k = synth.fill(2, 1, (B, H, s, D), device=dev)
    fq.flexq_append_kv(k, k, c, pos=0)
    q = synth.fill(2, 3, (B, H, D), device=dev)
    fq.flexq_append_decode_attention(q, q, q, c, s + n)
elif what == "gemm":
    K, N = 256, 512
    w = synth.fill(3, 1, (K, N), device=dev)
    cc, m = fq.flexq_quantize(w)
    p = fq.flexq_pack_weight(cc, m)
    for M in (20, 170):
        fq.flexq_dequant_gemm(synth.fill(3, 2 + M, (M, K), device=dev), p, N)
elif what == "variants":
    for (b, g, D, B, H, s, n) in ((3, 32, 128, 1, 3, 300, 3), (2, 64, 64, 8, 40, 61, 2)):
        c = fq.KVCache(B, H, D, s, n, device=dev, bits=b, group_size=g)
        k = synth.fill(4, b, (B, H, s, D), device=dev)
        fq.flexq_append_kv(k, k, c, pos=0)
        q = synth.fill(4, 9, (B, H, D), device=dev)
        fq.flexq_decode_attention(q, c, s)
torch.cuda.synchronize()
print("probe ok", what)
