"""Probe: can the kernels run on a KV cache in pinned host memory (zero-copy over PCIe)?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2303_06865_b200 import flexq as fq  # noqa: E402
from paper_2303_06865_b200 import synth  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    B, H, D, s, n = 16, 96, 128, 512, 32
    cd = fq.KVCache(B, H, D, s, n, device=dev)
    ch = fq.KVCache(B, H, D, s, n, device="cpu")
    ch.k = ch.k.pin_memory()
    ch.v = ch.v.pin_memory()
    k = synth.fill(5, 1, (B, H, s, D), device=dev)
    v = synth.fill(5, 2, (B, H, s, D), device=dev)
    fq.flexq_append_kv(k, v, cd, pos=0)
    fq.flexq_append_kv(k, v, ch, pos=0)
    torch.cuda.synchronize()
    print("append to host cache:", torch.equal(cd.k.cpu(), ch.k), torch.equal(cd.v.cpu(), ch.v))
    q = synth.fill(5, 3, (B, H, D), device=dev)
    kn = synth.fill(5, 4, (B, H, D), device=dev)
    vn = synth.fill(5, 5, (B, H, D), device=dev)
    od = fq.flexq_append_decode_attention(q, kn, vn, cd, s + 1)
    oh = fq.flexq_append_decode_attention(q, kn, vn, ch, s + 1)
    torch.cuda.synchronize()
    print("fused on host cache equal:", torch.equal(od, oh), torch.equal(cd.k.cpu(), ch.k), torch.equal(cd.v.cpu(), ch.v))
    ws = fq.make_workspace(cd)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for c, name in ((cd, "hbm"), (ch, "host")):
        fq.flexq_decode_attention(q, c, s + n, workspace=ws)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            fq.flexq_decode_attention(q, c, s + n, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 3
        nb = c.nbytes() * (s + n) / (c.t_stride)
        print(json.dumps({"cache": name, "us": round(us, 1), "GBps": round(nb / us / 1e3, 2)}))
    # pinned H2D copy bandwidth (the PCIe roofline)
    src = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
    dst = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(4):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"h2d_copy_GBps": round(4 * src.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)}))


if __name__ == "__main__":
    main()
