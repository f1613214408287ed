"""NEXT-4 measurement: decode steps over a host-offloaded compressed KV cache (OPT-175B shape),
Alg. 1 overlap, against the pinned host->device copy bandwidth (the PCIe roofline)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2303_06865_b200 import synth  # noqa: E402
from paper_2303_06865_b200.offload import OffloadedKV  # noqa: E402


def h2d_gbs(dev, nbytes=1 << 30):
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(3):                    # best of 3 trials of 4 back-to-back 1 GiB copies
        e0.record()
        for _ in range(4):
            dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 4 * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def run(layers=2, gpu_batches=1, B=144, H=96, D=128, s=512, n=32, steps=3, dev="cuda:0"):
    dev = torch.device(dev)
    peak = h2d_gbs(dev)
    off = OffloadedKV(layers, gpu_batches, B, H, D, s, n, dev, slots=2)
    seed = 230306865 + 3
    kp = synth.fill(seed, 1, (B, H, s, D), device=dev)
    vp = synth.fill(seed, 2, (B, H, s, D), device=dev)
    off.prefill(lambda j, k: kp, lambda j, k: vp)
    del kp, vp
    q = synth.fill(seed, 3, (B, H, D), device=dev)
    kn = synth.fill(seed, 4, (B, H, D), device=dev)
    vn = synth.fill(seed, 5, (B, H, D), device=dev)
    out = torch.empty_like(q)
    f = lambda t: (lambda j, k: t)  # noqa: E731
    off.decode_step(s + 1, f(q), f(kn), f(vn), f(out))        # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(2, 2 + steps):
        off.decode_step(s + i, f(q), f(kn), f(vn), f(out))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    blocks = layers * gpu_batches
    moved = blocks * off.block_bytes()                        # H2D per step
    return {"layers": layers, "gpu_batches": gpu_batches, "batch_per_gpu_batch": B, "ms_per_step": round(ms, 2),
            "ms_per_block": round(ms / blocks, 3), "h2d_bytes_per_step": moved,
            "h2d_gbs": round(moved / (ms * 1e-3) / 1e9, 2), "pinned_h2d_copy_gbs": round(peak, 2),
            "frac_of_pcie": round(moved / (ms * 1e-3) / 1e9 / peak, 4),
            "model_tokens_per_s": round(B * gpu_batches / (ms * 1e-3), 1),
            "attention_tokens_per_s_per_layer": round(B * gpu_batches * layers / (ms * 1e-3), 1),
            "fp16_equivalent_bytes_per_step": int(moved / 0.28125 * 1.0)}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--gpu-batches", type=int, default=1)
    ap.add_argument("--batch", type=int, default=144)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    print(json.dumps(run(a.layers, a.gpu_batches, a.batch, steps=a.steps)))
