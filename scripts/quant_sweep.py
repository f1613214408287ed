"""Time flexq_quantize / flexq_dequantize alone on the weight-sweep shapes (tuning helper)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2303_06865_b200 import flexq as fq  # noqa: E402
from paper_2303_06865_b200 import synth  # noqa: E402


def timed(fn, reps=10):
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    dev = torch.device("cuda:0")
    for (r, c) in ((12288, 49152), (12288, 12288), (4096, 4096)):
        x = synth.fill(7, 1, (r, c), device=dev)
        codes = torch.empty(r, c // 2, dtype=torch.uint8, device=dev)
        meta = torch.empty(r, c // 64, 2, dtype=torch.float16, device=dev)
        y = torch.empty_like(x)
        nb = r * c * 2 + r * c // 2 + r * c // 64 * 4
        tq = timed(lambda: fq.flexq_quantize(x, codes, meta))
        td = timed(lambda: fq.flexq_dequantize(codes, meta, y))
        print(json.dumps({"shape": f"{r}x{c}", "quantize_us": round(tq, 1), "quantize_gbs": round(nb / tq / 1e3, 1),
                          "dequantize_us": round(td, 1), "dequantize_gbs": round(nb / td / 1e3, 1)}))


def variants():
    """NEXT-3 variants on the OPT-175B w_Q-class matrix (12288 x 12288)."""
    dev = torch.device("cuda:0")
    r, c = 12288, 12288
    x = synth.fill(7, 1, (r, c), device=dev)
    y = torch.empty_like(x)
    for b in (2, 3, 4, 8):
        for g in (32, 64, 128):
            codes = torch.empty(r, c * b // 8, dtype=torch.uint8, device=dev)
            meta = torch.empty(r, c // g, 2, dtype=torch.float16, device=dev)
            nb = r * c * 2 + r * c * b // 8 + r * c // g * 4
            tq = timed(lambda: fq.flexq_quantize(x, codes, meta, bits=b, group_size=g))
            td = timed(lambda: fq.flexq_dequantize(codes, meta, y, bits=b, group_size=g))
            print(json.dumps({"shape": f"{r}x{c}", "bits": b, "group": g, "quantize_us": round(tq, 1),
                              "quantize_gbs": round(nb / tq / 1e3, 1), "dequantize_us": round(td, 1),
                              "dequantize_gbs": round(nb / td / 1e3, 1)}))


if __name__ == "__main__":
    if "--variants" in sys.argv:
        variants()
    else:
        main()
