"""Time flexq_dequant_gemm (NEXT-2) on the OPT-175B decode linear layers, beside the
library baselines: flexq_dequantize + cuBLAS (torch.matmul) and cuBLAS on the fp16 weight."""
import argparse
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
    best = 1e30
    for _ in range(3):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, nargs="*", default=[144])
    ap.add_argument("--only", action="store_true", help="flexq kernel only (for ncu)")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--shapes", nargs="*", default=["12288x49152", "12288x12288"], help="KxN")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    for (K, N) in [tuple(int(v) for v in sh.split("x")) for sh in a.shapes]:
        w = synth.fill(7, 1, (K, N), device=dev)
        codes, meta = fq.flexq_quantize(w)
        panels = fq.flexq_pack_weight(codes, meta)
        for M in a.m:
            x = synth.fill(7, 2, (M, K), device=dev)
            y = torch.empty(M, N, dtype=torch.float16, device=dev)
            ws = fq.make_gemm_workspace(M, K, N, dev)
            flops = 2.0 * M * K * N
            wbytes = K * N // 2 + K * N // 64 * 4
            t = timed(lambda: fq.flexq_dequant_gemm(x, panels, N, out=y, workspace=ws), a.reps)
            r = {"shape": f"{M}x{K}x{N}", "flexq_us": round(t, 1), "flexq_tflops": round(flops / t / 1e6, 1),
                 "flexq_weight_gbs": round(wbytes / t / 1e3, 1)}
            if not a.only:
                wd = torch.empty(K, N, dtype=torch.float16, device=dev)
                yd = torch.empty_like(y)
                t2 = timed(lambda: (fq.flexq_dequantize(codes, meta, wd), torch.matmul(x, wd, out=yd)), a.reps)
                t3 = timed(lambda: torch.matmul(x, w, out=yd), a.reps)
                r.update({"dequant_then_cublas_us": round(t2, 1), "cublas_fp16_weight_us": round(t3, 1),
                          "speedup_vs_dequant_cublas": round(t2 / t, 2), "speedup_vs_fp16_cublas": round(t3 / t, 2)})
                del wd, yd
            print(json.dumps(r), flush=True)
        del w, codes, meta, panels


if __name__ == "__main__":
    main()
