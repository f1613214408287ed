"""Pipeline trace of CTA 0 (tuning): run the FLEXQ_GEMM_TRACE=1 build and print stage timings."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_06865_b200 import flexq as fq  # noqa: E402
from paper_2303_06865_b200 import synth  # noqa: E402

dev = torch.device("cuda:0")
K, N = 12288, 256 * 148 * int(os.environ.get('TRACE_NMUL', '1'))
w = synth.fill(7, 1, (K, N), device=dev)
codes, meta = fq.flexq_quantize(w)
panels = fq.flexq_pack_weight(codes, meta)
for M in [int(a) for a in sys.argv[1:]] or [1, 144]:
    x = synth.fill(7, 2, (M, K), device=dev)
    ws = fq.make_gemm_workspace(M, K, N, dev)
    for _ in range(3):
        fq.flexq_dequant_gemm(x, panels, N, workspace=ws)
    torch.cuda.synchronize()
    tick = (N // 256 * 4 + 255) // 256 * 256
    t = ws[tick:tick + 8 * 256 * 8].view(torch.int64).view(8, 256).cpu().numpy().astype(np.int64)
    t = t - t[0, 0]
    names = ["mma_top", "mma_2iss", "mma_waited", "mma_commit", "dq_pre", "dq_pfull", "dq_aempty", "dq_afull"]
    print(f"M={M}: stages 100..110 (cycles from MMA start)")
    print("      " + " ".join(f"{n:>10s}" for n in names))
    for j in range(100, 106):
        print(f"{j:5d} " + " ".join(f"{t[i, j]:10d}" for i in range(8)))
    per = (t[3, 200] - t[3, 100]) / 100
    print(f"cycles per stage (MMA commit cadence 100..200): {per:.0f}")
