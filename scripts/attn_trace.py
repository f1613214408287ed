"""Per-warp timeline of one dense-attention launch (tuning helper, trace build only).

    python -m paper_2303_06865_b200.build --trace
    FLEXQ_LIB=paper_2303_06865_b200/libflexq_trace.so python scripts/attn_trace.py --config opt-6.7b

Replays a CUDA graph of `layers` launches, then reads the last launch's per-warp
%globaltimer stamps (resident, after griddepcontrol.wait, end) and prints where
the launch's time goes: the wait for the previous grid, the spread of warp end
times (tail), and the warp durations.
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_06865_b200 import flexq as fq  # noqa: E402
from paper_2303_06865_b200 import synth  # noqa: E402
from paper_2303_06865_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="opt-6.7b")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--fused", action="store_true")
    ap.add_argument("--dump", default="", help="save the raw per-warp stamps (.npy) for offline analysis")
    a = ap.parse_args()
    w = wl.CONFIGS[a.config]
    B = a.batch or w.batch
    H, D, s, n = w.heads, w.head_dim, w.prompt_len, w.gen_len
    dev = torch.device("cuda:0")
    caches = [fq.KVCache(B, H, D, s, n, device=dev) for _ in range(a.layers)]
    k = synth.fill(5, 1, (B, H, s + n - 1, D), device=dev)
    v = synth.fill(5, 2, (B, H, s + n - 1, D), device=dev)
    for c in caches:
        fq.flexq_append_kv(k, v, c, pos=0)
    del k, v
    q = synth.fill(5, 3, (B, H, D), device=dev)
    kn = synth.fill(5, 4, (B, H, D), device=dev)
    vn = synth.fill(5, 5, (B, H, D), device=dev)
    out = torch.empty_like(q)
    ws = fq.make_workspace(caches[0])
    cur = s + n - 1

    def call(c):
        if a.fused:
            fq.flexq_append_decode_attention(q, kn, vn, c, cur, out=out, workspace=ws)
        else:
            fq.flexq_decode_attention(q, c, cur, out=out, workspace=ws)
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
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    per_launch = e0.elapsed_time(e1) * 1e3 / a.layers
    W = 4096
    buf = np.zeros((W, 4), np.uint64)
    rc = fq.lib().flexq_debug_attn_trace(ctypes.c_void_p(buf.ctypes.data), W)
    assert rc == 0, rc
    used = buf[:, 2] > 0
    if a.dump:
        np.save(a.dump, buf[used])
    t = buf[used].astype(np.int64)
    t0 = t[:, 0].min()
    res, go, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
    dur = end - go
    q = lambda x: [round(float(np.percentile(x, p)), 2) for p in (0, 10, 50, 90, 100)]  # noqa: E731
    print(json.dumps({
        "config": a.config, "batch": B, "fused": a.fused, "warps": int(used.sum()), "us_per_launch": round(per_launch, 2),
        "resident_us_pct": q(res), "go_us_pct": q(go), "end_us_pct": q(end), "dur_us_pct": q(dur),
        "pieces_pct": q(t[:, 3] & 0xFFFFFFFF),
        "span_us": round(float(end.max()), 2)}))
    sm = (t[:, 3] >> 32).astype(np.int64)
    per_sm = np.array([dur[sm == i].mean() for i in np.unique(sm)])
    within = np.array([dur[sm == i].std() for i in np.unique(sm)])
    order = np.argsort(per_sm)
    print(json.dumps({"sms": int(len(per_sm)), "sm_mean_dur_pct": q(per_sm), "within_sm_std_mean": round(float(within.mean()), 2),
                      "slowest_sms": [int(np.unique(sm)[i]) for i in order[-8:]],
                      "fastest_sms": [int(np.unique(sm)[i]) for i in order[:8]],
                      "dur_by_warp_index_decile": [round(float(dur[(np.arange(len(dur)) * 10 // len(dur)) == d].mean()), 2) for d in range(10)]}))


if __name__ == "__main__":
    main()
