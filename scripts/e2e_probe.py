"""Where does the e2e step's time go (tuning helper)?  OPT-175B shape with a reduced layer count:
the device-resident step, the e2e step, the e2e step without D2H, and the copies alone."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2303_06865_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--slots", type=int, default=8)
    a = ap.parse_args()
    w = wl.CONFIGS["opt-175b"]
    w = wl.Workload(w.name, w.batch, w.heads, w.head_dim, w.prompt_len, w.gen_len, a.layers)
    dev = torch.device("cuda:0")
    st = torch.cuda.Stream()
    m = bench.DecodeModel(w, a.layers, w.batch, 0, w.batch, bench.synth_seed(), dev, st, True)
    m.capture()
    ms, _ = m.time_steps(2, 4, torch.cuda.synchronize)
    L = a.layers
    hin = torch.stack([m.qs, m.kn, m.vn], dim=1).cpu().pin_memory()
    outh = torch.empty(m.outs.shape, dtype=m.outs.dtype).pin_memory()
    NB = a.slots
    din = [torch.empty_like(hin[0], device=dev) for _ in range(NB)]
    dout = [torch.empty_like(m.outs[0]) for _ in range(NB)]
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    res = {"layers": L, "device_step_ms": round(ms / 4, 3)}

    def step(i, do_compute=True, do_d2h=True, do_h2d=True):
        cur = w.prompt_len + i
        ready = [torch.cuda.Event() for _ in range(L)]
        consumed = [torch.cuda.Event() for _ in range(L)]
        drained = [torch.cuda.Event() for _ in range(L)]
        fork = torch.cuda.Event()
        fork.record(st)
        h2d.wait_event(fork)
        d2h.wait_event(fork)
        for j in range(L):
            b = j % NB
            with torch.cuda.stream(h2d):
                if j >= NB:
                    h2d.wait_event(consumed[j - NB])
                if do_h2d:
                    din[b].copy_(hin[j], non_blocking=True)
                ready[j].record(h2d)
            st.wait_event(ready[j])
            if j >= NB:
                st.wait_event(drained[j - NB])
            if do_compute:
                m.layer_step(j, cur, din[b][0], din[b][1], din[b][2], dout[b], st)
            consumed[j].record(st)
            with torch.cuda.stream(d2h):
                d2h.wait_event(consumed[j])
                if do_d2h:
                    outh[j].copy_(dout[b], non_blocking=True)
                drained[j].record(d2h)
        st.wait_stream(h2d)
        st.wait_stream(d2h)

    for name, kw in (("e2e", {}), ("no_d2h", {"do_d2h": False}), ("copies_only", {"do_compute": False}),
                     ("h2d_only", {"do_compute": False, "do_d2h": False}), ("compute_only", {"do_h2d": False,
                                                                                             "do_d2h": False})):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            step(1, **kw)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            for _ in range(4):
                g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        res[name + "_ms"] = round(e0.elapsed_time(e1) / 4, 3)
    res["h2d_mb_per_layer"] = round(hin[0].nbytes / 1e6, 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
