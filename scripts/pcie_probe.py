"""Host<->device copy bandwidth on this box (e2e tuning helper): pinned H2D alone, D2H alone,
and both directions at once on two streams (is the link used full duplex?)."""
import json

import torch


def main():
    dev = torch.device("cuda:0")
    n = 1 << 30
    hs = torch.empty(n, dtype=torch.uint8).pin_memory()
    hd = torch.empty(n, dtype=torch.uint8).pin_memory()
    ds = torch.empty(n, dtype=torch.uint8, device=dev)
    dd = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=3):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e-3)
        return best

    def h2d():
        s1.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s1):
            ds.copy_(hs, non_blocking=True)

    def d2h():
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            hd.copy_(dd, non_blocking=True)

    def both():
        h2d()
        d2h()
    t_h, t_d, t_b = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"h2d_gbs": round(n / t_h / 1e9, 1), "d2h_gbs": round(n / t_d / 1e9, 1),
                      "both_ms": round(t_b * 1e3, 2), "sum_ms": round((t_h + t_d) * 1e3, 2),
                      "max_ms": round(max(t_h, t_d) * 1e3, 2),
                      "duplex": "full" if t_b < 0.6 * (t_h + t_d) else "shared"}))


if __name__ == "__main__":
    main()
