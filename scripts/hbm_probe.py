"""HBM read-only / write-only / copy bandwidth with torch ops (context for write-heavy kernels)."""
import torch
dev = torch.device("cuda:0")
n = 600 * 1024 * 1024
a = torch.empty(n, dtype=torch.float16, device=dev)
b = torch.empty(n, dtype=torch.float16, device=dev)
def t(fn, nbytes, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
print("write (fill_)  GB/s", round(t(lambda: a.fill_(1.0), 2 * n), 1))
print("read (sum)     GB/s", round(t(lambda: a.sum(), 2 * n), 1))
print("copy           GB/s", round(t(lambda: b.copy_(a), 4 * n), 1))
c = torch.empty(n // 4, dtype=torch.uint8, device=dev)
print("read 0.28 + write 1 (dequant-like: b = a[:n/4] expanded)", round(t(lambda: b.view(4, -1).copy_(a[: n // 4].view(1, -1).expand(4, -1)), n // 2 + 2 * n), 1))
